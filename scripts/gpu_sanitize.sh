#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small instances of
# every kernel family.  Logs -> gpurun_out/sanitize/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
for case in ${CASES:-jc5 dengue dengue_fp32 mmm yeast yeast_levels s122 s256 codon_fp32}; do
  for tool in memcheck racecheck synccheck; do
    log=gpurun_out/sanitize/${case}_${tool}.log
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 17 --print-limit 50 \
        python scripts/sanitize_case.py $case > $log 2>&1
    echo "$case $tool exit=$?" | tee -a gpurun_out/sanitize/summary.txt
    tail -3 $log
  done
done
