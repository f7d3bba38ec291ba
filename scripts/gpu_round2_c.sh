#!/bin/bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2c
O=gpurun_out/r2c
PG_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.log 2>&1
echo "tests exit $?" >> $O/gpu_tests.log; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log; cat $O/smoke.log
rm -rf gpurun_out/sanitize; CASES="mmm yeast s256 codon_fp32" bash scripts/gpu_sanitize.sh > $O/sanitize_stdout.txt 2>&1; cp -r gpurun_out/sanitize $O/
cat $O/sanitize/summary.txt
