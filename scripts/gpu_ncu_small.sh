#!/bin/bash
# ncu --set full of the small-S traversal: MMM (config 2) and dengue (config 1)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in ${CFGS:-2 1}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse_small -s 3 -c 1 -o gpurun_out/prof_small_c$cfg -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fp64-probe --no-flush --no-extra-configs --config $cfg > gpurun_out/ncu_small_c$cfg.log 2>&1; tail -1 gpurun_out/ncu_small_c$cfg.log
  python scripts/ncu_summary.py gpurun_out/prof_small_c$cfg.ncu-rep > gpurun_out/ncu_small_c$cfg.txt; cat gpurun_out/ncu_small_c$cfg.txt
  python scripts/ncu_lines.py gpurun_out/prof_small_c$cfg.ncu-rep traverse_small 60 > gpurun_out/ncu_small_c${cfg}_lines.txt
done
