#!/bin/bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_multi_gpu.py -q -x -k "mmm or codon or yeast or wnv or small_shapes or max_categories or nccl or two_process" > gpurun_out/d_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/d_tests.log; tail -3 gpurun_out/d_tests.log
rm -rf gpurun_out/sanitize; CASES="mmm yeast yeast_levels s122 dengue" bash scripts/gpu_sanitize.sh > /dev/null 2>&1; cat gpurun_out/sanitize/summary.txt
for c in 2 3 5; do timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --no-fp64-probe 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['kernel_ms'])"; done
