#!/bin/bash
# S = 16 traversal on the FP64 tensor path: parity, then MMM timings vs K
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "mmm or small_shapes or max_categories or partials or deep or config0 or dengue_reduced" > gpurun_out/mma_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/mma_tests.log
tail -3 gpurun_out/mma_tests.log
for k in 0 1 2 3 4 5; do
  if [ $k = 0 ]; then e=""; else e="PG_SMALL_K=$k"; fi
  env $e timeout 300 python bench.py --config 2 --steps 300 --warmup 20 --no-cpu-baseline --no-fp64-probe > gpurun_out/b.json 2>gpurun_out/b.err
  python - "$e" <<'PY'
import json,sys
try:
    d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
    r=d['roofline']; p=d['plan']
    print(f"{sys.argv[1]:14s} {d['ms_per_step']:.4f} ms  kern {d['kernel_ms']} frac {r['frac']} grid {p['grid']} block {p['block']} smem {p['smem_bytes']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e, open('gpurun_out/b.err').read()[-800:])
PY
done 2>&1 | tee gpurun_out/mma_bench.txt
