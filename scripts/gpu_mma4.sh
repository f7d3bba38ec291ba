#!/bin/bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "dengue or small_shapes or max_categories or partials or deep or config0 or caterpillar or zero or branch_lengths or device_path or mmm" > gpurun_out/mma4_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/mma4_tests.log
tail -3 gpurun_out/mma4_tests.log
for v in default old; do
  if [ $v = default ]; then lib=""; else lib="PHYLOGRAD_LIB=$PWD/paper_2303_04390_b200/lib/libphylograd_old.so"; fi
  env $lib timeout 300 python bench.py --config 1 --steps 300 --warmup 20 --no-cpu-baseline --no-fp64-probe --no-extra-configs > gpurun_out/b.json 2>gpurun_out/b.err
  python - "$v" <<'PY'
import json,sys
try:
    d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
    r=d['roofline']; p=d['plan']
    print(f"{sys.argv[1]:10s} {d['ms_per_step']:.4f} ms  kern {d['kernel_ms']} frac {r['frac']} grid {p['grid']} smem {p['smem_bytes']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e, open('gpurun_out/b.err').read()[-800:])
PY
done 2>&1 | tee gpurun_out/mma4_bench.txt
