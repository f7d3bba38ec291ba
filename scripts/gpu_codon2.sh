#!/bin/bash
# codon flow v2 (warp-specialised TMA ring): parity, then timings vs v1
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "codon or yeast or wnv or mmm122 or hmc or clock or extended" > gpurun_out/codon2_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/codon2_tests.log
tail -5 gpurun_out/codon2_tests.log
for v in 2 1; do
  for cfg in "--config 3" "--config 3 --virtual-shard 8" "--config 4" "--config 4 --virtual-shard 8" "--config 5" "--config 5 --virtual-shard 8"; do
    PG_CODON_FLOW=$v timeout 300 python bench.py $cfg --steps 200 --warmup 20 --no-cpu-baseline --no-fp64-probe > gpurun_out/b.json 2>gpurun_out/b.err
    python - "$v" "$cfg" <<'PY'
import json,sys
try:
    d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
    r=d['roofline']
    print(f"v{sys.argv[1]} {sys.argv[2]:32s} {d['ms_per_step']:.4f} ms  kern {d['kernel_ms']}  frac {r['frac']} eval_frac {r['eval_frac']}")
except Exception as e:
    print("v", sys.argv[1], sys.argv[2], "FAILED", e, open('gpurun_out/b.err').read()[-800:])
PY
  done
done 2>&1 | tee gpurun_out/codon2_bench.txt
