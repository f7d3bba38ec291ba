#!/bin/bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PG_PARITY_LOG=gpurun_out/parity_tc.jsonl timeout 1200 python -m pytest tests/test_parity_gpu.py -q -x -k "fp32" > gpurun_out/tc_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tc_tests.log; tail -4 gpurun_out/tc_tests.log
for args in "--config 3 --precision fp32" "--config 3 --precision fp64" "--config 4 --precision fp32" "--config 3 --precision fp32 --virtual-shard 8"; do
  timeout 300 python bench.py $args --steps 200 --warmup 10 --no-cpu-baseline --no-fp64-probe > gpurun_out/b.json 2>gpurun_out/b.err
  python - "$args" <<'PY'
import json,sys
try:
    d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
    r=d['roofline']; p=d['plan']
    print(f"{sys.argv[1]:42s} {d['ms_per_step']:.4f} ms {d['value']:.1f} evals/s kern {d['kernel_ms']} variant {p['kernel_variant']} frac {r['frac']} {r['unit']} peak {r['peak']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e, open('gpurun_out/b.err').read()[-800:])
PY
done 2>&1 | tee gpurun_out/tc_bench.txt
