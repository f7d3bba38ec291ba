#!/bin/bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
PG_PARITY_LOG=gpurun_out/parity_s256.jsonl timeout 1500 python -m pytest tests/test_s256_gpu.py -q -x > gpurun_out/s256_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/s256_tests.log
tail -5 gpurun_out/s256_tests.log
timeout 900 python bench.py --config 6 --steps 5 --warmup 3 --no-cpu-baseline --no-fp64-probe > gpurun_out/bench_c6.json 2>gpurun_out/bench_c6.err
tail -2 gpurun_out/bench_c6.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_c6.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'], d['roofline']['eval_frac'])"
