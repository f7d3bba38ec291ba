#!/bin/bash
# session-2 start: validate HEAD (all GPU tests, smoke, default bench)
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/r3a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
PG_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rf -x > $O/gpu_tests.log 2>&1
echo "tests exit $?" >> $O/gpu_tests.log; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench exit $?" >> $O/bench_default.err
tail -c 3000 $O/bench_default.json
