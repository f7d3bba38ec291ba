#!/bin/bash
# codon flow v2: A1 P / D readiness flags split (post items wait for P only)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_multi_gpu.py -q -x -k "codon or yeast or wnv or mmm122 or shard or nccl or two_process" > gpurun_out/codon7_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/codon7_tests.log
tail -3 gpurun_out/codon7_tests.log
run() {
    env $1 timeout 300 python bench.py $2 --steps 300 --warmup 20 --no-cpu-baseline --no-fp64-probe --no-extra-configs > gpurun_out/b.json 2>gpurun_out/b.err
    python - "$1" "$2" <<'PY'
import json,sys
try:
    d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
    r=d['roofline']; p=d['plan']
    print(f"{sys.argv[1]:34s} {sys.argv[2]:32s} {d['ms_per_step']:.4f} ms p50 {d['ms_step_p10_p50_p90'][1]:.4f} kern {d['kernel_ms']} frac {r['frac']} eval_frac {r['eval_frac']}")
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e, open('gpurun_out/b.err').read()[-800:])
PY
}
for cfg in "--config 3 --virtual-shard 8" "--config 4 --virtual-shard 8" "--config 5 --virtual-shard 8" "--config 3"; do
    run "PG_FLOW_PUB=1" "$cfg"
done 2>&1 | tee gpurun_out/codon7_bench.txt
python scripts/flow2_trace.py 3 8 > gpurun_out/trace_3_8.txt 2>&1; head -14 gpurun_out/trace_3_8.txt
