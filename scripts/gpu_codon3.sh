#!/bin/bash
# codon flow v2 variants: parity, then timings (NST 1/2, PDL on/off) vs v1
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_multi_gpu.py -q -x -k "codon or yeast or wnv or mmm122 or hmc or clock or extended or nccl" > gpurun_out/codon3_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/codon3_tests.log
tail -3 gpurun_out/codon3_tests.log
run() {
    env $1 timeout 300 python bench.py $2 --steps 200 --warmup 20 --no-cpu-baseline --no-fp64-probe > gpurun_out/b.json 2>gpurun_out/b.err
    python - "$1" "$2" <<'PY'
import json,sys
try:
    d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
    r=d['roofline']; p=d['plan']
    print(f"{sys.argv[1]:34s} {sys.argv[2]:32s} {d['ms_per_step']:.4f} ms p50 {d['ms_step_p10_p50_p90'][1]:.4f} kern {d['kernel_ms']} frac {r['frac']} eval_frac {r['eval_frac']} nst {p.get('flow_stages')} pdl {p.get('flow_pdl')}")
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e, open('gpurun_out/b.err').read()[-800:])
PY
}
for cfg in "--config 3" "--config 3 --virtual-shard 8" "--config 4" "--config 4 --virtual-shard 8" "--config 5" "--config 5 --virtual-shard 8"; do
  for e in "PG_CODON_FLOW=2" "PG_FLOW_RS=2"; do
    run "$e" "$cfg"
  done
done 2>&1 | tee gpurun_out/codon3_bench.txt
