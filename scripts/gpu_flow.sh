# codon schedule comparison: level kernels vs the one-launch flow kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -x > gpurun_out/gpu_tests.log 2>&1; tail -4 gpurun_out/gpu_tests.log
rm -f gpurun_out/flow.jsonl
run() { timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline "$@" >> gpurun_out/flow.jsonl 2>>gpurun_out/flow.err; }
for cfg in 3 4; do
  PG_CODON_FLOW=0 run --config $cfg
  for t in ${TCHS:-1 2 4}; do PG_FLOW_TCH=$t run --config $cfg; done
  PG_CODON_FLOW=0 run --config $cfg --virtual-shard 8
  for t in 1 2; do PG_FLOW_TCH=$t run --config $cfg --virtual-shard 8; done
done
python - <<'PY'
import json
for l in open("gpurun_out/flow.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"], d["config"]["parallelism"][:30], "tch", d["plan"].get("flow_tiles"), "ms", d["ms_per_step"],
          "trav", d["kernel_ms"]["traverse"], "frac", d["roofline"]["frac"])
PY
tail -5 gpurun_out/flow.err
