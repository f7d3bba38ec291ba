# session-3 re-verification of HEAD: gpu tests, smoke, default bench, all configs
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cp MEASURED_PEAKS.json gpurun_out/ 2>/dev/null
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -rf > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json | cut -c1-300
rm -f gpurun_out/bench_allcfg.jsonl
for args in "--config 1 --precision fp32" "--config 2" "--config 3" "--config 4" "--config 0" "--config 3 --virtual-shard 8" "--config 4 --virtual-shard 8"; do
  timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $args >> gpurun_out/bench_allcfg.jsonl 2>>gpurun_out/bench_allcfg.err
done
python - <<'PY'
import json
for l in open("gpurun_out/bench_allcfg.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"], d["dtype"], d["config"].get("parallelism","")[:30], "v", d["value"], "ms", d["ms_per_step"], "frac", d["roofline"]["frac"], d.get("roofline_alu",{}).get("frac"))
PY
