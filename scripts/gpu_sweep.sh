# pattern-count sweep (the Figure 6 analogue): evals/s
# and patterns/s against C for the yeast codon and dengue nucleotide workloads
mkdir -p gpurun_out
rm -f gpurun_out/pattern_sweep.jsonl
for C in 32 128 512 1024 2048 4000 8192 22151; do
  timeout 300 python bench.py --config 3 --patterns $C --steps 100 --warmup 10 --no-cpu-baseline >> gpurun_out/pattern_sweep.jsonl 2>>gpurun_out/sweep.err
done
for C in 128 1024 4096 10000 20000; do
  timeout 300 python bench.py --config 1 --patterns $C --steps 100 --warmup 10 --no-cpu-baseline >> gpurun_out/pattern_sweep.jsonl 2>>gpurun_out/sweep.err
done
python - <<'PY'
import json
for l in open("gpurun_out/pattern_sweep.jsonl"):
    d = json.loads(l)
    C = d["config"]["patterns"]
    print(d["config"]["workload"], C, "evals/s", d["value"], "ms", d["ms_per_step"], "patterns/s %.3g" % (d["value"] * C),
          "frac", d["roofline"]["frac"])
PY
tail -3 gpurun_out/sweep.err
