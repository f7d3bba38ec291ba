# round-end style evidence: tests, smoke, default bench, all configs (+ 8-way
# virtual shards), reference arm, launch lists (dengue, yeast, MMM, S=122) and
# ncu --set full captures of the dengue traversal and the codon flow kernel
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
rm -f gpurun_out/bench_allcfg.jsonl
for args in "--config 1 --precision fp32" "--config 2" "--config 3" "--config 4" "--config 5" "--config 0" \
            "--config 3 --virtual-shard 8" "--config 4 --virtual-shard 8" "--config 5 --virtual-shard 8"; do
  timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $args >> gpurun_out/bench_allcfg.jsonl 2>>gpurun_out/bench_allcfg.err
done
python - <<'PY'
import json
for l in open("gpurun_out/bench_allcfg.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"], d["dtype"], d["config"]["parallelism"][:24], "evals/s", d["value"], "ms", d["ms_per_step"],
          d["roofline"]["bound"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_dengue.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 40 --csv --log-file gpurun_out/launches_yeast.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_mmm.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_s122.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 5 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse -s 2 -c 1 -o gpurun_out/prof_trav -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codon_flow -s 3 -c 1 -o gpurun_out/prof_flow -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 3 > gpurun_out/ncu_flow.log 2>&1; tail -1 gpurun_out/ncu_flow.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codon_flow -s 3 -c 1 -o gpurun_out/prof_flow_wnv -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 4 > gpurun_out/ncu_flow_wnv.log 2>&1; tail -1 gpurun_out/ncu_flow_wnv.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codon_flow -s 3 -c 1 -o gpurun_out/prof_flow_s122 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 5 > gpurun_out/ncu_flow_s122.log 2>&1; tail -1 gpurun_out/ncu_flow_s122.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codon_flow -s 3 -c 1 -o gpurun_out/prof_flow8 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 3 --virtual-shard 8 > gpurun_out/ncu_flow8.log 2>&1; tail -1 gpurun_out/ncu_flow8.log
for r in prof_trav prof_flow prof_flow_wnv prof_flow_s122 prof_flow8; do
  [ -f gpurun_out/$r.ncu-rep ] && python scripts/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.txt
done
python scripts/ncu_lines.py gpurun_out/prof_flow.ncu-rep codon_flow 60 > gpurun_out/prof_flow_lines.txt 2>&1
python scripts/ncu_lines.py gpurun_out/prof_trav.ncu-rep traverse 60 > gpurun_out/prof_trav_lines.txt 2>&1
python scripts/update_traffic.py gpurun_out > gpurun_out/traffic.json 2>&1
# keep the copy-back under 64 MiB: only the yeast flow report stays as .ncu-rep
rm -f gpurun_out/prof_flow_wnv.ncu-rep gpurun_out/prof_flow_s122.ncu-rep gpurun_out/prof_flow8.ncu-rep gpurun_out/prof_trav.ncu-rep
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
timeout 300 python scripts/hmc_bench.py 1 3 > gpurun_out/hmc_bench.jsonl 2>&1; cat gpurun_out/hmc_bench.jsonl
timeout 300 python scripts/flow_trace.py 3 8 > gpurun_out/flow_trace_yeast8.txt 2>&1
bash scripts/gpu_sweep.sh
