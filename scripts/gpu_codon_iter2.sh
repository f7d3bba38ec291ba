mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -x -k "codon or clock or yeast or wnv or config3 or config4" > gpurun_out/gpu_tests_codon.log 2>&1; tail -2 gpurun_out/gpu_tests_codon.log
timeout 300 python scripts/flow_trace.py 3 8 > gpurun_out/flow_trace_yeast8.txt 2>&1; head -5 gpurun_out/flow_trace_yeast8.txt | grep -v Warn
for args in "--config 3" "--config 4" "--config 3 --virtual-shard 8" "--config 4 --virtual-shard 8"; do
  timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['config']['parallelism'][:20], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'])"
done
