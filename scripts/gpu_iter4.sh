mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x -k "codon or clock or yeast or wnv or mmm or hmc or determinism or partials" > gpurun_out/gpu_tests_i4.log 2>&1; tail -2 gpurun_out/gpu_tests_i4.log
for args in "--config 3 --virtual-shard 8" "--config 3" "--config 4 --virtual-shard 8" "--config 5"; do
  timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:12], d['config']['parallelism'][:10], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'])"
done
