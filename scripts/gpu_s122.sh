mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x -k "mmm122 or codon2" > gpurun_out/gpu_tests_s122.log 2>&1; tail -3 gpurun_out/gpu_tests_s122.log
for args in "--config 5" "--config 5 --precision fp32" "--config 5 --virtual-shard 8"; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline $args 2>gpurun_out/s122.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['dtype'], d['config']['parallelism'][:20], d['ms_per_step'], d['kernel_ms'], d['roofline'])"
done
tail -3 gpurun_out/s122.err
