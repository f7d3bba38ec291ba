mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x -k "codon or clock or yeast or wnv or mmm122 or determinism or device_path or virtual or small_shapes or partials" > gpurun_out/gpu_tests_s128.log 2>&1; tail -3 gpurun_out/gpu_tests_s128.log
for args in "--config 3" "--config 5" "--config 5 --virtual-shard 8" "--config 3 --virtual-shard 8"; do
  timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline $args 2>gpurun_out/s128.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['dtype'], d['config']['parallelism'][:20], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'], d['roofline']['bound'])"
done
tail -3 gpurun_out/s128.err
