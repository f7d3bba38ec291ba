mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -x > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
for args in "--config 3" "--config 4"; do
  echo "== $args"
  timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline $args 2>>gpurun_out/allcfg.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['dtype'], 'value', d['value'], 'ms', d['ms_per_step'], 'kernels', d['kernel_ms'], d.get('roofline_alu'), d['gpu_launches'])"
done
