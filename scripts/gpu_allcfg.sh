mkdir -p gpurun_out
for args in "--config 1 --precision fp32" "--config 2" "--config 3" "--config 4" "--config 0"; do
  echo "== $args"
  timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline $args 2>>gpurun_out/allcfg.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['dtype'], 'value', d['value'], 'ms', d['ms_per_step'], 'kernels', d['kernel_ms'], 'frac', d['roofline']['frac'], d.get('roofline_alu'), d['plan'])"
done
