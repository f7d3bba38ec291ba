# fp32 S = 4: three CTAs of 3 consumer warps per SM (auto) vs one CTA of 9 (PG_SMALL_K=9)
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x -k "fp32 or dengue or small_shapes or max_categories or jc5" > gpurun_out/gpu_tests_fp32k.log 2>&1; tail -1 gpurun_out/gpu_tests_fp32k.log
for rep in 1 2; do
  for k in 0 9; do
    PG_SMALL_K=$k timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --config 1 --precision fp32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PG_SMALL_K=$k', d['ms_per_step'], d['kernel_ms']['traverse'], d['plan']['grid'], d['plan']['block'], d['value'], d['roofline']['frac'])"
  done
done
timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --config 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fp64', d['ms_per_step'], d['kernel_ms']['traverse'], d['plan']['grid'], d['plan']['block'])"
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --config 1 --precision fp32 > gpurun_out/bench_fp32.json 2>/dev/null
