# consumer warps per CTA of the small-S traversal (2 CTAs per SM when K <= ~5)
for k in 9 6 5 4 3; do
  for args in "--config 1" "--config 2" "--config 1 --precision fp32"; do
    PG_SMALL_K=$k timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('K=$k', d['config']['workload'][:12], d['dtype'], d['ms_per_step'], d['kernel_ms']['traverse'], d['plan']['grid'], d['plan']['block'], d['plan']['smem_bytes'])"
  done
done
