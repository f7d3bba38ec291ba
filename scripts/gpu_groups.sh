# small-S traversal: one producer warp per CTA (default) vs two producer groups (PG_GROUPS=2)
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x -k "dengue or mmm or small_shapes or max_categories or partials or caterpillar or deep or jc5 or determinism" > gpurun_out/gpu_tests_g1.log 2>&1; tail -1 gpurun_out/gpu_tests_g1.log
PHYLOGRAD_LIB=$PWD/paper_2303_04390_b200/lib/libphylograd_vG2.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x -k "dengue or mmm or small_shapes or max_categories or partials or caterpillar or deep or jc5 or determinism" > gpurun_out/gpu_tests_g2.log 2>&1; tail -1 gpurun_out/gpu_tests_g2.log
for rep in 1 2; do
for f in "" vG2; do
  if [ -n "$f" ]; then export PHYLOGRAD_LIB=$PWD/paper_2303_04390_b200/lib/libphylograd_$f.so; else unset PHYLOGRAD_LIB; fi
  for args in "--config 1" "--config 2" "--config 1 --precision fp32"; do
    timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${f:-default}', d['config']['workload'][:12], d['dtype'], d['ms_per_step'], d['kernel_ms']['traverse'], d['plan']['block'], d['plan']['smem_bytes'])"
  done
done
done
