# A/B: HEAD library vs working tree on the same box (codon configs) + codon/S=122 parity
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x -k "codon or clock or yeast or wnv or mmm122 or partials or small_shapes" > gpurun_out/gpu_tests_ab.log 2>&1; tail -2 gpurun_out/gpu_tests_ab.log
for rep in 1 2; do
for lib in paper_2303_04390_b200/lib/libphylograd_head.so paper_2303_04390_b200/lib/libphylograd.so; do
  for args in "--config 3" "--config 3 --virtual-shard 8" "--config 4"; do
    PHYLOGRAD_LIB=$PWD/$lib timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], d['config']['workload'][:8], d['config']['parallelism'][:12], d['ms_per_step'], d['kernel_ms'])"
  done
done
done
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --config 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'])"
