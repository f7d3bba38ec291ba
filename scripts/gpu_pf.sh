# small-S traversal: L2 prefetch distance (PF) and gradient window (W)
for rep in 1 2; do
for f in "" vPF4 vPF8 vPF32 vW1; do
  if [ -n "$f" ]; then export PHYLOGRAD_LIB=$PWD/paper_2303_04390_b200/lib/libphylograd_$f.so; else unset PHYLOGRAD_LIB; fi
  for args in "--config 1" "--config 1 --precision fp32" "--config 2"; do
    timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${f:-default}', d['config']['workload'][:12], d['dtype'], d['ms_per_step'], d['kernel_ms']['traverse'])"
  done
done
done
