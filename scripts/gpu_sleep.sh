# flow-kernel dependency polling: nanosleep between acquire loads (default 40 ns) vs none / 400 ns
for f in "" vS0 vS400; do
  if [ -n "$f" ]; then export PHYLOGRAD_LIB=$PWD/paper_2303_04390_b200/lib/libphylograd_$f.so; else unset PHYLOGRAD_LIB; fi
  for args in "--config 3 --virtual-shard 8" "--config 3" "--config 4 --virtual-shard 8"; do
    timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${f:-default}', d['config']['workload'][:8], d['config']['parallelism'][:10], d['ms_per_step'], d['kernel_ms'])"
  done
done
