# ring depth / ops per stage for the S = 16 (MMM) traversal
for f in "" vD8 vD8o1 vD4o1; do
  if [ -n "$f" ]; then export PHYLOGRAD_LIB=$PWD/paper_2303_04390_b200/lib/libphylograd_$f.so; else unset PHYLOGRAD_LIB; fi
  timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --config 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${f:-default}', d['ms_per_step'], d['kernel_ms'], d['plan']['smem_bytes'], d['plan']['block'], d['plan']['grid'])"
done
