#!/bin/bash
set -u
cd "$(dirname "$0")/.."
for v in default s4 nopf s6 s12; do
  if [ $v = default ]; then lib=""; else lib="PHYLOGRAD_LIB=$PWD/paper_2303_04390_b200/lib/libphylograd_$v.so"; fi
  for k in 0 3; do
    if [ $k = 0 ]; then e=""; else e="PG_SMALL_K=$k"; fi
    env $lib $e timeout 300 python bench.py --config 2 --steps 300 --warmup 20 --no-cpu-baseline --no-fp64-probe > gpurun_out/b.json 2>gpurun_out/b.err
    python - "$v $e" <<'PY'
import json,sys
try:
    d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1])
    r=d['roofline']; p=d['plan']
    print(f"{sys.argv[1]:24s} {d['ms_per_step']:.4f} ms  kern {d['kernel_ms']} frac {r['frac']} grid {p['grid']} smem {p['smem_bytes']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e, open('gpurun_out/b.err').read()[-800:])
PY
  done
done 2>&1 | tee gpurun_out/mmm_var.txt
timeout 300 python -m pytest tests/test_parity_gpu.py -q -x -k "mmm" 2>&1 | tail -2
