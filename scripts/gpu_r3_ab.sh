#!/bin/bash
# A/B of library variants (paper_2303_04390_b200/lib/libphylograd_<v>.so): bench lines per config
# CFGS: ';'-separated bench argument sets (default "--config 1;--config 2")
cd "$(dirname "$0")/.."
O=gpurun_out/r3ab; mkdir -p $O
IFS=';' read -ra CF <<< "${CFGS:---config 1;--config 2}"
for v in ${VARIANTS:-base}; do
  L=$PWD/paper_2303_04390_b200/lib/libphylograd_$v.so; [ "$v" = base ] && L=$PWD/paper_2303_04390_b200/lib/libphylograd.so
  i=0
  for cfg in "${CF[@]}"; do
    i=$((i+1))
    PHYLOGRAD_LIB=$L timeout 300 python bench.py $cfg --steps ${STEPS:-300} --warmup 20 --no-cpu-baseline --no-fp64-probe --no-extra-configs > $O/b_${v}_$i.json 2>$O/b_${v}_$i.err
    python - $O/b_${v}_$i "$v" "$cfg" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]+'.json').read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:8s} {sys.argv[3]:30s} ms {d['ms_per_step']:.4f} p50 {d['ms_step_p10_p50_p90'][1]:.4f} kern {d['kernel_ms']} frac {d['roofline']['frac']} smem {d.get('plan',{}).get('smem_bytes')} grid {d.get('plan',{}).get('grid')}")
except Exception as e:
    print(sys.argv[2], sys.argv[3], 'FAILED', e, open(sys.argv[1]+'.err').read()[-1500:])
PY
  done
done
