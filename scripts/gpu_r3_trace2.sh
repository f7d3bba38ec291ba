#!/bin/bash
# producer phase trace: bulk-copy vs cp.async producer, one warp per CTA (C = 1184) and full dengue
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r3t
for v in ${TV:-trace trace_bulk}; do
  L=$PWD/paper_2303_04390_b200/lib/libphylograd_$v.so
  for C in 1184 10000; do
    echo "=== $v C=$C"
    TRACE_C=$C PHYLOGRAD_LIB=$L timeout 300 python scripts/trace_dengue.py 1 2>&1 
  done
done
