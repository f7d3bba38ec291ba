#!/bin/bash
# phase trace of the small-S traversal (trace build): dengue full, MMM
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r3t
L=$PWD/paper_2303_04390_b200/lib/libphylograd_trace.so
for c in ${TRACE_CFGS:-1 2}; do
PHYLOGRAD_LIB=$L timeout 300 python scripts/trace_dengue.py $c > gpurun_out/r3t/trace_c$c.log 2>&1
done
tail -n 50 gpurun_out/r3t/*.log
