#!/bin/bash
# phase trace of the small-S traversal: dengue full, dengue C=1184 (one warp per SM), MMM
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r3t
L=$PWD/paper_2303_04390_b200/lib/libphylograd_trace.so
PHYLOGRAD_LIB=$L timeout 300 python scripts/trace_dengue.py 1 > gpurun_out/r3t/trace_c1.log 2>&1
TRACE_C=1184 PHYLOGRAD_LIB=$L timeout 300 python scripts/trace_dengue.py 1 > gpurun_out/r3t/trace_c1_1184.log 2>&1
PHYLOGRAD_LIB=$L timeout 300 python scripts/trace_dengue.py 2 > gpurun_out/r3t/trace_c2.log 2>&1
tail -n 40 gpurun_out/r3t/*.log
