# phase trace of the small-S traversal (dengue, MMM) with the -DPG_TRACE library
mkdir -p gpurun_out
for c in ${TRACE_CFGS:-1 2}; do
PHYLOGRAD_LIB=$PWD/paper_2303_04390_b200/lib/libphylograd_trace.so timeout 300 python scripts/trace_dengue.py $c > gpurun_out/trace_cfg$c.log 2>&1; cat gpurun_out/trace_cfg$c.log
done
