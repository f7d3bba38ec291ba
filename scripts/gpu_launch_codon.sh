mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none -s 30 -c 26 --csv --log-file gpurun_out/launches_codon2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-flush --config 3 > /dev/null 2>&1
