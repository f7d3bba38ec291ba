mkdir -p gpurun_out
timeout 300 python scripts/flow_trace.py 3 8 > gpurun_out/flow_trace_yeast8.txt 2>&1; head -8 gpurun_out/flow_trace_yeast8.txt
timeout 300 python scripts/flow_trace.py 3 1 > gpurun_out/flow_trace_yeast1.txt 2>&1; head -4 gpurun_out/flow_trace_yeast1.txt
bash scripts/gpu_sweep.sh
