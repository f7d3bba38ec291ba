# ncu --set full of the codon flow kernel (one evaluation): full yeast and an 8-way shard
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codon_flow -s 3 -c 1 -o gpurun_out/prof_flow -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fp64-probe --no-flush --config 3 > gpurun_out/ncu_flow.log 2>&1; tail -1 gpurun_out/ncu_flow.log
python scripts/ncu_summary.py gpurun_out/prof_flow.ncu-rep > gpurun_out/ncu_flow_yeast.txt; cat gpurun_out/ncu_flow_yeast.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codon_flow -s 3 -c 1 -o gpurun_out/prof_flow8 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fp64-probe --no-flush --config 3 --virtual-shard 8 > gpurun_out/ncu_flow8.log 2>&1; tail -1 gpurun_out/ncu_flow8.log
python scripts/ncu_summary.py gpurun_out/prof_flow8.ncu-rep > gpurun_out/ncu_flow_yeast8.txt; cat gpurun_out/ncu_flow_yeast8.txt
