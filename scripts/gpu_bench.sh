mkdir -p gpurun_out
set -x
timeout 900 python bench.py --steps 500 --warmup 20 --cpu-seconds 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-flush > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse -s 2 -c 1 -o gpurun_out/prof_trav python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
