mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codon_pre -s 5 -c 1 -o gpurun_out/prof_pre -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 3 > gpurun_out/ncu_pre.log 2>&1; tail -2 gpurun_out/ncu_pre.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codon_post -s 0 -c 1 -o gpurun_out/prof_post -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 3 > gpurun_out/ncu_post.log 2>&1; tail -2 gpurun_out/ncu_post.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_codon.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-flush --config 3 > /dev/null 2>&1
