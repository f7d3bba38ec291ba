# quick iteration: parity tests, bench, one ncu --set full capture of the traversal kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -x > gpurun_out/gpu_tests.log 2>&1; tail -4 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 300 --warmup 10 --cpu-seconds 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse -s 2 -c 1 -o gpurun_out/prof_trav -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush ${BENCH_ARGS} > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
fi
