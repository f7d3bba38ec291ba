# round-end style evidence: tests, smoke, default bench, all configs, reference arm,
# launch lists (dengue, yeast incl. DMMA pipe + DRAM bytes, MMM) and ncu --set full
# captures of the dengue traversal and of one codon post / pre level kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -4 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -1 gpurun_out/bench_default.json
rm -f gpurun_out/bench_allcfg.jsonl
for args in "--config 1 --precision fp32" "--config 2" "--config 3" "--config 4" "--config 0"; do
  timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $args >> gpurun_out/bench_allcfg.jsonl 2>>gpurun_out/bench_allcfg.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_dengue.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 120 --csv --log-file gpurun_out/launches_yeast.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-flush --config 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_mmm.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:traverse -s 2 -c 1 -o gpurun_out/prof_trav -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codon_post -s 11 -c 1 -o gpurun_out/prof_codon_post -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-flush --config 3 > gpurun_out/ncu_codon_post.log 2>&1; tail -1 gpurun_out/ncu_codon_post.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:codon_pre -s 17 -c 1 -o gpurun_out/prof_codon_pre -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-flush --config 3 > gpurun_out/ncu_codon_pre.log 2>&1; tail -1 gpurun_out/ncu_codon_pre.log
