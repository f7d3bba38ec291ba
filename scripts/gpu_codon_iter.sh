# codon iteration: parity tests, yeast/WNV bench, per-launch durations + DMMA pipe utilisation
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
for c in 3 4; do timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['kernel_ms'], d['roofline']['frac'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:codon -c 120 --csv --log-file gpurun_out/launches_codon3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-flush --config 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_codon3.csv
