#!/bin/bash
# end-of-round evidence: GPU tests (+ parity log), smoke, default bench, ncu
# launch lists, ncu --set full of the top kernels, compute-sanitizer
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/r2f; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
PG_PARITY_LOG=$O/parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -rf > $O/gpu_tests.log 2>&1
echo "tests exit $?" >> $O/gpu_tests.log; tail -3 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench exit $?" >> $O/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file $O/launches_dengue.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-fp64-probe --no-extra-configs > /dev/null 2>&1
for cfg in 2 3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 60 --csv --log-file $O/launches_c$cfg.csv python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-fp64-probe > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 60 --csv --log-file $O/launches_c3_shard8.csv python bench.py --config 3 --virtual-shard 8 --steps 20 --warmup 3 --no-cpu-baseline --no-fp64-probe > /dev/null 2>&1
CFGS="1 2" bash scripts/gpu_ncu_small.sh > $O/ncu_small.out 2>&1
bash scripts/gpu_ncu_flow.sh > $O/ncu_flow.out 2>&1
cp gpurun_out/ncu_small_c*.txt gpurun_out/ncu_small_c*_lines.txt gpurun_out/ncu_flow_yeast*.txt $O/ 2>/dev/null
python scripts/ncu_lines.py gpurun_out/prof_flow.ncu-rep codon_flow 60 > $O/ncu_flow_yeast_lines.txt 2>/dev/null
rm -rf gpurun_out/sanitize; bash scripts/gpu_sanitize.sh > $O/sanitize.out 2>&1; cp -r gpurun_out/sanitize $O/
rm -f gpurun_out/*.ncu-rep
echo done
