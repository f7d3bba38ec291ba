# codon flow: half-tile post items (PG_FLOW_HALF=1) vs whole tiles
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x -k "codon_schedules or yeast_codon or wnv_codon or mmm122 or clock or hmc" > gpurun_out/gpu_tests_defer.log 2>&1; tail -2 gpurun_out/gpu_tests_defer.log
for rep in 1 2; do
for d in 0 1; do
  for args in "--config 3 --virtual-shard 8" "--config 4 --virtual-shard 8" "--config 5 --virtual-shard 8" "--config 3"; do
    PG_FLOW_HALF=$d timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('half=$d', d['config']['workload'][:10], d['config']['parallelism'][:10], d['ms_per_step'], d['kernel_ms']['traverse'])"
  done
done
done
