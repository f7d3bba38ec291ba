mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -x -k "codon or clock or yeast or wnv or determinism or device_path or virtual" > gpurun_out/gpu_tests_codon.log 2>&1; tail -2 gpurun_out/gpu_tests_codon.log
for pm in 1 0; do
for args in "--config 3" "--config 4" "--config 3 --virtual-shard 8" "--config 4 --virtual-shard 8"; do
  PG_FLOW_PMAT=$pm timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pmat-fold', $pm, d['config']['workload'], d['config']['parallelism'][:20], d['ms_per_step'], d['kernel_ms'], d['roofline']['frac'])"
done
done
