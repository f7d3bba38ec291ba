set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -rf > gpurun_out/gpu_tests.log 2>&1
tail -30 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
tail -5 gpurun_out/smoke.log
timeout 600 python bench.py --steps 200 --warmup 10 --cpu-seconds 8 > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/bench.log
