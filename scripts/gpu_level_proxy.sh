#!/bin/bash
# level-batched control (lower-bound proxy) for the dengue traversal design
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/level_proxy scripts/level_proxy.cu
python scripts/level_proxy_prep.py gpurun_out/level_proxy_dengue.bin
for i in 1 2 3; do ./gpurun_out/level_proxy gpurun_out/level_proxy_dengue.bin; done | tee gpurun_out/level_proxy.jsonl
rm -f gpurun_out/level_proxy gpurun_out/level_proxy_dengue.bin
