#!/bin/bash
# flow v2 item traces: full yeast, yeast 8-way shard, WNV
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TRACE_SUMMARY_ONLY=1 python scripts/flow2_trace.py 3 1 > gpurun_out/trace_3_1.txt 2>&1
python scripts/flow2_trace.py 3 8 > gpurun_out/trace_3_8.txt 2>&1
TRACE_SUMMARY_ONLY=1 python scripts/flow2_trace.py 4 1 > gpurun_out/trace_4_1.txt 2>&1
head -8 gpurun_out/trace_3_1.txt gpurun_out/trace_3_8.txt gpurun_out/trace_4_1.txt
