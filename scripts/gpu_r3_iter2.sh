#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/r3i; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "dengue or mmm or hky or jc or small or clock or hmc or nucleotide" > $O/tests.log 2>&1; echo "tests exit $?" >> $O/tests.log; tail -3 $O/tests.log
VARIANTS="base old" bash scripts/gpu_r3_ab.sh
bash scripts/gpu_r3_trace.sh 2>&1 | grep -A12 "== post\|== pre" | grep -v "3->4\|4->5\|5->6\|6->7" 
