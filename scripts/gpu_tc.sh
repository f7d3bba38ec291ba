#!/bin/bash
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 ./scripts/tc_probe > gpurun_out/tc_probe.log 2>&1; echo "probe exit $?" >> gpurun_out/tc_probe.log; cat gpurun_out/tc_probe.log
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "fp32 or codon_fp32" > gpurun_out/tc_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tc_tests.log; tail -15 gpurun_out/tc_tests.log
timeout 300 python - <<'PY' > gpurun_out/tc_small.log 2>&1
import numpy as np, oracle, phylo_synth as ps, paper_2303_04390_b200 as pg
for N, R, C in ((3, 1, 5), (5, 1, 130), (9, 2, 200), (20, 4, 300)):
    pb = ps.small_problem(N, "codon", R=R, C=C, seed=N + C, missing=0.1, simulate=True)
    pb.precision = "fp32"
    inst = pg.from_problem(pb, precision="fp32")
    info = inst.plan_info()
    l, g = inst.compute()
    ref = oracle.loglik_grad(pb, threads=4)
    el = abs(l - ref["logL"]) / abs(ref["logL"])
    eg = float(np.max(np.abs(g - ref["grad"]) / np.maximum(np.abs(ref["grad"]), ref["grad_abs"])))
    print(N, R, C, "variant", info["kernel_variant"], "logL", l, ref["logL"], "el %.2e eg %.2e" % (el, eg))
PY
cat gpurun_out/tc_small.log | tail -8
