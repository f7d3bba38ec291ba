#!/usr/bin/env python
"""One evaluation of a named workload through the C ABI, checked against the
oracle; the unit compute-sanitizer runs (scripts/gpu_sanitize.sh).

    python scripts/sanitize_case.py jc5|dengue|yeast|yeast_levels|s122|mmm
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import phylo_synth as ps  # noqa: E402

CASES = {
    "jc5": lambda: ps.config0_jc5(),
    "dengue": lambda: ps.config1_dengue(N=100, C=200),
    "dengue_fp32": lambda: ps.config1_dengue(N=100, C=200, precision="fp32"),
    "mmm": lambda: ps.config2_mmm(N=30, C=100),
    "yeast": lambda: ps.config3_yeast(N=20, C=77),
    "yeast_levels": lambda: ps.config3_yeast(N=20, C=77),
    "s122": lambda: ps.config5_yeast_mmm(N=10, C=40),
    "s256": lambda: ps.small_problem(5, "codon4", R=1, C=33, seed=7, simulate=True),
    "codon_fp32": lambda: _fp32(ps.small_problem(9, "codon", R=2, C=150, seed=5, missing=0.05, simulate=True)),
}


def _fp32(pb):
    pb.precision = "fp32"
    return pb


def main():
    name = sys.argv[1]
    if name == "yeast_levels":
        os.environ["PG_CODON_FLOW"] = "0"
    import paper_2303_04390_b200 as pg
    pb = CASES[name]()
    inst = pg.from_problem(pb, precision=pb.precision)
    logl, g = inst.compute()
    logl2, g2 = inst.compute()               # a replay of the captured graph
    ref = oracle.loglik_grad(pb, threads=4)
    tol = 1e-4 if pb.precision == "fp32" else 1e-10
    el = abs(logl - ref["logL"]) / abs(ref["logL"])
    eg = float(np.max(np.abs(g - ref["grad"]) / np.maximum(np.abs(ref["grad"]), ref["grad_abs"])))
    inst.close()
    print(f"{name}: logL rel {el:.2e}, grad C17 {eg:.2e}, replay identical {logl == logl2 and np.array_equal(g, g2)}")
    assert el <= tol and eg <= tol


if __name__ == "__main__":
    main()
