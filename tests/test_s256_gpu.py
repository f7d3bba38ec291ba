"""NEXT-2, the S = 256 class: 129..254 states padded to 256 on
the transpose-free level kernels (traverse_big.cuh), checked against the CPU
oracle (pytest -m gpu).

The model is the paper's Markov-modulated codon family widened to four rate
classes (4 x 61 = 244 states); tips are observed codons (state tips) or the
0/1 masks on the 4 hidden copies of the observed codon.  At the full size of
config 6 (10,001 tips, 20,000 branches) the oracle is far too slow (its
20,000 transition matrices alone are ~10^12 flops), so that instance is
checked through properties that hold at any size: the Euler identity
sum_i b_i g_i = d/dalpha logL(alpha b) (central difference of the CUDA
path's own logL), the pulley principle (the two root branches of a
reversible model with stationary root carry equal gradients), and finite
results; the oracle covers the same kernels on smaller trees.
"""
import numpy as np
import pytest

import oracle
import phylo_synth as ps

pytestmark = pytest.mark.gpu


def _cmp(pb, tol=1e-10):
    import paper_2303_04390_b200 as pg
    inst = pg.from_problem(pb)
    assert inst.plan_info()["kernel_variant"] == 3
    logl, g = inst.compute()
    inst.close()
    ref = oracle.loglik_grad(pb, threads=8)
    el = abs(logl - ref["logL"]) / abs(ref["logL"])
    scale = np.maximum(np.abs(ref["grad"]), ref["grad_abs"])
    eg = float(np.max(np.abs(g - ref["grad"]) / np.where(scale > 0, scale, 1.0)))
    import json
    import os
    path = os.environ.get("PG_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": "s256", "problem": pb.name, "precision": "fp64", "N": pb.n_tips, "C": pb.patterns,
                       "S": pb.states, "R": len(pb.cat_rates), "logl_rel_err": el, "grad_c17_err": eg,
                       "grad_plain_rel_err_max": eg, "tol": tol, "headroom": tol / max(el, eg, 1e-300),
                       "reference": "fp64 oracle"}) + "\n")
    assert el <= tol and eg <= tol, (pb.name, el, eg)


@pytest.mark.parametrize("N,R,C,missing", [(3, 1, 5, 0.1), (5, 2, 33, 0.1), (9, 1, 40, 0.0), (12, 4, 20, 0.05)])
def test_s256_state_tips(N, R, C, missing):
    pb = ps.small_problem(N, "codon4", R=R, C=C, seed=N + C, missing=missing, simulate=True)
    _cmp(pb)


@pytest.mark.parametrize("N,R,C", [(4, 1, 9), (10, 2, 37)])
def test_s256_hidden_class_masks(N, R, C):
    pb = ps.small_problem(N, "codon4", R=R, C=C, seed=3 * N, simulate=True, hidden_masks=4)
    _cmp(pb)


def test_s256_config6_reduced():
    """Config 6's generator at a reduced tree (several tiles, ragged tail)."""
    pb = ps.config6_codon_mmm4(N=60, C=70)
    _cmp(pb)


@pytest.mark.slow
def test_s256_config6_full_size_properties():
    """10,001 tips (20,000 branch lengths), 256 patterns, S = 244 -> 256."""
    import paper_2303_04390_b200 as pg
    pb = ps.config6_codon_mmm4()
    inst = pg.from_problem(pb)
    info = inst.plan_info()
    assert info["kernel_variant"] == 3
    logl, g = inst.compute()
    assert np.isfinite(logl) and np.all(np.isfinite(g))
    b = pb.branch_lengths.copy()
    # Euler identity (SURVEY §8(c) pins): d/dalpha logL(alpha b) at alpha = 1
    h = 1e-5
    vals = []
    for a in (1 + h, 1 - h):
        inst.set_branch_lengths(b * a)
        vals.append(inst.compute()[0])
    fd = (vals[0] - vals[1]) / (2 * h)
    euler = float(np.dot(b, g))
    assert abs(fd - euler) <= 1e-6 * max(abs(euler), np.sum(np.abs(b * g))), (fd, euler)
    # pulley principle: equal gradients on the two root branches
    d, ca, cb = pb.ops[-1]
    assert abs(g[ca] - g[cb]) <= 1e-8 * max(abs(g[ca]), 1.0), (g[ca], g[cb])
    inst.close()
