"""Host-side checks of the C ABI library that need no GPU (-m "not gpu").

The library must load and export every symbol include/phylograd.h declares;
topology validation and traversal planning run on the host.
"""
import ctypes
import subprocess

import numpy as np
import pytest

import phylo_synth as ps


@pytest.fixture(scope="module")
def pg():
    import paper_2303_04390_b200 as m
    return m


def test_library_exports_every_header_symbol(pg):
    syms = pg.header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(pg._lib, s)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", pg.LIB_PATH], capture_output=True, text=True).stdout
    for s in syms:
        assert f" T {s}" in nm, s


def test_library_is_sm100a(pg):
    out = subprocess.run(["cuobjdump", "--list-elf", pg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_strerror(pg):
    assert pg._lib.pg_version() >= 100
    assert pg._lib.pg_strerror(pg.PG_ERR_TOPOLOGY).decode() == "invalid tree topology"


def test_plan_check_depths(pg):
    assert pg.plan_check(5, ps.tree_from_newick_fixed5().ops) == (2, 2)
    for N in (49, 62, 104, 997, 4000):
        tr = ps.coalescent_tree(N, np.random.default_rng(N), 1.0)
        post, pre = pg.plan_check(N, tr.ops)
        # Sethi-Ullman / smaller-subtree-first bounds: O(log N) stack slots
        assert 1 <= post <= np.log2(N) + 2 and 1 <= pre <= np.log2(N) + 2, (N, post, pre)
    N = 500                                  # caterpillar: constant stack
    ops = [(N, 0, 1)] + [(N + k - 1, N + k - 2, k) for k in range(2, N)]
    assert pg.plan_check(N, ops) == (1, 1)


@pytest.mark.parametrize("bad", [
    [(5, 0, 1), (6, 2, 3), (7, 5, 6), (8, 7, 4)][:3],           # too few ops
    [(5, 0, 1), (6, 2, 3), (7, 5, 6), (8, 7, 7)],               # repeated child
    [(5, 0, 1), (6, 2, 3), (7, 5, 9), (8, 7, 4)],               # child out of range
    [(5, 0, 1), (6, 2, 7), (7, 5, 3), (8, 6, 4)],               # child used before defined
    [(5, 0, 1), (6, 0, 3), (7, 5, 6), (8, 7, 4)],               # two parents
    [(5, 0, 1), (6, 2, 3), (8, 5, 6), (7, 8, 4)],               # root not last
    [(4, 0, 1), (6, 2, 3), (7, 5, 6), (8, 7, 4)],               # dest is a tip
])
def test_plan_check_rejects_bad_topologies(pg, bad):
    with pytest.raises(pg.PhyloGradError) as ei:
        pg.plan_check(5, bad)
    assert ei.value.code in (pg.PG_ERR_TOPOLOGY, pg.PG_ERR_ARG)


def test_workspace_bytes(pg):
    b = pg.workspace_bytes(997, 10000, 4, 4)
    u = (997 - 2) * 4 * 10016 * 4 * 8
    assert u < b < u * 1.1
    assert pg.workspace_bytes(997, 10000, 4, 4, "fp32") < b
    with pytest.raises(pg.PhyloGradError) as ei:
        pg.workspace_bytes(10, 10, 300, 1)
    assert ei.value.code == pg.PG_ERR_UNSUPPORTED
    # S = 122 (two-class codon MMM) pads to 128 on the large-state kernel
    b122 = pg.workspace_bytes(49, 4000, 122, 1)
    assert (49 - 2) * 4000 * 128 * 8 < b122
    for S, R, prec in ((129, 1, "fp32"), (255, 1, "fp64"), (122, 9, "fp32"), (122, 17, "fp64")):
        with pytest.raises(pg.PhyloGradError) as ei:
            pg.workspace_bytes(10, 10, S, R, prec)
        assert ei.value.code == pg.PG_ERR_UNSUPPORTED


def test_s256_workspace_fits_without_stored_transposes(pg):
    """NEXT-2: 244 states padded to 256, 10,001 tips = 20,000
    branches.  The paper keeps P and its transpose for every branch (~10 GB of
    transposes alone); this build keeps ONE matrix per (branch, category),
    W = P' (traverse_big.cuh), so the matrices take B R 256^2 8 bytes once."""
    N, C, S = 10_001, 256, 244
    B, SP = 2 * N - 2, 256
    one_copy = B * SP * SP * 8                          # 10.5 GB
    for R in (1, 2):
        ws = pg.workspace_bytes(N, C, S, R, "fp64", tip_partials=True)
        mats = R * one_copy
        # u, q (N-2 internal nodes) and u of the partial tips, [R][C][256] each
        vecs = (2 * (N - 2) + N) * R * C * SP * 8
        assert ws >= mats + vecs
        assert ws < mats + vecs + R * one_copy // 4     # no second matrix layout
        assert ws < 180e9 / 2                           # fits a B200 with room to spare



def test_shard_range_covers_patterns(pg):
    for C, w in ((10000, 8), (37, 4), (5, 2)):
        spans = [pg.shard_range(C, w, r) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == C
        assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
    # balanced: sizes differ by at most one; C < world leaves some shards empty
    for C, w in ((9, 8), (10000, 8), (3, 8), (1, 2)):
        sizes = [hi - lo for lo, hi in (pg.shard_range(C, w, r) for r in range(w))]
        assert sum(sizes) == C and max(sizes) - min(sizes) <= 1


def test_setters_check_array_sizes(pg):
    """Short or long host arrays raise before the C call (the C side reads
    fixed counts: 2N-2, C, C*S, S*S, R)."""
    import numpy as np
    sig = pg._f64
    with pytest.raises(ValueError):
        sig(np.zeros(5), 6, "x")
    with pytest.raises(ValueError):
        pg._i32(np.zeros(7), 6, "y")
    assert sig(np.zeros((2, 3)), 6, "z").shape == (2, 3)
