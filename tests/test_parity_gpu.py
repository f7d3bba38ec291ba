"""CUDA path vs the CPU oracle, through the C ABI (pytest -m gpu).

Metric: logL relative error; every gradient
entry |g - g*| <= tol * max(|g*|, sum_c w_c |d*_c|) where the second term is
the oracle's condition scale (gradient entries are sums of mixed-sign
per-pattern terms).  tol = 1e-10 in fp64, 1e-4 in fp32 (BJ:north_star).
"""
import json
import os

import numpy as np
import pytest

import oracle
import phylo_synth as ps

pytestmark = pytest.mark.gpu


def record_parity(rec: dict):
    """Parity headroom record: with PG_PARITY_LOG=<file>, every comparison
    appends its maximum errors (scripts/parity_summary.py -> profiles/)."""
    path = os.environ.get("PG_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def _pg():
    import paper_2303_04390_b200 as pg
    return pg


def _compare(pb, precision="fp64", tol=None, threads=8, inst=None):
    pg = _pg()
    tol = tol or (1e-10 if precision == "fp64" else 1e-4)
    own = inst is None
    inst = inst or pg.from_problem(pb, precision=precision)
    logl, g = inst.compute()
    ref = oracle.loglik_grad(pb, threads=threads)
    el = abs(logl - ref["logL"]) / abs(ref["logL"])
    scale = np.maximum(np.abs(ref["grad"]), ref["grad_abs"])
    eg = np.abs(g - ref["grad"]) / np.where(scale > 0, scale, 1.0)
    record_parity({"test": os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0], "problem": pb.name,
                   "precision": precision, "N": pb.n_tips, "C": pb.patterns, "S": pb.states,
                   "R": len(pb.cat_rates), "logl_rel_err": el, "grad_c17_err": float(eg.max()),
                   "grad_plain_rel_err_max": float(np.max(np.abs(g - ref["grad"]) /
                                                          np.maximum(np.abs(ref["grad"]), 1e-300))),
                   "tol": tol, "headroom": tol / max(el, float(eg.max()), 1e-300), "reference": "fp64 oracle"})
    assert el <= tol, f"{pb.name} {precision}: logL {logl!r} vs {ref['logL']!r} (rel {el:.3e})"
    bad = np.argmax(eg)
    assert eg.max() <= tol, (f"{pb.name} {precision}: grad[{bad}] {g[bad]!r} vs {ref['grad'][bad]!r} "
                             f"(C17 err {eg.max():.3e})")
    if own:
        inst.close()
    return logl, g, ref


# --------------------------------------------------------------- configs ----

def test_config0_jc5_fp64():
    _compare(ps.config0_jc5())


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_dengue_reduced(precision):
    # several 32-pattern tiles plus a ragged tail, 1% gaps, Gamma-4
    _compare(ps.config1_dengue(N=150, C=333), precision)


@pytest.mark.parametrize("K,R", [(4, 1), (3, 1), (4, 4), (2, 2)])
def test_mmm_reduced(K, R):
    _compare(ps.config2_mmm(N=30, C=201, K=K, R=R))


def test_mmm_reduced_fp32():
    _compare(ps.config2_mmm(N=30, C=201), "fp32")


def test_yeast_codon_reduced():
    _compare(ps.config3_yeast(N=20, C=77))


def test_wnv_codon_reduced():
    _compare(ps.config4_wnv(N=30, C=45))


def test_codon_fp32_reduced():
    _compare(ps.config3_yeast(N=16, C=50, precision="fp32"), "fp32")


@pytest.mark.parametrize("N,R,C,missing,stationary", [(3, 1, 5, 0.1, True), (5, 1, 130, 0.1, True),
                                                      (9, 2, 200, 0.0, False), (20, 4, 300, 0.05, True),
                                                      (40, 3, 257, 0.02, False)])
def test_codon_fp32_tensor_core_shapes(N, R, C, missing, stationary):
    """fp32 codon on tcgen05 (kind::tf32, 3xTF32; kernel variant 4): ragged
    128-pattern tiles, missing data, several categories, non-stationary root."""
    pb = ps.small_problem(N, "codon", R=R, C=C, seed=N + C, missing=missing, simulate=True,
                          stationary_root=stationary)
    pb.precision = "fp32"
    inst = _pg().from_problem(pb, precision="fp32")
    assert inst.plan_info()["kernel_variant"] == 4
    _compare(pb, "fp32", inst=inst)
    inst.close()


@pytest.mark.slow
def test_codon_fp32_full():
    """BJ:configs[3] in fp32 at full size on the tcgen05 path, 1e-4 (BJ:north_star)."""
    _compare(ps.config3_yeast(precision="fp32"), "fp32", threads=16)


@pytest.mark.slow
def test_wnv_fp32_full():
    _compare(ps.config4_wnv(precision="fp32"), "fp32", threads=16)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_codon_mmm122_reduced(precision):
    # NEXT-2: two-class codon MMM, S = 122 padded to 128, tip partials
    _compare(ps.config5_yeast_mmm(N=12, C=45, precision=precision), precision)


@pytest.mark.slow
def test_dengue_full_fp64():
    """BJ:configs[1] at full size in the bench launch configuration."""
    _compare(ps.config1_dengue(), "fp64", threads=16)


@pytest.mark.slow
def test_dengue_full_fp32():
    _compare(ps.config1_dengue(precision="fp32"), "fp32", threads=16)


@pytest.mark.slow
def test_mmm_full():
    _compare(ps.config2_mmm(), threads=16)


@pytest.mark.slow
def test_yeast_full():
    _compare(ps.config3_yeast(), threads=16)


@pytest.mark.slow
def test_codon_mmm122_full():
    _compare(ps.config5_yeast_mmm(), threads=16)


@pytest.mark.slow
def test_wnv_full():
    _compare(ps.config4_wnv(), threads=16)


# ------------------------------------------------------------ edge cases ----

@pytest.mark.parametrize("model,N,R,C", [("jc", 2, 1, 1), ("hky", 3, 4, 31), ("gtr", 17, 3, 33),
                                         ("hky", 64, 2, 95), ("mmm2", 9, 3, 40), ("mmm4", 12, 2, 64),
                                         ("codon", 5, 1, 9), ("codon", 9, 4, 20), ("codon2", 7, 2, 33),
                                         ("codon2", 5, 8, 9)])
def test_small_shapes(model, N, R, C):
    pb = ps.small_problem(N, model, R=R, C=C, seed=N + C, missing=0.1, simulate=True)
    _compare(pb)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("seed", range(6))
def test_nucleotide_staging_shapes(seed, precision):
    """Randomised nucleotide shapes through the grouped post-order staging
    (per-step records, tip-code streams): tree sizes that are not multiples
    of the 8-step group, 1-16 categories (category pads with and without the
    P 1 column), several tiles per CTA and partial last CTAs."""
    rng = np.random.default_rng(100 + seed)
    N = int(rng.integers(2, 300))
    R = int(rng.choice([1, 2, 3, 4, 5, 8, 16]))
    C = int(rng.integers(1, 4000))
    pb = ps.small_problem(N, str(rng.choice(["jc", "hky", "gtr"])), R=R, C=C, seed=seed,
                          missing=float(rng.uniform(0, 0.3)), simulate=True)
    _compare(pb, precision=precision)


def test_large_tree_programs_not_staged():
    """A tree whose two traversal programs do not fit in shared memory beside
    the ring and stacks (4,000 tips: 128 KB of ops): the producer reads ops
    from global memory; grouped post-order staging still on."""
    pb = ps.small_problem(4000, "hky", R=4, C=600, seed=9, missing=0.05, simulate=True)
    # floor the coalescent's shortest branches (3.5e-6 here): on those the
    # literal fp64 Eq. 1 of the oracle is 2e-10 from exact while the CUDA
    # path's identity-split A1 is 2e-13 (measured against oracle/extended.py;
    # DESIGN.md R15b)
    pb.branch_lengths[:] = np.maximum(pb.branch_lengths, 1e-3)
    _compare(pb)


@pytest.mark.parametrize("model,R", [("mmm4", 8), ("mmm2", 16), ("hky", 16)])
def test_max_categories(model, R):
    # lane maps at their limits: S = 16 with 8 categories (4 lanes per vector x 8
    # categories = one pattern per warp), S = 8 / 4 with 16 categories
    pb = ps.small_problem(21, model, R=R, C=45, seed=R, missing=0.1, simulate=True)
    _compare(pb)


@pytest.mark.parametrize("model", ["hky", "mmm4", "codon"])
def test_tip_partials_nonstationary_root(model):
    pb = ps.small_problem(10, model, R=2, C=37, seed=5, partial_tips=True, stationary_root=False,
                          simulate=True)
    _compare(pb)


def test_caterpillar_tree():
    pb = ps.small_problem(60, "hky", R=4, C=50, seed=3, simulate=True)
    N = pb.n_tips
    ops, prev = [], 0
    for k in range(1, N):
        d = N + k - 1
        ops.append((d, prev, k))
        prev = d
    pb.ops = np.array(ops, np.int32)
    pb.branch_lengths = np.random.default_rng(0).uniform(0.01, 0.1, 2 * N - 2)
    _compare(pb)


def test_zero_branch_lengths_and_unrooted_convention():
    pb = ps.small_problem(12, "gtr", R=2, C=40, seed=9, simulate=True)
    d, a, b = pb.ops[-1]
    pb.branch_lengths[a] = 0.0          # unrooted tree as a zero root branch
    pb.branch_lengths[3] = 0.0
    _compare(pb)


def test_zero_weights_and_all_missing_patterns():
    pb = ps.small_problem(15, "hky", R=4, C=70, seed=4, simulate=True)
    pb.pattern_weights[::3] = 0.0
    pb.tip_states[:, 5] = pb.states
    _compare(pb)


def test_deep_tree_needs_rescaling():
    """Without rescaling these partials underflow double (logL < -745/pattern)."""
    pb = ps.small_problem(300, "mmm4", R=1, C=40, seed=2, root_height=3.0, simulate=True)
    _compare(pb)


def test_zero_likelihood_reports_pattern():
    pg = _pg()
    pb = ps.small_problem(6, "hky", R=1, C=40, seed=1)
    pb.branch_lengths[:] = 0.0
    pb.tip_states[:, :] = 0
    pb.tip_states[2, 33] = 1                      # impossible with P(0) = I
    inst = pg.from_problem(pb)
    with pytest.raises(pg.PhyloGradError) as ei:
        inst.compute()
    assert ei.value.code == pg.PG_ERR_ZERO_LIKELIHOOD
    assert "33" in str(ei.value)
    assert inst.check_status() == 33


# --------------------------------------------------- boundary behaviour ----

def test_branch_lengths_update_between_computes_and_determinism():
    pg = _pg()
    pb = ps.config1_dengue(N=80, C=200)
    inst = pg.from_problem(pb)
    l1, g1 = inst.compute()
    l1b, g1b = inst.compute()
    assert l1 == l1b and np.array_equal(g1, g1b)      # bitwise reproducible (no atomics)
    rng = np.random.default_rng(0)
    for _ in range(3):
        pb.branch_lengths = pb.branch_lengths * rng.uniform(0.9, 1.1, pb.branch_lengths.shape)
        inst.set_branch_lengths(pb.branch_lengths)
        _compare(pb, inst=inst)
    inst.close()


def test_device_path_matches_host_path():
    pg = _pg()
    import torch
    pb = ps.config1_dengue(N=60, C=150)
    inst = pg.from_problem(pb)
    logl, g = inst.compute()
    out = torch.zeros(2 * pb.n_tips - 1, dtype=torch.float64, device="cuda")
    bl = torch.tensor(pb.branch_lengths, dtype=torch.float64, device="cuda")
    with torch.cuda.stream(inst.stream):
        inst.set_branch_lengths_device(bl)
        inst.compute_device(out)
    inst.stream.synchronize()
    o = out.cpu().numpy()
    assert o[0] == logl and np.array_equal(o[1:], g)
    assert inst.check_status() == -1


def test_sequencing_errors_and_replanning():
    pg = _pg()
    pb = ps.small_problem(8, "hky", R=2, C=20, seed=1, simulate=True)
    inst = pg.Instance(pb.n_tips, pb.patterns, 4, 2)
    with pytest.raises(pg.PhyloGradError) as ei:
        inst.compute()
    assert ei.value.code == pg.PG_ERR_SEQUENCE
    inst.close()
    inst = pg.from_problem(pb)
    _compare(pb, inst=inst)
    # a different topology on the same instance re-plans and re-captures
    pb2 = ps.small_problem(8, "hky", R=2, C=20, seed=77, simulate=True)
    pb2.tip_states, pb2.pattern_weights = pb.tip_states, pb.pattern_weights
    pb2.evec, pb2.ievec, pb2.evals, pb2.Q, pb2.pi = pb.evec, pb.ievec, pb.evals, pb.Q, pb.pi
    pb2.cat_rates, pb2.cat_weights = pb.cat_rates, pb.cat_weights
    inst.set_operations(pb2.ops)
    inst.set_branch_lengths(pb2.branch_lengths)
    _compare(pb2, inst=inst)
    with pytest.raises(pg.PhyloGradError) as ei:
        inst.set_branch_lengths(-np.ones(14))
    assert ei.value.code == pg.PG_ERR_DOMAIN
    inst.close()


@pytest.mark.parametrize("gpost", ["1", "0"])
def test_tip_updates_between_computes(gpost, monkeypatch):
    """New tip states after an evaluation reach the next one: the grouped
    post-order staging (PG_GPOST=1, S = 4) rebuilds its per-CTA tip-code
    streams; several CTAs of K > 1 tiles and a partial last CTA."""
    monkeypatch.setenv("PG_GPOST", gpost)
    pg = _pg()
    pb = ps.small_problem(60, "hky", R=4, C=3000, seed=11, missing=0.05, simulate=True)
    inst = pg.from_problem(pb)
    _compare(pb, inst=inst)
    rng = np.random.default_rng(3)
    for t in rng.choice(pb.n_tips, 7, replace=False):
        pb.tip_states[t] = rng.integers(0, 5, size=pb.patterns)   # code 4 = missing
        inst.set_tip_states(int(t), pb.tip_states[t])
    _compare(pb, inst=inst)
    inst.close()


def test_caller_owned_stream_and_virtual_sharding():
    """T3(a): g instances over disjoint pattern shards on one GPU, summed,
    equal the unsharded evaluation (the multi-GPU maths without g GPUs)."""
    pg = _pg()
    pb = ps.config1_dengue(N=100, C=500)
    full = pg.from_problem(pb)
    l0, g0 = full.compute()
    lt, gt = 0.0, np.zeros_like(g0)
    for rank in range(4):
        lo, hi = pg.shard_range(pb.patterns, 4, rank)
        inst = pg.from_problem(pb, lo=lo, hi=hi)
        l, g = inst.compute()
        lt += l
        gt += g
        inst.close()
    assert abs(lt - l0) <= 1e-13 * abs(l0)
    ref = oracle.loglik_grad(pb, threads=8)
    assert np.max(np.abs(gt - g0) / ref["grad_abs"]) < 1e-13


# ------------------------------------------- time-tree parameterisation ----

def _clock_ref(pb, model):
    """The fp64 oracle (R15b: A1's identity-split form keeps the
    CUDA codon path closer to the exact result than the oracle itself)."""
    return oracle.loglik_grad(pb, threads=4)


@pytest.mark.parametrize("model,N,R,C", [("hky", 40, 4, 75), ("mmm4", 20, 1, 40), ("codon", 14, 2, 37)])
def test_clock_gradient_parity(model, N, R, C):
    """b = rho (h_parent - h) formed on the device, and dlogL/drho, dlogL/dh
    and branch-set sums (include/phylograd.h) vs the oracle's chain rule on
    the oracle's g; C17-style scale: sums of |terms| with sum_c w_c |d_c|."""
    pg = _pg()
    import torch
    pb = ps.small_problem(N, model, R=R, C=C, seed=N + C)
    rng = np.random.default_rng(N)
    h = np.zeros(2 * N - 1)
    h[2 * N - 2] = 0.8
    for d, a, b in pb.ops[::-1]:
        for c in (a, b):
            h[c] = h[d] * rng.uniform(0.3, 0.95)
    rho = rng.lognormal(0.0, 0.3, size=2 * N - 2)
    sets = rng.integers(-1, 4, size=2 * N - 2)
    pb.branch_lengths[:] = oracle.clock_branch_lengths(N, pb.ops, h, rho)
    ref = _clock_ref(pb, model)
    cref = oracle.clock_gradient(N, pb.ops, h, rho, (ref["grad"], ref["grad_abs"]), sets, 4)
    inst = pg.from_problem(pb)
    inst.set_branch_lengths(np.full(2 * N - 2, 0.123))       # replaced by the heights below
    inst.set_node_heights(h, rho)
    inst.set_branch_sets(sets, 4)
    logl, g, gr, gh, ss = inst.clock_gradient(n_sets=4)
    assert abs(logl - ref["logL"]) <= 1e-10 * abs(ref["logL"])
    for got, key, akey in ((gr, "grad_rates", "abs_rates"), (gh, "grad_heights", "abs_heights"),
                           (ss, "set_sums", "abs_sets")):
        scale = np.maximum(np.abs(cref[key]), cref[akey])
        err = np.abs(got - cref[key]) / np.where(scale > 0, scale, 1.0)
        assert err.max() <= 1e-10, (key, int(np.argmax(err)), err.max())
    # device-pointer path (rates NULL = all 1) and host path agree
    dev = torch.device("cuda", 0)
    pb.branch_lengths[:] = oracle.clock_branch_lengths(N, pb.ops, h, None)
    ref1 = _clock_ref(pb, model)
    inst.set_node_heights_device(torch.tensor(h, device=dev))
    out = torch.empty(2 * N - 1, dtype=torch.float64, device=dev)
    gh1 = torch.empty(2 * N - 1, dtype=torch.float64, device=dev)
    with torch.cuda.stream(inst.stream):
        inst.compute_device(out)
        inst.clock_gradient_device(out, grad_heights=gh1)
    inst.stream.synchronize()
    c1 = oracle.clock_gradient(N, pb.ops, h, None, (ref1["grad"], ref1["grad_abs"]))
    scale = np.maximum(np.abs(c1["grad_heights"]), c1["abs_heights"])
    assert np.max(np.abs(gh1.cpu().numpy() - c1["grad_heights"]) / scale) <= 1e-10
    assert abs(out[0].item() - ref1["logL"]) <= 1e-10 * abs(ref1["logL"])
    inst.close()


def test_clock_errors():
    pg = _pg()
    pb = ps.small_problem(6, "hky", R=1, C=5, seed=3)
    inst = pg.from_problem(pb)
    N = 6
    h = np.linspace(0, 1, 2 * N - 1)
    h[:N] = 0.0
    bad = h.copy()
    bad[0] = 5.0                                           # tip above its parent
    with pytest.raises(pg.PhyloGradError) as e:
        inst.set_node_heights(bad)
    assert e.value.code == pg.PG_ERR_DOMAIN
    with pytest.raises(pg.PhyloGradError) as e:
        inst.set_node_heights(h, -np.ones(2 * N - 2))
    assert e.value.code == pg.PG_ERR_DOMAIN
    with pytest.raises(pg.PhyloGradError) as e:
        inst.set_branch_sets(np.full(2 * N - 2, 3), 2)
    assert e.value.code == pg.PG_ERR_ARG
    import torch
    out = torch.zeros(2 * N - 1, dtype=torch.float64, device="cuda")
    with pytest.raises(pg.PhyloGradError) as e:             # heights never set
        inst.clock_gradient_device(out, grad_rates=out)
    assert e.value.code == pg.PG_ERR_SEQUENCE
    inst.close()


# ------------------------------------------------------- HMC (NEXT-4) ----

def _leapfrog_oracle(pb, theta, p, eps, n_steps):
    """Reference leapfrog over theta = log b with the oracle's gradient
    (target logL(e^theta) + sum(theta); include/phylograd.h pg_hmc_leapfrog)."""
    def grad(th):
        pb.branch_lengths[:] = np.exp(th)
        r = oracle.loglik_grad(pb, threads=4)
        return r["logL"], np.exp(th) * r["grad"] + 1.0
    th, pp = theta.copy(), p.copy()
    lg, g = grad(th)
    if n_steps > 0:
        pp += 0.5 * eps * g
    for s in range(n_steps):
        th += eps * pp
        lg, g = grad(th)
        pp += (eps if s + 1 < n_steps else 0.5 * eps) * g
    return th, pp, lg, g


@pytest.mark.parametrize("model,N,R,C", [("hky", 12, 4, 40), ("codon", 7, 2, 15)])
def test_hmc_leapfrog_matches_oracle_trajectory(model, N, R, C):
    import torch
    pg = _pg()
    pb = ps.small_problem(N, model, R=R, C=C, seed=3, simulate=True)
    rng = np.random.default_rng(7)
    theta0 = np.log(pb.branch_lengths.copy())
    p0 = rng.standard_normal(2 * N - 2)
    eps, L = 0.02, 6
    th_ref, p_ref, lg_ref, g_ref = _leapfrog_oracle(pb, theta0, p0, eps, L)
    inst = pg.from_problem(pb)
    dev = torch.device("cuda", 0)
    th = torch.tensor(theta0, device=dev)
    pm = torch.tensor(p0, device=dev)
    out = torch.empty(2 * N - 1, dtype=torch.float64, device=dev)
    gt = torch.empty(2 * N - 2, dtype=torch.float64, device=dev)
    with torch.cuda.stream(inst.stream):
        inst.hmc_leapfrog(th, pm, eps, L, out, grad_theta=gt)
    inst.stream.synchronize()
    assert inst.check_status() == -1
    # the trajectory only propagates gradient rounding (~1e-12 relative)
    scale = np.maximum(np.abs(p_ref), 1.0)
    assert np.max(np.abs(th.cpu().numpy() - th_ref)) < 1e-10
    assert np.max(np.abs(pm.cpu().numpy() - p_ref) / scale) < 1e-10
    assert abs(out[0].item() - lg_ref) <= 1e-10 * abs(lg_ref)
    assert np.max(np.abs(gt.cpu().numpy() - g_ref) / np.maximum(np.abs(g_ref), 1.0)) < 1e-9
    # zero steps: one evaluation at the current position, momenta unchanged
    p_before = pm.clone()
    with torch.cuda.stream(inst.stream):
        inst.hmc_leapfrog(th, pm, eps, 0, out)
    inst.stream.synchronize()
    assert torch.equal(pm, p_before)
    assert abs(out[0].item() - lg_ref) <= 1e-10 * abs(lg_ref)
    inst.close()


@pytest.mark.parametrize("env", [{"PG_CODON_FLOW": "0"}, {"PG_CODON_FLOW": "2"}, {"PG_CODON_FLOW": "1"},
                                 {"PG_FLOW_NST": "1"}, {"PG_FLOW_NST": "2"}, {"PG_FLOW_PDL": "1"},
                                 {"PG_FLOW_NST": "1", "PG_FLOW_PDL": "1"}, {"PG_FLOW_SPLIT": "1"},
                                 {"PG_FLOW_RS": "2"}, {"PG_FLOW_RS": "2", "PG_FLOW_SPLIT": "1"},
                                 {"PG_FLOW_RS": "2", "PG_FLOW_SPLIT": "0"},
                                 {"PG_FLOW_SPLIT": "0", "PG_FLOW_PDL": "1"}, {"PG_FLOW_SPLIT": "1", "PG_FLOW_NST": "1"},
                                 {"PG_FLOW_PPROD": "1"}, {"PG_FLOW_PPROD": "1", "PG_FLOW_SPLIT": "1"},
                                 {"PG_FLOW_PPROD": "1", "PG_FLOW_NST": "1"}, {"PG_FLOW_PUB": "0"},
                                 {"PG_FLOW_PUB": "0", "PG_FLOW_SPLIT": "1"}, {"PG_FLOW_PUB": "1", "PG_FLOW_RS": "2"},
                                 {"PG_CODON_FLOW": "1", "PG_FLOW_TCH": "3"},
                                 {"PG_CODON_FLOW": "1", "PG_FLOW_TCH": "1"},
                                 {"PG_CODON_FLOW": "1", "PG_FLOW_DEFER": "1"},
                                 {"PG_CODON_FLOW": "1", "PG_FLOW_HALF": "1"},
                                 {"PG_CODON_FLOW": "1", "PG_FLOW_HALF": "1", "PG_FLOW_DEFER": "1"},
                                 {"PG_FUSED_A6": "1"}, {"PG_FUSED_A6": "0"},
                                 {"PG_FUSED_A6": "1", "PG_FLOW_PUB": "0"}])
def test_codon_schedules(env, monkeypatch):
    """Every codon schedule gives the same parity: the level-by-level kernels
    (PG_CODON_FLOW=0), the round-1 one-launch flow kernel (=1, with its chunk
    / deferral / half-tile options) and the default warp-specialised TMA flow
    kernel (=2) (read when the instance plans its launches)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _compare(ps.config3_yeast(N=24, C=150))
    _compare(ps.config5_yeast_mmm(N=10, C=70))


@pytest.mark.parametrize("model,N,R,C,seed", [("codon", 14, 2, 37, 51), ("codon", 8, 4, 30, 3),
                                              ("mmm4", 10, 2, 30, 4), ("hky", 12, 4, 40, 5)])
def test_error_vs_extended_precision(model, N, R, C, seed):
    """Distance of the CUDA path and of the fp64 oracle from the exact result
    of the same inputs (oracle/extended.py: long double, complex-step
    gradient), C17 metric.  The CUDA path must be within 1e-10 of exact, and
    is recorded next to the oracle's own distance (parity headroom)."""
    from oracle import extended
    pg = _pg()
    pb = ps.small_problem(N, model, R=R, C=C, seed=seed)
    if model == "codon" and N == 14:          # the clock-test instance (short branches)
        rng = np.random.default_rng(N)
        h = np.zeros(2 * N - 1)
        h[2 * N - 2] = 0.8
        for d, a, b in pb.ops[::-1]:
            for c in (a, b):
                h[c] = h[d] * rng.uniform(0.3, 0.95)
        rho = rng.lognormal(0.0, 0.3, size=2 * N - 2)
        pb.branch_lengths[:] = oracle.clock_branch_lengths(N, pb.ops, h, rho)
    ex = extended.loglik_grad(pb)
    ref = oracle.loglik_grad(pb, threads=4)
    inst = pg.from_problem(pb)
    logl, g = inst.compute()
    inst.close()
    exg, exl = ex["grad"].astype(float), float(ex["logL"])
    scale = np.maximum(np.abs(exg), ref["grad_abs"])
    e_gpu = float(np.max(np.abs(g - exg) / scale))
    e_orc = float(np.max(np.abs(ref["grad"] - exg) / scale))
    l_gpu, l_orc = abs(logl - exl) / abs(exl), abs(ref["logL"] - exl) / abs(exl)
    record_parity({"test": "error_vs_extended", "problem": pb.name, "N": N, "C": C, "S": pb.states, "R": R,
                   "cuda_grad_c17_vs_exact": e_gpu, "oracle_grad_c17_vs_exact": e_orc,
                   "cuda_logl_rel_vs_exact": l_gpu, "oracle_logl_rel_vs_exact": l_orc, "tol": 1e-10,
                   "reference": "oracle/extended.py (long double, complex step)"})
    assert e_gpu <= 1e-10 and l_gpu <= 1e-10, (e_gpu, l_gpu)
