"""ctypes wrapper of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` legs, never by the product
package `paper_2303_04390_b200`.  See oracle.c's header for what is computed
and which PAPER.md passages each function follows.

Parity-pin status (details in DESIGN.md §Oracle):
  oracle_transition        pinned: JC69 closed form, scipy expm (Padé)
  oracle_loglik_grad logL  pinned: two-taxon JC closed form, brute force over
                           internal states (numpy + scipy expm), compression
  oracle_loglik_grad grad  pinned: two-taxon JC closed-form derivative, brute
                           force with dP, central finite differences, pulley
                           principle, Euler identity
  node likelihoods (Eq. 5) pinned: equality to L_c at every node
  oracle_grad_quadratic    pinned: brute force, finite differences
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


class _Problem(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int), ("S", ctypes.c_int), ("R", ctypes.c_int), ("C", ctypes.c_int),
                ("ops", _ip), ("branch_lengths", _dp), ("evec", _dp), ("ievec", _dp),
                ("evals", _dp), ("pi", _dp), ("cat_rates", _dp), ("cat_weights", _dp),
                ("pattern_weights", _dp), ("tip_states", _ip), ("tip_partials", _dp)]


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain gcc -O2, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.oracle_transition.argtypes = [ctypes.c_int, _dp, _dp, _dp, ctypes.c_double, _dp]
        lib.oracle_transition_deriv.argtypes = [ctypes.c_int, _dp, _dp, _dp, ctypes.c_double,
                                                ctypes.c_double, _dp]
        lib.oracle_loglik_grad.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, _dp, _dp, _dp, _dp, _dp, _ip]
        lib.oracle_grad_quadratic.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int,
                                              ctypes.c_int, _dp]
        _lib = lib
    return _lib


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


class _Bound:
    """A Problem marshalled into C arrays (kept alive with the struct)."""

    def __init__(self, pb):
        # implicit hidden-copy masks (phylo_synth config 6) as explicit partials
        tp = pb.tip_partials_dense() if getattr(pb, "mask_K", 0) else pb.tip_partials
        self.arrs = dict(
            ops=_c(pb.ops, np.int32), bl=_c(pb.branch_lengths, np.float64),
            V=_c(pb.evec, np.float64), Vi=_c(pb.ievec, np.float64),
            lam=_c(pb.evals, np.float64), pi=_c(pb.pi, np.float64),
            g=_c(pb.cat_rates, np.float64), cw=_c(pb.cat_weights, np.float64),
            w=_c(pb.pattern_weights, np.float64),
            ts=_c(pb.tip_states, np.int32) if tp is None else None,
            tp=_c(tp, np.float64))
        a = self.arrs
        self.S = int(pb.states)
        self.N = int(pb.n_tips)
        self.C = int(a["w"].shape[0])
        self.st = _Problem(self.N, self.S, int(a["g"].shape[0]), self.C,
                           _ptr(a["ops"], _ip), _ptr(a["bl"]), _ptr(a["V"]), _ptr(a["Vi"]),
                           _ptr(a["lam"]), _ptr(a["pi"]), _ptr(a["g"]), _ptr(a["cw"]),
                           _ptr(a["w"]), _ptr(a["ts"], _ip), _ptr(a["tp"]))


def transition(evec, ievec, evals, t):
    """Eq. 1 for one (branch, category): P = V diag(exp(lambda t)) V^-1."""
    lib = _load()
    S = len(evals)
    V, Vi, lam = (np.ascontiguousarray(x, np.float64) for x in (evec, ievec, evals))
    P = np.zeros((S, S))
    lib.oracle_transition(S, _ptr(V), _ptr(Vi), _ptr(lam), float(t), _ptr(P))
    return P


def transition_deriv(evec, ievec, evals, rate, b):
    """d/db exp(rate b Q) = rate Q P."""
    lib = _load()
    S = len(evals)
    V, Vi, lam = (np.ascontiguousarray(x, np.float64) for x in (evec, ievec, evals))
    dP = np.zeros((S, S))
    lib.oracle_transition_deriv(S, _ptr(V), _ptr(Vi), _ptr(lam), float(rate), float(b), _ptr(dP))
    return dP


def _run_block(bound, c0, c1, rescale, want_nodes):
    lib = _load()
    N, B = bound.N, 2 * bound.N - 2
    logL = ctypes.c_double(0.0)
    g = np.zeros(B)
    ga = np.zeros(B)
    site = np.zeros(c1 - c0)
    nodes = np.zeros((2 * N - 1, c1 - c0)) if want_nodes else None
    zp = ctypes.c_int(-1)
    rc = lib.oracle_loglik_grad(ctypes.byref(bound.st), c0, c1, int(rescale), ctypes.byref(logL),
                                _ptr(g), _ptr(ga), _ptr(site), _ptr(nodes), ctypes.byref(zp))
    if rc < 0:
        raise ValueError(f"oracle_loglik_grad failed ({rc})")
    return rc, logL.value, g, ga, site, nodes, zp.value


def loglik_grad(pb, lo: int = 0, hi: int | None = None, rescale: bool = True,
                node_likelihoods: bool = False, threads: int = 1, block: int = 256):
    """logL, gradient and diagnostics over patterns [lo, hi) (Eq. 3, Eq. 6-8).

    threads > 1 splits the pattern range into blocks run concurrently (ctypes
    releases the GIL); partial sums are combined in block order.
    """
    bound = _Bound(pb)
    hi = bound.C if hi is None else hi
    blocks = [(c, min(hi, c + block)) for c in range(lo, hi, block)] if threads > 1 else [(lo, hi)]
    if threads > 1:
        with ThreadPoolExecutor(threads) as ex:
            res = list(ex.map(lambda b: _run_block(bound, b[0], b[1], rescale, node_likelihoods),
                              blocks))
    else:
        res = [_run_block(bound, lo, hi, rescale, node_likelihoods)]
    B = 2 * bound.N - 2
    out = dict(logL=0.0, grad=np.zeros(B), grad_abs=np.zeros(B), zero_pattern=-1, status=0)
    sites, nodes = [], []
    for rc, lg, g, ga, site, nd, zp in res:
        out["logL"] += lg
        out["grad"] += g
        out["grad_abs"] += ga
        sites.append(site)
        if nd is not None:
            nodes.append(nd)
        if rc == 1 and out["status"] == 0:
            out["status"], out["zero_pattern"] = 1, zp
    out["site_logL"] = np.concatenate(sites) if sites else np.zeros(0)
    if node_likelihoods:
        out["node_logL"] = np.concatenate(nodes, axis=1)
    return out


def grad_quadratic(pb, lo: int = 0, hi: int | None = None):
    """O(N^2) derivative-substitution gradient."""
    lib = _load()
    bound = _Bound(pb)
    hi = bound.C if hi is None else hi
    g = np.zeros(2 * bound.N - 2)
    rc = lib.oracle_grad_quadratic(ctypes.byref(bound.st), lo, hi, _ptr(g))
    if rc < 0:
        raise ValueError(f"oracle_grad_quadratic failed ({rc})")
    return g


# ---------------------------------------------------------------------------
# Time-tree ("clock") parameterisation, SURVEY §8(f) NEXT-1 and C23.
# "Each branch length b_i ... can ... be the difference
# between the parent and child node heights measured in time-units multiplied
# by a (possibly branch-specific) evolutionary rate scalar":
#     b_i = rho_i * (h_parent(i) - h_i).
# for a strict clock "further reduce the partial derivatives across
# a set of branches and report a single value".  The gradients below are the
# chain rule written out term by term; pinned in tests/test_oracle_pins.py by
# central finite differences of logL in h, rho and a global clock rate, and
# by the scaling identity sum_k h_k dlogL/dh_k = sum_i b_i g_i.
# ---------------------------------------------------------------------------

def parents(N: int, ops) -> np.ndarray:
    """parent[v] of every node (-1 for the root) from the post-order op list."""
    par = np.full(2 * N - 1, -1, dtype=np.int64)
    for d, a, b in np.asarray(ops).reshape(-1, 3):
        par[a] = d
        par[b] = d
    return par


def clock_branch_lengths(N: int, ops, heights, rates=None) -> np.ndarray:
    """b_i = rho_i (h_parent(i) - h_i), i = 0..2N-3."""
    par = parents(N, ops)
    B = 2 * N - 2
    b = np.zeros(B)
    for i in range(B):
        rho = 1.0 if rates is None else rates[i]
        b[i] = rho * (heights[par[i]] - heights[i])
    return b


def clock_gradient(N: int, ops, heights, rates, g, set_of_branch=None, n_sets: int = 1):
    """Chain rule of logL(b(h, rho)) from g = dlogL/db:
      dlogL/drho_i = (h_parent(i) - h_i) g_i
      dlogL/dh_k   = sum over children c of k: rho_c g_c   (b_c grows with h_k)
                     - rho_k g_k if k is not the root      (b_k shrinks)
      set sums     = sum over branches i of set s of (h_parent(i) - h_i) g_i
                     (= dlogL/dr for b_i = r tau_i on that set).
    Also returns the condition-aware magnitudes (same sums of |terms|, with
    `g_abs` in place of g when given via g=(g, g_abs))."""
    g_abs = None
    if isinstance(g, tuple):
        g, g_abs = g
    par = parents(N, ops)
    B = 2 * N - 2
    rho = np.ones(B) if rates is None else np.asarray(rates, float)
    sets = np.zeros(B, dtype=np.int64) if set_of_branch is None else np.asarray(set_of_branch)
    d_rho = np.zeros(B)
    d_h = np.zeros(2 * N - 1)
    s_sum = np.zeros(n_sets)
    a_rho, a_h, a_s = np.zeros(B), np.zeros(2 * N - 1), np.zeros(n_sets)
    for i in range(B):
        tau = heights[par[i]] - heights[i]
        d_rho[i] = tau * g[i]
        d_h[par[i]] += rho[i] * g[i]
        d_h[i] -= rho[i] * g[i]
        if sets[i] >= 0:
            s_sum[sets[i]] += tau * g[i]
        if g_abs is not None:
            a_rho[i] = abs(tau) * g_abs[i]
            a_h[par[i]] += abs(rho[i]) * g_abs[i]
            a_h[i] += abs(rho[i]) * g_abs[i]
            if sets[i] >= 0:
                a_s[sets[i]] += abs(tau) * g_abs[i]
    out = dict(grad_rates=d_rho, grad_heights=d_h, set_sums=s_sum)
    if g_abs is not None:
        out.update(abs_rates=a_rho, abs_heights=a_h, abs_sets=a_s)
    return out
