"""Extended-precision reference for logL and its branch-length gradient.

TEST INFRASTRUCTURE ONLY (same rule as oracle/__init__.py): imported by tests/
only, never by the product package.

Why it exists.  The fp64 oracle (oracle.c) follows Eq. 1-8 literally; on codon
instances whose eigenvector matrix V is ill-conditioned, P = V diag(e) V^-1
(Eq. 1) carries rounding errors of order eps |V| |V^-1|, so the
fp64 oracle itself sits up to ~5e-11 (C17 scale) from the exact gradient of the
given inputs.  A parity bound of 1e-10 between two fp64 evaluations of such an
instance then has no headroom (R15).  This module computes the same
quantities with the inputs (V, V^-1, lambda, rates, weights, b, tips) taken as
exact and every operation in numpy long double (64-bit mantissa, unit
roundoff 5.4e-20):

  logL(b)  = sum_c w_c log sum_r P(gamma_r) pi' p_root        (Eq. 2-3)
  dlogL/db_i by the complex step  Im logL(b + i h e_i) / h,  h = 1e-40:
             exact to working precision (no subtraction, so no cancellation);
             P(b + ih) = V diag(exp(gamma lambda (b + ih))) V^-1 is Eq. 1 at
             complex b.

No rescaling is needed at the small sizes it is used for (the long double
exponent range is 2^-16382).  Cost: one pruning pass per branch; use on small
instances only (N <= ~30, C <= ~100).
"""
from __future__ import annotations

import numpy as np

_LD = np.longdouble
_CLD = np.clongdouble


def _loglik(pb, bl):
    """Eq. 2-3 in complex long double for branch lengths `bl` ([2N-2], complex)."""
    N, S, R, C = pb.n_tips, pb.states, len(pb.cat_rates), len(pb.pattern_weights)
    V = pb.evec.astype(_LD)
    Vi = pb.ievec.astype(_LD).astype(_CLD)
    lam = pb.evals.astype(_LD)
    part = {}
    for t in range(N):
        if pb.tip_partials is not None:
            v = pb.tip_partials[t].astype(_LD).astype(_CLD)
        else:
            v = np.zeros((C, S), dtype=_CLD)
            st = pb.tip_states[t]
            obs = st < S
            v[np.nonzero(obs)[0], st[obs]] = 1
            v[~obs, :] = 1                         # missing: all-ones partial
        for r in range(R):
            part[t, r] = v
    Pm = {}
    for i in range(2 * N - 2):
        for r in range(R):
            e = np.exp(lam * _LD(pb.cat_rates[r]) * bl[i])          # Eq. 1
            Pm[i, r] = (V * e[None, :]) @ Vi
    for d, a, b in pb.ops:                                         # Eq. 2
        for r in range(R):
            part[d, r] = (part[a, r] @ Pm[a, r].T) * (part[b, r] @ Pm[b, r].T)
    root = int(pb.ops[-1][0])
    pi = pb.pi.astype(_LD).astype(_CLD)
    L = sum(_LD(pb.cat_weights[r]) * (part[root, r] @ pi) for r in range(R))   # Eq. 3
    return np.sum(pb.pattern_weights.astype(_LD) * np.log(L))


def loglik_grad(pb, branches=None):
    """logL and dlogL/db_i (for `branches`, default all 2N-2) in long double."""
    B = 2 * pb.n_tips - 2
    b0 = pb.branch_lengths[:B].astype(_LD).astype(_CLD)
    logl = _loglik(pb, b0).real
    h = _LD(1e-40)
    idx = range(B) if branches is None else branches
    g = np.zeros(B, dtype=_LD)
    for i in idx:
        bb = b0.copy()
        bb[i] += 1j * h
        g[i] = _loglik(pb, bb).imag / h
    return dict(logL=logl, grad=g)
