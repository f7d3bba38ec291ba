"""Independent brute-force likelihood and gradient for tiny trees (test-only).

Marginalises the latent states of all N-1 internal nodes (incl. the root)
explicitly (P:213-218 data augmentation; S:240 / S:321), with transition
matrices from scipy's Padé expm (not the eigensystem the oracle uses), so a
mistake in the oracle's pruning, pre-order, orientation or eigen path shows
up as a mismatch.  Shares nothing with oracle/ or the CUDA path.
"""
from __future__ import annotations

import itertools

import numpy as np
from scipy.linalg import expm


def site_likelihoods(pb, branch_override=None):
    """L_c for every pattern and dL_c/db_i for every branch, by enumeration.

    Returns (L [C], dL [2N-2, C]).
    """
    N, S, C = pb.n_tips, pb.states, pb.patterns
    R = len(pb.cat_rates)
    B = 2 * N - 2
    Q = pb.Q
    bl = pb.branch_lengths if branch_override is None else branch_override
    parent = {}
    for d, a, b in pb.ops:
        parent[int(a)] = int(d)
        parent[int(b)] = int(d)
    root = 2 * N - 2
    internal = list(range(N, 2 * N - 1))
    tips = pb.tip_partials_dense()                       # [N, C, S]
    L = np.zeros(C)
    dL = np.zeros((B, C))
    for r in range(R):
        g, w = pb.cat_rates[r], pb.cat_weights[r]
        P = [expm(g * bl[i] * Q) for i in range(B)]
        dP = [g * Q @ P[i] for i in range(B)]
        # tip factor for edge i: F_i[s, c] = sum_t P_i[s, t] tip_i[c, t]
        Ftip = [P[i] @ tips[i].T for i in range(N)]          # [S, C]
        dFtip = [dP[i] @ tips[i].T for i in range(N)]
        for assign in itertools.product(range(S), repeat=len(internal)):
            st = dict(zip(internal, assign))
            # edge factors for this assignment, per pattern
            fac = []
            dfac = []
            for i in range(B):
                sp = st[parent[i]]
                if i < N:
                    fac.append(Ftip[i][sp])
                    dfac.append(dFtip[i][sp])
                else:
                    fac.append(np.full(C, P[i][sp, st[i]]))
                    dfac.append(np.full(C, dP[i][sp, st[i]]))
            fac = np.array(fac)                          # [B, C]
            prior = pb.pi[st[root]]
            L += w * prior * np.prod(fac, axis=0)
            for i in range(B):
                others = np.prod(np.delete(fac, i, axis=0), axis=0)
                dL[i] += w * prior * dfac[i] * others
    return L, dL


def loglik_grad(pb):
    L, dL = site_likelihoods(pb)
    W = pb.pattern_weights
    return float(np.sum(W * np.log(L))), (dL / L[None, :]) @ W
