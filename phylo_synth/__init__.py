"""Seeded synthetic inputs shaped like the paper's workloads.

This module produces INPUTS only: substitution-rate matrices and their
eigensystems, discrete-Gamma rate categories, trees, simulated alignments and
their site-pattern compression.  It holds none of the method's arithmetic
(no Eq. 1 transition matrices, no pruning, no pre-order, no gradient): the
alignment is simulated by the CTMC jump chain (exponential holding times and
the embedded jump matrix of Q), never through exp(tQ).  Both the oracle side
(`oracle/`) and the CUDA side (`paper_2303_04390_b200`) consume what it makes;
neither is imported here.

Paper references (PAPER.md line numbers, arXiv 2303.04390):
  * data, site patterns and weights ................. P:191-193
  * node numbering (tips, internals, root, branches) . P:197-201
  * rate categories gamma_r, P(gamma_r) .............. P:203-206
  * GTR / Yang codon models, Gamma-4 ................. P:888
  * Markov-modulated models ........................... P:196
  * WNV example (104 taxa, 1999-2007, kappa, omega) .. P:962-996

Node numbering used everywhere in this repo is the paper's shifted
to 0-based: tips 0..N-1, internal nodes N..2N-3, root 2N-2; branch i is the
edge above node i.  `ops` is the post-order operation list: (N-1) triples
(dest, child1, child2), children defined before parents, last dest = root.
"""
from __future__ import annotations

import dataclasses
import hashlib
import itertools
from typing import Optional

import numpy as np
from scipy import special

MASTER_SEED = 2303043900

NUC = "ACGT"
# NCBI translation table 1 (universal), codons enumerated in TCAG order.
_UNIVERSAL_AA = "FFLLSSSSYY**CC*WLLLLPPPPHHQQRRRRIIIMTTTTNNKKSSRRVVVVAAAADDEEGGGG"
_TCAG = "TCAG"


# --------------------------------------------------------------------------
# Rate matrices (input production; the library takes only their eigensystem)
# --------------------------------------------------------------------------

def normalize_rate(Q: np.ndarray, pi: np.ndarray) -> np.ndarray:
    """Scale Q so the expected substitution rate -sum_s pi_s Q_ss is 1."""
    mu = -float(np.dot(pi, np.diag(Q)))
    return Q / mu


def _fill_diag(Q: np.ndarray) -> np.ndarray:
    Q = Q.copy()
    np.fill_diagonal(Q, 0.0)
    np.fill_diagonal(Q, -Q.sum(axis=1))
    return Q


def gtr(exch, pi) -> np.ndarray:
    """GTR generator; exch = (AC, AG, AT, CG, CT, GT), pi over ACGT."""
    pi = np.asarray(pi, float)
    a = np.zeros((4, 4))
    for (i, j), e in zip(itertools.combinations(range(4), 2), exch):
        a[i, j] = a[j, i] = e
    Q = a * pi[None, :]
    return normalize_rate(_fill_diag(Q), pi)


def hky(kappa: float, pi) -> np.ndarray:
    """HKY85 = GTR with exchangeabilities 1 except kappa on transitions."""
    return gtr((1.0, kappa, 1.0, 1.0, kappa, 1.0), pi)


def jc69() -> np.ndarray:
    return gtr((1.0,) * 6, (0.25,) * 4)


def sense_codons(code: str = "universal"):
    """Sense codons (as 3-char strings over ACGT) and their amino acids."""
    if code != "universal":
        raise ValueError("only the universal code is provided")
    cod, aa = [], []
    for k, (x, y, z) in enumerate(itertools.product(_TCAG, repeat=3)):
        if _UNIVERSAL_AA[k] != "*":
            cod.append(x + y + z)
            aa.append(_UNIVERSAL_AA[k])
    # canonical order: lexicographic over ACGT
    order = sorted(range(len(cod)), key=lambda i: [NUC.index(c) for c in cod[i]])
    return [cod[i] for i in order], [aa[i] for i in order]


def gy94(kappa: float, omega: float, codon_freqs: np.ndarray, code="universal") -> np.ndarray:
    """Goldman-Yang 1994 / M0 codon generator (P:888 'Yang codon model')."""
    cod, aa = sense_codons(code)
    S = len(cod)
    pi = np.asarray(codon_freqs, float)
    assert pi.shape == (S,)
    Q = np.zeros((S, S))
    transitions = {frozenset("AG"), frozenset("CT")}
    for i in range(S):
        for j in range(S):
            diff = [p for p in range(3) if cod[i][p] != cod[j][p]]
            if len(diff) != 1:
                continue
            p = diff[0]
            r = pi[j]
            if frozenset((cod[i][p], cod[j][p])) in transitions:
                r *= kappa
            if aa[i] != aa[j]:
                r *= omega
            Q[i, j] = r
    return normalize_rate(_fill_diag(Q), pi)


def f3x4_freqs(pos_freqs: np.ndarray, code="universal") -> np.ndarray:
    """F3x4 codon frequencies from 3 x 4 position-specific nucleotide freqs."""
    cod, _ = sense_codons(code)
    f = np.array([np.prod([pos_freqs[p, NUC.index(c[p])] for p in range(3)]) for c in cod])
    return f / f.sum()


def markov_modulated(Qbase: np.ndarray, pibase: np.ndarray, class_rates, delta: float):
    """Markov-modulated model: K hidden rate classes over a base model.

    State s = n*K + k (observed base state n, hidden class k).  Within class k
    the base process runs at rate class_rates[k]; the class switches at rate
    delta (uniform stationary class distribution).  Reversible.
    """
    Sb = Qbase.shape[0]
    rho = np.asarray(class_rates, float)
    K = len(rho)
    S = Sb * K
    Q = np.zeros((S, S))
    for n in range(Sb):
        for k in range(K):
            s = n * K + k
            for n2 in range(Sb):
                if n2 != n:
                    Q[s, n2 * K + k] = rho[k] * Qbase[n, n2]
            for k2 in range(K):
                if k2 != k:
                    Q[s, n * K + k2] = delta
    pi = np.repeat(pibase, K) / K
    return normalize_rate(_fill_diag(Q), pi), pi


def eigen_reversible(Q: np.ndarray, pi: np.ndarray):
    """Real eigensystem Q = V diag(lam) V^{-1} via the pi^(1/2) symmetrisation.

    Returns (V, Vinv, lam), row-major S x S, S x S, S.  This is the ABI's
    `pg_set_eigen` input (C13: real eigensystems only).
    """
    d = np.sqrt(pi)
    B = (d[:, None] * Q) / d[None, :]
    B = 0.5 * (B + B.T)
    lam, U = np.linalg.eigh(B)
    V = U / d[:, None]
    Vinv = U.T * d[None, :]
    return V, Vinv, lam


def discrete_gamma(alpha: float, R: int):
    """Equal-weight discrete Gamma (Yang 1994) with mean-of-bin rates, mean one.

    P:204-206 (the paper does not pin the variant; SURVEY C12 / SPEC S:114).
    """
    if R == 1:
        return np.ones(1), np.ones(1)
    edges = special.gammaincinv(alpha, np.arange(1, R) / R) / alpha
    cdf1 = np.concatenate([[0.0], special.gammainc(alpha + 1.0, edges * alpha), [1.0]])
    rates = R * np.diff(cdf1)
    rates = rates / rates.mean()
    return rates, np.full(R, 1.0 / R)


# --------------------------------------------------------------------------
# Trees
# --------------------------------------------------------------------------

@dataclasses.dataclass
class Tree:
    n_tips: int
    ops: np.ndarray            # int32 [N-1, 3] post-order (dest, c1, c2)
    heights: np.ndarray        # float64 [2N-1] node heights (time or subs)
    branch_lengths: np.ndarray  # float64 [2N-1], index = child node; root entry 0

    @property
    def root(self) -> int:
        return 2 * self.n_tips - 2

    def parent(self) -> np.ndarray:
        par = np.full(2 * self.n_tips - 1, -1, np.int64)
        for d, a, b in self.ops:
            par[a] = d
            par[b] = d
        return par


def tree_from_newick_fixed5() -> Tree:
    """BJ:configs[0] tree ((A:0.10,B:0.20):0.05,(C:0.15,(D:0.30,E:0.25):0.10):0.07);

    Tips A..E = 0..4; internals (A,B)=5, (D,E)=6, (C,(D,E))=7; root 8.
    """
    ops = np.array([[5, 0, 1], [6, 3, 4], [7, 2, 6], [8, 5, 7]], np.int32)
    b = np.array([0.10, 0.20, 0.15, 0.30, 0.25, 0.05, 0.10, 0.07, 0.0])
    return Tree(5, ops, np.zeros(9), b)


def coalescent_tree(N: int, rng: np.random.Generator, root_height: float,
                    tip_times: Optional[np.ndarray] = None) -> Tree:
    """Kingman random-joining tree (optionally serially sampled tips).

    Internal nodes are numbered in creation (i.e. post-) order N..2N-2, the
    last one being the root, so `ops` is a valid post-order list.  Heights are
    rescaled so the root sits at `root_height`.
    """
    tip_h = np.zeros(N) if tip_times is None else np.asarray(tip_times, float)
    order = np.argsort(tip_h, kind="stable")
    heights = np.zeros(2 * N - 1)
    heights[:N] = tip_h
    active: list[int] = []
    pending = list(order)
    t = 0.0
    nxt = N
    ops = []
    while nxt < 2 * N - 1:
        while pending and tip_h[pending[0]] <= t:
            active.append(pending.pop(0))
        k = len(active)
        if k < 2:
            t = tip_h[pending[0]]
            continue
        rate = k * (k - 1) / 2.0
        dt = rng.exponential(1.0 / rate)
        if pending and t + dt > tip_h[pending[0]]:
            t = tip_h[pending[0]]
            continue
        t += dt
        i, j = rng.choice(k, size=2, replace=False)
        a, b = active[i], active[j]
        for x in sorted((i, j), reverse=True):
            active.pop(x)
        heights[nxt] = t
        ops.append((nxt, a, b))
        active.append(nxt)
        nxt += 1
    ops = np.array(ops, np.int32)
    scale = root_height / (heights[2 * N - 2] - heights[:N].min())
    heights = (heights - heights[:N].min()) * scale
    tr = Tree(N, ops, heights, np.zeros(2 * N - 1))
    par = tr.parent()
    bl = np.zeros(2 * N - 1)
    for v in range(2 * N - 2):
        bl[v] = heights[par[v]] - heights[v]
    tr.branch_lengths = bl
    return tr


# --------------------------------------------------------------------------
# Alignment simulation (CTMC jump chain) and site-pattern compression
# --------------------------------------------------------------------------

def simulate_alignment(tree: Tree, Q: np.ndarray, pi: np.ndarray, rates: np.ndarray,
                       weights: np.ndarray, n_sites: int, rng: np.random.Generator,
                       branch_scale: Optional[np.ndarray] = None) -> np.ndarray:
    """Simulate states [N, n_sites] by Gillespie along each branch.

    Holding time in state s ~ Exp(-Q_ss * gamma_r); jump to t with prob
    Q_st / -Q_ss.  `branch_scale` multiplies branch lengths (relaxed clock).
    """
    S = Q.shape[0]
    out_rate = -np.diag(Q)
    J = np.where(np.eye(S, dtype=bool), 0.0, Q) / np.maximum(out_rate, 1e-300)[:, None]
    Jcum = np.cumsum(J, axis=1)
    Jcum[:, -1] = 1.0
    cat = rng.choice(len(rates), size=n_sites, p=weights)
    site_rate = rates[cat]
    N = tree.n_tips
    states = np.zeros((2 * N - 1, n_sites), np.int64)
    states[tree.root] = rng.choice(S, size=n_sites, p=pi)
    bl = tree.branch_lengths if branch_scale is None else tree.branch_lengths * branch_scale
    for d, a, b in tree.ops[::-1]:
        for c in (a, b):
            x = states[d].copy()
            tleft = bl[c] * site_rate
            idx = np.arange(n_sites)
            while idx.size:
                r = out_rate[x[idx]]
                w = rng.exponential(1.0, size=idx.size) / np.maximum(r, 1e-300)
                jump = w < tleft[idx]
                idx = idx[jump]
                if not idx.size:
                    break
                tleft[idx] -= w[jump]
                u = rng.random(idx.size)
                rows = Jcum[x[idx]]
                x[idx] = np.minimum((rows < u[:, None]).sum(axis=1), S - 1)
            states[c] = x
    return states[:N]


def compress_patterns(aln: np.ndarray, n_patterns: Optional[int] = None):
    """Unique columns in first-occurrence order with integer counts.

    Returns (patterns [N, C] int, weights [C] float64).  When `n_patterns` is
    given, the first n_patterns unique columns are kept (their counts over the
    whole simulated alignment are the weights).
    """
    u, first, inv, cnt = np.unique(aln.T, axis=0, return_index=True,
                                   return_inverse=True, return_counts=True)
    order = np.argsort(first, kind="stable")
    pats = u[order].T
    w = cnt[order].astype(np.float64)
    if n_patterns is not None:
        if pats.shape[1] < n_patterns:
            raise ValueError(f"only {pats.shape[1]} unique patterns (< {n_patterns})")
        pats, w = pats[:, :n_patterns], w[:n_patterns]
    return pats, w


# --------------------------------------------------------------------------
# Problem instances (the BJ configs)
# --------------------------------------------------------------------------

@dataclasses.dataclass
class Problem:
    """One likelihood/gradient instance, in the library's input vocabulary."""
    name: str
    n_tips: int
    states: int                       # S (unpadded)
    ops: np.ndarray                   # int32 [N-1, 3]
    branch_lengths: np.ndarray        # float64 [2N-2] by child node
    evec: np.ndarray                  # float64 [S, S]
    ievec: np.ndarray                 # float64 [S, S]
    evals: np.ndarray                 # float64 [S]
    Q: np.ndarray                     # float64 [S, S] (for reference/tests)
    pi: np.ndarray                    # float64 [S] root prior (Eq. 3)
    cat_rates: np.ndarray             # float64 [R]
    cat_weights: np.ndarray           # float64 [R]
    pattern_weights: np.ndarray       # float64 [C]
    tip_states: Optional[np.ndarray] = None    # int32 [N, C], S = missing
    tip_partials: Optional[np.ndarray] = None  # float64 [N, C, S]
    precision: str = "fp64"
    rate_scalars: Optional[np.ndarray] = None  # relaxed clock rho [2N-2]
    branch_times: Optional[np.ndarray] = None  # tau [2N-2]
    # Markov-modulated models with the hidden class unobserved at the tips:
    # tip (n, c) is the 0/1 mask with ones on the mask_K hidden copies
    # mask_K * obs + k of the observed base state obs = tip_obs[n, c]
    # (kept implicit: a dense [N, C, S] array is ~5 GB at S = 244, N = 10^4)
    tip_obs: Optional[np.ndarray] = None       # int32 [N, C]
    mask_K: int = 0

    @property
    def patterns(self) -> int:
        return int(self.pattern_weights.shape[0])

    @property
    def has_partials(self) -> bool:
        return self.tip_partials is not None or self.mask_K > 0

    def tip_partial_rows(self, n: int, lo: int = 0, hi: Optional[int] = None) -> np.ndarray:
        """Dense partials [hi-lo, S] of tip n (explicit, or the hidden-copy mask)."""
        hi = self.patterns if hi is None else hi
        if self.tip_partials is not None:
            return self.tip_partials[n, lo:hi]
        obs = self.tip_obs[n, lo:hi]
        part = np.zeros((hi - lo, self.states))
        for k in range(self.mask_K):
            part[np.arange(hi - lo), obs * self.mask_K + k] = 1.0
        return part

    def subset(self, lo: int, hi: int) -> "Problem":
        """The same tree and model on patterns [lo, hi), tips materialised
        (explicit partials for mask problems: oracle input)."""
        import dataclasses
        kw = dict(pattern_weights=self.pattern_weights[lo:hi].copy(), name=f"{self.name}_p{lo}_{hi}")
        if self.has_partials:
            kw.update(tip_partials=np.stack([self.tip_partial_rows(n, lo, hi) for n in range(self.n_tips)]),
                      tip_states=None, tip_obs=None, mask_K=0)
        else:
            kw.update(tip_states=self.tip_states[:, lo:hi].copy())
        return dataclasses.replace(self, **kw)

    @property
    def categories(self) -> int:
        return int(self.cat_rates.shape[0])

    def digest(self) -> str:
        h = hashlib.sha256()
        for a in (self.ops, self.branch_lengths, self.evec, self.ievec, self.evals,
                  self.pi, self.cat_rates, self.cat_weights, self.pattern_weights,
                  self.tip_states, self.tip_partials):
            if a is not None:
                h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()[:16]

    def tip_partials_dense(self) -> np.ndarray:
        """[N, C, S] partials; a state code S (missing) becomes all-ones."""
        if self.tip_partials is not None:
            return self.tip_partials
        if self.mask_K > 0:
            return np.stack([self.tip_partial_rows(n) for n in range(self.n_tips)])
        N, C, S = self.n_tips, self.patterns, self.states
        out = np.zeros((N, C, S))
        st = self.tip_states
        for n in range(N):
            obs = st[n] < S
            out[n, np.arange(C)[obs], st[n][obs]] = 1.0
            out[n, ~obs, :] = 1.0
        return out


def _finish(name, tree, Q, pi, rates, cw, pats, w, S, **kw) -> Problem:
    V, Vi, lam = eigen_reversible(Q, pi)
    return Problem(name=name, n_tips=tree.n_tips, states=S, ops=tree.ops.copy(),
                   branch_lengths=tree.branch_lengths[:-1].copy(), evec=V, ievec=Vi,
                   evals=lam, Q=Q, pi=pi, cat_rates=rates, cat_weights=cw,
                   pattern_weights=w, **kw)


def _simulate_until(tree, Q, pi, rates, cw, C, rng, branch_scale=None, start=None,
                    project=None):
    n = start or max(2 * C, 64)
    for _ in range(12):
        aln = simulate_alignment(tree, Q, pi, rates, cw, n, rng, branch_scale)
        obs = aln if project is None else project(aln)
        u = np.unique(obs.T, axis=0).shape[0]
        if u >= C:
            return aln
        n = int(n * max(2.0, 1.5 * C / max(u, 1)))
    raise RuntimeError("could not reach the requested number of unique patterns")


def config0_jc5(C: int = 200, seed: Optional[int] = None) -> Problem:
    """BJ:configs[0]: 5-taxon fixed tree, JC69, 200 unique patterns, R=1."""
    rng = np.random.default_rng(MASTER_SEED + 0 if seed is None else seed)
    tree = tree_from_newick_fixed5()
    Q = jc69()
    pi = np.full(4, 0.25)
    rates, cw = np.ones(1), np.ones(1)
    # long-ish branches relative to the tree so 200 of the 1024 patterns appear
    aln = _simulate_until(tree, Q, pi, rates, cw, C, rng, start=200_000)
    pats, w = compress_patterns(aln, C)
    return _finish("jc5", tree, Q, pi, rates, cw, pats, w, 4,
                   tip_states=pats.astype(np.int32))


def config1_dengue(N: int = 997, C: int = 10_000, precision: str = "fp64",
                   seed: Optional[int] = None, gap_frac: float = 0.01) -> Problem:
    """BJ:configs[1]: dengue-shaped, HKY+Gamma4, Kingman tree, ~10k patterns."""
    rng = np.random.default_rng(MASTER_SEED + 1 if seed is None else seed)
    tree = coalescent_tree(N, rng, root_height=0.25)
    pi = np.array([0.33, 0.21, 0.25, 0.21])
    Q = hky(8.0, pi)
    rates, cw = discrete_gamma(0.5, 4)
    aln = _simulate_until(tree, Q, pi, rates, cw, C, rng, start=int(1.6 * C))
    if gap_frac > 0:
        # missing data as sequence-end blocks (incomplete genomes), so gapped
        # columns still repeat; ~gap_frac of all cells overall
        L = aln.shape[1]
        ntax = max(1, int(round(gap_frac / 0.2 * N)))
        for n in rng.choice(N, size=ntax, replace=False):
            ln = int(rng.uniform(0.1, 0.3) * L)
            if rng.random() < 0.5:
                aln[n, :ln] = 4
            else:
                aln[n, L - ln:] = 4
    pats, w = compress_patterns(aln, C)
    return _finish(f"dengue{N}", tree, Q, pi, rates, cw, pats, w, 4,
                   tip_states=pats.astype(np.int32), precision=precision)


def config2_mmm(N: int = 62, C: int = 5_000, K: int = 4, R: int = 1,
                precision: str = "fp64", seed: Optional[int] = None) -> Problem:
    """BJ:configs[2]: carnivore-shaped 4xK Markov-modulated HKY, tip partials."""
    rng = np.random.default_rng(MASTER_SEED + 2 if seed is None else seed)
    tree = coalescent_tree(N, rng, root_height=0.6)
    pib = np.array([0.30, 0.20, 0.20, 0.30])
    Qb = hky(4.0, pib)
    cls = np.array([0.1, 0.5, 1.2, 2.2][:K] if K <= 4 else np.linspace(0.1, 2.2, K))
    cls = cls / cls.mean()
    Q, pi = markov_modulated(Qb, pib, cls, 0.5)
    if R == 1:
        rates, cw = np.ones(1), np.ones(1)
    else:
        rates, cw = discrete_gamma(0.5, R)
    hidden = _simulate_until(tree, Q, pi, rates, cw, C, rng, start=3 * C,
                             project=lambda a: a // K)
    obs = hidden // K
    pats, w = compress_patterns(obs, C)
    S = 4 * K
    part = np.zeros((N, C, S))
    for n in range(N):
        for k in range(K):
            part[n, np.arange(C), pats[n] * K + k] = 1.0
    return _finish(f"mmm{N}_K{K}", tree, Q, pi, rates, cw, pats, w, S,
                   tip_partials=part, precision=precision)


def _codon_freqs(rng) -> np.ndarray:
    pos = rng.dirichlet(np.full(4, 8.0), size=3)
    return f3x4_freqs(pos)


def config3_yeast(N: int = 49, C: int = 4_000, precision: str = "fp64",
                  seed: Optional[int] = None) -> Problem:
    """BJ:configs[3]: yeast-shaped GY94 codon (61 states), Gamma4."""
    rng = np.random.default_rng(MASTER_SEED + 3 if seed is None else seed)
    tree = coalescent_tree(N, rng, root_height=1.0)
    pi = _codon_freqs(rng)
    Q = gy94(2.5, 0.1, pi)
    rates, cw = discrete_gamma(0.5, 4)
    aln = _simulate_until(tree, Q, pi, rates, cw, C, rng, start=int(1.3 * C))
    pats, w = compress_patterns(aln, C)
    return _finish(f"yeast{N}", tree, Q, pi, rates, cw, pats, w, 61,
                   tip_states=pats.astype(np.int32), precision=precision)


def config4_wnv(N: int = 104, C: int = 3_700, precision: str = "fp64",
                seed: Optional[int] = None) -> Problem:
    """BJ:configs[4]: WNV-shaped GY94 (kappa 11.34, omega 0.14),
    Gamma4, serially sampled time tree 1999-2007 with root ~1998.6 (P:964,
    P:994), uncorrelated lognormal relaxed clock b_i = rho_i * tau_i.
    """
    rng = np.random.default_rng(MASTER_SEED + 4 if seed is None else seed)
    ages = rng.uniform(0.0, 8.0, size=N)          # years before 2007.0
    ages[np.argmax(ages)] = 8.0                    # one 1999 sample
    tree = coalescent_tree(N, rng, root_height=8.4, tip_times=ages)  # root ~1998.6
    tau = tree.branch_lengths[:-1].copy()
    sd = 0.3
    s2 = np.log(1 + sd * sd)
    rho = rng.lognormal(-s2 / 2, np.sqrt(s2), size=2 * N - 2)   # mean 1, sd 0.3
    clock = 0.05                                   # codon subs / codon / year
    b = rho * tau * clock
    pi = _codon_freqs(rng)
    Q = gy94(11.34, 0.14, pi)
    rates, cw = discrete_gamma(0.5, 4)
    tree2 = Tree(N, tree.ops, tree.heights, np.concatenate([b, [0.0]]))
    aln = _simulate_until(tree2, Q, pi, rates, cw, C, rng, start=int(2 * C))
    pats, w = compress_patterns(aln, C)
    return _finish(f"wnv{N}", tree2, Q, pi, rates, cw, pats, w, 61,
                   tip_states=pats.astype(np.int32), precision=precision,
                   rate_scalars=rho * clock, branch_times=tau)


def config5_yeast_mmm(N: int = 49, C: int = 4_000, precision: str = "fp64",
                      seed: Optional[int] = None) -> Problem:
    """the paper's state-space test, a
    Markov-modulated model of two GY94 codon models (2 x 61 = 122 states,
    padded to 128) on the yeast-shaped tree; hidden class unobserved at the
    tips (partials with 1 on both copies of the observed codon)."""
    rng = np.random.default_rng(MASTER_SEED + 5 if seed is None else seed)
    tree = coalescent_tree(N, rng, root_height=1.0)
    pib = _codon_freqs(rng)
    Qb = gy94(2.5, 0.1, pib)
    K = 2
    Q, pi = markov_modulated(Qb, pib, np.array([0.4, 1.6]), 0.5)
    rates, cw = np.ones(1), np.ones(1)
    hidden = _simulate_until(tree, Q, pi, rates, cw, C, rng, start=int(1.3 * C),
                             project=lambda a: a // K)
    obs = hidden // K
    pats, w = compress_patterns(obs, C)
    S = 61 * K
    part = np.zeros((N, C, S))
    for n in range(N):
        for k in range(K):
            part[n, np.arange(C), pats[n] * K + k] = 1.0
    return _finish(f"yeastmmm{N}", tree, Q, pi, rates, cw, pats, w, S,
                   tip_partials=part, precision=precision)


def config6_codon_mmm4(N: int = 10_001, C: int = 256, precision: str = "fp64",
                       seed: Optional[int] = None) -> Problem:
    """SURVEY §8(f) NEXT-2, the S = 256 class with over 20,000 branch lengths
    (P:1022-1024): a Markov-modulated model of four GY94 codon classes (4 x 61
    = 244 states, padded to 256) on a 10,001-tip Kingman tree (20,000
    branches); the hidden class is unobserved at the tips (0/1 masks on the 4
    copies of the observed codon, kept implicit: `tip_obs`, `mask_K`)."""
    rng = np.random.default_rng(MASTER_SEED + 6 if seed is None else seed)
    tree = coalescent_tree(N, rng, root_height=1.0)
    pib = _codon_freqs(rng)
    K = 4
    Q, pi = markov_modulated(gy94(2.5, 0.1, pib), pib, np.array([0.25, 0.75, 1.25, 1.75]), 0.5)
    rates, cw = np.ones(1), np.ones(1)
    hidden = _simulate_until(tree, Q, pi, rates, cw, C, rng, start=int(1.2 * C),
                             project=lambda a: a // K)
    pats, w = compress_patterns(hidden // K, C)
    return _finish(f"codonmmm4_{N}", tree, Q, pi, rates, cw, pats, w, 61 * K,
                   tip_obs=pats.astype(np.int32), mask_K=K, precision=precision)


CONFIGS = {
    0: config0_jc5,
    1: config1_dengue,
    2: config2_mmm,
    3: config3_yeast,
    4: config4_wnv,
    5: config5_yeast_mmm,
    6: config6_codon_mmm4,
}


def make_config(idx: int, **kw) -> Problem:
    return CONFIGS[idx](**kw)


def shard_patterns(C: int, world: int, rank: int, align: int = 1):
    """Contiguous pattern shard [lo, hi) of rank `rank` out of `world`.

    Shards are balanced to within `align` patterns.
    """
    per = -(-C // world)
    per = -(-per // align) * align
    lo = min(C, rank * per)
    hi = min(C, lo + per)
    return lo, hi


def subset_patterns(pb: Problem, lo: int, hi: int) -> Problem:
    """The same problem restricted to patterns [lo, hi)."""
    kw = dataclasses.asdict(pb)
    kw["pattern_weights"] = pb.pattern_weights[lo:hi].copy()
    if pb.tip_states is not None:
        kw["tip_states"] = pb.tip_states[:, lo:hi].copy()
    if pb.tip_partials is not None:
        kw["tip_partials"] = pb.tip_partials[:, lo:hi].copy()
    kw["name"] = f"{pb.name}[{lo}:{hi}]"
    return Problem(**kw)


def small_problem(N: int = 5, model: str = "hky", R: int = 1, C: int = 7,
                  seed: int = 0, missing: float = 0.0, partial_tips: bool = False,
                  root_height: float = 0.5, stationary_root: bool = True,
                  simulate: bool = False, hidden_masks: int = 0) -> Problem:
    """Small random instance for pins and parity tests.

    model: 'jc' | 'hky' | 'gtr' | 'mmm2' (S=8) | 'mmm4' (S=16) | 'codon' (S=61)
           | 'codon2' (S=122, two-class codon MMM).
    Tip states are uniform random (or simulated when `simulate`), with a
    `missing` fraction of state code S; `partial_tips` gives random masks.
    """
    rng = np.random.default_rng(seed)
    if model == "jc":
        Q, pi = jc69(), np.full(4, 0.25)
    elif model in ("hky", "gtr"):
        pi = rng.dirichlet(np.full(4, 5.0))
        Q = hky(3.0, pi) if model == "hky" else gtr(rng.uniform(0.5, 3.0, 6), pi)
    elif model.startswith("mmm"):
        K = int(model[3:])
        pib = rng.dirichlet(np.full(4, 5.0))
        Q, pi = markov_modulated(hky(2.0, pib), pib, np.linspace(0.2, 1.8, K), 0.4)
    elif model == "codon":
        pi = _codon_freqs(rng)
        Q = gy94(2.5, 0.2, pi)
    elif model == "codon2":                   # 2-class codon MMM, S = 122
        pib = _codon_freqs(rng)
        Q, pi = markov_modulated(gy94(2.5, 0.2, pib), pib, np.array([0.4, 1.6]), 0.5)
    elif model == "codon4":                   # 4-class codon MMM, S = 244 (padded to 256)
        pib = _codon_freqs(rng)
        Q, pi = markov_modulated(gy94(2.5, 0.2, pib), pib, np.array([0.25, 0.75, 1.25, 1.75]), 0.5)
    else:
        raise ValueError(model)
    S = Q.shape[0]
    tree = coalescent_tree(N, rng, root_height=root_height)
    rates, cw = discrete_gamma(0.5, R) if R > 1 else (np.ones(1), np.ones(1))
    if R > 1:
        cw = rng.dirichlet(np.full(R, 4.0))   # unequal weights exercise P(gamma_r)
    if simulate:
        aln = simulate_alignment(tree, Q, pi, rates, cw, C, rng)
        states = aln.astype(np.int32)
    else:
        states = rng.integers(0, S, size=(N, C)).astype(np.int32)
    if missing > 0:
        states = np.where(rng.random(states.shape) < missing, S, states).astype(np.int32)
    w = rng.integers(1, 5, size=C).astype(np.float64)
    root_pi = pi if stationary_root else rng.dirichlet(np.full(S, 2.0))
    V, Vi, lam = eigen_reversible(Q, pi)
    kw = dict(tip_states=states)
    if hidden_masks:                          # MMM: 0/1 masks on the K hidden copies of an observed state
        K = hidden_masks
        obs = np.minimum(states, S - 1) // K
        part = np.zeros((N, C, S))
        for k in range(K):
            part[np.arange(N)[:, None], np.arange(C)[None, :], obs * K + k] = 1.0
        kw = dict(tip_partials=part)
    elif partial_tips:
        part = (rng.random((N, C, S)) < 0.4).astype(np.float64)
        part[np.arange(N)[:, None], np.arange(C)[None, :], states % S] = 1.0
        kw = dict(tip_partials=part)
    return Problem(name=f"small_{model}_N{N}_R{R}_C{C}_s{seed}", n_tips=N, states=S,
                   ops=tree.ops.copy(), branch_lengths=tree.branch_lengths[:-1].copy(),
                   evec=V, ievec=Vi, evals=lam, Q=Q, pi=root_pi, cat_rates=rates,
                   cat_weights=cw, pattern_weights=w, **kw)


def two_taxon_jc(b1: float, b2: float, tips) -> Problem:
    """N=2 rooted tree (tip0:b1, tip1:b2) under JC69; tips = [(s0, s1), ...]."""
    Q, pi = jc69(), np.full(4, 0.25)
    V, Vi, lam = eigen_reversible(Q, pi)
    st = np.array(tips, np.int32).T.copy()
    return Problem(name="jc2", n_tips=2, states=4, ops=np.array([[2, 0, 1]], np.int32),
                   branch_lengths=np.array([b1, b2], float), evec=V, ievec=Vi, evals=lam,
                   Q=Q, pi=pi, cat_rates=np.ones(1), cat_weights=np.ones(1),
                   pattern_weights=np.ones(st.shape[1]), tip_states=st)
