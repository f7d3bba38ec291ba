/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU reference (fp64).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2303_04390_b200/csrc); it depends on libc/libm only.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, arXiv 2303.04390):
 *   Eq. 1  P^{(r)}(b_i) = exp(gamma_r b_i Q), evaluated from the
 *                       eigensystem Q = V diag(lambda) V^{-1}.
 *   Eq. 2  post-order  p_k = (P_i p_i) o (P_j p_j).
 *   Eq. 3  L_c = sum_r P(gamma_r) pi' p_{root,r,c};
 *                       logL = sum_c w_c log L_c   (w_c: pattern weights).
 *   Eq. 4  pre-order   q_root = pi,  q_i = P_i' (q_k o P_j p_j).
 *   Eq. 5  sum_r P(gamma_r) p_i' q_i = L_c for every node i
 *                       (returned per node so tests can check it).
 *   Eq. 6-8 d/db_i log P(Y) = sum_c w_c
 *                          [sum_r gamma_r P(gamma_r) p' Q' q] / [sum_r P(gamma_r) p' q]
 *                       Eq. 8 orientation p'Q'q (Alg. 2's literal
 *                       p'Qq is not used).
 *   O(N^2) derivative substitution: re-prune with dP_i/db in place
 *                       of P_i (an independent cross-check of Eq. 8).
 *
 * Rescaling against underflow is not in the paper: after every
 * post-order (and pre-order) step the vector of pattern c at node k is
 * divided by m = max_{r,s}, and log m is accumulated, shared across rate
 * categories.  Set `rescale = 0` to switch it off (tests check invariance).
 *
 * Patterns are conditionally independent, so everything runs one
 * pattern at a time over [c_begin, c_end); results for a sub-range are the
 * corresponding partial sums, which lets tests sample patterns or split the
 * range across threads.
 *
 * Numbering (P:197-201, 0-based): tips 0..N-1, internal N..2N-3, root 2N-2;
 * branch i is the edge above node i; ops = (N-1) post-order triples
 * (dest, child1, child2), last dest = root.  Tip state code S = missing
 * (all-ones partial).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int N, S, R, C;
    const int *ops;               /* [N-1][3]                              */
    const double *branch_lengths; /* [2N-2]                                */
    const double *evec;           /* V      [S][S] row-major               */
    const double *ievec;          /* V^{-1} [S][S] row-major               */
    const double *evals;          /* lambda [S]                            */
    const double *pi;             /* [S]                                   */
    const double *cat_rates;      /* gamma_r [R]                           */
    const double *cat_weights;    /* P(gamma_r) [R]                        */
    const double *pattern_weights;/* w_c [C]                               */
    const int *tip_states;        /* [N][C] or NULL; S = missing           */
    const double *tip_partials;   /* [N][C][S] or NULL                     */
} oracle_problem;

enum { OR_OK = 0, OR_ZERO_LIKELIHOOD = 1, OR_ERR_ARG = -1, OR_ERR_MEM = -2 };

/* Eq. 1: P = V diag(exp(lambda * t)) V^{-1};  t = gamma_r * b_i. */
int oracle_transition(int S, const double *V, const double *Vi, const double *lam,
                      double t, double *P)
{
    if (S < 1 || !V || !Vi || !lam || !P) return OR_ERR_ARG;
    for (int s = 0; s < S; ++s)
        for (int u = 0; u < S; ++u) {
            double acc = 0.0;
            for (int k = 0; k < S; ++k)
                acc += V[s * S + k] * exp(lam[k] * t) * Vi[k * S + u];
            P[s * S + u] = acc;
        }
    return OR_OK;
}

/* d/db exp(rate * b * Q) = V diag(rate * lambda * exp(rate * b * lambda)) V^{-1}
 * (= rate * Q * P, the factor used in Eq. 8). */
int oracle_transition_deriv(int S, const double *V, const double *Vi, const double *lam,
                            double rate, double b, double *dP)
{
    if (S < 1 || !V || !Vi || !lam || !dP) return OR_ERR_ARG;
    for (int s = 0; s < S; ++s)
        for (int u = 0; u < S; ++u) {
            double acc = 0.0;
            for (int k = 0; k < S; ++k)
                acc += V[s * S + k] * rate * lam[k] * exp(rate * b * lam[k]) * Vi[k * S + u];
            dP[s * S + u] = acc;
        }
    return OR_OK;
}

static int check_problem(const oracle_problem *pb, int c0, int c1)
{
    if (!pb || pb->N < 2 || pb->S < 1 || pb->R < 1 || pb->C < 0) return 0;
    if (!pb->ops || !pb->branch_lengths || !pb->evec || !pb->ievec || !pb->evals ||
        !pb->pi || !pb->cat_rates || !pb->cat_weights || !pb->pattern_weights) return 0;
    if (!pb->tip_states && !pb->tip_partials) return 0;
    if (c0 < 0 || c1 > pb->C || c0 > c1) return 0;
    return 1;
}

/* All transition matrices P[i][r] (and optionally dP[i][r]) for the 2N-2 branches. */
static double *all_matrices(const oracle_problem *pb, int deriv)
{
    int S = pb->S, R = pb->R, B = 2 * pb->N - 2;
    double *M = malloc(sizeof(double) * (size_t)B * R * S * S);
    if (!M) return NULL;
    for (int i = 0; i < B; ++i)
        for (int r = 0; r < R; ++r) {
            double *dst = M + ((size_t)i * R + r) * S * S;
            if (deriv)
                oracle_transition_deriv(S, pb->evec, pb->ievec, pb->evals,
                                        pb->cat_rates[r], pb->branch_lengths[i], dst);
            else
                oracle_transition(S, pb->evec, pb->ievec, pb->evals,
                                  pb->cat_rates[r] * pb->branch_lengths[i], dst);
        }
    return M;
}

/* Tip post-order partial of tip n, pattern c: indicator of the observed state,
 * all-ones when missing, or the given partial vector. */
static void tip_partial(const oracle_problem *pb, int n, int c, double *out /*[R][S]*/)
{
    int S = pb->S, R = pb->R;
    for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) {
            double v;
            if (pb->tip_partials)
                v = pb->tip_partials[((size_t)n * pb->C + c) * S + s];
            else {
                int st = pb->tip_states[(size_t)n * pb->C + c];
                v = (st >= S || st < 0) ? 1.0 : (st == s ? 1.0 : 0.0);
            }
            out[r * S + s] = v;
        }
}

/* y[s] = sum_t M[s][t] x[t] for one category (S x S matrix). */
static void matvec(int S, const double *M, const double *x, double *y)
{
    for (int s = 0; s < S; ++s) {
        double acc = 0.0;
        for (int t = 0; t < S; ++t) acc += M[s * S + t] * x[t];
        y[s] = acc;
    }
}

/* y[t] = sum_s M[s][t] x[s]  (transpose). */
static void matvec_t(int S, const double *M, const double *x, double *y)
{
    for (int t = 0; t < S; ++t) {
        double acc = 0.0;
        for (int s = 0; s < S; ++s) acc += M[s * S + t] * x[s];
        y[t] = acc;
    }
}

/* Divide v[0..n) by its max m (if m > 0) and return m (1 if rescale off). */
static double rescale_vec(double *v, int n, int rescale)
{
    if (!rescale) return 1.0;
    double m = 0.0;
    for (int k = 0; k < n; ++k) if (v[k] > m) m = v[k];
    if (!(m > 0.0)) return 1.0;
    for (int k = 0; k < n; ++k) v[k] /= m;
    return m;
}

/*
 * Post-order pass for one pattern (Eq. 2): fills p[node][r][s] for all nodes
 * and lsP[node] (accumulated log scale factors), and mscale[node] = the
 * factor each internal node was divided by.  Pmat = matrices to use (the
 * quadratic oracle passes a set with one branch substituted), `fixed_scale`
 * non-NULL => divide by those factors instead of computing new ones.
 */
static void post_order(const oracle_problem *pb, int c, const double *Pmat,
                       double *p, double *lsP, double *mscale,
                       const double *fixed_scale, int rescale, double *tmp)
{
    int N = pb->N, S = pb->S, R = pb->R, RS = R * S;
    for (int n = 0; n < N; ++n) {
        tip_partial(pb, n, c, p + (size_t)n * RS);
        lsP[n] = 0.0;
    }
    double *a = tmp, *b = tmp + S;
    for (int o = 0; o < N - 1; ++o) {
        int k = pb->ops[3 * o], i = pb->ops[3 * o + 1], j = pb->ops[3 * o + 2];
        for (int r = 0; r < R; ++r) {
            matvec(S, Pmat + ((size_t)i * R + r) * S * S, p + (size_t)i * RS + r * S, a);
            matvec(S, Pmat + ((size_t)j * R + r) * S * S, p + (size_t)j * RS + r * S, b);
            for (int s = 0; s < S; ++s) p[(size_t)k * RS + r * S + s] = a[s] * b[s];
        }
        double m;
        if (fixed_scale) {
            m = fixed_scale[k];
            for (int x = 0; x < RS; ++x) p[(size_t)k * RS + x] /= m;
        } else {
            m = rescale_vec(p + (size_t)k * RS, RS, rescale);
            if (mscale) mscale[k] = m;
        }
        lsP[k] = log(m) + lsP[i] + lsP[j];
    }
}

/* Eq. 3 at the root, in the scaled units of p_root. */
static double root_likelihood(const oracle_problem *pb, const double *proot)
{
    int S = pb->S, R = pb->R;
    double L = 0.0;
    for (int r = 0; r < R; ++r) {
        double acc = 0.0;
        for (int s = 0; s < S; ++s) acc += pb->pi[s] * proot[r * S + s];
        L += pb->cat_weights[r] * acc;
    }
    return L;
}

/*
 * logL, gradient (Eq. 6-8) and diagnostics over patterns [c0, c1).
 *   logL        : sum_c w_c log L_c                                   (Eq. 3)
 *   grad[i]     : sum_c w_c d_ic   for branches i = 0..2N-3           (Eq. 6-8)
 *   grad_abs[i] : sum_c w_c |d_ic| (condition scale for the parity metric, C17)
 *   site_logL[c-c0]           : log L_c
 *   node_logL[i*(c1-c0)+c-c0] : log sum_r P(gamma_r) p_i'q_i, i = 0..2N-2 (Eq. 5)
 * Any output pointer may be NULL.  Returns OR_ZERO_LIKELIHOOD (and logL =
 * -inf, gradient not accumulated for that pattern) if some L_c == 0; the
 * first such pattern index is written to *zero_pattern if non-NULL.
 */
int oracle_loglik_grad(const oracle_problem *pb, int c0, int c1, int rescale,
                       double *logL, double *grad, double *grad_abs,
                       double *site_logL, double *node_logL, int *zero_pattern)
{
    if (!check_problem(pb, c0, c1)) return OR_ERR_ARG;
    int N = pb->N, S = pb->S, R = pb->R, RS = R * S, nn = 2 * N - 1, B = 2 * N - 2;
    int root = 2 * N - 2;
    double *Pmat = all_matrices(pb, 0);
    double *p = malloc(sizeof(double) * (size_t)nn * RS);
    double *q = malloc(sizeof(double) * (size_t)nn * RS);
    double *lsP = malloc(sizeof(double) * nn), *lsQ = malloc(sizeof(double) * nn);
    double *tmp = malloc(sizeof(double) * 4 * S);
    double *Q = malloc(sizeof(double) * S * S);
    if (!Pmat || !p || !q || !lsP || !lsQ || !tmp || !Q) {
        free(Pmat); free(p); free(q); free(lsP); free(lsQ); free(tmp); free(Q);
        return OR_ERR_MEM;
    }
    /* Q = V diag(lambda) V^{-1} (the generator whose eigensystem was given). */
    for (int s = 0; s < S; ++s)
        for (int u = 0; u < S; ++u) {
            double acc = 0.0;
            for (int k = 0; k < S; ++k)
                acc += pb->evec[s * S + k] * pb->evals[k] * pb->ievec[k * S + u];
            Q[s * S + u] = acc;
        }
    if (grad) memset(grad, 0, sizeof(double) * B);
    if (grad_abs) memset(grad_abs, 0, sizeof(double) * B);
    double total = 0.0;
    int status = OR_OK;
    int nc = c1 - c0;
    for (int c = c0; c < c1; ++c) {
        /* ---- post-order (Eq. 2) ---- */
        post_order(pb, c, Pmat, p, lsP, NULL, NULL, rescale, tmp);
        /* ---- likelihood (Eq. 3) ---- */
        double L = root_likelihood(pb, p + (size_t)root * RS);
        double site = log(L) + lsP[root];
        if (site_logL) site_logL[c - c0] = site;
        if (!(L > 0.0)) {
            if (status == OR_OK && zero_pattern) *zero_pattern = c;
            status = OR_ZERO_LIKELIHOOD;
            total = -INFINITY;
            if (node_logL)
                for (int i = 0; i < nn; ++i) node_logL[(size_t)i * nc + c - c0] = -INFINITY;
            continue;
        }
        total += pb->pattern_weights[c] * site;
        /* ---- pre-order (Eq. 4), ops in reverse = parents before children ---- */
        for (int r = 0; r < R; ++r)
            for (int s = 0; s < S; ++s) q[(size_t)root * RS + r * S + s] = pb->pi[s];
        lsQ[root] = 0.0;
        for (int o = N - 2; o >= 0; --o) {
            int k = pb->ops[3 * o];
            for (int side = 0; side < 2; ++side) {
                int i = pb->ops[3 * o + 1 + side];       /* child whose q we form */
                int j = pb->ops[3 * o + 2 - side];       /* its sibling           */
                for (int r = 0; r < R; ++r) {
                    double *x = tmp, *y = tmp + S;
                    matvec(S, Pmat + ((size_t)j * R + r) * S * S, p + (size_t)j * RS + r * S, y);
                    for (int s = 0; s < S; ++s) x[s] = q[(size_t)k * RS + r * S + s] * y[s];
                    matvec_t(S, Pmat + ((size_t)i * R + r) * S * S, x, q + (size_t)i * RS + r * S);
                }
                double m = rescale_vec(q + (size_t)i * RS, RS, rescale);
                lsQ[i] = log(m) + lsQ[k] + lsP[j];
            }
        }
        /* ---- Eq. 5 per node (diagnostic) ---- */
        if (node_logL)
            for (int i = 0; i < nn; ++i) {
                double acc = 0.0;
                for (int r = 0; r < R; ++r) {
                    double d = 0.0;
                    for (int s = 0; s < S; ++s)
                        d += p[(size_t)i * RS + r * S + s] * q[(size_t)i * RS + r * S + s];
                    acc += pb->cat_weights[r] * d;
                }
                node_logL[(size_t)i * nc + c - c0] = log(acc) + lsP[i] + lsQ[i];
            }
        /* ---- gradient (Eq. 8): p' Q' q = sum_s p_s sum_t Q_ts q_t ---- */
        if (grad || grad_abs)
            for (int i = 0; i < B; ++i) {
                double num = 0.0, den = 0.0;
                for (int r = 0; r < R; ++r) {
                    const double *pi_ = p + (size_t)i * RS + r * S;
                    const double *qi_ = q + (size_t)i * RS + r * S;
                    double pq = 0.0, pQq = 0.0;
                    for (int s = 0; s < S; ++s) {
                        double Qtq = 0.0;
                        for (int t = 0; t < S; ++t) Qtq += Q[t * S + s] * qi_[t];
                        pQq += pi_[s] * Qtq;
                        pq += pi_[s] * qi_[s];
                    }
                    num += pb->cat_rates[r] * pb->cat_weights[r] * pQq;
                    den += pb->cat_weights[r] * pq;
                }
                double d = num / den;
                if (grad) grad[i] += pb->pattern_weights[c] * d;
                if (grad_abs) grad_abs[i] += pb->pattern_weights[c] * fabs(d);
            }
    }
    if (logL) *logL = total;
    free(Pmat); free(p); free(q); free(lsP); free(lsQ); free(tmp); free(Q);
    return status;
}

/*
 * O(N^2) gradient by derivative substitution: for each branch i,
 * re-run Eq. 2 with P_i replaced by dP_i/db_i and take
 *     d_ic = [sum_r P(gamma_r) pi' dp_root] / [sum_r P(gamma_r) pi' p_root],
 * both in the scaled units of the original pass (same per-node factors).
 */
int oracle_grad_quadratic(const oracle_problem *pb, int c0, int c1, double *grad)
{
    if (!check_problem(pb, c0, c1) || !grad) return OR_ERR_ARG;
    int N = pb->N, S = pb->S, R = pb->R, RS = R * S, nn = 2 * N - 1, B = 2 * N - 2;
    int root = 2 * N - 2;
    size_t msz = (size_t)S * S;
    double *Pmat = all_matrices(pb, 0), *dPmat = all_matrices(pb, 1);
    double *Psub = malloc(sizeof(double) * (size_t)B * R * msz);
    double *p = malloc(sizeof(double) * (size_t)nn * RS);
    double *dp = malloc(sizeof(double) * (size_t)nn * RS);
    double *lsP = malloc(sizeof(double) * nn), *mscale = malloc(sizeof(double) * nn);
    double *tmp = malloc(sizeof(double) * 4 * S);
    if (!Pmat || !dPmat || !Psub || !p || !dp || !lsP || !mscale || !tmp) {
        free(Pmat); free(dPmat); free(Psub); free(p); free(dp); free(lsP); free(mscale); free(tmp);
        return OR_ERR_MEM;
    }
    memset(grad, 0, sizeof(double) * B);
    int status = OR_OK;
    memcpy(Psub, Pmat, sizeof(double) * (size_t)B * R * msz);
    for (int c = c0; c < c1; ++c) {
        for (int n = 0; n < nn; ++n) mscale[n] = 1.0;
        post_order(pb, c, Pmat, p, lsP, mscale, NULL, 1, tmp);
        double L = root_likelihood(pb, p + (size_t)root * RS);
        if (!(L > 0.0)) { status = OR_ZERO_LIKELIHOOD; continue; }
        for (int i = 0; i < B; ++i) {
            memcpy(Psub + (size_t)i * R * msz, dPmat + (size_t)i * R * msz, sizeof(double) * R * msz);
            post_order(pb, c, Psub, dp, lsP, NULL, mscale, 1, tmp);
            memcpy(Psub + (size_t)i * R * msz, Pmat + (size_t)i * R * msz, sizeof(double) * R * msz);
            double dL = root_likelihood(pb, dp + (size_t)root * RS);
            grad[i] += pb->pattern_weights[c] * dL / L;
        }
    }
    free(Pmat); free(dPmat); free(Psub); free(p); free(dp); free(lsP); free(mscale); free(tmp);
    return status;
}
