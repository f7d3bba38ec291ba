// aux_kernels.cuh -- transition matrices (A1) and the site/branch reduction (A6).
#pragma once
#include "common.cuh"

namespace pg {

// First statement of the small-S A1 kernels: lets the traversal (launched
// with programmatic stream serialization) start its setup while A1 runs --
// the traversal waits (griddepcontrol.wait) before it reads any matrix --
// and resets the evaluation's status words (first zero-likelihood pattern,
// stall flag) in place of two memset nodes.
__device__ __forceinline__ void pdl_trigger_and_reset(int *status) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (status && blockIdx.x == 0 && threadIdx.x == 0) {
        status[0] = 0x7f7f7f7f;
        status[1] = 0;
        status[2] = 0;                  // finished-CTA count of a fused A6
    }
}

// A1 -- Eq. 1: P^{(r)}(b_i) = V diag(exp(gamma_r b_i lambda)) V^{-1}
// for every branch i and category r, in the compute precision, zero padded to
// SP x SP (category blocks `cs` Reals apart).  One CTA per (branch, category): the S exponentials go to shared
// memory, then every thread forms entries of P and (optionally) P'.  Padded
// rows/columns are exactly 0.  The work is ~2% of an evaluation.
// Evaluated as P = M0 + V diag(expm1(gamma_r b_i lambda)) V^{-1} with
// M0 = V V^{-1} formed once on the host (equal to Eq. 1 in exact arithmetic;
// the summed terms shrink with |gamma b lambda|, so short branches lose less
// to cancellation, R15b).
template <typename Real, int SP>
__global__ void __launch_bounds__(256) pmat_kernel(const double *__restrict__ V,
                                                   const double *__restrict__ Vi,
                                                   const double *__restrict__ M0,
                                                   const double *__restrict__ lam,
                                                   const double *__restrict__ rates,
                                                   const double *__restrict__ bl, int S, int R,
                                                   int cs, Real *__restrict__ P, Real *__restrict__ PT,
                                                   int *__restrict__ status, unsigned char *__restrict__ recp,
                                                   const int *__restrict__ pdst, unsigned char *__restrict__ recq,
                                                   const int *__restrict__ qdst) {
    __shared__ double e[SP];
    pdl_trigger_and_reset(status);
    const int br = blockIdx.x;          // branch * R + r
    const int r = br % R, b = br / R;
    const double t = rates[r] * bl[b];
    for (int k = threadIdx.x; k < SP; k += blockDim.x) e[k] = k < S ? expm1(lam[k] * t) : 0.0;
    __syncthreads();
    Real *Pm = P + (size_t)br * cs;     // cs = category stride (>= SP*SP, zero padded)
    // grouped small-S staging: the branch's slot in its post-order step record
    Real *Rm = nullptr, *Qm = nullptr;
    if (recp && pdst[b] >= 0) Rm = reinterpret_cast<Real *>(recp + pdst[b]) + (size_t)r * cs;
    if (recq && qdst[b] >= 0) Qm = reinterpret_cast<Real *>(recq + qdst[b]) + (size_t)r * cs;   // pre-order record
    Real *PTm = PT ? PT + (size_t)br * SP * SP : nullptr;
    for (int idx = threadIdx.x; idx < SP * SP; idx += blockDim.x) {
        const int s = idx / SP, u = idx % SP;
        double acc = 0.0;
        if (s < S && u < S) {
            for (int k = 0; k < S; ++k) acc += V[s * S + k] * e[k] * Vi[k * S + u];
            acc += M0[idx];
        }
        Pm[idx] = (Real)acc;
        if (Rm) Rm[idx] = (Real)acc;
        if (Qm) Qm[idx] = (Real)acc;
        if (PTm) PTm[u * SP + s] = (Real)acc;
    }
    // a category pad that holds SP Reals carries P 1 (row sums, summed in
    // column order like the traversal's missing-state tip gather): the
    // small-S kernel then reads column `state` or this vector without a branch
    if (cs >= SP * SP + SP) {
        __syncthreads();
        for (int s = threadIdx.x; s < SP; s += blockDim.x) {
            Real acc = Pm[s * SP];
            for (int u = 1; u < SP; ++u) acc += Pm[s * SP + u];
            Pm[SP * SP + s] = acc;
            if (Rm) Rm[SP * SP + s] = acc;
            if (Qm) Qm[SP * SP + s] = acc;
        }
    }
}

// A1 for the FP64 tensor-core S = 16 traversal (traverse_small.cuh,
// small_mma): P = M0 + V diag(expm1(gamma_r b_i lambda)) V^{-1} as above,
// written as the branch's three layouts [B of u = P p][B of q = x P][row-major,
// stride 17, column 16 = P 1] (fragment order: element (kt, nt, lane) at
// (kt * 2 + nt) * 32 + lane, k = 4 kt + lane % 4, n = 8 nt + lane / 4, output
// state sigma(n)).  One CTA per branch (R = 1).
__global__ void __launch_bounds__(256) pmat16_mma_kernel(const double *__restrict__ V, const double *__restrict__ Vi,
                                                         const double *__restrict__ M0,
                                                         const double *__restrict__ lam,
                                                         const double *__restrict__ rates,
                                                         const double *__restrict__ bl, int S, int rec,
                                                         double *__restrict__ P, int *__restrict__ status,
                                                         const MaskTable mt, unsigned char *__restrict__ recp,
                                                         const int *__restrict__ pdst, unsigned char *__restrict__ recq,
                                                         const int *__restrict__ qdst) {
    __shared__ double e[16], Ps[16][17], Vs[256], Vis[256];
    pdl_trigger_and_reset(status);
    const int b = blockIdx.x;
    const double t = rates[0] * bl[b];
    // V and V^-1 staged once (one load per thread) instead of 2 S loads per
    // thread from L2 inside the sum
    if (threadIdx.x < S * S) {
        Vs[threadIdx.x] = V[threadIdx.x];
        Vis[threadIdx.x] = Vi[threadIdx.x];
    }
    const double m0 = M0[threadIdx.x];
    for (int k = threadIdx.x; k < 16; k += blockDim.x) e[k] = k < S ? expm1(lam[k] * t) : 0.0;
    __syncthreads();
    {
        const int s = threadIdx.x >> 4, u = threadIdx.x & 15;
        double acc = 0.0;
        if (s < S && u < S) {
            for (int k = 0; k < S; ++k) acc += Vs[s * S + k] * e[k] * Vis[k * S + u];
            acc += m0;
        }
        Ps[s][u] = acc;
    }
    __syncthreads();
    double *R0 = P + (size_t)b * rec;
    // element i of layout lay (0: B of u = P p, 1: B of q = x P, both in
    // fragment order over 256 entries; 2: row-major, stride 17, column 16 =
    // P 1, mask-tip columns as sums), straight from the shared-memory P
    auto elem = [&](int lay, int i) -> double {
        if (lay < 2) {
            if (i >= 256) return 0.0;
            const int f = i >> 5, l = i & 31;
            const int k = 4 * (f >> 1) + (l & 3), n = 8 * (f & 1) + (l >> 2);
            const int sg = 4 * (2 * (n >> 3) + (n & 1)) + ((n & 7) >> 1);
            return lay == 0 ? Ps[sg][k] : Ps[k][sg];
        }
        const int row = i / 17, col = i % 17;
        double v = 0.0;
        if (col == 16) {
            for (int c = 0; c < 16; ++c) v += Ps[row][c];
        } else if (mt.n < 0) {
            v = Ps[row][col];
        } else if (col < mt.n) {                 // coded mask tips: column m = sum over mask m's states
            for (int c = 0; c < 16; ++c)
                if (mt.mask[col] >> c & 1) v += Ps[row][c];
        }
        return v;
    };
    // the branch's three layouts, and the staging-record slots that read it
    // (traverse_small_kernel GRP variant; destination = byte offset * 4 + layout)
    const int dp = recp ? pdst[b] : -1, dq = recp ? qdst[b] : -1;
    for (int i = threadIdx.x; i < 16 * 17; i += blockDim.x) {
        if (i < 256) {
            R0[i] = elem(0, i);
            R0[16 * 17 + i] = elem(1, i);
        }
        R0[2 * 16 * 17 + i] = elem(2, i);
        if (dp >= 0) reinterpret_cast<double *>(recp + (dp >> 2))[i] = elem(dp & 3, i);
        if (dq >= 0) reinterpret_cast<double *>(recq + (dq >> 2))[i] = elem(dq & 3, i);
    }
}

// A1 for the FP64 tensor-core S = 4, R = 4 traversal (traverse_small.cuh,
// small_tc): thread (category r, lane l) forms the two B-operand entries
// P_r[(l/4)/2][l%4] (u = P p) and P_r[l%4][(l/4)/2] (q = x P), each as
// M0 + sum_k V diag(expm1(gamma_r b lambda)) V^{-1}.  One CTA per branch.
__global__ void __launch_bounds__(128) pmat4_mma_kernel(const double *__restrict__ V, const double *__restrict__ Vi,
                                                        const double *__restrict__ M0,
                                                        const double *__restrict__ lam,
                                                        const double *__restrict__ rates,
                                                        const double *__restrict__ bl, int S, int rec,
                                                        double *__restrict__ P, int *__restrict__ status) {
    pdl_trigger_and_reset(status);
    const int b = blockIdx.x, r = threadIdx.x >> 5, l = threadIdx.x & 31;
    const double t = rates[r] * bl[b];
    double e[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) e[k] = k < S ? expm1(lam[k] * t) : 0.0;
    auto entry = [&](int s, int u) {
        if (s >= S || u >= S) return 0.0;
        double acc = 0.0;
        for (int k = 0; k < S; ++k) acc += V[s * S + k] * e[k] * Vi[k * S + u];
        return acc + M0[s * 4 + u];
    };
    double *R0 = P + (size_t)b * rec;
    R0[r * 32 + l] = entry((l >> 2) >> 1, l & 3);
    R0[128 + r * 32 + l] = entry(l & 3, (l >> 2) >> 1);
}

// A6 -- Eq. 6 column sum, deterministic: block b < B sums the
// per-tile gradient partials of branch b, block B the per-tile logL partials,
// in a fixed order (strided serial sums, then a fixed smem tree).  No atomics,
// so fp64 results are bitwise reproducible run to run.
// Grouped post-order staging of the small-S traversal: tip-code windows per
// (CTA, post step, child) -> ts[cta][m][2][tipw] (child = tip with state
// codes; other entries left as they are).  Window = the tip's codes of the
// CTA's patterns from its first pattern rounded down to 16 (the same window
// the per-step copies take); bytes past the padded row are not read.
__global__ void tipstream_kernel(const Op4 *__restrict__ post, const uint8_t *__restrict__ tips,
                                 uint8_t *__restrict__ ts, int N, int Cpad, int cta_pats, int tipw) {
    const int m = blockIdx.x, cta = blockIdx.y;     // steps on x (N - 1 may exceed 65535)
    const Op4 op = post[m];
    const int p0 = cta * cta_pats, lead = p0 & 15;
    for (int c = 0; c < 2; ++c) {
        const int code = c ? op.z : op.y;
        if (code < 0 || (code & kTipPartialBit)) continue;
        const uint8_t *src = tips + (size_t)code * Cpad + (p0 - lead);
        uint8_t *dst = ts + (((size_t)cta * (N - 1) + m) * 2 + c) * tipw;
        for (int i = threadIdx.x; i < tipw; i += blockDim.x) dst[i] = (p0 - lead + i < Cpad) ? src[i] : (uint8_t)0;
    }
}

__global__ void __launch_bounds__(256) reduce_kernel(const double *__restrict__ grad_part,
                                                     const double *__restrict__ logl_part,
                                                     int B, int n_tiles, double *__restrict__ out) {
    __shared__ double sh[256];
    asm volatile("griddepcontrol.wait;" ::: "memory");     // the traversal's partials (PDL launch)
    const int b = blockIdx.x;
    const double *src = (b < B) ? grad_part + (size_t)b * n_tiles : logl_part;
    double acc = 0.0;
    for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) acc += src[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[b < B ? 1 + b : 0] = sh[0];
}

// NEXT-4: leapfrog pieces over theta = log b (include/phylograd.h pg_hmc_leapfrog)
// drift: theta += eps M^-1 p, b = exp(theta) into the instance's branch lengths
__global__ void hmc_drift_kernel(double *__restrict__ theta, const double *__restrict__ p,
                                 const double *__restrict__ inv_mass, double eps, double *__restrict__ bl, int B) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    const double th = theta[i] + eps * (inv_mass ? inv_mass[i] : 1.0) * p[i];
    theta[i] = th;
    bl[i] = exp(th);
}
// kick: grad = b o dlogL/db + 1 (from out = [logL, g]); p += coef grad
__global__ void hmc_kick_kernel(const double *__restrict__ bl, const double *__restrict__ out, double coef,
                                double *__restrict__ p, double *__restrict__ grad_theta, int B) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    const double g = bl[i] * out[1 + i] + 1.0;
    if (grad_theta) grad_theta[i] = g;
    p[i] += coef * g;
}

}  // namespace pg

namespace pg {

// ---- time-tree (clock) parameterisation, SURVEY §8(f) NEXT-1 / C23 ---------
// b_i = rho_i (h_parent(i) - h_i).  One thread per node: copies
// the heights and rate scalars into the instance (src may equal dst; rho_src
// NULL = all 1) and forms b for the 2N-2 branches.
__global__ void __launch_bounds__(256) clock_bl_kernel(const int *__restrict__ parent, const double *h_src,
                                                       const double *rho_src, int N, double *h_dst,
                                                       double *rho_dst, double *__restrict__ bl) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int B = 2 * N - 2;
    if (i > B) return;
    const double hi = h_src[i];
    if (i < B) {
        const double r = rho_src ? rho_src[i] : 1.0;
        const double tau = h_src[parent[i]] - hi;
        bl[i] = r * tau;
        rho_dst[i] = r;
    }
    h_dst[i] = hi;
}

// Chain rule on g = out[1..2N-2] (out[0] = logL), one thread per node k:
//   dlogL/drho_k = tau_k g_k;
//   dlogL/dh_k   = sum over children c of rho_c g_c (tau_c grows with h_k)
//                  - rho_k g_k (tau_k shrinks), the root having no branch.
__global__ void __launch_bounds__(256) clock_grad_kernel(const int *__restrict__ parent, const int *__restrict__ ca,
                                                         const int *__restrict__ cb, const double *__restrict__ h,
                                                         const double *__restrict__ rho, int N,
                                                         const double *__restrict__ out, double *grad_rho,
                                                         double *grad_h) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int B = 2 * N - 2;
    if (k > B) return;
    const double *g = out + 1;
    const double own = k < B ? rho[k] * g[k] : 0.0;
    if (grad_rho && k < B) grad_rho[k] = (h[parent[k]] - h[k]) * g[k];
    if (grad_h) {
        double d = 0.0;
        if (k >= N) d = rho[ca[k]] * g[ca[k]] + rho[cb[k]] * g[cb[k]];
        grad_h[k] = d - own;
    }
}

// Set sums sum_{i in set s} tau_i g_i: one CTA per set, fixed-order strided
// sums then a fixed shared-memory tree (deterministic, no atomics).
__global__ void __launch_bounds__(256) clock_set_kernel(const int *__restrict__ parent, const double *__restrict__ h,
                                                        const int *__restrict__ bset, int N,
                                                        const double *__restrict__ out, double *set_sums) {
    __shared__ double sh[256];
    const int s = blockIdx.x, B = 2 * N - 2;
    double acc = 0.0;
    for (int i = threadIdx.x; i < B; i += blockDim.x)
        if (bset[i] == s) acc += (h[parent[i]] - h[i]) * out[1 + i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) set_sums[s] = sh[0];
}

}  // namespace pg
