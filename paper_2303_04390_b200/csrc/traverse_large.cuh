// traverse_large.cuh -- fused post-order + pre-order + per-edge gradient for
// large state spaces (SP = 32, 64: codon models, padded 61 -> 64).
//
// Same per-pattern programs as traverse_small.cuh (schedule.hpp), but one
// (pattern, category) vector of SP states is spread over G = SP/4 threads
// (4 states each) and lives in shared memory, because a matvec needs the
// whole input vector:  u = P p reads the transposed copy P' (so each thread's
// 4 outputs are 4 consecutive words for every input state t), q = P' x reads
// P row-major, Q u reads Q'.  A CTA owns TPL patterns x R categories.
// SIMT FMA with CTA barriers between phases.  Used only where no tensor-core
// variant applies: fp32 with partial tips, or fp32 with
// 64 < S <= 128; fp64 codon runs on DMMA (traverse_codon2.cuh), fp32 codon
// with state tips on tcgen05 TF32 (traverse_tc.cuh).
#pragma once
#include "common.cuh"

namespace pg {

template <typename Real, int SP>
struct LargeCfg {
    static constexpr int G = SP / 4;   // threads per vector
    static __host__ __device__ int tpl(int R) {   // patterns per CTA (power of two, <= 32)
        int t = 256 / (R * G);
        int p = 1;
        while (p * 2 <= t && p * 2 <= 32) p *= 2;
        return p;
    }
    static __host__ __device__ int threads(int R) { return tpl(R) * R * G; }
    static __host__ __device__ size_t vec_bytes(int R) { return (size_t)tpl(R) * R * SP * sizeof(Real); }
    // A, B, X0, X1, T buffers + stack + reduction scratch
    static __host__ __device__ size_t smem(int R, int depth) {
        return (5 + (size_t)depth) * vec_bytes(R) + (size_t)tpl(R) * R * (4 * sizeof(double) + 2 * sizeof(int)) +
               (size_t)tpl(R) * sizeof(double) * 2;
    }
};

template <typename Real>
__device__ __forceinline__ Real group_sum(Real v, int G) {
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ int group_max_int(int v, int G) {
    for (int o = G / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <typename Real, int SP>
__global__ void __launch_bounds__(256) traverse_large_kernel(const TravArgs a) {
    using Cfg = LargeCfg<Real, SP>;
    constexpr int G = Cfg::G;
    extern __shared__ __align__(16) unsigned char smem[];
    const int R = a.R, N = a.N, S = a.S;
    const int TPL = Cfg::tpl(R);
    const int nvec = TPL * R;
    const int tid = threadIdx.x;
    const int g = tid % G;                 // state chunk: states 4g .. 4g+3
    const int vec = tid / G;               // = pl * R + r
    const int r = vec % R, pl = vec / R;
    const int tile = blockIdx.x;
    const int pat = tile * TPL + pl;
    const int root = 2 * N - 2;
    const size_t Cpad = (size_t)a.Cpad, mat = (size_t)SP * SP;
    const int s0 = 4 * g;

    Real *bufA = reinterpret_cast<Real *>(smem);
    Real *bufB = bufA + (size_t)nvec * SP;
    Real *bufX0 = bufB + (size_t)nvec * SP;
    Real *bufX1 = bufX0 + (size_t)nvec * SP;
    Real *bufT = bufX1 + (size_t)nvec * SP;
    Real *stack = bufT + (size_t)nvec * SP;
    double *rd = reinterpret_cast<double *>(stack + (size_t)a.depth * nvec * SP);   // [4][nvec]
    int *ri = reinterpret_cast<int *>(rd + 4 * nvec);                               // [2][nvec]
    double *pd = reinterpret_cast<double *>(ri + 2 * nvec + (2 * nvec & 1));         // [2][TPL]

    const Real *__restrict__ P = static_cast<const Real *>(a.P);
    const Real *__restrict__ PT = static_cast<const Real *>(a.PT);
    const Real *__restrict__ QT = static_cast<const Real *>(a.QT);
    const Real *__restrict__ pig = static_cast<const Real *>(a.pi);
    const Real *__restrict__ tipP = static_cast<const Real *>(a.tip_partials);
    Real *__restrict__ U = static_cast<Real *>(a.u);
    const double wr = a.cat_w[r], gr = a.cat_g[r];
    const double Wc = a.pat_w[pat];

    auto vslot = [&](Real *buf) -> Real * { return buf + (size_t)vec * SP; };
    auto stack_at = [&](int slot) -> Real * { return stack + ((size_t)slot * nvec + vec) * SP; };
    auto u_global = [&](int node) -> Real * { return U + (((size_t)(node - N) * R + r) * Cpad + pat) * SP; };

    // chunk of y = M x where Mt = M' is given (y[s] = sum_t Mt[t][s] x[t]), x full in smem
    auto mv_from_T = [&](Real (&y)[4], const Real *__restrict__ Mt, const Real *x) {
        y[0] = y[1] = y[2] = y[3] = 0;
        for (int t = 0; t < SP; ++t) {
            const Real xt = x[t];
            const Real *row = Mt + (size_t)t * SP + s0;
            y[0] = fma(__ldg(row + 0), xt, y[0]);
            y[1] = fma(__ldg(row + 1), xt, y[1]);
            y[2] = fma(__ldg(row + 2), xt, y[2]);
            y[3] = fma(__ldg(row + 3), xt, y[3]);
        }
    };
    // tip vector chunk for `code` (state: column of P; missing: P 1; partial: P p)
    auto tip_chunk = [&](Real (&u)[4], int code, Real *scratch) {
        const int node = code & ~kTipPartialBit;
        const Real *PTm = PT + ((size_t)node * R + r) * mat;
        if (code & kTipPartialBit) {
            const Real *src = tipP + ((size_t)node * Cpad + pat) * SP;
            Real *x = vslot(scratch);
            for (int k = 0; k < 4; ++k) x[s0 + k] = src[s0 + k];
            __syncwarp();
            mv_from_T(u, PTm, x);
        } else {
            const int st = a.tip_states[(size_t)node * Cpad + pat];
            if (st < S) {
                for (int k = 0; k < 4; ++k) u[k] = __ldg(PTm + (size_t)st * SP + s0 + k);
            } else {
                for (int k = 0; k < 4; ++k) u[k] = 0;
                for (int t = 0; t < SP; ++t)
                    for (int k = 0; k < 4; ++k) u[k] += __ldg(PTm + (size_t)t * SP + s0 + k);
            }
        }
    };

    // ---------------- post program (Eq. 2, Eq. 3) ----------------------------
    int E = 0;
    double logl_local = 0.0;
    for (int n = 0; n < N - 1; ++n) {
        const Op4 op = a.post[n];
        const int cs[2] = {op.y, op.z};
        Real uc[2][4];
        for (int c = 0; c < 2; ++c) {
            if (cs[c] < 0) {
                const Real *src = stack_at(-cs[c] - 1);
                for (int k = 0; k < 4; ++k) uc[c][k] = src[s0 + k];
            } else {
                tip_chunk(uc[c], cs[c], c == 0 ? bufT : bufX1);
            }
        }
        Real p[4];
        for (int k = 0; k < 4; ++k) p[k] = uc[0][k] * uc[1][k];
        if (op.x == root) {
            double Lr = 0.0;
            for (int k = 0; k < 4; ++k) Lr += (double)__ldg(pig + s0 + k) * (double)p[k];
            Lr = group_sum(Lr, G);
            if (g == 0) rd[vec] = wr * Lr;
            __syncthreads();
            if (g == 0 && r == 0) {
                double L = 0.0;
                for (int q = 0; q < R; ++q) L += rd[pl * R + q];
                if (pat < a.C) {
                    if (!(L > 0.0) || !isfinite(L)) atomicMin(a.status, pat);
                    logl_local = Wc * (log(L) + (double)E * 0.69314718055994530942);
                }
                pd[pl] = logl_local;
            }
            __syncthreads();
            if (tid == 0) {
                double v = 0.0;
                for (int q = 0; q < TPL; ++q) v += pd[q];
                a.logl_part[tile] = v;
            }
        } else {
            Real m = p[0];
            for (int k = 1; k < 4; ++k) m = p[k] > m ? p[k] : m;
            int e = group_max_int(exponent_of(m), G);
            if (g == 0) ri[vec] = e;
            __syncthreads();
            e = ri[pl * R];
            for (int q = 1; q < R; ++q) e = max(e, ri[pl * R + q]);
            E += e;
            Real *x = vslot(bufX0);
            for (int k = 0; k < 4; ++k) x[s0 + k] = scale_pow2(p[k], -e);
            __syncwarp();
            Real u[4];
            mv_from_T(u, PT + ((size_t)op.x * R + r) * mat, x);
            Real *dst = u_global(op.x), *st = stack_at(op.w);
            for (int k = 0; k < 4; ++k) { dst[s0 + k] = u[k]; st[s0 + k] = u[k]; }
        }
        __syncthreads();
    }
    __threadfence_block();
    __syncthreads();

    // ---------------- pre program (Eq. 4) + gradient (Eq. 8) ------------------
    for (int n = 0; n < N - 1; ++n) {
        const Op4 op = a.pre[n];
        Real q[4];
        if (op.x < 0) for (int k = 0; k < 4; ++k) q[k] = __ldg(pig + s0 + k);
        else { const Real *src = stack_at(op.x); for (int k = 0; k < 4; ++k) q[k] = src[s0 + k]; }
        const int cs[2] = {op.y, op.z};
        const int slots[2] = {(op.w & 0xffff) - 1, (op.w >> 16) - 1};
        int node[2];
        Real *ubuf[2] = {vslot(bufA), vslot(bufB)};
        for (int c = 0; c < 2; ++c) {
            node[c] = cs[c] & ~kTipPartialBit;
            Real u[4];
            if (node[c] >= N) {
                const Real *src = u_global(node[c]);
                for (int k = 0; k < 4; ++k) u[k] = src[s0 + k];
            } else {
                tip_chunk(u, cs[c], c == 0 ? bufT : bufX1);
            }
            for (int k = 0; k < 4; ++k) ubuf[c][s0 + k] = u[k];
        }
        __syncthreads();
        Real *xbuf[2] = {vslot(bufX0), vslot(bufX1)};
        for (int c = 0; c < 2; ++c)
            for (int k = 0; k < 4; ++k) xbuf[c][s0 + k] = q[k] * ubuf[1 - c][s0 + k];
        __syncwarp();
        __syncthreads();
        for (int c = 0; c < 2; ++c) {
            Real Qu[4];
            mv_from_T(Qu, QT, ubuf[c]);                      // (Q u)[s] = sum_t Q[s][t] u[t]
            Real num = 0, den = 0;
            for (int k = 0; k < 4; ++k) {
                num = fma(xbuf[c][s0 + k], Qu[k], num);
                den = fma(xbuf[c][s0 + k], ubuf[c][s0 + k], den);
            }
            double dn = group_sum((double)num, G), dd = group_sum((double)den, G);
            if (g == 0) { rd[(2 * c) * nvec + vec] = gr * wr * dn; rd[(2 * c + 1) * nvec + vec] = wr * dd; }
            if (slots[c] >= 0) {
                // q_c[t] = sum_s P[s][t] x[s]: row-major P gives 4 consecutive t
                const Real *Pm = P + ((size_t)node[c] * R + r) * mat;
                Real qc[4] = {0, 0, 0, 0};
                for (int s = 0; s < SP; ++s) {
                    const Real xs = xbuf[c][s];
                    const Real *row = Pm + (size_t)s * SP + s0;
                    for (int k = 0; k < 4; ++k) qc[k] = fma(__ldg(row + k), xs, qc[k]);
                }
                Real m = qc[0];
                for (int k = 1; k < 4; ++k) m = qc[k] > m ? qc[k] : m;
                int e = group_max_int(exponent_of(m), G);
                if (g == 0) ri[c * nvec + vec] = e;
                Real *dst = stack_at(slots[c]);
                for (int k = 0; k < 4; ++k) dst[s0 + k] = qc[k];
            }
        }
        __syncthreads();
        for (int c = 0; c < 2; ++c) {
            if (g == 0 && r == 0) {
                double num = 0.0, den = 0.0;
                for (int q2 = 0; q2 < R; ++q2) {
                    num += rd[(2 * c) * nvec + pl * R + q2];
                    den += rd[(2 * c + 1) * nvec + pl * R + q2];
                }
                pd[c * TPL + pl] = (Wc != 0.0) ? Wc * (num / den) : 0.0;
            }
            if (slots[c] >= 0) {
                int e = ri[c * nvec + pl * R];
                for (int q2 = 1; q2 < R; ++q2) e = max(e, ri[c * nvec + pl * R + q2]);
                Real *dst = stack_at(slots[c]);
                for (int k = 0; k < 4; ++k) dst[s0 + k] = scale_pow2(dst[s0 + k], -e);
            }
        }
        __syncthreads();
        if (tid < 2) {
            double v = 0.0;
            for (int q2 = 0; q2 < TPL; ++q2) v += pd[tid * TPL + q2];
            a.grad_part[(size_t)node[tid] * a.n_tiles + tile] = v;
        }
        __syncthreads();
    }
}

}  // namespace pg
