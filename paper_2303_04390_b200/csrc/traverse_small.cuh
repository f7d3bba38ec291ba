// traverse_small.cuh -- fused post-order + pre-order + per-edge gradient for
// small state spaces (SP = 4, 8, 16): the HBM-bound nucleotide and
// Markov-modulated paths.
//
// Design.  Site patterns are independent, so
// a CTA owns a tile of 32 patterns for ALL rate categories and walks the whole
// tree for them in one launch -- no per-level launches, no grid-wide sync:
//   * warp w = rate category r (CTA = R warps), lane = pattern of the tile;
//     every lane of a warp reads the same transition matrix (broadcast loads)
//     and each thread keeps the SP states of its (pattern, category) vector
//     in registers.
//   * post program (Eq. 2): p_k = u_a o u_b, exact power-of-two rescale shared
//     across categories, u_k = P_k p_k is streamed to HBM once (16-B vector
//     stores) and kept on a per-thread shared-memory stack for the parent.
//   * root (Eq. 3): L_c = sum_r P(gamma_r) pi' p_root; logL partial per tile.
//   * pre program (Eq. 4 in the branch-top form of SURVEY §0): for parent k
//     with children a, b: x_a = q_k o u_b, x_b = q_k o u_a;
//       Eq. 8 numerator   sum_r gamma_r P(gamma_r) x_a' Q u_a   (= p'Q'q)
//       Eq. 8 denominator sum_r P(gamma_r) x_a' u_a             (= p'q)
//     and q_a = P_a' x_a for internal children (pushed on the stack).  u_a,
//     u_b are the only HBM reads; the static program lets every thread
//     prefetch them `prefetch` steps ahead with cp.async into a smem ring.
//   * cross-category sums/maxima go through a double-buffered smem exchange
//     with one __syncthreads per step.
// HBM traffic per evaluation is 2 (N-2) R C SP sizeof(Real) (u written once,
// read once) + tip codes, versus 5 (N-2) V for a level-batched schedule.
#pragma once
#include "common.cuh"

namespace pg {

template <typename Real, int SP>
struct SmallSmem {
    // byte offsets inside dynamic smem
    static __host__ __device__ size_t red_bytes(int R) { return (size_t)2 * 4 * R * 32 * sizeof(double) + 2 * 2 * R * 32 * sizeof(int); }
    static __host__ __device__ size_t ring_bytes(int R, int D) { return (size_t)D * 2 * R * 32 * SP * sizeof(Real); }
    static __host__ __device__ size_t stack_bytes(int R, int depth) { return (size_t)depth * R * 32 * SP * sizeof(Real); }
    static __host__ __device__ size_t total(int R, int D, int depth) {
        return red_bytes(R) + ring_bytes(R, D) + stack_bytes(R, depth);
    }
};

template <typename Real, int SP>
struct VecT { Real v[SP]; };

template <typename Real, int SP>
__device__ __forceinline__ void load_vec(Real (&d)[SP], const Real *src) {
    if constexpr (sizeof(Real) * SP % 16 == 0) {
#pragma unroll
        for (int i = 0; i < SP * (int)sizeof(Real) / 16; ++i) {
            float4 t = *reinterpret_cast<const float4 *>((const char *)src + 16 * i);
            memcpy((char *)d + 16 * i, &t, 16);
        }
    } else {
#pragma unroll
        for (int i = 0; i < SP; ++i) d[i] = src[i];
    }
}
// read-only (texture path) vector load of SP values from global memory
template <typename Real, int SP>
__device__ __forceinline__ void ldg_vec(Real (&d)[SP], const Real *src) {
    if constexpr (sizeof(Real) * SP % 16 == 0) {
#pragma unroll
        for (int i = 0; i < SP * (int)sizeof(Real) / 16; ++i) {
            float4 t = __ldg(reinterpret_cast<const float4 *>((const char *)src + 16 * i));
            memcpy((char *)d + 16 * i, &t, 16);
        }
    } else {
#pragma unroll
        for (int i = 0; i < SP; ++i) d[i] = __ldg(src + i);
    }
}

template <typename Real, int SP>
__device__ __forceinline__ void store_vec(Real *dst, const Real (&d)[SP]) {
    if constexpr (sizeof(Real) * SP % 16 == 0) {
#pragma unroll
        for (int i = 0; i < SP * (int)sizeof(Real) / 16; ++i) {
            float4 t;
            memcpy(&t, (const char *)d + 16 * i, 16);
            *reinterpret_cast<float4 *>((char *)dst + 16 * i) = t;
        }
    } else {
#pragma unroll
        for (int i = 0; i < SP; ++i) dst[i] = d[i];
    }
}

// u = column `s` of P (observed tip state), or P * 1 (missing, s >= S).
template <typename Real, int SP>
__device__ __forceinline__ void tip_column(Real (&u)[SP], const Real *__restrict__ Pm, int s, int S) {
    if (s < S) {
#pragma unroll
        for (int x = 0; x < SP; ++x) u[x] = ldg(Pm + x * SP + s);
    } else {
#pragma unroll
        for (int x = 0; x < SP; ++x) {
            Real acc = 0;
#pragma unroll
            for (int t = 0; t < SP; ++t) acc += ldg(Pm + x * SP + t);
            u[x] = acc;
        }
    }
}

// y = P x  (y[s] = sum_t P[s][t] x[t]) -- Eq. 2 / branch-top post vector.
template <typename Real, int SP>
__device__ __forceinline__ void matvec(Real (&y)[SP], const Real *__restrict__ Pm, const Real (&x)[SP]) {
#pragma unroll
    for (int s = 0; s < SP; ++s) {
        Real row[SP];
        ldg_vec<Real, SP>(row, Pm + s * SP);   // broadcast (same address in the warp)
        Real acc = 0;
#pragma unroll
        for (int t = 0; t < SP; ++t) acc = fma(row[t], x[t], acc);
        y[s] = acc;
    }
}

// y = P' x  (y[t] = sum_s P[s][t] x[s]) -- Eq. 4.
template <typename Real, int SP>
__device__ __forceinline__ void matvec_t(Real (&y)[SP], const Real *__restrict__ Pm, const Real (&x)[SP]) {
#pragma unroll
    for (int t = 0; t < SP; ++t) y[t] = 0;
#pragma unroll
    for (int s = 0; s < SP; ++s) {
        Real row[SP];
        ldg_vec<Real, SP>(row, Pm + s * SP);
#pragma unroll
        for (int t = 0; t < SP; ++t) y[t] = fma(row[t], x[s], y[t]);
    }
}

template <typename Real, int SP>
__device__ __forceinline__ Real vmax(const Real (&v)[SP]) {
    Real m = v[0];
#pragma unroll
    for (int i = 1; i < SP; ++i) m = v[i] > m ? v[i] : m;
    return m;
}

template <typename Real, int SP>
__global__ void __launch_bounds__(SP <= 8 ? 512 : 256) traverse_small_kernel(const TravArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int R = a.R, N = a.N, D = a.prefetch;
    const int nthr = R * 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r = warp;                                  // rate category of this warp
    const int tid = threadIdx.x;
    const int tile = blockIdx.x;
    const int pat = tile * 32 + lane;                    // < Cpad
    const int root = 2 * N - 2;
    const size_t Cpad = (size_t)a.Cpad;
    const size_t mat = (size_t)SP * SP;

    double *redd = reinterpret_cast<double *>(smem);                       // [2][4][R*32]
    int *redi = reinterpret_cast<int *>(smem + (size_t)2 * 4 * nthr * sizeof(double));  // [2][2][R*32]
    Real *ring = reinterpret_cast<Real *>(smem + SmallSmem<Real, SP>::red_bytes(R));    // [D][2][R*32][SP]
    Real *stack = ring + (size_t)D * 2 * nthr * SP;                                       // [depth][R*32][SP]

    const Real *__restrict__ P = static_cast<const Real *>(a.P);
    const Real *__restrict__ Qg = static_cast<const Real *>(a.Q);
    const Real *__restrict__ pig = static_cast<const Real *>(a.pi);
    const Real *__restrict__ tipP = static_cast<const Real *>(a.tip_partials);
    Real *__restrict__ U = static_cast<Real *>(a.u);
    const double wr = a.cat_w[r], gr = a.cat_g[r];
    const double Wc = a.pat_w[pat];

    auto ring_at = [&](int n, int child) -> Real * {
        return ring + (((size_t)(n % D) * 2 + child) * nthr + tid) * SP;
    };
    auto stack_at = [&](int slot) -> Real * { return stack + ((size_t)slot * nthr + tid) * SP; };
    auto u_global = [&](int node) -> Real * {
        return U + (((size_t)(node - N) * R + r) * Cpad + pat) * SP;
    };
    auto tip_word = [&](int node) -> const uint8_t * { return a.tip_states + (size_t)node * Cpad + (pat & ~3); };
    auto tip_state = [&](const Real *slot) -> int {
        uint32_t w = *reinterpret_cast<const uint32_t *>(slot);
        return (int)((w >> (8 * (pat & 3))) & 0xffu);
    };
    auto tip_vec = [&](int node) -> const Real * { return tipP + ((size_t)node * Cpad + pat) * SP; };

    // ---------------- post program (Eq. 2, Eq. 3) ----------------------------
    auto issue_post = [&](int n) {
        if (n < N - 1) {
            const Op4 op = a.post[n];
            const int cs[2] = {op.y, op.z};
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int code = cs[c];
                if (code >= 0) {
                    const int node = code & ~kTipPartialBit;
                    if (code & kTipPartialBit) cp_async_vec<SP * sizeof(Real)>(ring_at(n, c), tip_vec(node));
                    else cp_async4(ring_at(n, c), tip_word(node));
                }
            }
        }
        cp_async_commit();
    };
    for (int n = 0; n < D - 1; ++n) issue_post(n);

    int E = 0;              // accumulated scale exponent of this pattern (post-order)
    int parity = 0;
    double logl_local = 0.0;
    for (int n = 0; n < N - 1; ++n) {
        issue_post(n + D - 1);
        cp_async_wait_dyn(D - 1);
        const Op4 op = a.post[n];
        Real uc[2][SP];
        const int cs[2] = {op.y, op.z};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int code = cs[c];
            if (code < 0) {
                load_vec<Real, SP>(uc[c], stack_at(-code - 1));
            } else {
                const int node = code & ~kTipPartialBit;
                const Real *Pm = P + ((size_t)node * R + r) * mat;
                if (code & kTipPartialBit) {
                    Real tp[SP];
                    load_vec<Real, SP>(tp, ring_at(n, c));
                    matvec<Real, SP>(uc[c], Pm, tp);
                } else {
                    tip_column<Real, SP>(uc[c], Pm, tip_state(ring_at(n, c)), a.S);
                }
            }
        }
        Real p[SP];
#pragma unroll
        for (int s = 0; s < SP; ++s) p[s] = uc[0][s] * uc[1][s];
        double *rd = redd + (size_t)parity * 4 * nthr;
        int *ri = redi + (size_t)parity * 2 * nthr;
        if (op.x == root) {
            double Lr = 0.0;
#pragma unroll
            for (int s = 0; s < SP; ++s) Lr += (double)ldg(pig + s) * (double)p[s];
            rd[tid] = wr * Lr;
            __syncthreads();
            if (warp == 0) {
                double L = 0.0;
                for (int q = 0; q < R; ++q) L += rd[q * 32 + lane];
                if (pat < a.C) {
                    if (!(L > 0.0) || !isfinite(L)) atomicMin(a.status, pat);
                    logl_local = Wc * (log(L) + (double)E * 0.69314718055994530942);
                }
            }
        } else {
            ri[tid] = exponent_of(vmax<Real, SP>(p));
            __syncthreads();
            int e = ri[lane];
            for (int q = 1; q < R; ++q) e = max(e, ri[q * 32 + lane]);
            E += e;
#pragma unroll
            for (int s = 0; s < SP; ++s) p[s] = scale_pow2(p[s], -e);
            Real u[SP];
            matvec<Real, SP>(u, P + ((size_t)op.x * R + r) * mat, p);
            store_vec<Real, SP>(u_global(op.x), u);
            store_vec<Real, SP>(stack_at(op.w), u);
        }
        parity ^= 1;
    }
    // logL partial of this tile (warp 0 holds it)
    if (warp == 0) {
        double v = logl_local;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) a.logl_part[tile] = v;
    }
    cp_async_wait<0>();
    __threadfence_block();

    // ---------------- pre program (Eq. 4) + gradient (Eq. 8) ------------------
    auto issue_pre = [&](int n) {
        if (n < N - 1) {
            const Op4 op = a.pre[n];
            const int cs[2] = {op.y, op.z};
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int code = cs[c];
                const int node = code & ~kTipPartialBit;
                if (node >= N) cp_async_vec<SP * sizeof(Real)>(ring_at(n, c), u_global(node));
                else if (code & kTipPartialBit) cp_async_vec<SP * sizeof(Real)>(ring_at(n, c), tip_vec(node));
                else cp_async4(ring_at(n, c), tip_word(node));
            }
        }
        cp_async_commit();
    };
    for (int n = 0; n < D - 1; ++n) issue_pre(n);

    for (int n = 0; n < N - 1; ++n) {
        issue_pre(n + D - 1);
        cp_async_wait_dyn(D - 1);
        const Op4 op = a.pre[n];
        Real q[SP];
        if (op.x < 0) ldg_vec<Real, SP>(q, pig);
        else load_vec<Real, SP>(q, stack_at(op.x));
        const int cs[2] = {op.y, op.z};
        const int slots[2] = {(op.w & 0xffff) - 1, (op.w >> 16) - 1};
        int node[2];
        Real uc[2][SP];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int code = cs[c];
            node[c] = code & ~kTipPartialBit;
            if (node[c] >= N) {
                load_vec<Real, SP>(uc[c], ring_at(n, c));
            } else {
                const Real *Pm = P + ((size_t)node[c] * R + r) * mat;
                if (code & kTipPartialBit) {
                    Real tp[SP];
                    load_vec<Real, SP>(tp, ring_at(n, c));
                    matvec<Real, SP>(uc[c], Pm, tp);
                } else {
                    tip_column<Real, SP>(uc[c], Pm, tip_state(ring_at(n, c)), a.S);
                }
            }
        }
        double *rd = redd + (size_t)parity * 4 * nthr;
        int *ri = redi + (size_t)parity * 2 * nthr;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            Real x[SP];
#pragma unroll
            for (int s = 0; s < SP; ++s) x[s] = q[s] * uc[1 - c][s];
            // Eq. 8 terms for branch node[c] in the branch-top form:
            //   num_r = gamma_r P(gamma_r) x' Q u,  den_r = P(gamma_r) x' u
            Real Qu[SP];
            matvec<Real, SP>(Qu, Qg, uc[c]);
            Real num = 0, den = 0;
#pragma unroll
            for (int s = 0; s < SP; ++s) {
                num = fma(x[s], Qu[s], num);
                den = fma(x[s], uc[c][s], den);
            }
            rd[(2 * c) * nthr + tid] = gr * wr * (double)num;
            rd[(2 * c + 1) * nthr + tid] = wr * (double)den;
            if (slots[c] >= 0) {      // q_c = P_c' x_c (Eq. 4), rescaled after the exchange
                Real qc[SP];
                matvec_t<Real, SP>(qc, P + ((size_t)node[c] * R + r) * mat, x);
                ri[c * nthr + tid] = exponent_of(vmax<Real, SP>(qc));
                store_vec<Real, SP>(stack_at(slots[c]), qc);
            }
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            if (warp == (c % R)) {
                double num = 0.0, den = 0.0;
                for (int q2 = 0; q2 < R; ++q2) {
                    num += rd[(2 * c) * nthr + q2 * 32 + lane];
                    den += rd[(2 * c + 1) * nthr + q2 * 32 + lane];
                }
                double d = (Wc != 0.0) ? Wc * (num / den) : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                if (lane == 0) a.grad_part[(size_t)node[c] * a.n_tiles + tile] = d;
            }
            if (slots[c] >= 0) {
                int e = ri[c * nthr + lane];
                for (int q2 = 1; q2 < R; ++q2) e = max(e, ri[c * nthr + q2 * 32 + lane]);
                Real v[SP];
                load_vec<Real, SP>(v, stack_at(slots[c]));
#pragma unroll
                for (int s = 0; s < SP; ++s) v[s] = scale_pow2(v[s], -e);
                store_vec<Real, SP>(stack_at(slots[c]), v);
            }
        }
        parity ^= 1;
    }
    cp_async_wait<0>();
}

}  // namespace pg
