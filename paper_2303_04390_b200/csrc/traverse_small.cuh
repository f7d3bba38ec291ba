// traverse_small.cuh -- fused post-order + pre-order + per-edge gradient for
// small state spaces (SP = 4, 8, 16): the HBM-bound nucleotide and
// Markov-modulated paths.
//
// Design.  Site patterns are independent, so
// every WARP owns a tile of TP = 32/RP patterns for all R rate categories and
// walks the whole tree for them -- one launch, no grid or CTA barriers:
//   * lane = (pattern, category), category fastest (RP = R rounded up to a
//     power of two; lanes with category >= R shadow category R-1 with zero
//     weight).  Each lane keeps the SP states of its vector in registers.
//   * The two per-pattern programs (schedule.hpp) are static, so every input
//     of a step is fetched ahead of time by lane 0 with 1-D bulk copies (TMA
//     engine, mbarrier completion) into a D-stage shared-memory ring: ops in
//     32-op chunks, the R transition matrices of each branch involved (one
//     contiguous copy) and the warp's contiguous u chunk or tip codes of each
//     child.  HBM-resident u chunks are also pulled into L2 PF steps ahead
//     (bulk prefetch).  The dependent chain of a step touches only registers
//     and shared memory.
//   * post program (Eq. 2): p_k = u_a o u_b; u_k = P_k p_k streamed to HBM
//     once and kept on a per-lane stack for the parent.
//   * root (Eq. 3): L_c = sum_r P(gamma_r) pi' p_root; logL partial per tile.
//   * pre program (Eq. 4, branch-top form SURVEY §0): for parent k with
//     children a, b: x_a = q_k o u_b, x_b = q_k o u_a,
//       num_r = gamma_r P(gamma_r) x_a' Q u_a   (= gamma_r P(gamma_r) p'Q'q)
//       den_r = P(gamma_r) x_a' u_a             (= P(gamma_r) p'q)
//     and q_a = P_a' x_a pushed for internal children.  (num_r, den_r) go to a
//     small smem window; every W steps the warp forms sum_r num / sum_r den
//     (Eq. 8), weights it by w_c and sums the tile's patterns (Eq. 6) with
//     all 32 lanes busy.
//   * Underflow (R4): a vector is multiplied by 2^-e (e = exponent of
//     the max over its pattern's categories) when a warp vote finds one below
//     2^-256 (fp64) / 2^-64 (fp32).  Powers of two are exact, so results do
//     not depend on when rescaling happens; post-order exponents are summed
//     per pattern for logL, pre-order ones cancel in the Eq. 8 ratio.
// HBM traffic per evaluation: 2 (N-2) R C SP sizeof(Real) (u written once,
// read once) + 2 N C tip-code bytes, vs 5 (N-2) V for level batching.
#pragma once
#include "common.cuh"

namespace pg {

// ---- compile-time shape of one warp's work --------------------------------
// Global layout of the transition matrices for this kernel: per branch, R
// category blocks of SP*SP Reals padded to CS bytes (16 extra bytes when
// R > 1 so the categories of a warp hit distinct shared-memory banks); one
// branch's matrices are one contiguous bulk copy.
template <typename Real, int SP, int RP>
struct SmallCfg {
    static constexpr int TP = 32 / RP;                        // patterns per warp tile
    static constexpr int D = (SP <= 8) ? 4 : 2;                // bulk-copy ring depth
    static constexpr int PF = 16;                              // L2 prefetch distance (steps)
    static constexpr int W = 2;                                // gradient window (steps)
    static constexpr int VB = SP * (int)sizeof(Real);          // vector bytes
    static constexpr int MATB = SP * SP * (int)sizeof(Real);   // one category's matrix
    static constexpr int CS = MATB + (RP > 1 ? 16 : 0);        // padded category stride
    static constexpr int TIPW = TP > 16 ? TP : 16;             // tip-code window bytes
    static constexpr int OPS = 64 * 16;                        // 2 x 32-op chunks
    static constexpr int ND = W * 2 * 32 * 16;                 // (num, den) window
    static __host__ __device__ int mat_slot(int R) { return R * CS; }
    static __host__ __device__ int vss() { return TP * VB > TIPW ? TP * VB : TIPW; }      // post vec slot
    static __host__ __device__ int vsb(int R) { return TP * R * VB > vss() ? TP * R * VB : vss(); }  // pre
    static __host__ __device__ int stage(int R) {
        const int a = 3 * mat_slot(R) + 2 * vss(), b = 2 * mat_slot(R) + 2 * vsb(R);
        return ((a > b ? a : b) + 15) / 16 * 16;
    }
    static __host__ __device__ size_t smem(int R, int depth) {
        return 64 + (size_t)OPS + ND + (size_t)D * stage(R) + (size_t)depth * 32 * VB + TP * 8;
    }
};

// ---- vector access helpers ------------------------------------------------
template <typename Real, int SP>
__device__ __forceinline__ void lds_vec(Real (&d)[SP], const void *src) {
    if constexpr (sizeof(Real) == 8) {
#pragma unroll
        for (int i = 0; i < SP / 2; ++i) {
            const double2 t = reinterpret_cast<const double2 *>(src)[i];
            d[2 * i] = t.x;
            d[2 * i + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < SP / 4; ++i) {
            const float4 t = reinterpret_cast<const float4 *>(src)[i];
            d[4 * i] = t.x; d[4 * i + 1] = t.y; d[4 * i + 2] = t.z; d[4 * i + 3] = t.w;
        }
    }
}
template <typename Real, int SP>
__device__ __forceinline__ void sts_vec(void *dst, const Real (&d)[SP]) {
    if constexpr (sizeof(Real) == 8) {
#pragma unroll
        for (int i = 0; i < SP / 2; ++i) reinterpret_cast<double2 *>(dst)[i] = make_double2(d[2 * i], d[2 * i + 1]);
    } else {
#pragma unroll
        for (int i = 0; i < SP / 4; ++i)
            reinterpret_cast<float4 *>(dst)[i] = make_float4(d[4 * i], d[4 * i + 1], d[4 * i + 2], d[4 * i + 3]);
    }
}
template <typename Real, int SP>
__device__ __forceinline__ void stg_vec(void *dst, const Real (&d)[SP]) {
    if constexpr (sizeof(Real) == 8) {
#pragma unroll
        for (int i = 0; i < SP / 2; ++i) __stcg(reinterpret_cast<double2 *>(dst) + i, make_double2(d[2 * i], d[2 * i + 1]));
    } else {
#pragma unroll
        for (int i = 0; i < SP / 4; ++i)
            __stcg(reinterpret_cast<float4 *>(dst) + i, make_float4(d[4 * i], d[4 * i + 1], d[4 * i + 2], d[4 * i + 3]));
    }
}

// y = M x (y[s] = sum_t M[s][t] x[t]), M row-major in shared memory
template <typename Real, int SP>
__device__ __forceinline__ void mv(Real (&y)[SP], const Real *M, const Real (&x)[SP]) {
#pragma unroll
    for (int s = 0; s < SP; ++s) {
        Real row[SP];
        lds_vec<Real, SP>(row, M + s * SP);
        Real acc = row[0] * x[0];
#pragma unroll
        for (int t = 1; t < SP; ++t) acc = fma(row[t], x[t], acc);
        y[s] = acc;
    }
}
// y = M' x (y[t] = sum_s M[s][t] x[s])
template <typename Real, int SP>
__device__ __forceinline__ void mvt(Real (&y)[SP], const Real *M, const Real (&x)[SP]) {
#pragma unroll
    for (int s = 0; s < SP; ++s) {
        Real row[SP];
        lds_vec<Real, SP>(row, M + s * SP);
#pragma unroll
        for (int t = 0; t < SP; ++t) y[t] = s == 0 ? row[t] * x[0] : fma(row[t], x[s], y[t]);
    }
}
// u = column s of M (observed tip state) or M 1 (missing, s >= S)
template <typename Real, int SP>
__device__ __forceinline__ void mcol(Real (&u)[SP], const Real *M, int s, int S) {
    if (s < S) {
#pragma unroll
        for (int x = 0; x < SP; ++x) u[x] = M[x * SP + s];
    } else {
#pragma unroll
        for (int x = 0; x < SP; ++x) {
            Real row[SP];
            lds_vec<Real, SP>(row, M + x * SP);
            Real acc = row[0];
#pragma unroll
            for (int t = 1; t < SP; ++t) acc += row[t];
            u[x] = acc;
        }
    }
}

// ---- exact power-of-two rescaling -----------------------------------------
__device__ __forceinline__ int expfield(double x) { return __double2hiint(x) >> 20; }   // x >= 0
__device__ __forceinline__ int expfield(float x) { return __float_as_int(x) >> 23; }
template <typename Real, int SP>
__device__ __forceinline__ int max_expfield(const Real (&v)[SP]) {
    int m = expfield(v[0]);
#pragma unroll
    for (int i = 1; i < SP; ++i) m = max(m, expfield(v[i]));
    return m;
}
template <typename Real> struct ScaleTraits;
template <> struct ScaleTraits<double> {
    static constexpr int THRESH = 1023 - 256;   // rescale once a max drops below 2^-256
    static __device__ __forceinline__ int exponent(int field) { return min(max(field - 1022, -1021), 1022); }
    static __device__ __forceinline__ double factor(int e) { return __longlong_as_double((long long)(1023 - e) << 52); }
};
template <> struct ScaleTraits<float> {
    static constexpr int THRESH = 127 - 64;      // 2^-64
    static __device__ __forceinline__ int exponent(int field) { return min(max(field - 126, -125), 126); }
    static __device__ __forceinline__ float factor(int e) { return __int_as_float((127 - e) << 23); }
};
template <int RP, typename T>
__device__ __forceinline__ T cat_max(T v) {
#pragma unroll
    for (int o = 1; o < RP; o <<= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <int RP>
__device__ __forceinline__ double cat_sum(double v) {
#pragma unroll
    for (int o = 1; o < RP; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// Rescale v (exactly) if any vector of the warp fell below the threshold;
// returns the exponent removed (shared by the categories of a pattern).
template <typename Real, int SP, int RP>
__device__ __forceinline__ int maybe_rescale(Real (&v)[SP]) {
    const int f = max_expfield<Real, SP>(v);
    if (!__any_sync(0xffffffffu, f < ScaleTraits<Real>::THRESH)) return 0;
    const int e = ScaleTraits<Real>::exponent(cat_max<RP>(f));
    const Real s = ScaleTraits<Real>::factor(e);
#pragma unroll
    for (int i = 0; i < SP; ++i) v[i] *= s;
    return e;
}


template <typename Real, int SP, int RP>
__global__ void __launch_bounds__(32) traverse_small_kernel(const TravArgs a) {
    using Cfg = SmallCfg<Real, SP, RP>;
    constexpr int TP = Cfg::TP, D = Cfg::D, PF = Cfg::PF, W = Cfg::W, VB = Cfg::VB, CS = Cfg::CS;
    extern __shared__ __align__(16) unsigned char smem[];
    const int R = a.R, N = a.N, S = a.S;
    const int lane = threadIdx.x;
    const int cat = lane & (RP - 1);
    const int r = min(cat, R - 1);                  // shadow lanes reuse category R-1
    const bool live = cat < R;
    const int pl = lane / RP;                       // pattern within the tile
    const int tile = blockIdx.x;
    const int pat0 = tile * TP;
    const int pat = pat0 + pl;                      // < Cpad
    const int root = 2 * N - 2;
    const int nops = N - 1;
    const int MS = Cfg::mat_slot(R), VSS = Cfg::vss(), VSB = Cfg::vsb(R), ST = Cfg::stage(R);

    uint64_t *bars = reinterpret_cast<uint64_t *>(smem);                          // [D] stages + [1] prologue
    Op4 *opbuf = reinterpret_cast<Op4 *>(smem + 64);
    double2 *nd = reinterpret_cast<double2 *>(smem + 64 + Cfg::OPS);              // [W][2][32]
    unsigned char *stages = smem + 64 + Cfg::OPS + Cfg::ND;
    unsigned char *stackb = stages + D * ST;
    double *wbuf = reinterpret_cast<double *>(stackb + (size_t)a.depth * 32 * VB); // [TP]

    const char *__restrict__ Pb = static_cast<const char *>(a.P);
    const char *__restrict__ tipP = static_cast<const char *>(a.tip_partials);
    const uint8_t *__restrict__ tipS = a.tip_states;
    char *__restrict__ Ub = static_cast<char *>(a.u);
    const double wr = live ? a.cat_w[r] : 0.0;
    const double gwr = wr * a.cat_g[r];
    Real pi[SP];
#pragma unroll
    for (int s = 0; s < SP; ++s) pi[s] = static_cast<const Real *>(a.pi)[s];
    if (lane < TP) wbuf[lane] = a.pat_w[pat0 + lane];
    if (lane == 0) {
        for (int i = 0; i <= D; ++i) mbar_init(bars + i, 1);
        fence_mbar_init();
    }
    __syncwarp();

    // constant offsets
    const size_t Cpad = (size_t)a.Cpad;
    const size_t u_node = Cpad * R * VB;                           // one node's u block (bytes)
    const size_t u_warp = (size_t)pat0 * R * VB;                   // this warp's contiguous chunk
    const unsigned u_chunk = TP * R * VB;
    const unsigned u_vec = (pl * R + r) * VB;                      // my vector inside a u chunk
    const int tip_off = pat0 & 15;                                 // my tile inside a tip window
    const unsigned mat_lane = r * CS;

    auto op_at = [&](int n) -> Op4 { return opbuf[(n >> 5 & 1) * 32 + (n & 31)]; };
    auto stage_at = [&](int t) -> unsigned char * { return stages + (t & (D - 1)) * ST; };
    auto bar_at = [&](int t) -> uint64_t * { return bars + (t & (D - 1)); };
    auto parity_at = [&](int t) -> uint32_t { return (uint32_t)(t / D) & 1u; };
    auto stack_at = [&](int slot) -> unsigned char * { return stackb + (slot * 32 + lane) * VB; };
    auto tip_bytes = [&](int code) -> unsigned { return (code & kTipPartialBit) ? TP * VB : Cfg::TIPW; };
    // lane 0: bulk copy of tip data (16-B window of codes, or the tile's partial vectors)
    auto copy_tip = [&](unsigned char *dst, int code, uint64_t *bar) {
        const int node = code & ~kTipPartialBit;
        if (code & kTipPartialBit) bulk_g2s(dst, tipP + ((size_t)node * Cpad + pat0) * VB, TP * VB, bar);
        else bulk_g2s(dst, tipS + (((size_t)node * Cpad + pat0) & ~(size_t)15), Cfg::TIPW, bar);
    };
    auto ops_bytes = [&](int chunk) -> unsigned {
        const int n = nops - chunk * 32;
        return n <= 0 ? 0u : (unsigned)(n < 32 ? n : 32) * 16u;
    };
    auto copy_ops = [&](const Op4 *prog, int chunk, uint64_t *bar) {
        const unsigned b = ops_bytes(chunk);
        if (b) bulk_g2s(opbuf + (chunk & 1) * 32, prog + chunk * 32, b, bar);
    };
    // child vector from a stage: state tip (column of P), partial tip (P p)
    auto child_tip = [&](Real (&u)[SP], const unsigned char *M_, const unsigned char *vs, int code) {
        const Real *M = reinterpret_cast<const Real *>(M_ + mat_lane);
        if (code & kTipPartialBit) {
            Real tp[SP];
            lds_vec<Real, SP>(tp, vs + pl * VB);
            mv<Real, SP>(u, M, tp);
        } else {
            mcol<Real, SP>(u, M, vs[tip_off + pl], S);
        }
    };
    auto load_prologue_ops = [&](const Op4 *prog, uint32_t parity) {
        if (lane == 0) {
            mbar_arrive_expect_tx(bars + D, ops_bytes(0) + ops_bytes(1));
            copy_ops(prog, 0, bars + D);
            copy_ops(prog, 1, bars + D);
        }
        mbar_wait(bars + D, parity);
    };

    // ====================== post program (Eq. 2, Eq. 3) =======================
    // stage layout: [P_k][P_a][P_b][tip a][tip b]
    auto issue_post = [&](int m) {           // lane 0 only
        if (m >= nops) return;
        unsigned char *st = stage_at(m);
        uint64_t *bar = bar_at(m);
        const Op4 op = op_at(m);
        const bool ops_next = (m & 31) == D - 1;     // op chunk (m/32)+1 rides on stage m
        const int chunk = m / 32 + 1;
        unsigned bytes = (op.x != root ? MS : 0) + (op.y >= 0 ? MS + tip_bytes(op.y) : 0) +
                         (op.z >= 0 ? MS + tip_bytes(op.z) : 0) + ((ops_next && chunk >= 2) ? ops_bytes(chunk) : 0);
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(bar, bytes);
        if (op.x != root) bulk_g2s(st, Pb + (size_t)op.x * MS, MS, bar);
        if (op.y >= 0) {
            bulk_g2s(st + MS, Pb + (size_t)(op.y & ~kTipPartialBit) * MS, MS, bar);
            copy_tip(st + 3 * MS, op.y, bar);
        }
        if (op.z >= 0) {
            bulk_g2s(st + 2 * MS, Pb + (size_t)(op.z & ~kTipPartialBit) * MS, MS, bar);
            copy_tip(st + 3 * MS + VSS, op.z, bar);
        }
        if (ops_next && chunk >= 2) copy_ops(a.post, chunk, bar);
    };
    load_prologue_ops(a.post, 0);
    if (lane == 0)
        for (int m = 0; m < D - 1; ++m) issue_post(m);

    int E = 0;                    // post-order exponents removed from this pattern
    double logl_local = 0.0;
    for (int n = 0; n < nops; ++n) {
        __syncwarp();                                       // stage (n-1) consumed by all lanes
        if (lane == 0) issue_post(n + D - 1);
        mbar_wait(bar_at(n), parity_at(n));
        const Op4 op = op_at(n);
        const unsigned char *st = stage_at(n);
        Real ua[SP], ub[SP];
        if (op.y < 0) lds_vec<Real, SP>(ua, stack_at(-op.y - 1));
        else child_tip(ua, st + MS, st + 3 * MS, op.y);
        if (op.z < 0) lds_vec<Real, SP>(ub, stack_at(-op.z - 1));
        else child_tip(ub, st + 2 * MS, st + 3 * MS + VSS, op.z);
        Real p[SP];
#pragma unroll
        for (int s = 0; s < SP; ++s) p[s] = ua[s] * ub[s];
        if (op.x == root) {
            double L = 0.0;
#pragma unroll
            for (int s = 0; s < SP; ++s) L = fma((double)pi[s], (double)p[s], L);
            L = cat_sum<RP>(wr * L);
            if (cat == 0 && pat < a.C) {
                if (!(L > 0.0) || !isfinite(L)) atomicMin(a.status, pat);
                logl_local = wbuf[pl] * (log(L) + (double)E * 0.69314718055994530942);
            }
        } else {
            E += maybe_rescale<Real, SP, RP>(p);
            Real u[SP];
            mv<Real, SP>(u, reinterpret_cast<const Real *>(st + mat_lane), p);
            if (live) stg_vec<Real, SP>(Ub + (size_t)(op.x - N) * u_node + u_warp + u_vec, u);
            sts_vec<Real, SP>(stack_at(op.w), u);
        }
    }
    {
        double v = logl_local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) a.logl_part[tile] = v;
    }
    fence_proxy_async_global();          // u stores (generic proxy) before bulk reads (async proxy)
    __syncwarp();

    // =============== pre program (Eq. 4) + gradient (Eq. 6-8) =================
    // stage layout: [P_a][P_b][vec a][vec b]; step t = nops + n for ring/parity
    auto issue_pre = [&](int m) {            // lane 0 only
        if (m >= nops) return;
        const int t = nops + m;
        unsigned char *st = stage_at(t);
        uint64_t *bar = bar_at(t);
        const Op4 op = op_at(m);
        const int cs[2] = {op.y, op.z};
        const bool ops_next = (m & 31) == D - 1;
        const int chunk = m / 32 + 1;
        unsigned bytes = (ops_next && chunk >= 2) ? ops_bytes(chunk) : 0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int node = cs[c] & ~kTipPartialBit;
            bytes += MS + (node >= N ? u_chunk : tip_bytes(cs[c]));
        }
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(bar, bytes);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int node = cs[c] & ~kTipPartialBit;
            bulk_g2s(st + c * MS, Pb + (size_t)node * MS, MS, bar);
            unsigned char *vs = st + 2 * MS + c * VSB;
            if (node >= N) bulk_g2s(vs, Ub + (size_t)(node - N) * u_node + u_warp, u_chunk, bar);
            else copy_tip(vs, cs[c], bar);
        }
        if (ops_next && chunk >= 2) copy_ops(a.pre, chunk, bar);
    };
    auto prefetch_pre = [&](int m) {         // lane 0: pull step m's u chunks into L2
        if (m >= nops) return;
        const Op4 op = op_at(m);
        const int ny = op.y & ~kTipPartialBit, nz = op.z & ~kTipPartialBit;
        if (ny >= N) prefetch_l2(Ub + (size_t)(ny - N) * u_node + u_warp, u_chunk);
        if (nz >= N) prefetch_l2(Ub + (size_t)(nz - N) * u_node + u_warp, u_chunk);
    };
    // W steps of per-lane (num_r, den_r) -> Eq. 8 ratio per pattern, weighted by
    // w_c and summed over the tile's patterns (Eq. 6): all 32 lanes busy.
    auto flush = [&](int n_last) {
        __syncwarp();
        constexpr int PAIRS = 2 * W, LPP = 32 / PAIRS, PPL = TP / LPP > 0 ? TP / LPP : 1;
        const int pair = lane / LPP, sub = lane % LPP;
        const int wstep = pair >> 1, c = pair & 1;
        const int n = n_last - (n_last % W) + wstep;
        double acc = 0.0;
        if (n <= n_last && sub * PPL < TP) {
#pragma unroll
            for (int k = 0; k < PPL; ++k) {
                const int p = sub * PPL + k;
                const double2 *src = nd + ((wstep * 2 + c) * 32 + p * RP);
                double num = 0.0, den = 0.0;
#pragma unroll
                for (int q = 0; q < RP; ++q) { const double2 v = src[q]; num += v.x; den += v.y; }
                const double w = wbuf[p];
                acc += (w != 0.0) ? w * (num / den) : 0.0;
            }
        }
#pragma unroll
        for (int o = 1; o < LPP; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (sub == 0 && n <= n_last) {
            const Op4 op = op_at(n);
            const int node = (c == 0 ? op.y : op.z) & ~kTipPartialBit;
            a.grad_part[(size_t)node * a.n_tiles + tile] = acc;
        }
    };

    load_prologue_ops(a.pre, 1);
    if (lane == 0) {
        for (int m = 0; m < PF; ++m) prefetch_pre(m);
        for (int m = 0; m < D - 1; ++m) issue_pre(m);
    }

    Real Qr[SP][SP <= 4 ? SP : 1];
    if constexpr (SP <= 4) {
#pragma unroll
        for (int s = 0; s < SP; ++s)
#pragma unroll
            for (int t = 0; t < SP; ++t) Qr[s][t] = static_cast<const Real *>(a.Q)[s * SP + t];
    }
    const Real *Qg = static_cast<const Real *>(a.Q);

    for (int n = 0; n < nops; ++n) {
        __syncwarp();
        if (lane == 0) {
            prefetch_pre(n + PF);
            issue_pre(n + D - 1);
        }
        mbar_wait(bar_at(nops + n), parity_at(nops + n));
        const Op4 op = op_at(n);
        const unsigned char *st = stage_at(nops + n);
        Real q[SP];
        if (op.x < 0) {
#pragma unroll
            for (int s = 0; s < SP; ++s) q[s] = pi[s];
        } else {
            lds_vec<Real, SP>(q, stack_at(op.x));
        }
        const int cs[2] = {op.y, op.z};
        const int slots[2] = {(op.w & 0xffff) - 1, (op.w >> 16) - 1};
        Real uc[2][SP];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const unsigned char *vs = st + 2 * MS + c * VSB;
            if ((cs[c] & ~kTipPartialBit) >= N) lds_vec<Real, SP>(uc[c], vs + u_vec);
            else child_tip(uc[c], st + c * MS, vs, cs[c]);
        }
        double2 *ndw = nd + (n % W) * 64 + lane;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            Real x[SP];
#pragma unroll
            for (int s = 0; s < SP; ++s) x[s] = q[s] * uc[1 - c][s];
            Real num = 0, den = 0;
#pragma unroll
            for (int s = 0; s < SP; ++s) {
                Real Qu;
                if constexpr (SP <= 4) {
                    Qu = Qr[s][0] * uc[c][0];
#pragma unroll
                    for (int t = 1; t < SP; ++t) Qu = fma(Qr[s][t], uc[c][t], Qu);
                } else {
                    Qu = __ldg(Qg + s * SP) * uc[c][0];
#pragma unroll
                    for (int t = 1; t < SP; ++t) Qu = fma(__ldg(Qg + s * SP + t), uc[c][t], Qu);
                }
                num = fma(x[s], Qu, num);
                den = fma(x[s], uc[c][s], den);
            }
            ndw[c * 32] = make_double2(gwr * (double)num, wr * (double)den);
            if (slots[c] >= 0) {               // q_c = P_c' x_c (Eq. 4), pushed
                Real qc[SP];
                mvt<Real, SP>(qc, reinterpret_cast<const Real *>(st + c * MS + mat_lane), x);
                maybe_rescale<Real, SP, RP>(qc);
                sts_vec<Real, SP>(stack_at(slots[c]), qc);
            }
        }
        if (n % W == W - 1 || n == nops - 1) flush(n);
    }
}

}  // namespace pg
