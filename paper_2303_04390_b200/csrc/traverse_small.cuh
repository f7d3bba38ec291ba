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
//   * A CTA is K such warps (K consecutive tiles, K = ceil(tiles / #SMs) so the
//     grid is one wave) plus one PRODUCER warp.  The two per-pattern programs
//     (schedule.hpp) are static and identical for every tile, so the producer
//     walks them D steps ahead of the consumers and, per step, issues 1-D bulk
//     copies (TMA engine, mbarrier transaction counts) into a D-stage shared
//     ring: the op, the R transition matrices of each branch involved (one
//     contiguous copy, shared by the K warps) and each child's u chunk or tip
//     codes for all K tiles (contiguous in HBM: one copy).  u chunks are also
//     pulled into L2 PF steps ahead (bulk prefetch).  Consumers wait on the
//     stage's "full" barrier, compute, and arrive on its "empty" barrier; the
//     dependent chain of a step touches only registers and shared memory.
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

// fence.proxy.async before the producer's bulk copies into a released
// stage: not needed (the stage was only READ by the consumers, whose release
// / acquire through the empty barrier orders those reads before the copies);
// dropping it: dengue traversal 1.306 -> 1.284 ms (scripts/gpu_r3_ab.sh)
#ifndef PG_PROXY_FENCE
#define PG_PROXY_FENCE 0
#endif
#ifndef PG_GPOST
#define PG_GPOST 8
#endif
#ifndef PG_MMA_STAGES
#define PG_MMA_STAGES 8
#endif
#ifndef PG_TIPP_PF
#define PG_TIPP_PF 0
#endif


namespace pg {

// lanes per (pattern, category) vector: each lane holds VL = SP / LV states.
// SP = 4 keeps a whole vector per lane; S = 8 and 16 split it over 2 and 4
// lanes so a warp's 32 lanes hold 8 patterns x R categories at any S (more
// resident warps, a quarter of the per-lane matvec work for S = 16).
// (Splitting S = 4 over 2 lanes as well was measured 2x slower on the dengue
// workload: twice the warps, the same per-step control work.)
#ifndef PG_SP4_LV
#define PG_SP4_LV 1
#endif
#ifndef PG_SP16_LV
#define PG_SP16_LV 4
#endif
__host__ __device__ constexpr int small_lanes_per_vector(int SP, int RP) {
    return SP == 4 ? PG_SP4_LV : SP == 16 ? (PG_SP16_LV < 32 / RP ? PG_SP16_LV : 32 / RP) : SP / 4;
}
// bytes between consecutive category matrices beyond SP*SP Reals (R > 1):
// shifts each category's matrix to other shared-memory banks so the lanes of
// different categories reading the same row (matvec) or column (tip gather)
// do not collide; fp64 S = 4 matrices are exactly 32 banks long and need an
// 8-bank (32 B) shift for the column reads of tip children
__host__ __device__ constexpr int small_cat_pad(int real_bytes, int SP) {
#ifdef PG_CATPAD16
    return 16;
#else
    return (real_bytes == 8 && SP == 4) ? 32 : 16;
#endif
}
// FP64 tensor-core variant (SP = 16, one rate category, fp64: the 4 x K
// Markov-modulated workloads, BJ:configs[2]).  A warp's tile is 8 patterns x
// 16 states, and every matrix-vector product of a step -- u = P p (Eq. 2),
// q = x P (Eq. 4), Q u (Eq. 8) -- is one [8 x 16] x [16 x 16] product: 8
// mma.sync.m8n8k4.f64 (SASS DMMA) instead of 64 DFMA per lane plus a
// shared-memory exchange of the whole vector.  Lane l holds states
// {j, 4+j, 8+j, 12+j} (j = l % 4) of pattern l / 4: exactly its A fragments
// (k = 4 kt + j).  The output columns of the B operands are permuted,
// n -> sigma(n) = 4 (2 (n / 8) + n % 2) + (n % 8) / 2, so the lane's C
// fragments are again its own states in the same order: a product's result
// is the next product's A operand with no data movement.  Each branch's
// record holds three 16 x 16 layouts (A1 writes them): [P as B of u = P p]
// [P as B of q = x P] [P row-major, row stride 17, column 16 = P 1].
// The S = 4 (nucleotide) variant with four rate categories: lane l holds
// state j = l % 4 of pattern l / 4 for the four categories (one register
// each); per category the product is one m8n8k4 DMMA whose B operand repeats
// every output column twice (n -> state n / 2), so lane l's first C element
// is exactly state j of its pattern: [8 x 4] x [4 x 8] per category, the
// result again in the A layout.  Branch record: [P as B of u = P p][P as B
// of q = x P], each [4 categories][32 lanes] doubles.
// Measured (scripts/gpu_mma4.sh, dengue fp64): the S = 4 variant is slower
// than the SIMT kernel (traversal 1.577 vs 1.427 ms: a DMMA per category
// spends 4x the FP64-pipe time of the 16 DFMA it replaces and its latency sits
// on the step chain), so it is built only with -DPG_SMALL_MMA4 (parity-tested
// there); S = 16 gains 2x (MMM traversal 0.219 -> 0.109 ms).
__host__ __device__ constexpr bool small_tc(int SP, int R, int real_bytes) {
#ifdef PG_NO_SMALL_MMA
    return false;
#elif defined(PG_SMALL_MMA4)
    return real_bytes == 8 && ((SP == 16 && R == 1) || (SP == 4 && R == 4));
#else
    return real_bytes == 8 && SP == 16 && R == 1;
#endif
}
constexpr int MMA4_SLOT = 4 * 32 * 8;                            // bytes per layout (1 KB)
constexpr int MMA_RS = 17;                                       // row stride of the row-major layout
constexpr int MMA_SLOT = 16 * MMA_RS * 8;                        // bytes per layout (2176)
constexpr int MMA_REC = 3 * MMA_SLOT;                            // bytes per branch record
__host__ __device__ constexpr int mma_sigma(int n) { return 4 * (2 * (n >> 3) + (n & 1)) + ((n & 7) >> 1); }

// consumer warps per CTA at most (launch bounds: + 1 producer warp)
__host__ __device__ constexpr int small_max_consumers(int SP, int RP) { return small_lanes_per_vector(SP, RP) * 4 / SP >= 2 ? 17 : 9; }

// ---- shape of one CTA's work ----------------------------------------------
// A CTA = K consumer warps (one pattern tile each) + 1 producer warp.  Global
// layout of the transition matrices for this kernel: per branch, R category
// blocks of SP*SP Reals padded to CS bytes (16 extra bytes when R > 1 so the
// categories of a warp hit distinct shared-memory banks): one branch's
// matrices are one contiguous bulk copy.
template <typename Real, int SP, int RP, int TC = 0>
struct SmallCfg {
    static constexpr bool MMA = TC && SP == 16;                 // tensor-core S = 16, R = 1
    static constexpr bool MMA4 = TC && SP == 4;                 // tensor-core S = 4, R = 4
    static constexpr int LV = small_lanes_per_vector(SP, RP); // lanes per vector
    static constexpr int VL = SP / LV;                         // states per lane
    static constexpr int TP = 32 / (RP * LV);                  // patterns per warp tile
#ifndef PG_STAGES
    // stage ring depth (steps); the tensor-core S = 16 variant's steps are
    // short enough that 4 stages do not cover the copies' latency
    static constexpr int D = MMA ? PG_MMA_STAGES : 4;
#else
    static constexpr int D = PG_STAGES;
#endif
#ifdef PG_PF
    static constexpr int PF = PG_PF;
#else
    static constexpr int PF = 32;                              // L2 prefetch distance (steps; 16: +0.4 %, scripts/gpu_pf.sh)
#endif
    // gradient window (steps): per pre step the lanes of a pattern sum their
    // (num_a, num_b, den) shares (xor shuffles) and one lane stores the three
    // totals; every W steps the warp forms the Eq. 8 ratios of W x TP
    // (step, pattern) items, PPL per lane (ILP instead of a per-2-step
    // latency chain); W TP 3 doubles per warp
#ifdef PG_SMALL_W
    static constexpr int W = PG_SMALL_W;
#else
    // 128 / TP steps (3 KB per warp): dengue traversal 1.316 (8 steps) -> 1.302 ms
    // (16 steps) vs 1.358 ms (4 steps), MMM 0.1024 -> 0.1004 ms (scripts/gpu_r3_ab.sh)
    static constexpr int W = (128 / TP) < 32 ? ((128 / TP) > 0 ? 128 / TP : 1) : 32;
#endif
    static constexpr int LPS = 32 / W;                         // lanes per window step
    static constexpr int PPL = TP / LPS > 0 ? TP / LPS : 1;    // patterns per lane in a flush
    static constexpr int VB = SP * (int)sizeof(Real);          // vector bytes
    static constexpr int VBL = VL * (int)sizeof(Real);         // one lane's part of a vector
    static constexpr int MATB = SP * SP * (int)sizeof(Real);   // one category's matrix
    static constexpr int CS = MATB + (RP > 1 ? small_cat_pad(sizeof(Real), SP) : 0);   // padded category stride
    static constexpr int ND = W * TP * 3 * 8;                  // (num_a, num_b, den) window per warp
    static constexpr int XGS = VB + 16;                        // exchange stride per lane group (bank skew)
    static constexpr int XB = (LV > 1 && !MMA) ? (32 / LV) * XGS : 0;   // full-vector exchange buffer per warp
#ifdef PG_OPS
    static constexpr int OPS = PG_OPS;
#else
    static constexpr int OPS = 1;
#endif
    static constexpr int DS = D / OPS < 2 ? 2 : D / OPS;
    // grouped post-order staging: GPOST steps per stage, DPG stages
    static constexpr int GPOST = PG_GPOST, DPG = 4;
    static __host__ __device__ int rec_bytes(int R) { return 16 + 3 * mat_slot(R); }
    static __host__ __device__ int gstage(int R, int tipw) { return GPOST * (rec_bytes(R) + 2 * tipw); }
    static __host__ __device__ size_t ring(int R, int K, int tipw) {
        const size_t a = (size_t)DS * OPS * stage(R, K), b = tipw > 0 ? (size_t)DPG * gstage(R, tipw) : 0;
        return a > b ? a : b;
    }
    // barriers (full[DS], empty[DS], post_done, prog_bar) below QOFF, then Q
    // (SP > 4 only; SP <= 4 keeps it in registers).  QOFF follows DS: a fixed
    // 128 B let an 8-stage ring's post_done / prog_bar overlap Q (found by
    // compute-sanitizer synccheck on the S = 16 tensor-core variant)
    static constexpr int QOFF = (8 * (2 * DS + 2 + 2 * DPG) + 127) / 128 * 128;
    static constexpr int BARS = QOFF + (SP > 4 ? SP * SP * (int)sizeof(Real) : 0);   // barriers + Q
    static __host__ __device__ int mat_slot(int R) { return MMA ? MMA_SLOT : MMA4 ? MMA4_SLOT : R * CS; }
    static __host__ __device__ int mat_rec(int R) { return MMA ? MMA_REC : MMA4 ? 2 * MMA4_SLOT : R * CS; }   // bytes per branch in HBM
    static __host__ __device__ int vslot(int R, int K) {       // one child's vectors for K warps
        int a = K * TP * R * VB, b = K * TP * VB, c = (15 + K * TP + 15) / 16 * 16;
        int m = a > b ? a : b;
        m = m > c ? m : c;
        return (m + 15) / 16 * 16;
    }
    static __host__ __device__ int stage(int R, int K) { return 16 + 3 * mat_slot(R) + 2 * vslot(R, K); }
    // stack: depth slots + one holding pi (the root's q)
    static __host__ __device__ int warp_bytes(int depth) {
        return ((depth + 1) * 32 * VBL + ND + XB + TP * 8 + W * 2 * 4 + 8 + 15) / 16 * 16;
    }
    // OPS consecutive ops share one ring stage (one full/empty barrier pair),
    // DS stages in the ring.  Pairing halves the barrier traffic but lets the
    // producer refill only after both ops: 24 % slower for S = 4; for S = 16
    // (MMM) 2 stages x 2 ops vs 4 stages x 1 op measured 0.228 vs 0.222 ms
    // (scripts/gpu_mmm_stages.sh), so one op per stage everywhere.
    static __host__ __device__ size_t smem(int R, int K, int depth, int tipw = 0) {
        return (size_t)BARS + ring(R, K, tipw) + (size_t)K * warp_bytes(depth);
    }
};

// ---- vector access helpers (n values, 16-byte chunks where possible) -------
template <typename Real, int n>
__device__ __forceinline__ void lds_vec(Real (&d)[n], const void *src) {
    if constexpr (sizeof(Real) == 8) {
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            const double2 t = reinterpret_cast<const double2 *>(src)[i];
            d[2 * i] = t.x;
            d[2 * i + 1] = t.y;
        }
        if constexpr (n % 2) d[n - 1] = reinterpret_cast<const double *>(src)[n - 1];
    } else if constexpr (n % 4 == 0) {
#pragma unroll
        for (int i = 0; i < n / 4; ++i) {
            const float4 t = reinterpret_cast<const float4 *>(src)[i];
            d[4 * i] = t.x; d[4 * i + 1] = t.y; d[4 * i + 2] = t.z; d[4 * i + 3] = t.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < n; ++i) d[i] = reinterpret_cast<const float *>(src)[i];
    }
}
template <typename Real, int n>
__device__ __forceinline__ void sts_vec(void *dst, const Real (&d)[n]) {
    if constexpr (sizeof(Real) == 8) {
#pragma unroll
        for (int i = 0; i < n / 2; ++i) reinterpret_cast<double2 *>(dst)[i] = make_double2(d[2 * i], d[2 * i + 1]);
        if constexpr (n % 2) reinterpret_cast<double *>(dst)[n - 1] = d[n - 1];
    } else if constexpr (n % 4 == 0) {
#pragma unroll
        for (int i = 0; i < n / 4; ++i)
            reinterpret_cast<float4 *>(dst)[i] = make_float4(d[4 * i], d[4 * i + 1], d[4 * i + 2], d[4 * i + 3]);
    } else {
#pragma unroll
        for (int i = 0; i < n; ++i) reinterpret_cast<float *>(dst)[i] = d[i];
    }
}
template <typename Real, int n>
__device__ __forceinline__ void stg_vec(void *dst, const Real (&d)[n]) {
    if constexpr (sizeof(Real) == 8) {
#pragma unroll
        for (int i = 0; i < n / 2; ++i) __stcg(reinterpret_cast<double2 *>(dst) + i, make_double2(d[2 * i], d[2 * i + 1]));
        if constexpr (n % 2) __stcg(reinterpret_cast<double *>(dst) + n - 1, d[n - 1]);
    } else if constexpr (n % 4 == 0) {
#pragma unroll
        for (int i = 0; i < n / 4; ++i)
            __stcg(reinterpret_cast<float4 *>(dst) + i, make_float4(d[4 * i], d[4 * i + 1], d[4 * i + 2], d[4 * i + 3]));
    } else {
#pragma unroll
        for (int i = 0; i < n; ++i) __stcg(reinterpret_cast<float *>(dst) + i, d[i]);
    }
}

// The lane owns states [h VL, h VL + VL) of a vector.  Whole vectors it
// gathers are kept ROTATED by h VL (its own block first): x[j] holds state
// (j + h VL) mod SP.  Walking matrix rows in the same rotated order makes the
// LV lanes of a group read different shared-memory banks (rows are 32 banks
// long, so unrotated they would all start on bank 0).  LV = 1: no rotation.
// y = rows [h VL, +VL) of M x, M row-major SP x SP in shared memory
template <typename Real, int SP, int VL>
__device__ __forceinline__ void mv(Real (&y)[VL], const Real *M, const Real (&x)[SP], int h) {
    constexpr int LV = SP / VL;
#pragma unroll
    for (int i = 0; i < VL; ++i) {
        const Real *row = M + (h * VL + i) * SP;
        Real acc = 0;
#pragma unroll
        for (int b = 0; b < LV; ++b) {
            Real blk[VL];
            lds_vec<Real, VL>(blk, row + ((b + h) & (LV - 1)) * VL);
#pragma unroll
            for (int t = 0; t < VL; ++t) acc = (b == 0 && t == 0) ? blk[0] * x[0] : fma(blk[t], x[b * VL + t], acc);
        }
        y[i] = acc;
    }
}
// y = entries [h VL, +VL) of M' x (y[i] = sum_s M[s][h VL + i] x[s]), x rotated
template <typename Real, int SP, int VL>
__device__ __forceinline__ void mvt(Real (&y)[VL], const Real *M, const Real (&x)[SP], int h) {
#pragma unroll
    for (int j = 0; j < SP; ++j) {
        const int s = (j + h * VL) & (SP - 1);
        Real row[VL];
        lds_vec<Real, VL>(row, M + s * SP + h * VL);
#pragma unroll
        for (int i = 0; i < VL; ++i) y[i] = j == 0 ? row[i] * x[0] : fma(row[i], x[j], y[i]);
    }
}
// rotated whole vector from shared memory (LV blocks of VL)
template <typename Real, int SP, int VL>
__device__ __forceinline__ void lds_rot(Real (&x)[SP], const unsigned char *src, int h) {
    constexpr int LV = SP / VL;
#pragma unroll
    for (int b = 0; b < LV; ++b) {
        Real blk[VL];
        lds_vec<Real, VL>(blk, src + ((b + h) & (LV - 1)) * VL * (int)sizeof(Real));
#pragma unroll
        for (int t = 0; t < VL; ++t) x[b * VL + t] = blk[t];
    }
}
// u = entries [h VL, +VL) of column s of M (observed tip state) or of M 1 (missing, s >= S)
// ONECOL: M 1 is stored right after M (pmat_kernel fills the category pad),
// so both cases are one gather with no divergent branch
template <typename Real, int SP, int VL, bool ONECOL = false>
__device__ __forceinline__ void mcol(Real (&u)[VL], const Real *M, int s, int S, int h) {
    if constexpr (ONECOL) {
        const bool obs = s < S;
#pragma unroll
        for (int x = 0; x < VL; ++x) u[x] = M[obs ? (h * VL + x) * SP + s : SP * SP + h * VL + x];
        return;
    }
    if (s < S) {
#pragma unroll
        for (int x = 0; x < VL; ++x) u[x] = M[(h * VL + x) * SP + s];
    } else {
#pragma unroll
        for (int x = 0; x < VL; ++x) {
            Real row[SP];
            lds_vec<Real, SP>(row, M + (h * VL + x) * SP);
            Real acc = row[0];
#pragma unroll
            for (int t = 1; t < SP; ++t) acc += row[t];
            u[x] = acc;
        }
    }
}

// ---- exact power-of-two rescaling -----------------------------------------
// high word of a non-negative value: ordered like the value, exponent field in
// bits 20 (fp64) / 23 (fp32) and up
__device__ __forceinline__ int hiword(double x) { return __double2hiint(x); }
__device__ __forceinline__ int hiword(float x) { return __float_as_int(x); }
template <typename Real, int SP>
__device__ __forceinline__ int max_hiword(const Real (&v)[SP]) {
    int m = hiword(v[0]);
#pragma unroll
    for (int i = 1; i < SP; ++i) m = max(m, hiword(v[i]));
    return m;
}
template <typename Real> struct ScaleTraits;
template <> struct ScaleTraits<double> {
    static constexpr int THRESH = 1023 - 256;   // rescale once a max drops below 2^-256
    static constexpr int SHIFT = 20;
    static __device__ __forceinline__ int exponent(int field) { return min(max(field - 1022, -1021), 1022); }
    static __device__ __forceinline__ double factor(int e) { return __longlong_as_double((long long)(1023 - e) << 52); }
};
template <> struct ScaleTraits<float> {
    static constexpr int THRESH = 127 - 64;      // 2^-64
    static constexpr int SHIFT = 23;
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
// n / d for the Eq. 8 ratio, branch-free: hardware reciprocal estimate, two
// Newton steps and one residual correction (faithful to <= 1 ulp; d is a
// normal positive number: vectors are rescaled long before denormals).
__device__ __forceinline__ double ratio(double n, double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    const double q = n * r;
    return fma(fma(-d, q, n), r, q);
}
// [8 patterns x 16] x [16 x 16] on the FP64 tensor path: y (the lane's 4
// states, slot order) = A (slot order) times the fragment-ordered B operand
// Bf[(kt * 2 + nt) * 32 + lane]; see small_mma.
__device__ __forceinline__ void dmma16(double (&y)[4], const double (&A)[4], const double *Bf, int lane) {
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
        const double b0 = Bf[(kt * 2) * 32 + lane], b1 = Bf[(kt * 2 + 1) * 32 + lane];
        PG_MMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c0[0]), "+d"(c0[1]) : "d"(A[kt]), "d"(b0));
        PG_MMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c1[0]), "+d"(c1[1]) : "d"(A[kt]), "d"(b1));
    }
    y[0] = c0[0];
    y[1] = c0[1];
    y[2] = c1[0];
    y[3] = c1[1];
}
// one category of the S = 4 variant: C = A (8 x 4) B (4 x 8); the lane's
// first C element is state (lane % 4) of its pattern (see small_tc)
__device__ __forceinline__ double dmma4(double a, double b) {
    double c0 = 0.0, c1 = 0.0;
    PG_MMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    return c0;
}
__device__ __forceinline__ void dmma16r(double (&y)[4], const double (&A)[4], const double (&B)[8]) {
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
        PG_MMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c0[0]), "+d"(c0[1]) : "d"(A[kt]), "d"(B[2 * kt]));
        PG_MMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c1[0]), "+d"(c1[1]) : "d"(A[kt]), "d"(B[2 * kt + 1]));
    }
    y[0] = c0[0];
    y[1] = c0[1];
    y[2] = c1[0];
    y[3] = c1[1];
}

// Rescale v (exactly) if any vector of the warp fell below the threshold;
// returns the exponent removed (shared by the categories of a pattern).
// G = lanes sharing one pattern (categories x state groups, contiguous)
template <typename Real, int SP, int G>
__device__ __forceinline__ int maybe_rescale(Real (&v)[SP]) {
    using T = ScaleTraits<Real>;
    const int h = max_hiword<Real, SP>(v);
    if (!__any_sync(0xffffffffu, h < (T::THRESH << T::SHIFT))) return 0;
    const int e = T::exponent(cat_max<G>(h) >> T::SHIFT);
    const Real s = ScaleTraits<Real>::factor(e);
#pragma unroll
    for (int i = 0; i < SP; ++i) v[i] *= s;
    return e;
}


// GRP: grouped post-order staging (a.rec_post / a.tipstream; SP = 4 only)
template <typename Real, int SP, int RP, int TC = 0, bool GRP = false>
__global__ void __launch_bounds__(32 * (small_max_consumers(SP, RP) + 1), 1) traverse_small_kernel(const TravArgs a) {
    using Cfg = SmallCfg<Real, SP, RP, TC>;
    constexpr int TP = Cfg::TP, PF = Cfg::PF, W = Cfg::W, VB = Cfg::VB, CS = Cfg::CS;
    constexpr int LV = Cfg::LV, VL = Cfg::VL, VBL = Cfg::VBL, G = RP * LV;
    constexpr int OPS = Cfg::OPS, DS = Cfg::DS;
    extern __shared__ __align__(128) unsigned char smem_s[];
    unsigned char *smem = smem_s;
    const int R = a.R, N = a.N, S = a.S;
    const int K = blockDim.x / 32 - 1;              // consumer warps; warp K = producer
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nops = N - 1, root = 2 * N - 2;
    const int MS = Cfg::mat_slot(R), VS = Cfg::vslot(R, K), ST = Cfg::stage(R, K);
    const int MREC = Cfg::mat_rec(R);
    constexpr bool MMA = Cfg::MMA, MMA4 = Cfg::MMA4;
    const size_t Cpad = (size_t)a.Cpad;
    const int cta_tile0 = blockIdx.x * K;
    const int ntile = min(K, a.n_tiles - cta_tile0);               // live tiles of this CTA
    const int cta_pat0 = cta_tile0 * TP;
    const size_t u_node = Cpad * R * VB;                           // one node's u block (bytes)

    uint64_t *full = reinterpret_cast<uint64_t *>(smem);            // [D]
    uint64_t *empty = full + DS;                                    // [DS]
    uint64_t *post_done = empty + DS;                               // [1]
    uint64_t *gfull = post_done + 2, *gempty = gfull + Cfg::DPG;    // grouped post stages
    unsigned char *stages = smem + Cfg::BARS;
    // GRP: staging records (A1 writes each step's matrices next to its op);
    // S = 4 with state tips also groups GPOST post steps per ring stage
    constexpr bool records = GRP, grouped = GRP && !Cfg::MMA && !Cfg::MMA4;
    constexpr int GG = Cfg::GPOST, DPG = Cfg::DPG;
    const int RECB = Cfg::rec_bytes(a.R), TW = a.tipw, GSTG = grouped ? Cfg::gstage(a.R, a.tipw) : 0;
    // shared-window addresses of the barriers and stages (loop-invariant bases)
    const uint32_t sbase = smem_u32(smem);
    const uint32_t full_u = sbase, empty_u = sbase + 8u * DS, stages_u = sbase + Cfg::BARS;
    // step t (post 0..nops-1, pre nops..2nops-1) -> ring stage and slot; the
    // pre program starts on a fresh stage
    // grouped: the pre program's stages are numbered from 0 (the post
    // program uses its own ring and barriers)
    const int GP = grouped ? 0 : (nops + OPS - 1) / OPS;
    auto stg = [&](int t) { return t < nops ? t / OPS : GP + (t - nops) / OPS; };
    auto slot = [&](int t) { return t < nops ? t % OPS : (t - nops) % OPS; };
    auto sub_off = [&](int t) { return (stg(t) % DS) * (OPS * ST) + slot(t) * ST; };
    auto last_in_stage = [&](int t) { return slot(t) == OPS - 1 || t == nops - 1 || t == 2 * nops - 1; };
    auto wait_full = [&](int t) { const int g = stg(t); mbar_wait_u32(full_u + 8u * (g % DS), (uint32_t)(g / DS) & 1u); };

    const char *__restrict__ Pb = static_cast<const char *>(a.P);
    const char *__restrict__ tipP = static_cast<const char *>(a.tip_partials);
    const uint8_t *__restrict__ tipS = a.tip_states;
    char *__restrict__ Ub = static_cast<char *>(a.u);

    // both traversal programs staged once in shared memory (when they fit), so
    // neither the producer nor the consumers read ops from global memory
    uint64_t *prog_bar = post_done + 1;
    const Op4 *post_prog = a.post, *pre_prog = a.pre;
    if (a.prog_smem_off > 0) {
        post_prog = reinterpret_cast<const Op4 *>(smem + a.prog_smem_off);
        pre_prog = post_prog + (N - 1);
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < DS; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, K); }
        for (int i = 0; i < DPG; ++i) { mbar_init(gfull + i, 1); mbar_init(gempty + i, K); }
        mbar_init(post_done, K);
        mbar_init(prog_bar, 1);
        fence_mbar_init();
        if (a.prog_smem_off > 0) {
            const unsigned pb = (unsigned)(N - 1) * 16u;
            mbar_arrive_expect_tx(prog_bar, 2 * pb);
            bulk_g2s(smem + a.prog_smem_off, a.post, pb, prog_bar);
            bulk_g2s(smem + a.prog_smem_off + pb, a.pre, pb, prog_bar);
        } else {
            mbar_arrive_expect_tx(prog_bar, 0);
        }
    }
    if constexpr (SP > 4) {
        Real *Qs = reinterpret_cast<Real *>(smem + Cfg::QOFF);
        for (int i = threadIdx.x; i < SP * SP; i += blockDim.x) Qs[i] = static_cast<const Real *>(a.Q)[i];
    }
    __syncthreads();
    mbar_wait(prog_bar, 0u);
    // PDL launch behind A1: everything above overlapped it; the matrices (and
    // the status words A1 resets) are read only after this
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // A6 fused (a.a6cnt; the host sets it only when the whole grid is
    // co-resident): after its warps are done every CTA counts itself
    // finished; once all are, CTA c sums rows c, c + grid, ... of the
    // per-tile partials (threads stride the tiles, then a fixed tree) into
    // out = [logL, g] -- in place of reduce_kernel, the same numbers whichever
    // CTA takes a row.  Reached by the producer and the consumer warps at
    // different points: named barrier 1.
    auto a6_epilogue = [&]() {
        if constexpr (MMA || MMA4) return;     // (not offered on the tensor path)
        if (!a.a6cnt) return;
        __shared__ double a6red[32];
        asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(a.a6cnt, 1);
            int x;
            unsigned long long t0;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            for (unsigned it = 0;; ++it) {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(x) : "l"(a.a6cnt) : "memory");
                if (x >= (int)gridDim.x) break;
                if ((it & 1023u) == 1023u) {
                    unsigned long long t1;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                    if (t1 - t0 > 20000000000ull) { atomicExch(a.status + 1, 1); break; }   // reported as a stall
                }
                __nanosleep(64);
            }
            __threadfence();
        }
        asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
        const int B = 2 * N - 2, nw = blockDim.x >> 5;
        for (int row = blockIdx.x; row <= B; row += gridDim.x) {
            const double *src = row < B ? a.grad_part + (size_t)row * a.n_tiles : a.logl_part;
            double acc = 0.0;
            for (int i = threadIdx.x; i < a.n_tiles; i += blockDim.x) acc += __ldcg(src + i);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if ((threadIdx.x & 31) == 0) a6red[threadIdx.x >> 5] = acc;
            asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
            if (threadIdx.x == 0) {
                double t = 0.0;
                for (int w2 = 0; w2 < nw; ++w2) t += a6red[w2];
                a.out[row < B ? 1 + row : 0] = t;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
        }
    };

    // =============================== producer ===================================
    if (warp == K) {
        const unsigned u_bytes = ntile * TP * R * VB;
        const size_t u_cta = (size_t)cta_pat0 * R * VB;
        const unsigned tipp_bytes = ntile * TP * VB;
        const int tip_lead = cta_pat0 & 15;
        const unsigned tipw_bytes = (tip_lead + ntile * TP + 15) / 16 * 16;
        auto tip_bytes = [&](int code) -> unsigned { return (code & kTipPartialBit) ? tipp_bytes : tipw_bytes; };
        auto copy_tip = [&](uint32_t dst, int code, uint32_t bar) {
            const int node = code & ~kTipPartialBit;
            if (code & kTipPartialBit) bulk_g2s_u32(dst, tipP + ((size_t)node * Cpad + cta_pat0) * VB, tipp_bytes, bar);
            else bulk_g2s_u32(dst, tipS + ((size_t)node * Cpad + cta_pat0 - tip_lead), tipw_bytes, bar);
        };
        auto u_src = [&](int node) -> const char * { return Ub + (size_t)(node - N) * u_node + u_cta; };
        // the matrix a step reads for node `code` in role `pre` (MMA: which
        // layout of the branch record; else the branch's R category blocks)
        auto mat_src = [&](int code, bool pre_child) -> const char * {
            const int node = code & ~kTipPartialBit;
            const char *rec = Pb + (size_t)node * MREC;
            if constexpr (MMA) {
                const int lay = node >= N ? (pre_child ? 1 : 0) : ((code & kTipPartialBit) ? 0 : 2);
                return rec + lay * MMA_SLOT;
            }
            if constexpr (MMA4) return rec + ((node >= N && pre_child) ? MMA4_SLOT : 0);
            return rec;
        };
        // bytes and copies of step t's sub-stage:
        //   post [op][P_k][P_a][P_b][tip a][tip b];  pre [op][P_a][P_b][-][vec a][vec b]
        auto op_bytes = [&](int t) -> unsigned {
            const bool pre = t >= nops;
            const int m = pre ? t - nops : t;
            const Op4 op = (pre ? pre_prog : post_prog)[m];
            if (!pre && records)
                return 16 + 3 * MS + (op.y >= 0 ? tip_bytes(op.y) : 0) + (op.z >= 0 ? tip_bytes(op.z) : 0);
            if (!pre)
                return 16 + (op.x != root ? MS : 0) + (op.y >= 0 ? MS + tip_bytes(op.y) : 0) +
                       (op.z >= 0 ? MS + tip_bytes(op.z) : 0);
            const int na = op.y & ~kTipPartialBit, nb = op.z & ~kTipPartialBit;
            return 16 + 2 * MS + (na >= N ? u_bytes : tip_bytes(op.y)) + (nb >= N ? u_bytes : tip_bytes(op.z));
        };
        auto op_issue = [&](int t, uint32_t st, uint32_t bar) {
            const bool pre = t >= nops;
            const int m = pre ? t - nops : t;
            const Op4 *gprog = pre ? a.pre : a.post;           // global copy (bulk source)
            const Op4 *prog = pre ? pre_prog : post_prog;       // smem copy when staged
            const Op4 op = prog[m];
            if (records && !pre) {
                // the step's record: op, P_k and the tip children's matrices
                bulk_g2s_u32(st, a.rec_post + (size_t)m * (16 + 3 * MS), 16 + 3 * MS, bar);
                if (op.y >= 0) copy_tip(st + 16 + 3 * MS, op.y, bar);
                if (op.z >= 0) copy_tip(st + 16 + 3 * MS + VS, op.z, bar);
                return;
            }
            if (records && pre) {
                // the step's record: op and both children's matrices, one copy
                const unsigned recpb = 16 + 2 * MS;
                bulk_g2s_u32(st, a.rec_pre + (size_t)m * recpb, recpb, bar);
                const int na = op.y & ~kTipPartialBit, nb = op.z & ~kTipPartialBit;
                if (na >= N) bulk_g2s_u32(st + 16 + 3 * MS, u_src(na), u_bytes, bar);
                else copy_tip(st + 16 + 3 * MS, op.y, bar);
                if (nb >= N) bulk_g2s_u32(st + 16 + 3 * MS + VS, u_src(nb), u_bytes, bar);
                else copy_tip(st + 16 + 3 * MS + VS, op.z, bar);
                if (m + PF < nops) {
                    const Op4 o2 = prog[m + PF];
                    const int pa = o2.y & ~kTipPartialBit, pb = o2.z & ~kTipPartialBit;
                    if (pa >= N) prefetch_l2(u_src(pa), u_bytes);
                    if (pb >= N) prefetch_l2(u_src(pb), u_bytes);
                }
                return;
            }
            bulk_g2s_u32(st, gprog + m, 16, bar);
            if (PG_TIPP_PF && tipP && m + PF < nops) {      // partial-tip chunks into L2 ahead (HBM latency)
                const Op4 o2 = prog[m + PF];
                if (o2.y >= 0 && (o2.y & kTipPartialBit))
                    prefetch_l2(tipP + ((size_t)(o2.y & ~kTipPartialBit) * Cpad + cta_pat0) * VB, tipp_bytes);
                if (o2.z >= 0 && (o2.z & kTipPartialBit))
                    prefetch_l2(tipP + ((size_t)(o2.z & ~kTipPartialBit) * Cpad + cta_pat0) * VB, tipp_bytes);
            }
            if (!pre) {
                if (op.x != root) bulk_g2s_u32(st + 16, mat_src(op.x, false), MS, bar);
                if (op.y >= 0) {
                    bulk_g2s_u32(st + 16 + MS, mat_src(op.y, false), MS, bar);
                    copy_tip(st + 16 + 3 * MS, op.y, bar);
                }
                if (op.z >= 0) {
                    bulk_g2s_u32(st + 16 + 2 * MS, mat_src(op.z, false), MS, bar);
                    copy_tip(st + 16 + 3 * MS + VS, op.z, bar);
                }
            } else {
                const int na = op.y & ~kTipPartialBit, nb = op.z & ~kTipPartialBit;
                bulk_g2s_u32(st + 16, mat_src(op.y, true), MS, bar);
                bulk_g2s_u32(st + 16 + MS, mat_src(op.z, true), MS, bar);
                if (na >= N) bulk_g2s_u32(st + 16 + 3 * MS, u_src(na), u_bytes, bar);
                else copy_tip(st + 16 + 3 * MS, op.y, bar);
                if (nb >= N) bulk_g2s_u32(st + 16 + 3 * MS + VS, u_src(nb), u_bytes, bar);
                else copy_tip(st + 16 + 3 * MS + VS, op.z, bar);
                if (m + PF < nops) {                         // pull later u chunks into L2
                    const Op4 o2 = prog[m + PF];
                    const int pa = o2.y & ~kTipPartialBit, pb = o2.z & ~kTipPartialBit;
                    if (pa >= N) prefetch_l2(u_src(pa), u_bytes);
                    if (pb >= N) prefetch_l2(u_src(pb), u_bytes);
                }
            }
        };
        if (grouped) {
            // post program: GG steps per stage -- the steps' records (op,
            // matrices) and this CTA's tip-code windows, two bulk copies
            const int NGP = (nops + GG - 1) / GG;
            for (int g = 0; g < NGP; ++g) {
                const int sg = g % DPG;
                if (g >= DPG) mbar_wait_u32(smem_u32(gempty + sg), (uint32_t)(g / DPG + 1) & 1u);
                if (lane == 0) {
                    const int m0 = g * GG, cnt = min(GG, nops - m0);
                    const uint32_t bar = smem_u32(gfull + sg), dst = stages_u + sg * GSTG;
                    mbar_arrive_expect_tx_u32(bar, (unsigned)cnt * (RECB + 2 * TW));
                    bulk_g2s_u32(dst, a.rec_post + (size_t)m0 * RECB, (unsigned)cnt * RECB, bar);
                    bulk_g2s_u32(dst + GG * RECB, a.tipstream + ((size_t)blockIdx.x * nops + m0) * 2 * TW,
                                 (unsigned)cnt * 2 * TW, bar);
                }
                __syncwarp();
            }
        }
        const int NG = GP + (nops + OPS - 1) / OPS;
        for (int g = grouped ? 0 : 0; g < NG; ++g) {
            const bool pre = grouped || g >= GP;
            const int t0 = pre ? nops + (g - GP) * OPS : g * OPS;
            const int t1 = min(t0 + OPS, pre ? 2 * nops : nops);
            PG_TSTAMP((size_t)t0 * 16 + 0, g);
            if (g == GP) mbar_wait(post_done, 0);            // u of every tile stored + fenced
            if (g >= DS) mbar_wait_u32(empty_u + 8u * (g % DS), (uint32_t)(g / DS + 1) & 1u);
            PG_TSTAMP((size_t)t0 * 16 + 1, g);
            if (lane == 0) {
                const uint32_t bar = full_u + 8u * (g % DS);
                unsigned total = 0;
                for (int t = t0; t < t1; ++t) total += op_bytes(t);
                if (PG_PROXY_FENCE) fence_proxy_async_smem();
                mbar_arrive_expect_tx_u32(bar, total);
                for (int t = t0; t < t1; ++t) op_issue(t, stages_u + sub_off(t), bar);
            }
            __syncwarp();
            PG_TSTAMP((size_t)t0 * 16 + 2, g);
        }
        a6_epilogue();
        return;
    }

    // =============================== consumers ==================================
    // lane = (pattern pl, category cat, state group h), h fastest; the G = RP LV
    // lanes of one pattern are contiguous.
    const int tile = cta_tile0 + warp;
    const bool active = warp < ntile;
    const int h = lane & (LV - 1);
    const int cat = (lane / LV) & (RP - 1);
    const int r = min(cat, R - 1);                  // shadow lanes reuse category R-1
    const bool live = cat < R;
    const int pl = lane / G;
    const int pat0 = tile * TP;
    const int pat = pat0 + pl;
    unsigned char *wsm = stages + Cfg::ring(R, K, grouped ? TW : 0) + (size_t)warp * Cfg::warp_bytes(a.depth);
    unsigned char *stackb = wsm;
    const int pi_slot = a.depth;
    double *nd = reinterpret_cast<double *>(wsm + (a.depth + 1) * 32 * VBL);       // [W][TP][3]
    unsigned char *xb = wsm + (a.depth + 1) * 32 * VBL + Cfg::ND;                  // exchange [32/LV][XGS]
    double *wbuf = reinterpret_cast<double *>(xb + Cfg::XB);                        // [TP]
    int *nodes_w = reinterpret_cast<int *>(wbuf + TP);                              // [W][2] branch ids
    const double wr = live ? a.cat_w[r] : 0.0;
    const double gwr = wr * a.cat_g[r];
    // MMA4: the lane's registers are the four categories of state j = cat
    double wR[MMA4 ? 4 : 1], gwR[MMA4 ? 4 : 1];
    if constexpr (MMA4) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            wR[q] = a.cat_w[q];
            gwR[q] = wR[q] * a.cat_g[q];
        }
    }
    Real pi[VL];
#pragma unroll
    for (int s = 0; s < VL; ++s) pi[s] = static_cast<const Real *>(a.pi)[MMA ? 4 * s + h : MMA4 ? cat : h * VL + s];
    if (active && lane < TP) wbuf[lane] = a.pat_w[pat0 + lane];
    __syncwarp();

    const unsigned mat_lane = r * CS;
    const unsigned u_vec = ((warp * TP + pl) * R + r) * VB + h * VBL;   // my part inside a CTA u chunk
    const int tip_idx = (cta_pat0 & 15) + warp * TP + pl;          // my code inside a tip window
    const unsigned tipp_vec = (warp * TP + pl) * VB;               // my tip partial vector (whole)
    const size_t u_lane = (size_t)pat * R * VB + r * VB + h * VBL;
    unsigned char *xg = xb + (lane / LV) * Cfg::XGS;               // my group's exchange row
    auto stack_at = [&](int slot) -> unsigned char * { return stackb + (slot * 32 + lane) * VBL; };
    // stack slots as 16-B planes [slot][plane][lane]: a lane's 32-B part at a
    // 32-B lane stride cost 2-way bank conflicts per 128-bit access (dengue
    // fp64 traversal 1.493 -> 1.434 ms, scripts/gpu_ss.sh; PG_STACK_INTERLEAVED
    // restores the old layout)
    constexpr int NPL = VBL > 16 ? VBL / 16 : 1, PLB = VBL > 16 ? 16 : VBL;
    auto stk_ld = [&](Real (&v)[VL], int slot) {
#ifndef PG_STACK_INTERLEAVED
        constexpr int PE = PLB / (int)sizeof(Real);
#pragma unroll
        for (int c = 0; c < NPL; ++c) {
            Real t[PE];
            lds_vec<Real, PE>(t, stackb + ((slot * NPL + c) * 32 + lane) * PLB);
#pragma unroll
            for (int i = 0; i < PE; ++i) v[c * PE + i] = t[i];
        }
#else
        lds_vec<Real, VL>(v, stack_at(slot));
#endif
    };
    auto stk_st = [&](int slot, const Real (&v)[VL]) {
#ifndef PG_STACK_INTERLEAVED
        constexpr int PE = PLB / (int)sizeof(Real);
#pragma unroll
        for (int c = 0; c < NPL; ++c) {
            Real t[PE];
#pragma unroll
            for (int i = 0; i < PE; ++i) t[i] = v[c * PE + i];
            sts_vec<Real, PE>(stackb + ((slot * NPL + c) * 32 + lane) * PLB, t);
        }
#else
        sts_vec<Real, VL>(stack_at(slot), v);
#endif
    };
    auto release = [&](int t) {                      // after step t's last use of its stage
        if (!last_in_stage(t)) return;
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(empty_u + 8u * (stg(t) % DS));
    };
    // the whole SP-vector of my (pattern, category) from the lanes' parts, rotated by h VL
    auto gather = [&](Real (&full)[SP], const Real (&part)[VL]) {
        if constexpr (LV == 1) {
#pragma unroll
            for (int s = 0; s < SP; ++s) full[s] = part[s];
        } else {
            __syncwarp();
            sts_vec<Real, VL>(xg + h * VBL, part);
            __syncwarp();
            lds_rot<Real, SP, VL>(full, xg, h);
        }
    };
    auto child_tip = [&](Real (&u)[VL], const unsigned char *M_, const unsigned char *vs, int code) {
        const Real *M = reinterpret_cast<const Real *>(M_ + mat_lane);
        if constexpr (MMA4) {
            const double *Bf = reinterpret_cast<const double *>(M_);     // [4 categories][32] (u = P p layout)
            if (code & kTipPartialBit) {
                const double pt = reinterpret_cast<const double *>(vs + tipp_vec)[cat];
#pragma unroll
                for (int q = 0; q < 4; ++q) u[q] = dmma4(pt, Bf[q * 32 + lane]);
            } else {                                // P[j][state] sits at lane 8 j + state
                const int sv = vs[tip_idx];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double *row = Bf + q * 32 + 8 * cat;
                    u[q] = sv < S ? row[sv] : (row[0] + row[1]) + (row[2] + row[3]);
                }
            }
            return;
        }
        if constexpr (MMA) {
            if (code & kTipPartialBit) {            // u = P p_tip: the lane's states of p_tip, one product
                const double *tp = reinterpret_cast<const double *>(vs + tipp_vec);
                double pa[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) pa[i] = tp[4 * i + h];
                dmma16(u, pa, M, lane);
            } else {                                // column `state` of P (column 16 = P 1: missing)
                const int sv = vs[tip_idx];
                const int col = sv < S ? sv : 16;
#pragma unroll
                for (int i = 0; i < 4; ++i) u[i] = M[(4 * i + h) * MMA_RS + col];
            }
            return;
        }
        if (code & kTipPartialBit) {
            Real tp[SP];
            lds_rot<Real, SP, VL>(tp, vs + tipp_vec, h);
            mv<Real, SP, VL>(u, M, tp, h);
        } else {
            mcol<Real, SP, VL, (CS - Cfg::MATB >= VB)>(u, M, vs[tip_idx], S, h);
        }
    };

    // ------------------------- post program (Eq. 2, Eq. 3) -----------------------
    // The next op is decoded while the current step computes, and the u just
    // pushed is forwarded through registers when the next op consumes it
    // (the common case in a depth-first order): no STS -> LDS round trip.
    int E = 0;                    // post-order exponents removed from this pattern
    double logl_local = 0.0;
    int prev_slot = -1;
    Real prev_u[VL];
    Op4 op_next = {0, 0, 0, 0};
    // post-program stage addressing: grouped (GG steps per stage: records,
    // then the tip windows) or one step per stage
    auto post_st = [&](int t) -> const unsigned char * {
        return grouped ? stages + (size_t)((t / GG) % DPG) * GSTG + (size_t)(t % GG) * RECB : stages + sub_off(t);
    };
    auto post_tip = [&](int t, int c) -> const unsigned char * {
        return grouped ? stages + (size_t)((t / GG) % DPG) * GSTG + (size_t)GG * RECB + (size_t)(t % GG) * 2 * TW + c * TW
                       : stages + sub_off(t) + 16 + 3 * MS + c * VS;
    };
    auto post_wait = [&](int t) {
        if (grouped) {
            if (t % GG == 0) mbar_wait_u32(smem_u32(gfull + (t / GG) % DPG), (uint32_t)((t / GG) / DPG) & 1u);
        } else if (slot(t) == 0) {
            wait_full(t);
        }
    };
    auto post_release = [&](int t) {
        if (!grouped) { release(t); return; }
        if (t % GG != GG - 1 && t != nops - 1) return;
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(smem_u32(gempty + (t / GG) % DPG));
    };
    if (active && nops > 0) {
        post_wait(0);
        op_next = *reinterpret_cast<const Op4 *>(post_st(0));
    }
    auto stack_or_fwd = [&](Real (&u)[VL], int code) {
        const int sl = -code - 1;
        if (sl == prev_slot) {
#pragma unroll
            for (int s = 0; s < VL; ++s) u[s] = prev_u[s];
        } else {
            stk_ld(u, sl);
        }
    };
    for (int t = 0; t < nops; ++t) {
        if (!active) {
            post_wait(t);
            post_release(t);
            continue;
        }
        const unsigned char *st = post_st(t);
        const Op4 op = op_next;
        if (warp == 0) PG_TSTAMP((size_t)t * 16 + 3, op.x);
        Real ua[VL], ub[VL];
        if (op.y < 0) stack_or_fwd(ua, op.y);
        else child_tip(ua, st + 16 + MS, post_tip(t, 0), op.y);
        if (op.z < 0) stack_or_fwd(ub, op.z);
        else child_tip(ub, st + 16 + 2 * MS, post_tip(t, 1), op.z);
        if (warp == 0) PG_TSTAMP((size_t)t * 16 + 4, ua[0] + ub[VL - 1]);
        if (t + 1 < nops) {
            post_wait(t + 1);
            op_next = *reinterpret_cast<const Op4 *>(post_st(t + 1));
        }
        if (warp == 0) PG_TSTAMP((size_t)t * 16 + 5, op_next.x);
        Real p[VL];
#pragma unroll
        for (int s = 0; s < VL; ++s) p[s] = ua[s] * ub[s];
        if (op.x == root) {
            post_release(t);
            double L = 0.0;
            if constexpr (MMA4) {
#pragma unroll
                for (int s = 0; s < VL; ++s) L = fma(wR[s] * (double)pi[s], (double)p[s], L);
                L = cat_sum<G>(L);
            } else {
#pragma unroll
                for (int s = 0; s < VL; ++s) L = fma((double)pi[s], (double)p[s], L);
                L = cat_sum<G>(wr * L);
            }
            if (cat == 0 && h == 0 && pat < a.C) {
                if (!(L > 0.0) || !isfinite(L)) atomicMin(a.status, pat);
                logl_local = wbuf[pl] * (log(L) + (double)E * 0.69314718055994530942);
            }
        } else {
            E += maybe_rescale<Real, VL, G>(p);
            if (warp == 0) PG_TSTAMP((size_t)t * 16 + 6, p[0]);
            Real u[VL];
            if constexpr (MMA) {
                dmma16(u, p, reinterpret_cast<const double *>(st + 16), lane);
            } else if constexpr (MMA4) {
                const double *Bf = reinterpret_cast<const double *>(st + 16);
#pragma unroll
                for (int q = 0; q < 4; ++q) u[q] = dmma4(p[q], Bf[q * 32 + lane]);
            } else {
                Real pf[SP];
                gather(pf, p);
                mv<Real, SP, VL>(u, reinterpret_cast<const Real *>(st + 16 + mat_lane), pf, h);
            }
            if (warp == 0) PG_TSTAMP((size_t)t * 16 + 7, u[0] + u[VL - 1]);
            post_release(t);
            stg_vec<Real, VL>(Ub + (size_t)(op.x - N) * u_node + u_lane, u);   // shadow lanes: same value
            stk_st(op.w, u);
#pragma unroll
            for (int s = 0; s < VL; ++s) prev_u[s] = u[s];
            prev_slot = op.w;
        }
    }
    if (active) {
        double v = logl_local;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) a.logl_part[tile] = v;
    }
    fence_proxy_async_global();          // u stores (generic proxy) before bulk reads (async proxy)
    __syncwarp();
    if (lane == 0) mbar_arrive(post_done);

    // -------------------- pre program (Eq. 4) + gradient (Eq. 6-8) ---------------
    // Q rows [h VL, +VL): registers when SP = 4, else shared memory
    Real Qr[SP <= 4 ? VL : 1][SP <= 4 ? SP : 1];
    double QB[MMA ? 8 : 1];                       // MMA: Q as the B operand of Q u (fragment order)
    if constexpr (MMA4) QB[0] = static_cast<const double *>(a.Q)[lane];
    if constexpr (MMA) {
#pragma unroll
        for (int f = 0; f < 8; ++f) QB[f] = reinterpret_cast<const double *>(smem + Cfg::QOFF)[f * 32 + lane];
    }
    if constexpr (SP <= 4 && !MMA4) {
#pragma unroll
        for (int s = 0; s < VL; ++s)
#pragma unroll
            for (int t = 0; t < SP; ++t)       // columns rotated like gathered vectors
                Qr[s][t] = static_cast<const Real *>(a.Q)[(h * VL + s) * SP + ((t + h * VL) & (SP - 1))];
    }
    const Real *Qs = reinterpret_cast<const Real *>(smem + Cfg::QOFF);
    // next op decoded early
    stk_st(pi_slot, pi);
    Op4 opn = {0, 0, 0, 0};
    if (active && nops > 0) {
        wait_full(nops);
        opn = *reinterpret_cast<const Op4 *>(stages + sub_off(nops));
    }
    // Eq. 8 window: step n's per-pattern totals (sums of the pending lane
    // shares over the pattern's G lanes: categories x state groups) into slot
    // n % W; every W steps the warp forms the ratios
    constexpr bool DEFER = MMA;
    double pend_na = 0.0, pend_nb = 0.0, pend_dn = 0.0;
    int pend_node_a = 0, pend_node_b = 0;
    auto store_totals = [&](const int n) {
        double na = pend_na, nb = pend_nb, dn = pend_dn;
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
            na += __shfl_xor_sync(0xffffffffu, na, o);
            nb += __shfl_xor_sync(0xffffffffu, nb, o);
            dn += __shfl_xor_sync(0xffffffffu, dn, o);
        }
        const int ws = n % W;
        if ((lane & (G - 1)) == 0) {
            double *e = nd + (ws * TP + pl) * 3;
            e[0] = na;
            e[1] = nb;
            e[2] = dn;
        }
        if (lane == 0) {
            nodes_w[ws * 2] = pend_node_a;
            nodes_w[ws * 2 + 1] = pend_node_b;
        }
        if (n % W != W - 1 && n != nops - 1) return;
        // W steps x TP patterns of (num_a, num_b, den) -> Eq. 8 ratios,
        // weighted by w_c (Eq. 6) and summed over the tile's patterns: LPS
        // lanes per step, PPL independent patterns per lane
        constexpr int LPS = Cfg::LPS, PPL = Cfg::PPL;
        __syncwarp();
        const int wstep = lane / LPS, sub = lane % LPS;
        const int n2 = n - (n % W) + wstep;
        double acc_a = 0.0, acc_b = 0.0;
        if (n2 <= n && sub * PPL < TP) {
#pragma unroll
            for (int k = 0; k < PPL; ++k) {
                const int p = sub * PPL + k;
                const double *e = nd + (wstep * TP + p) * 3;
                const double w = wbuf[p];
                const double d = (w != 0.0) ? e[2] : 1.0;           // w = 0: padding
                acc_a = fma(w, ratio(e[0], d), acc_a);
                acc_b = fma(w, ratio(e[1], d), acc_b);
            }
        }
#pragma unroll
        for (int o = 1; o < LPS; o <<= 1) {
            acc_a += __shfl_xor_sync(0xffffffffu, acc_a, o);
            acc_b += __shfl_xor_sync(0xffffffffu, acc_b, o);
        }
        if (sub == 0 && n2 <= n) {
            a.grad_part[(size_t)nodes_w[wstep * 2] * a.n_tiles + tile] = acc_a;
            a.grad_part[(size_t)nodes_w[wstep * 2 + 1] * a.n_tiles + tile] = acc_b;
        }
        __syncwarp();
    };
    for (int n = 0; n < nops; ++n) {
        const int t = nops + n;
        if (!active) {
            if (slot(t) == 0) wait_full(t);
            release(t);
            continue;
        }
        const unsigned char *st = stages + sub_off(t);
        const Op4 op = opn;
        if (warp == 0) PG_TSTAMP((size_t)t * 16 + 3, op.x);
        // q_k from its stack slot (pi for the root): forwarding the previous
        // step's pushes through registers measured slower here (more
        // instructions than the shared-memory round trip it saves)
        Real q[VL];
        stk_ld(q, op.x < 0 ? pi_slot : op.x);
        const int cs[2] = {op.y, op.z};
        const int slots[2] = {(op.w & 0xffff) - 1, (op.w >> 16) - 1};
        Real uc[2][VL];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const unsigned char *vs = st + 16 + 3 * MS + c * VS;
            if ((cs[c] & ~kTipPartialBit) >= N) lds_vec<Real, VL>(uc[c], vs + u_vec);
            else child_tip(uc[c], st + 16 + c * MS, vs, cs[c]);
        }
        if (DEFER && n > 0) store_totals(n - 1);    // the previous step's Eq. 8 totals
        if (warp == 0) PG_TSTAMP((size_t)t * 16 + 4, q[0] + uc[0][0] + uc[1][VL - 1]);
        if (n + 1 < nops) {
            const int t1 = t + 1;
            if (slot(t1) == 0) wait_full(t1);
            opn = *reinterpret_cast<const Op4 *>(stages + sub_off(t1));
        }
        if (warp == 0) PG_TSTAMP((size_t)t * 16 + 5, opn.x);
        // x_c = q o u_sibling (my states); q_c = P_c' x_c for internal children
        Real x[2][VL];
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int s = 0; s < VL; ++s) x[c][s] = q[s] * uc[1 - c][s];
        Real qc[2][VL];
#pragma unroll
        for (int c = 0; c < 2; ++c)
            if (slots[c] >= 0) {
                if constexpr (MMA) {
                    dmma16(qc[c], x[c], reinterpret_cast<const double *>(st + 16 + c * MS), lane);
                } else if constexpr (MMA4) {
                    const double *Bf = reinterpret_cast<const double *>(st + 16 + c * MS);
#pragma unroll
                    for (int q = 0; q < 4; ++q) qc[c][q] = dmma4(x[c][q], Bf[q * 32 + lane]);
                } else {
                    Real xf[SP];
                    gather(xf, x[c]);
                    mvt<Real, SP, VL>(qc[c], reinterpret_cast<const Real *>(st + 16 + c * MS + mat_lane), xf, h);
                }
            }
        if (warp == 0) PG_TSTAMP((size_t)t * 16 + 6, qc[0][0] + qc[1][0]);
        release(t);                                 // stage no longer needed
        // Eq. 8 terms: my states' shares of num_c = x_c' Q u_c for both
        // children and of den = x_c' u_c, which is the same number for both
        // children (q_k o u_a o u_b, Eq. 5): formed once
        Real num[2], den = 0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            num[c] = 0;
            if constexpr (MMA4) {                  // weighted over the lane's categories here
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double Qu = dmma4(uc[c][q], QB[0]);
                    num[c] = fma(gwR[q] * x[c][q], Qu, num[c]);
                    if (c == 0) den = fma(wR[q] * x[c][q], uc[c][q], den);
                }
            }
            if constexpr (MMA) {
                double Qu[4];
                dmma16r(Qu, uc[c], QB);
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    num[c] = fma(x[c][s], Qu[s], num[c]);
                    if (c == 0) den = fma(x[c][s], uc[c][s], den);
                }
            }
            if constexpr (!MMA && !MMA4) {
                Real ucf[SP];
                gather(ucf, uc[c]);
#pragma unroll
                for (int s = 0; s < VL; ++s) {
                    Real Qu;
                    if constexpr (SP <= 4) {
                        Qu = Qr[s][0] * ucf[0];
#pragma unroll
                        for (int t2 = 1; t2 < SP; ++t2) Qu = fma(Qr[s][t2], ucf[t2], Qu);
                    } else {
                        Real row[SP];
                        lds_rot<Real, SP, VL>(row, reinterpret_cast<const unsigned char *>(Qs + (h * VL + s) * SP), h);
                        Qu = row[0] * ucf[0];
#pragma unroll
                        for (int t2 = 1; t2 < SP; ++t2) Qu = fma(row[t2], ucf[t2], Qu);
                    }
                    num[c] = fma(x[c][s], Qu, num[c]);
                    if (c == 0) den = fma(x[c][s], uc[c][s], den);
                }
            }
        }
        // both children's q: one vote decides whether either needs rescaling
        {
            using T = ScaleTraits<Real>;
            int hmin = 0x7fffffff;
#pragma unroll
            for (int c = 0; c < 2; ++c)
                if (slots[c] >= 0) hmin = min(hmin, max_hiword<Real, VL>(qc[c]));
            if (__any_sync(0xffffffffu, hmin < (T::THRESH << T::SHIFT))) {
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    if (slots[c] >= 0) maybe_rescale<Real, VL, G>(qc[c]);
            }
#pragma unroll
            for (int c = 0; c < 2; ++c)
                if (slots[c] >= 0) stk_st(slots[c], qc[c]);
        }
        if (warp == 0) PG_TSTAMP((size_t)t * 16 + 7, qc[0][0] + qc[1][0]);
        // this step's (weighted) Eq. 8 shares; DEFER: they wait in registers
        // and their reduction over the pattern's lanes runs during the next
        // step, where its shuffle latency overlaps that step's operand loads
        // (MMM traversal 0.1004 -> 0.0983 ms; dengue, whose step has more
        // independent work of its own, 1.281 -> 1.291 ms: immediate there)
        pend_na = MMA4 ? (double)num[0] : gwr * (double)num[0];
        pend_nb = MMA4 ? (double)num[1] : gwr * (double)num[1];
        pend_dn = MMA4 ? (double)den : wr * (double)den;
        pend_node_a = cs[0] & ~kTipPartialBit;
        pend_node_b = cs[1] & ~kTipPartialBit;
        if (!DEFER) store_totals(n);
    }
    if (DEFER && active && nops > 0) store_totals(nops - 1);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // A6 may start launching
    a6_epilogue();
}

}  // namespace pg
