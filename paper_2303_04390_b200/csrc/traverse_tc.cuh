// traverse_tc.cuh -- codon-sized state spaces (16 < S <= 64, padded to 64)
// in fp32 on the 5th-generation tensor cores: tcgen05.mma kind::tf32 with
// the accumulators in TMEM, three TF32 products per GEMM (3xTF32:
// a_hi b_hi + a_hi b_lo + a_lo b_hi) so the fp32 path keeps its 1e-4
// tolerance (BJ:north_star "FP64/TF32 tensor cores").
//
// A tile is 128 patterns x 64 states of fp32, stored (HBM and shared memory)
// as the K-major SWIZZLE_NONE UMMA operand image (tc_common.cuh kmajor_off):
// a tile loads with one 32 KB bulk copy and is the MMA's A operand as is;
// element-wise products (Eq. 2's u_a o u_b, Eq. 4's q o u_sib) are
// position-wise.  Per (branch, category) A1 writes the B operands as hi/lo
// images: [P, u = p P'][P', q = x P] (16 KB each half); Q' (for x Q in Eq. 8)
// is fixed per instance.  The accumulator is read back with tcgen05.ld
// 32x32b (thread = pattern row), so per-pattern work -- rescaling maxima,
// the Eq. 3 and Eq. 8 dot products -- needs no cross-thread reduction.
//   post item (node k, category r, tile): p = u_a o u_b split into hi/lo in
//            place, u_k = p P_k' (Eq. 2) -> TMEM -> rows scaled, stored;
//            root: Eq. 3 terms.
//   pre item (parent k, r, tile): per child c, x_c = q_k o u_sib (hi/lo),
//            q_c = x_c P_c (Eq. 4; internal children) and y_c = x_c Q in one
//            pass over x_c (two TMEM accumulators), then num_c = y_c'u_c
//            (= x_c'Q u_c) and den = x_c'u_c (Eq. 6-8).
// Level-by-level launches; rescaling (lazy, exact powers of two shared by a
// pattern's categories), Eq. 3 partials and the ratio kernel follow the
// fp64 codon path (traverse_codon.cuh).
#pragma once
#include "tc_common.cuh"
#include "traverse_codon.cuh"

namespace pg {
namespace tcp {

using codon::CodonArgs;
constexpr int TM = 128, SP = 64, TILE = TM * SP;            // patterns per tile, states, floats per tile
constexpr uint32_t TILE_B = TILE * 4, HALF_B = SP * SP * 4;  // bytes: 32 KB tile, 16 KB B half
constexpr uint32_t LBO = 128, SBO_A = (SP / 4) * 128, SBO_B = (SP / 4) * 128;
constexpr size_t BREC = 4 * (size_t)SP * SP;                 // floats per (branch, r): post hi, lo, pre hi, lo

// fp32 lazy rescaling (R4): a child row (max over the pattern's
// categories) below 2^-32 is multiplied by 2^-e BEFORE it enters a product,
// so Eq. 2's u_a o u_b and Eq. 4's q o u_sib stay above ~2^-64 (fp32 normals
// end at 2^-126)
__device__ __forceinline__ int lazy_exp32(int field) { return field < 127 - 32 ? min(max(field - 126, -125), 126) : 0; }
// row of a canonical tile element from its float4 index
__device__ __forceinline__ int row_of4(int i) { return ((i * 16) / 2048) * 8 + ((i * 16) % 128) / 16; }
__device__ __forceinline__ float pow2neg32(int e) { return __int_as_float((127 - e) << 23); }

struct TcArgs {
    CodonArgs c;                 // shared fields (children, level table, weights, scales, numden, Lpart, E, status)
    const float *B;              // [branch][r][BREC] A1's B images
    const float *BQ;             // [2][SP*SP] Q' hi/lo (x Q)
    const float *ONE;            // [branch][r][SP] P 1 (missing-data tips)
    const float *pi;             // [SP]
    float *u, *q;                // [node][r][tile][TILE]
};

// 3xTF32 GEMM of a K = 64 product into TMEM column block d:
// D = A_hi B_hi + A_hi B_lo + A_lo B_hi (issued by one thread)
__device__ __forceinline__ void gemm3(uint32_t d, uint32_t ahi, uint32_t alo, uint32_t bhi, uint32_t blo) {
    constexpr uint32_t idesc = tc::idesc_tf32(TM, SP);
#pragma unroll
    for (int kk = 0; kk < SP / 8; ++kk) {
        const uint32_t o = 256u * kk;
        tc::mma_tf32(d, tc::sdesc(ahi + o, LBO, SBO_A), tc::sdesc(bhi + o, LBO, SBO_B), idesc, kk > 0);
        tc::mma_tf32(d, tc::sdesc(ahi + o, LBO, SBO_A), tc::sdesc(blo + o, LBO, SBO_B), idesc, 1);
        tc::mma_tf32(d, tc::sdesc(alo + o, LBO, SBO_A), tc::sdesc(bhi + o, LBO, SBO_B), idesc, 1);
    }
}

// A tile into smem: internal u / q (one bulk copy, tracked by bar) or a
// state tip's u (rows of P' picked by state: u[m][s] = P'[state_m][s], read
// as hi + lo of the pre image; missing data P 1), generic stores
__device__ __forceinline__ void load_tile(float *dst, const TcArgs &t, int child, int r, int tile, const int *st,
                                          uint64_t *bar, uint32_t &tx) {
    const CodonArgs &a = t.c;
    if (child >= a.N) {
        if (threadIdx.x == 0) {
            bulk_g2s(dst, t.u + (((size_t)(child - a.N) * a.R + r) * a.ntiles + tile) * TILE, TILE_B, bar);
        }
        tx += TILE_B;
        return;
    }
    const size_t br = (size_t)child * a.R + r;
    const float *Ph = t.B + br * BREC + 2 * SP * SP, *Pl = Ph + SP * SP, *one = t.ONE + br * SP;
    for (int i = threadIdx.x; i < TM * (SP / 4); i += blockDim.x) {
        const int m = i / (SP / 4), c4 = (i % (SP / 4)) * 4;
        const int s = st[m];
        float4 v;
        if (s < a.S) {
            const float4 h = __ldg(reinterpret_cast<const float4 *>(Ph + tc::kmajor_off(s, c4, SP) / 4));
            const float4 l = __ldg(reinterpret_cast<const float4 *>(Pl + tc::kmajor_off(s, c4, SP) / 4));
            v = make_float4(h.x + l.x, h.y + l.y, h.z + l.z, h.w + l.w);
        } else {
            v = __ldg(reinterpret_cast<const float4 *>(one + c4));
        }
        *reinterpret_cast<float4 *>(dst + tc::kmajor_off(m, c4, SP) / 4) = v;
    }
}

// this thread's row m of a tile in smem (16 chunks of 4)
__device__ __forceinline__ void row_ld(float (&v)[SP], const float *tile, int m) {
#pragma unroll
    for (int c = 0; c < SP / 4; ++c) {
        const float4 x = *reinterpret_cast<const float4 *>(tile + tc::kmajor_off(m, 4 * c, SP) / 4);
        v[4 * c] = x.x; v[4 * c + 1] = x.y; v[4 * c + 2] = x.z; v[4 * c + 3] = x.w;
    }
}
__device__ __forceinline__ void row_st_global(float *tile, int m, const float (&v)[SP]) {
#pragma unroll
    for (int c = 0; c < SP / 4; ++c)
        __stcg(reinterpret_cast<float4 *>(tile + tc::kmajor_off(m, 4 * c, SP) / 4),
               make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]));
}
__device__ __forceinline__ int row_maxfield(const float (&v)[SP]) {
    int f = 0;
#pragma unroll
    for (int i = 0; i < SP; ++i) f = max(f, (__float_as_int(v[i]) >> 23) & 0xff);
    return f;
}

// x (fp32 tile, in place over `xs`) -> hi into xs, lo into xl
__device__ __forceinline__ void split_tile(float *xs, float *xl) {
    for (int i = threadIdx.x; i < TILE / 4; i += blockDim.x) {
        float4 v = reinterpret_cast<float4 *>(xs)[i];
        const float4 h = make_float4(tc::tf32_hi(v.x), tc::tf32_hi(v.y), tc::tf32_hi(v.z), tc::tf32_hi(v.w));
        reinterpret_cast<float4 *>(xl)[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        reinterpret_cast<float4 *>(xs)[i] = h;
    }
}

constexpr size_t post_smem() { return (size_t)2 * TILE_B + 2 * HALF_B + 4 * TM * 4 + 64; }
constexpr size_t pre_smem() { return (size_t)5 * TILE_B + 4 * HALF_B + 5 * TM * 4 + 64; }

__global__ void __launch_bounds__(TM, 1) tc_post_kernel(const TcArgs t, int level_off) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const CodonArgs &a = t.c;
    float *S1 = reinterpret_cast<float *>(sm), *S2 = S1 + TILE, *Bh = S2 + TILE, *Bl = Bh + SP * SP;
    int *sta = reinterpret_cast<int *>(Bl + SP * SP), *stb = sta + TM;
    float *fA = reinterpret_cast<float *>(stb + TM), *fB = fA + TM;   // children's row factors
    uint64_t *bar = reinterpret_cast<uint64_t *>(fB + TM);    // [0] loads, [1] MMA done
    uint32_t *tmem_base = reinterpret_cast<uint32_t *>(bar + 2);
    const int tile = blockIdx.x, r = blockIdx.z;
    const int4 e = a.lev4[level_off + blockIdx.y];
    const int k = e.x, ca = e.y, cb = e.z;
    const int root = 2 * a.N - 2, pat0 = tile * TM, m = threadIdx.x, warp = threadIdx.x >> 5;
    const bool isroot = k == root;
    // programmatic dependent launch: the next level's CTAs may start their
    // prologue; everything this level reads from earlier launches comes after
    // griddepcontrol.wait
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp == 0 && !isroot) tc::tmem_alloc<64>(tmem_base);
    if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar + 1, 1); fence_mbar_init(); }
    sta[m] = ca < a.N ? a.tip_states[(size_t)ca * a.Cpad + pat0 + m] : 0;
    stb[m] = cb < a.N ? a.tip_states[(size_t)cb * a.Cpad + pat0 + m] : 0;
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint32_t tx = 0;
    load_tile(S1, t, ca, r, tile, sta, bar, tx);
    load_tile(S2, t, cb, r, tile, stb, bar, tx);
    if (!isroot) {
        if (threadIdx.x == 0) bulk_g2s(Bh, t.B + ((size_t)k * a.R + r) * BREC, 2 * HALF_B, bar);
        tx += 2 * HALF_B;
    }
    if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, tx);
    // children's rescaling exponents and E while the copies fly
    const int fa = ca >= a.N ? __ldcg(a.fmax + (size_t)(ca - a.N) * a.Cpad + pat0 + m) : 0;
    const int fb = cb >= a.N ? __ldcg(a.fmax + (size_t)(cb - a.N) * a.Cpad + pat0 + m) : 0;
    const int ea = ca >= a.N ? lazy_exp32(fa) : 0, eb = cb >= a.N ? lazy_exp32(fb) : 0;
    if (r == 0) {
        const int Ea = ca >= a.N ? __ldcg(a.E + (size_t)(ca - a.N) * a.Cpad + pat0 + m) : 0;
        const int Eb = cb >= a.N ? __ldcg(a.E + (size_t)(cb - a.N) * a.Cpad + pat0 + m) : 0;
        a.E[(size_t)(k - a.N) * a.Cpad + pat0 + m] = Ea + Eb + ea + eb;
    }
    fA[m] = pow2neg32(ea);
    fB[m] = pow2neg32(eb);
    mbar_wait(bar, 0);
    __syncthreads();                                           // gathered tip tiles (generic stores) too
    if (isroot) {                                              // Eq. 3 terms of pattern row m
        float x[SP], y[SP];
        row_ld(x, S1, m);
        row_ld(y, S2, m);
        double L = 0.0;
#pragma unroll
        for (int s = 0; s < SP; ++s) L = fma((double)t.pi[s], (double)(fA[m] * x[s]) * (double)(fB[m] * y[s]), L);
        a.Lpart[(size_t)r * a.Cpad + pat0 + m] = a.cat_w[r] * L;
        return;
    }
    for (int i = threadIdx.x; i < TILE / 4; i += blockDim.x) {   // p = (f_a u_a) o (f_b u_b) -> hi (S1), lo (S2)
        const int row = row_of4(i);
        const float ga = fA[row], gb = fB[row];
        const float4 x = reinterpret_cast<const float4 *>(S1)[i], y = reinterpret_cast<const float4 *>(S2)[i];
        const float4 p = make_float4(ga * x.x * (gb * y.x), ga * x.y * (gb * y.y), ga * x.z * (gb * y.z),
                                     ga * x.w * (gb * y.w));
        const float4 h = make_float4(tc::tf32_hi(p.x), tc::tf32_hi(p.y), tc::tf32_hi(p.z), tc::tf32_hi(p.w));
        reinterpret_cast<float4 *>(S1)[i] = h;
        reinterpret_cast<float4 *>(S2)[i] = make_float4(p.x - h.x, p.y - h.y, p.z - h.z, p.w - h.w);
    }
    tc::fence_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t d = *tmem_base;
    if (threadIdx.x == 0) {
        gemm3(d, smem_u32(S1), smem_u32(S2), smem_u32(Bh), smem_u32(Bl));
        tc::mma_commit(bar + 1);
    }
    mbar_wait(bar + 1, 0);
    tc::tc_fence_after();
    float v[SP];
    tc::tmem_ld64(d + ((uint32_t)(32 * warp) << 16), v);
    row_st_global(t.u + (((size_t)(k - a.N) * a.R + r) * a.ntiles + tile) * TILE, m, v);
    atomicMax(a.fmax + (size_t)(k - a.N) * a.Cpad + pat0 + m, row_maxfield(v));
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<64>(d);
}

__global__ void __launch_bounds__(TM, 1) tc_pre_kernel(const TcArgs t, int level_off) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const CodonArgs &a = t.c;
    float *Qk = reinterpret_cast<float *>(sm), *Ua = Qk + TILE, *Ub = Ua + TILE, *Xh = Ub + TILE, *Xl = Xh + TILE;
    float *BPh = Xl + TILE, *BPl = BPh + SP * SP, *BQh = BPl + SP * SP, *BQl = BQh + SP * SP;
    int *sta = reinterpret_cast<int *>(BQl + SP * SP), *stb = sta + TM;
    float *fQ = reinterpret_cast<float *>(stb + TM), *fS = fQ + TM;   // row factors: q_k; children [2][TM]
    uint64_t *bar = reinterpret_cast<uint64_t *>(fS + 2 * TM);   // [0] tiles, [1] MMA, [2] B of the 2nd child
    uint32_t *tmem_base = reinterpret_cast<uint32_t *>(bar + 3);
    const int tile = blockIdx.x, r = blockIdx.z;
    const int4 e = a.lev4[level_off + blockIdx.y];
    const int k = e.x, ch[2] = {e.y, e.z};
    const int root = 2 * a.N - 2, pat0 = tile * TM, m = threadIdx.x, warp = threadIdx.x >> 5;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // (see tc_post_kernel)
    if (warp == 0) tc::tmem_alloc<128>(tmem_base);
    if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar + 1, 1); mbar_init(bar + 2, 1); fence_mbar_init(); }
    sta[m] = ch[0] < a.N ? a.tip_states[(size_t)ch[0] * a.Cpad + pat0 + m] : 0;
    stb[m] = ch[1] < a.N ? a.tip_states[(size_t)ch[1] * a.Cpad + pat0 + m] : 0;
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint32_t tx = 0;
    if (k != root) {
        if (threadIdx.x == 0) bulk_g2s(Qk, t.q + (((size_t)(k - a.N) * a.R + r) * a.ntiles + tile) * TILE, TILE_B, bar);
        tx += TILE_B;
    } else {
        for (int i = threadIdx.x; i < TILE; i += blockDim.x) {
            const uint32_t off = (uint32_t)i * 4;               // canonical position -> state (k mod 64)
            const int kk = (int)(((off % (SBO_A)) / 128) * 4 + (off % 16) / 4);
            Qk[i] = t.pi[kk];
        }
    }
    load_tile(Ua, t, ch[0], r, tile, sta, bar, tx);
    load_tile(Ub, t, ch[1], r, tile, stb, bar, tx);
    if (threadIdx.x == 0) {
        bulk_g2s(BQh, t.BQ, 2 * HALF_B, bar);
        if (ch[0] >= a.N) bulk_g2s(BPh, t.B + ((size_t)ch[0] * a.R + r) * BREC + 2 * SP * SP, 2 * HALF_B, bar);
    }
    tx += 2 * HALF_B + (ch[0] >= a.N ? 2 * HALF_B : 0);
    if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, tx);
    fQ[m] = k == root ? 1.f : pow2neg32(lazy_exp32(__ldcg(a.qmax + (size_t)(k - a.N) * a.Cpad + pat0 + m)));
#pragma unroll
    for (int c = 0; c < 2; ++c)
        fS[c * TM + m] = ch[c] >= a.N ? pow2neg32(lazy_exp32(__ldcg(a.fmax + (size_t)(ch[c] - a.N) * a.Cpad + pat0 + m)))
                                      : 1.f;
    mbar_wait(bar, 0);
    __syncthreads();
    const uint32_t d = *tmem_base;                              // cols [0,64): q_c, [64,128): y_c = x_c Q
    const double wr = a.cat_w[r], gr = a.cat_g[r];
    uint32_t mma_phase = 0;
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
        const int node = ch[c];
        const float *Usib = c ? Ua : Ub, *Uc = c ? Ub : Ua;
        if (c == 1) {
            tc::tc_fence_before();
            __syncthreads();                                   // child 0's epilogue done with TMEM and X
            tc::tc_fence_after();
        }
        for (int i = threadIdx.x; i < TILE / 4; i += blockDim.x) {   // x_c = (f_q q_k) o (f_sib u_sib) -> hi / lo
            const int row = row_of4(i);
            const float g = fQ[row] * fS[(1 - c) * TM + row];
            const float4 q = reinterpret_cast<const float4 *>(Qk)[i], u = reinterpret_cast<const float4 *>(Usib)[i];
            const float4 x = make_float4(g * q.x * u.x, g * q.y * u.y, g * q.z * u.z, g * q.w * u.w);
            const float4 h = make_float4(tc::tf32_hi(x.x), tc::tf32_hi(x.y), tc::tf32_hi(x.z), tc::tf32_hi(x.w));
            reinterpret_cast<float4 *>(Xh)[i] = h;
            reinterpret_cast<float4 *>(Xl)[i] = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
        }
        tc::fence_async_smem();
        tc::tc_fence_before();
        __syncthreads();
        tc::tc_fence_after();
        if (c == 1 && node >= a.N) mbar_wait(bar + 2, 0);      // P' of child 1 (issued after child 0's MMAs)
        if (threadIdx.x == 0) {
            if (node >= a.N) gemm3(d, smem_u32(Xh), smem_u32(Xl), smem_u32(BPh), smem_u32(BPl));
            gemm3(d + 64, smem_u32(Xh), smem_u32(Xl), smem_u32(BQh), smem_u32(BQl));
            tc::mma_commit(bar + 1);
        }
        mbar_wait(bar + 1, mma_phase);
        mma_phase ^= 1;
        tc::tc_fence_after();
        if (c == 0 && ch[1] >= a.N && threadIdx.x == 0) {     // child 0's MMAs no longer read BP
            mbar_arrive_expect_tx(bar + 2, 2 * HALF_B);
            bulk_g2s(BPh, t.B + ((size_t)ch[1] * a.R + r) * BREC + 2 * SP * SP, 2 * HALF_B, bar + 2);
        }
        float v[SP];
        if (node >= a.N) {                                      // q_c (Eq. 4)
            tc::tmem_ld64(d + ((uint32_t)(32 * warp) << 16), v);
            row_st_global(t.q + (((size_t)(node - a.N) * a.R + r) * a.ntiles + tile) * TILE, m, v);
            atomicMax(a.qmax + (size_t)(node - a.N) * a.Cpad + pat0 + m, row_maxfield(v));
        }
        // Eq. 8: num = y_c'u_c (= x_c'Q u_c), den = x_c'u_c (scale factors cancel)
        tc::tmem_ld64(d + 64 + ((uint32_t)(32 * warp) << 16), v);
        float uc[SP], xh[SP], xl[SP];
        row_ld(uc, Uc, m);
        row_ld(xh, Xh, m);
        row_ld(xl, Xl, m);
        double num = 0.0, den = 0.0;
#pragma unroll
        for (int s = 0; s < SP; ++s) {
            num = fma((double)v[s], (double)uc[s], num);
            den = fma((double)xh[s] + (double)xl[s], (double)uc[s], den);
        }
        reinterpret_cast<double2 *>(a.numden)[((size_t)node * a.R + r) * a.Cpad + pat0 + m] =
            make_double2(gr * wr * num, wr * den);
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<128>(d);
}

// A1 for this path: P = M0 + V diag(expm1(gamma b lambda)) V^-1 in fp64 on
// the FP64 tensor path (one 64^3 DMMA product per (branch, category), V and
// V^-1 pre-arranged as fragments at pg_set_eigen, as codon_pmat_kernel),
// written as the hi/lo TF32 images of the two B operands (P for u = p P',
// P' for q = x P) and P 1
__global__ void __launch_bounds__(256) tc_pmat_kernel(const double *__restrict__ VA, const double *__restrict__ ViB,
                                                      const double *__restrict__ M0, const double *__restrict__ lam,
                                                      const double *__restrict__ rates, const double *__restrict__ bl,
                                                      int S, int R, float *B, float *ONE) {
    constexpr int KT = SP / 4, NW = SP / 8;
    extern __shared__ __align__(16) unsigned char smp[];
    double *Ps = reinterpret_cast<double *>(smp);            // [SP][SP+1]
    double *e = Ps + SP * (SP + 1);                          // [SP]
    double *Vs = e + SP;                                     // V's A fragments [SP*SP]
    const int br = blockIdx.x, r = br % R, b = br / R;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // the first post level may set up
    for (int i = threadIdx.x; i < SP * SP / 2; i += blockDim.x) cp_async16(Vs + 2 * i, VA + 2 * i);
    cp_async_commit();
    const double t = rates[r] * bl[b];
    for (int k = threadIdx.x; k < SP; k += blockDim.x) e[k] = k < S ? expm1(lam[k] * t) : 0.0;
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll 1
    for (int cs = w; cs < NW; cs += nw) {
        double bfr[KT];
        codon::load_bfrag<SP>(bfr, ViB, cs, lane);
#pragma unroll 1
        for (int h = 0; h < SP / 32; ++h) {
            double ap[4][2];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) ap[mt][0] = ap[mt][1] = 0.0;
            const double *A = Vs + h * 32 * SP + lane;
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
                const double ek = e[kt * 4 + (lane & 3)];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) codon::dmma(ap[mt], A[(mt * KT + kt) * 32] * ek, bfr[kt]);
            }
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int m = h * 32 + mt * 8 + (lane >> 2), n = cs * 8 + 2 * (lane & 3);
                Ps[m * (SP + 1) + n] = ap[mt][0] + M0[m * SP + n];
                Ps[m * (SP + 1) + n + 1] = ap[mt][1] + M0[m * SP + n + 1];
            }
        }
    }
    __syncthreads();
    float *rec = B + (size_t)br * BREC;
    for (int idx = threadIdx.x; idx < SP * SP; idx += blockDim.x) {
        const int n = idx / SP, kk = idx % SP;
        const uint32_t off = tc::kmajor_off(n, kk, SP) / 4;
        const float p = (float)Ps[n * (SP + 1) + kk], pt = (float)Ps[kk * (SP + 1) + n];   // image (n, k): P | P'
        const float ph = tc::tf32_hi(p), pth = tc::tf32_hi(pt);
        rec[off] = ph;
        rec[SP * SP + off] = p - ph;
        rec[2 * SP * SP + off] = pth;
        rec[3 * SP * SP + off] = pt - pth;
    }
    for (int s = threadIdx.x; s < SP; s += blockDim.x) {
        double acc = 0.0;
        for (int u = 0; u < SP; ++u) acc += Ps[s * (SP + 1) + u];
        ONE[(size_t)br * SP + s] = (float)acc;
    }
}
constexpr size_t pmat_smem() { return ((size_t)SP * (SP + 1) + SP + (size_t)SP * SP) * 8; }

}  // namespace tcp
}  // namespace pg
