// traverse_codon.cuh -- codon-sized state spaces (S <= 64, padded to 64) in
// fp64 on the FP64 tensor path: level-batched post-order and pre-order
// kernels whose inner operation is a [32 patterns x 64] x [64 x 64] product per
// rate category, issued as mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).
//
// Layout ("fragment order").  A 32-pattern x 64-state tile of partials is
// stored as [mt 4][kt 16][lane 32] doubles so that the m8n8k4 A fragment of
// (mt, kt) is 32 consecutive doubles: element (m, k) lives at
//     apos<SP>(m, k) = ((m/8)*16 + k/4)*32 + (m%8)*4 + k%4.
// u and q are stored per (node, category, tile) in this order in HBM, so a
// tile is one contiguous 16 KB block, and element-wise products (Eq. 2's
// u_a o u_b, Eq. 4's q o u) are plain position-wise products.  B operands
// (64 x 64) are stored as [nt 8][kt 16][lane 32] with element
// B[k = kt*4 + lane%4][n = nt*8 + lane/4]:
//   post  u_k = p P'      : B[t][s] = P[s][t]          (PBpost)
//   pre   q_c = x P       : B[s][t] = P[s][t]          (PBpre)
//   grad  Qu  = u Q'      : B[t][s] = Q[s][t]          (QB)
// Tip vectors are gathered from P' rows (u_tip[s] = P[s][state]) and, for
// the gradient, from D' rows with D = gamma_r Q P (Eq. 8's factor), so tips
// need no product at all.  Warp w of 8 computes output columns 8w..8w+7.
#pragma once
#include "common.cuh"

namespace pg {
namespace codon {

// Geometry of the SP-state path, SP = 64 (codon, 61 states) or 128 (two-class
// codon MMM, 122 states): a 32-pattern tile is
// [mt 4][kt SP/4][lane 32]; NW = SP/8 warps, warp w owns output columns
// 8w..8w+7 (B fragments of KT = SP/4 doubles per lane in registers).
constexpr int T = 32;
#define CODON_GEO                                                              \
    constexpr int TILE = T * SP, NW = SP / 8, NT = NW * 32, KT = SP / 4;       \
    constexpr size_t MAT = (size_t)SP * SP;                                    \
    (void)TILE; (void)NW; (void)NT; (void)KT; (void)MAT
template <int SP> constexpr int codon_threads() { return SP / 8 * 32; }
template <int SP> constexpr int codon_ctas_per_sm() { return SP == 64 ? 3 : 1; }

template <int SP>
__host__ __device__ __forceinline__ int apos(int m, int k) {
    return (((m >> 3) * (SP / 4) + (k >> 2)) << 5) + ((m & 7) << 2) + (k & 3);
}
// inverse of apos
template <int SP>
__device__ __forceinline__ void apos_inv(int idx, int &m, int &k) {
    const int lane = idx & 31, kt = (idx >> 5) & (SP / 4 - 1), mt = (int)((unsigned)idx / (8u * SP));
    m = mt * 8 + (lane >> 2);
    k = kt * 4 + (lane & 3);
}

struct CodonArgs {
    const int *child_a, *child_b;     // [2N-1] children of internal nodes (-1 for tips)
    const int *levels;                // node lists of all levels
    const int4 *lev4;                 // per level entry {node, child a, child b, kinds} (host-built)
    const double *PBpost, *PBpre;     // [B][R][MAT] fragment-ordered B operands
    const double *PT, *DT;            // [B][R][SP][SP]  P' and (gamma Q P)' row-major
    const double *PONE;               // [B][R][SP]      P 1 (missing-data tips)
    const double *QB;                 // [MAT]           Q as B operand of Qu = u Q'
    const double *pi;                 // [SP]
    const double *cat_w, *cat_g;      // [R]
    const double *pat_w;              // [Cpad]
    const uint8_t *tip_states;        // [N][Cpad]
    const double *tip_partials;       // [N][Cpad][SP] or null
    const uint8_t *tip_is_partial;    // [N]
    double *utip;                     // [N][R][ntiles][TILE] u = P p of partial tips (codon_tipu_kernel)
    const uint8_t *tip_mask;          // [N][Cpad][4] states of 0/1 mask partials (255 = none)
    const uint8_t *tip_masked;        // [N] 1: the tip's partials are such masks
    double *u;                        // [N-2][R][ntiles][TILE]
    double *q;                        // [N-2][R][ntiles][TILE]
    int *E;                           // [N-1][Cpad] cumulative exponent inside the stored u (internal + root)
    int *fmax;                        // [N-1][Cpad] max exponent field of u over categories (atomicMax)
    int *qmax;                        // [N-2][Cpad] same for q
    double *numden;                   // [B][R][Cpad][2] Eq. 8 terms per category
    // per-category exponents (codon_flow2_kernel; null elsewhere): E, fmax and
    // qmax above are then [node][R][Cpad]; EQ [N-2][R][Cpad] cumulative
    // exponent inside the stored q; Y [B][R][Cpad] exponent of a branch's
    // Eq. 8 terms (EQ of the parent + E of both children), reconciled over
    // categories in A6
    int *EQ, *Y;
    double *Lpart;                    // [R][Cpad] root likelihood terms per category
    double *grad_part;                // [B][ntiles]
    double *logl_part;                // [ntiles]
    int *status;
    int N, S, R, Cpad, C, ntiles;
};

// flow-schedule diagnostics (PG_FLOW_TRACE): u64 words per item, device clock
constexpr int TRW = 8;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    PG_MMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// B fragments of warp w (output columns 8w..8w+7) straight from L2 into
// registers: 16 independent coalesced 256-B loads per warp.
template <int SP>
__device__ __forceinline__ void load_bfrag(double (&b)[SP / 4], const double *__restrict__ Bg, int w, int lane) {
    const double *Bw = Bg + w * (SP / 4) * 32 + lane;
#pragma unroll
    for (int kt = 0; kt < SP / 4; ++kt) b[kt] = __ldg(Bw + kt * 32);
}

// acc[mt] (rows mt*8 + lane/4, cols w*8 + 2*(lane%4) + {0,1}) = A(32x64) * B(64x64)[:, 8w..8w+7]
template <int SP, int MT = 4>
__device__ __forceinline__ void gemm_tile(double (&acc)[MT][2], const double *As, const double (&b)[SP / 4], int lane) {
    constexpr int KT = SP / 4;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) dmma(acc[mt], As[(mt * KT + kt) * 32 + lane], b[kt]);
}

// copy n doubles (n % 2 == 0, 16-B aligned) global -> shared with all threads
__device__ __forceinline__ void load_block(double *dst, const double *src, int n) {
    for (int i = threadIdx.x; i < n / 2; i += blockDim.x)
        reinterpret_cast<double2 *>(dst)[i] = __ldg(reinterpret_cast<const double2 *>(src) + i);
}


// Fill a tile with child vectors for category r: internal (u from HBM) or tip
// (rows of P' picked by the pattern's state: u_tip[s] = P[s][state]).  Flat
// position loop (conflict-free smem stores), two states per 16-B load.
// `stbuf` (>= T ints of smem) receives the tile's tip states.
template <int SP>
__device__ void load_child(double *dst, const CodonArgs &a, int child, int r, int tile, int *stbuf) {
    CODON_GEO;
    if (child >= a.N) {
        load_block(dst, a.u + (((size_t)(child - a.N) * a.R + r) * a.ntiles + tile) * TILE, TILE);
        return;
    }
    const size_t br = (size_t)child * a.R + r;
    const int pat0 = tile * T;
    const double *PT = a.PT + br * MAT;
    if (a.tip_is_partial[child]) {          // u = P p, formed once per evaluation (codon_tipu_kernel)
        load_block(dst, a.utip + (((size_t)child * a.R + r) * a.ntiles + tile) * TILE, TILE);
        return;
    }
    if (threadIdx.x < T) stbuf[threadIdx.x] = a.tip_states[(size_t)child * a.Cpad + pat0 + threadIdx.x];
    __syncthreads();
    const double *ONE = a.PONE + br * SP;
    for (int i2 = threadIdx.x; i2 < TILE / 2; i2 += blockDim.x) {
        const int idx = 2 * i2;
        int m, k;
        apos_inv<SP>(idx, m, k);
        const int s = stbuf[m];
        const double2 v = __ldg(reinterpret_cast<const double2 *>(s < a.S ? PT + s * SP + k : ONE + k));
        reinterpret_cast<double2 *>(dst)[i2] = v;
    }
}

// Lazy exact rescaling across categories (R4).  Categories of a node run in
// different CTAs, so the stored u / q tiles are unscaled; every CTA atomically
// maxes the IEEE exponent field of its values into fmax/qmax[node][pattern],
// and the consumer at the next level multiplies by 2^-e with
// e = exponent of that max when it fell below 2^-256 (else e = 0).
__device__ __forceinline__ int lazy_exp(int field) {
    return field < 1023 - 256 ? min(max(field - 1022, -1021), 1022) : 0;
}
__device__ __forceinline__ double pow2neg(int e) { return __longlong_as_double((long long)(1023 - e) << 52); }

// per-pattern scale of a child tile (1 for tips)
__device__ __forceinline__ void child_scale(double *sc, const CodonArgs &a, int child, const int *mx, int pat0) {
    if (threadIdx.x < T) sc[threadIdx.x] = child >= a.N ? pow2neg(lazy_exp(__ldcg(mx + (size_t)(child - a.N) * a.Cpad + pat0 + threadIdx.x))) : 1.0;
}

// ---------------------------------------------------------------------------
// post-order level, persistent: each CTA walks a contiguous range of the
// level's work items (node, category r, tile), tile fastest, so the B
// fragments of P_k (registers) are reloaded only when (node, r) changes.
// Child tiles stream into a PST-stage shared-memory ring with cp.async
// (internal u tiles: contiguous 16 KB; tips: rows of P' picked by the
// pattern's state), issued PST-1 items ahead of the tensor-core GEMM.
// u_k[r] = (u_a o u_b) P_k' (Eq. 2), children rescaled in the epilogue;
// root: P(gamma_r) pi' p (Eq. 3) per pattern -> Lpart.
// ---------------------------------------------------------------------------
constexpr int PST = 2;                                           // post data stages
template <int SP> constexpr int pstage() { return 2 * T * SP * 8 + 2 * T * 4; }   // A, B tiles + children's fmax
constexpr int PSS = 3;                                           // state-code slots (2 children x 32 B)
template <int SP> constexpr size_t post_smem() { return (size_t)PST * pstage<SP>() + PSS * 2 * T + T * 8; }   // + row scales

// The level's nodes and their children, staged in shared memory at kernel
// start: {k, child a, child b, kinds}, kind = 0 internal, 1 tip states,
// 2 tip partials (child a in bits 0-1, child b in bits 2-3).
struct Item { int k, r, tile, ro, ca, cb, kinds; };
__device__ __forceinline__ int child_kind(const CodonArgs &a, int c) {
    return c >= a.N ? 0 : (a.tip_is_partial[c] ? 2 : 1);
}
__device__ __forceinline__ void stage_level(int4 *tab, const CodonArgs &a, int level_off, int cnt) {
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) tab[i] = a.lev4[level_off + i];
}
// Items are (node, r, tile, row block), row block fastest: MH m-tiles (8 MH
// patterns) of a 32-pattern tile.  Narrow levels use MH = 2 (twice the items,
// half the latency each); rows of a tile are contiguous in fragment order.
template <int MH>
__device__ __forceinline__ Item level_item(const CodonArgs &a, const int4 *tab, int item) {
    constexpr int HALF = 4 / MH;
    Item it;
    const int sub = item % (a.ntiles * HALF);
    it.tile = sub / HALF;
    it.ro = (sub % HALF) * 8 * MH;
    const int nr = item / (a.ntiles * HALF);
    it.r = nr % a.R;
    const int4 e = tab[nr / a.R];
    it.k = e.x;
    it.ca = e.y;
    it.cb = e.z;
    it.kinds = e.w;
    return it;
}
// Start the copy of child tile `child` (category r) into dst; fmax of an
// internal child's patterns into fm.  A tip's state codes for the tile (32
// bytes) were staged in shared memory one item earlier (`st`), so the
// gather addresses need no global round trip.  Tip partials (rare) are
// computed here.
template <int SP, int MH>
__device__ __forceinline__ void issue_child(double *dst, int *fm, const unsigned char *st, const CodonArgs &a,
                                            int child, int kind, int r, int tile, int ro) {
    CODON_GEO;
    const int tid = threadIdx.x;
    if (kind == 0) {
        const double *src = a.u + (((size_t)(child - a.N) * a.R + r) * a.ntiles + tile) * TILE + ro * SP;
#pragma unroll
        for (int j = 0; j < MH; ++j) cp_async16(dst + 2 * (tid + j * NT), src + 2 * (tid + j * NT));
        if (tid < 2 * MH) cp_async16(fm + 4 * tid, a.fmax + (size_t)(child - a.N) * a.Cpad + tile * T + ro + 4 * tid);
        return;
    }
    const size_t br = (size_t)child * a.R + r;
    const double *PT = a.PT + br * MAT;
    if (kind == 2) {                        // u = P p of a partial tip (codon_tipu_kernel)
        const double *src = a.utip + ((br * a.ntiles + tile) * TILE + ro * SP);
#pragma unroll
        for (int j = 0; j < MH; ++j) cp_async16(dst + 2 * (tid + j * NT), src + 2 * (tid + j * NT));
        return;
    }
    // thread tid needs patterns m = 8j + c, c = (tid & 15) / 2 (fragment order, any SP)
    const int c = (tid & 15) >> 1;
    const double *ONE = a.PONE + br * SP;
#pragma unroll
    for (int j = 0; j < MH; ++j) {
        int m, k;
        apos_inv<SP>(2 * (tid + j * NT), m, k);
        const int s = st[8 * j + c];
        cp_async16(dst + 2 * (tid + j * NT), s < a.S ? PT + s * SP + k : ONE + k);
    }
}
// stage a tip child's 8 MH state codes of the row block (16-B pieces)
template <int MH>
__device__ __forceinline__ void issue_states(unsigned char *st, const CodonArgs &a, int child, int kind, int tile, int ro) {
    if (kind == 1 && threadIdx.x < MH / 2)
        cp_async16(st + 16 * threadIdx.x, a.tip_states + (size_t)child * a.Cpad + tile * T + ro + 16 * threadIdx.x);
}
__device__ __forceinline__ double child_sc(const CodonArgs &a, int child, const int *fm, int m) {
    return child >= a.N ? pow2neg(lazy_exp(fm[m])) : 1.0;
}

// Items [beg, end) of a level whose node table `tab` is in shared memory.
// CACHE_B: keep P_k's B fragments in registers across consecutive items of
// the same (node, category) (persistent level kernel); the flow kernel runs
// one or two items per call and reloads them (fewer live registers)
template <int SP, int MH, bool CACHE_B = true>
__device__ __forceinline__ void post_range(const CodonArgs &a, const int4 *tab, int beg, int end, unsigned char *smem_c,
                                           unsigned long long *stamp = nullptr) {
    CODON_GEO;
    constexpr int PSTAGE = pstage<SP>();
    constexpr int TI = 8 * MH;               // patterns per item
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int root = 2 * a.N - 2;
    auto stage_A = [&](int s) { return reinterpret_cast<double *>(smem_c + (size_t)s * PSTAGE); };
    auto stage_B = [&](int s) { return reinterpret_cast<double *>(smem_c + (size_t)s * PSTAGE) + TILE; };
    auto stage_F = [&](int s) { return reinterpret_cast<int *>(smem_c + (size_t)s * PSTAGE + 2 * TILE * 8); };
    auto stage_S = [&](int item) { return smem_c + (size_t)PST * PSTAGE + ((item - beg) % PSS) * 2 * T; };
    // data of `item` into stage s (its states are staged); states of `item2`
    auto issue = [&](int item, int s, int item2) {
        if (item < end) {
            const Item it = level_item<MH>(a, tab, item);
            const unsigned char *st = stage_S(item);
            issue_child<SP, MH>(stage_A(s), stage_F(s), st, a, it.ca, it.kinds & 3, it.r, it.tile, it.ro);
            issue_child<SP, MH>(stage_B(s), stage_F(s) + T, st + T, a, it.cb, it.kinds >> 2, it.r, it.tile, it.ro);
        }
        if (item2 < end) {
            const Item it = level_item<MH>(a, tab, item2);
            unsigned char *st = stage_S(item2);
            issue_states<MH>(st, a, it.ca, it.kinds & 3, it.tile, it.ro);
            issue_states<MH>(st + T, a, it.cb, it.kinds >> 2, it.tile, it.ro);
        }
        cp_async_commit();
    };
    // prologue: states of items beg, beg+1; data of beg
    if (beg < end) {
        const Item it = level_item<MH>(a, tab, beg);
        issue_states<MH>(stage_S(beg), a, it.ca, it.kinds & 3, it.tile, it.ro);
        issue_states<MH>(stage_S(beg) + T, a, it.cb, it.kinds >> 2, it.tile, it.ro);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    issue(beg, 0, beg + 1);
    double bc[CACHE_B ? SP / 4 : 1];
    int cur = -1;                            // (node, r) whose B fragments are in bc
    for (int i = beg; i < end; ++i) {
        cp_async_wait<0>();                  // item i's data and item i+1's states (own thread) landed
        __syncthreads();                     // ... everyone's; stage of item i-1 is free
        if (stamp && threadIdx.x == 0) stamp[0] = gtimer();
        issue(i + 1, (i + 1 - beg) % PST, i + 2);
        const int s = (i - beg) % PST;
        const Item it = level_item<MH>(a, tab, i);
        const int k = it.k, r = it.r, ca = it.ca, cb = it.cb;
        const int pat0 = it.tile * T + it.ro;     // first pattern of the item
        const double *As = stage_A(s), *Ts = stage_B(s);
        const int *fa = stage_F(s), *fb = fa + T;
        // cumulative exponent inside u_k (and at the root): the children's E
        // loads are issued here and consumed after the GEMM (off the chain)
        const bool doE = r == 0 && threadIdx.x < TI;
        int Ea = 0, Eb = 0;
        if (doE) {
            const int m = threadIdx.x;
            if (ca >= a.N) Ea = __ldcg(a.E + (size_t)(ca - a.N) * a.Cpad + pat0 + m);
            if (cb >= a.N) Eb = __ldcg(a.E + (size_t)(cb - a.N) * a.Cpad + pat0 + m);
        }
        auto storeE = [&]() {
            const int m = threadIdx.x;
            const int Ek = Ea + Eb + (ca >= a.N ? lazy_exp(fa[m]) : 0) + (cb >= a.N ? lazy_exp(fb[m]) : 0);
            a.E[(size_t)(k - a.N) * a.Cpad + pat0 + m] = Ek;
        };
        if (k == root) {
            if (doE) storeE();
            // thread -> (pattern m = tid/8, 8 states); deterministic shuffle sum
            const int m = threadIdx.x >> 3, j = threadIdx.x & 7;
            double sum = 0.0;
            if (m < TI)
                for (int kk = j; kk < SP; kk += 8) {
                    const int p = apos<SP>(m, kk);
                    sum = fma(a.pi[kk], As[p] * Ts[p], sum);
                }
            sum += __shfl_xor_sync(0xffffffffu, sum, 1);
            sum += __shfl_xor_sync(0xffffffffu, sum, 2);
            sum += __shfl_xor_sync(0xffffffffu, sum, 4);
            if (j == 0 && m < TI)
                a.Lpart[(size_t)r * a.Cpad + pat0 + m] = a.cat_w[r] * sum * (child_sc(a, ca, fa, m) * child_sc(a, cb, fb, m));
            continue;
        }
        const int kr = k * a.R + r;
        double bl[CACHE_B ? 1 : SP / 4];
        if constexpr (CACHE_B) {
            if (kr != cur) {
                load_bfrag<SP>(bc, a.PBpost + (size_t)kr * MAT, w, lane);
                cur = kr;
            }
        } else {
            load_bfrag<SP>(bl, a.PBpost + (size_t)kr * MAT, w, lane);
        }
        // p = u_a o u_b in place (one A operand for the GEMM: half the
        // shared-memory traffic per DMMA of forming it on the fly)
        double *Pm = stage_A(s);
        double *f2s = reinterpret_cast<double *>(smem_c + (size_t)PST * PSTAGE + PSS * 2 * T);
        if (threadIdx.x < TI) f2s[threadIdx.x] = child_sc(a, ca, fa, threadIdx.x) * child_sc(a, cb, fb, threadIdx.x);
#pragma unroll
        for (int j = 0; j < MH; ++j) {
            double2 *pa = reinterpret_cast<double2 *>(Pm) + threadIdx.x + j * NT;
            const double2 tb = reinterpret_cast<const double2 *>(Ts)[threadIdx.x + j * NT];
            double2 v = *pa;
            v.x *= tb.x;
            v.y *= tb.y;
            *pa = v;
        }
        __syncthreads();
        double acc[MH][2];
        if constexpr (CACHE_B) gemm_tile<SP, MH>(acc, Pm, bc, lane);
        else gemm_tile<SP, MH>(acc, Pm, bl, lane);
        if (stamp && threadIdx.x == 0) stamp[1] = gtimer();
        if (doE) storeE();
        double *out = a.u + (((size_t)(k - a.N) * a.R + r) * a.ntiles + it.tile) * TILE + it.ro * SP;
        int *fm = a.fmax + (size_t)(k - a.N) * a.Cpad + pat0;
#pragma unroll
        for (int mt = 0; mt < MH; ++mt) {
            const int m = mt * 8 + (lane >> 2), n = w * 8 + 2 * (lane & 3);
            const double f2 = f2s[m];                         // children's scales (row)
            const double c0 = acc[mt][0] * f2, c1 = acc[mt][1] * f2;
            *reinterpret_cast<double2 *>(out + apos<SP>(m, n)) = make_double2(c0, c1);
            int f = max(__double2hiint(c0) >> 20, __double2hiint(c1) >> 20);
            f = max(f, __shfl_xor_sync(0xffffffffu, f, 1));
            f = max(f, __shfl_xor_sync(0xffffffffu, f, 2));
            if ((lane & 3) == 0) atomicMax(fm + m, f);
        }
    }
    cp_async_wait<0>();
}

template <int SP, int MH>
__global__ void __launch_bounds__(codon_threads<SP>(), codon_ctas_per_sm<SP>()) codon_post_kernel(const CodonArgs a, int level_off, int cnt) {
    extern __shared__ __align__(16) unsigned char smem_c[];
    const int nitems = cnt * a.R * a.ntiles * (4 / MH);
    int4 *tab = reinterpret_cast<int4 *>(smem_c + post_smem<SP>());
    stage_level(tab, a, level_off, cnt);
    __syncthreads();
    const int per = (nitems + gridDim.x - 1) / gridDim.x;
    const int beg = blockIdx.x * per, end = min(nitems, beg + per);
    post_range<SP, MH>(a, tab, beg, end, smem_c);
}

struct FlowArgs {
    int *ctr;          // item counter (reset per evaluation)
    int *rpost;        // [N-1][nch] completed post items per (internal node, chunk)
    int *rpre;         // [N-1][nch] completed q writes per (internal node, chunk)
    int npost, ntask, tch, nch;
    int defer;         // 1: pre items compute q only; Eq. 8 items (one per pre item) come after all of them
    int phalf;         // 2: post items are half tiles (16 patterns; needs tch == 1): shorter chain links
    unsigned long long *trace;   // diagnostics (PG_FLOW_TRACE): [item][TRW] = {smid, t_take, t_ready, t_done, phase stamps}
    const int *pready;           // codon_flow2_kernel under PDL: [B][R] A1 done flags (null: A1 finished before launch)
    int split;                   // codon_flow2_kernel: one pre item per child (latency-bound shards)
    const int *task_off;         // split schedule: [ntask + 1] first item of each task
    int pprod;                   // codon_flow2_kernel: the producer forms p = u_a o u_b of post items
    int pub;                     // codon_flow2_kernel: a publisher warp raises the completion flags
    // codon_flow2_kernel: A6 fused at the end of the launch (no ratio
    // kernel): a6cnt = finished-CTA counter, out = [logL, g]
    int *a6cnt;
    double *out;
};

// ---------------------------------------------------------------------------
// pre-order level: one CTA per (tile, parent of the level, category r).
// x_c = q_k o u_sibling; q_c = x_c P_c (Eq. 4) for internal children;
// Eq. 8 terms num_r = gamma_r P(gamma_r) x_c'Q u_c (internal: Qu = u Q' on the
// tensor path; tip: D' row gather), den_r = P(gamma_r) x_c'u_c per pattern ->
// numden[child][r][pattern]; the ratio over categories is formed afterwards.
// All inputs use the same per-pattern scales in every category, so the
// category sums stay consistent (the ratio itself is scale invariant).
// ---------------------------------------------------------------------------
template <int SP>
__device__ __forceinline__ void pre_tile(const CodonArgs &a, const int4 lv, int r, int tile, unsigned char *smem_c,
                                        unsigned long long *stamp = nullptr, const FlowArgs *fl = nullptr,
                                        int fch = 0, int mode = 0) {
    // mode 0: q of the children and their Eq. 8 terms; 1: q only (phase A);
    // 2: Eq. 8 terms only (phase B; q_k read back from HBM)
    CODON_GEO;
    double *Qs = reinterpret_cast<double *>(smem_c);
    double *Us[2] = {Qs + TILE, Qs + 2 * TILE};
    double *X = Qs + 3 * TILE;                               // x_c = q_k o u_sibling
    double *part = Qs + 4 * TILE;                            // [3: num a, num b, den][NW][T]
    double *sc = part + 3 * NW * T;                          // [3][T]: q_k, u_a, u_b scales
    int *stb = reinterpret_cast<int *>(sc + 3 * T);          // [2][T] tip states
    const int k = lv.x;
    const int root = 2 * a.N - 2;
    const int ch[2] = {lv.y, lv.z};
    const int kinds = lv.w;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pat0 = tile * T;
    if (threadIdx.x < T)
        sc[threadIdx.x] = k == root ? 1.0 : pow2neg(lazy_exp(__ldcg(a.qmax + (size_t)(k - a.N) * a.Cpad + pat0 + threadIdx.x)));
    child_scale(sc + T, a, ch[0], a.fmax, pat0);
    child_scale(sc + 2 * T, a, ch[1], a.fmax, pat0);
    // tip state codes of both children (one pass), then every tile copy in
    // flight at once with cp.async (16-B pieces; tips: rows of P' by state)
    if (threadIdx.x < 2 * T) {
        const int c = threadIdx.x / T, m = threadIdx.x % T, node = ch[c];
        stb[threadIdx.x] = (node < a.N) ? a.tip_states[(size_t)node * a.Cpad + pat0 + m] : 0;
    }
    __syncthreads();
    if (k == root) {
        for (int idx = threadIdx.x; idx < TILE; idx += NT) Qs[idx] = a.pi[((idx >> 5) & (KT - 1)) * 4 + (idx & 3)];
    } else {
        const double *src = a.q + (((size_t)(k - a.N) * a.R + r) * a.ntiles + tile) * TILE;
#pragma unroll
        for (int j = 0; j < TILE / 2 / NT; ++j) cp_async16(Qs + 2 * (threadIdx.x + j * NT), src + 2 * (threadIdx.x + j * NT));
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int node = ch[c];
        double *dst = Us[c];
        if (node >= a.N) {
            const double *src = a.u + (((size_t)(node - a.N) * a.R + r) * a.ntiles + tile) * TILE;
#pragma unroll
            for (int j = 0; j < TILE / 2 / NT; ++j) cp_async16(dst + 2 * (threadIdx.x + j * NT), src + 2 * (threadIdx.x + j * NT));
        } else if (((kinds >> (2 * c)) & 3) == 2) {
            load_child<SP>(dst, a, node, r, tile, stb + c * T);
        } else {
            const size_t br = (size_t)node * a.R + r;
            const double *PT = a.PT + br * MAT, *ONE = a.PONE + br * SP;
#pragma unroll
            for (int j = 0; j < TILE / 2 / NT; ++j) {
                int m, kk;
                apos_inv<SP>(2 * (threadIdx.x + j * NT), m, kk);
                const int st = stb[c * T + m];
                cp_async16(dst + 2 * (threadIdx.x + j * NT), st < a.S ? PT + st * SP + kk : ONE + kk);
            }
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[0] = gtimer();
    // Tiles stay unscaled: the Eq. 8 terms of a pattern carry the same factor
    // sc_q sc_a sc_b in numerator and denominator of every category (cancels);
    // the stored q_c rows are multiplied by sc_q sc_sibling below.
    const double wr = a.cat_w[r], gr = a.cat_g[r];
    // --- phase A (the pre-order chain): q_c = x_c P_c (Eq. 4) for internal
    // children, x_c = q_k o u_sibling formed in X; published (flow schedule)
    // before the Eq. 8 terms, which no later item waits for ---------------
#pragma unroll 1
    for (int c = 0; c < 2 && mode != 2; ++c) {
        const int node = ch[c];
        if (node < a.N) continue;
        const size_t br = (size_t)node * a.R + r;
        double bq[SP / 4], acc[4][2];
        load_bfrag<SP>(bq, a.PBpre + br * MAT, w, lane);
        __syncthreads();                                  // X free (previous child's GEMM done)
#pragma unroll
        for (int j = 0; j < TILE / 2 / NT; ++j) {
            const int i2 = threadIdx.x + j * NT;
            const double2 q2 = reinterpret_cast<const double2 *>(Qs)[i2];
            const double2 us = reinterpret_cast<const double2 *>(Us[1 - c])[i2];
            reinterpret_cast<double2 *>(X)[i2] = make_double2(q2.x * us.x, q2.y * us.y);
        }
        __syncthreads();
        gemm_tile<SP>(acc, X, bq, lane);
        double *out = a.q + (((size_t)(node - a.N) * a.R + r) * a.ntiles + tile) * TILE;
        int *qm = a.qmax + (size_t)(node - a.N) * a.Cpad + pat0;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int m = mt * 8 + (lane >> 2), n = w * 8 + 2 * (lane & 3);
            const double f2 = sc[m] * sc[(2 - c) * T + m];   // q_k and sibling scales
            acc[mt][0] *= f2;
            acc[mt][1] *= f2;
            *reinterpret_cast<double2 *>(out + apos<SP>(m, n)) = make_double2(acc[mt][0], acc[mt][1]);
            int f = max(__double2hiint(acc[mt][0]) >> 20, __double2hiint(acc[mt][1]) >> 20);
            f = max(f, __shfl_xor_sync(0xffffffffu, f, 1));
            f = max(f, __shfl_xor_sync(0xffffffffu, f, 2));
            if ((lane & 3) == 0) atomicMax(qm + m, f);
        }
    }
    if (stamp && threadIdx.x == 0) stamp[1] = gtimer();
    if (fl) {                                             // q of the internal children complete
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (ch[0] >= a.N) atomicAdd(fl->rpre + (size_t)(ch[0] - a.N) * fl->nch + fch, 1);
            if (ch[1] >= a.N) atomicAdd(fl->rpre + (size_t)(ch[1] - a.N) * fl->nch + fch, 1);
        }
    }
    if (mode == 1) return;
    // --- phase B: Eq. 8 terms of both children ---------------------------
    // num_c = x_c'(Q u_c) with x_c = q_k o u_sibling; den = x_c'u_c is the
    // same for both children (q_k o u_a o u_b, Eq. 5).
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
        const int node = ch[c];
        const size_t br = (size_t)node * a.R + r;
        double acc[4][2];
        if (node >= a.N || ((kinds >> (2 * c)) & 3) == 2) {
            // internal child or partial tip (u tile in smem): Q u on the tensor path
            double b[SP / 4];
            load_bfrag<SP>(b, a.QB, w, lane);
            gemm_tile<SP>(acc, Us[c], b, lane);
        } else {
            // tip: gamma (Q u)[s] = D[s][state]; missing data: D 1 = gamma Q 1 = 0
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) {
                const int m = mt * 8 + (lane >> 2), n = w * 8 + 2 * (lane & 3);
                {
                    const int s = stb[c * T + m];              // staged above
                    if (s < a.S) {
                        const double2 v = __ldg(reinterpret_cast<const double2 *>(a.DT + br * MAT + s * SP + n));
                        acc[mt][0] = v.x;
                        acc[mt][1] = v.y;
                    } else {
                        acc[mt][0] = acc[mt][1] = 0.0;
                    }
                }
            }
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int m = mt * 8 + (lane >> 2), n = w * 8 + 2 * (lane & 3);
            const int p = apos<SP>(m, n);
            const double2 q2 = *reinterpret_cast<const double2 *>(Qs + p);
            const double2 o2 = *reinterpret_cast<const double2 *>(Us[1 - c] + p);
            const double x0 = q2.x * o2.x, x1 = q2.y * o2.y;     // x_c = q_k o u_sibling
            double sn = x0 * acc[mt][0] + x1 * acc[mt][1];
            sn += __shfl_xor_sync(0xffffffffu, sn, 1);
            sn += __shfl_xor_sync(0xffffffffu, sn, 2);
            if ((lane & 3) == 0) part[(c * NW + w) * T + m] = sn;
            if (c == 0) {
                const double2 u2 = *reinterpret_cast<const double2 *>(Us[0] + p);
                double sd = x0 * u2.x + x1 * u2.y;
                sd += __shfl_xor_sync(0xffffffffu, sd, 1);
                sd += __shfl_xor_sync(0xffffffffu, sd, 2);
                if ((lane & 3) == 0) part[(2 * NW + w) * T + m] = sd;
            }
        }
    }
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[2] = gtimer();
    if (threadIdx.x < T) {                    // fixed-order sums over the 8 warps
        const int m = threadIdx.x;
        double sd = 0.0, sn0 = 0.0, sn1 = 0.0;
        for (int ww = 0; ww < NW; ++ww) {
            sn0 += part[ww * T + m];
            sn1 += part[(NW + ww) * T + m];
            sd += part[(2 * NW + ww) * T + m];
        }
        double2 *nd = reinterpret_cast<double2 *>(a.numden);
        // internal children and partial tips: Q u (times gamma_r here); state
        // tips: the D' row already carries gamma_r
        const bool qa = ch[0] >= a.N || (kinds & 3) == 2, qb = ch[1] >= a.N || ((kinds >> 2) & 3) == 2;
        const double s0 = qa ? gr * wr : wr, s1 = qb ? gr * wr : wr;
        nd[((size_t)ch[0] * a.R + r) * a.Cpad + pat0 + m] = make_double2(s0 * sn0, wr * sd);
        nd[((size_t)ch[1] * a.R + r) * a.Cpad + pat0 + m] = make_double2(s1 * sn1, wr * sd);
    }

}
template <int SP>
__global__ void __launch_bounds__(codon_threads<SP>(), codon_ctas_per_sm<SP>()) codon_pre_kernel(const CodonArgs a, int level_off) {
    extern __shared__ __align__(16) unsigned char smem_c[];
    // one CTA per (tile, parent of the level, category): {node, children, kinds} in one load
    pre_tile<SP>(a, a.lev4[level_off + blockIdx.y], blockIdx.z, blockIdx.x, smem_c);
}

// ---------------------------------------------------------------------------
// Eq. 6-8 ratio over categories, weighted by w_c, summed over patterns in a
// fixed order (block b < B: branch b); block B: logL from the root terms.
// ---------------------------------------------------------------------------
// Pattern slices per branch: block (b, slice) sums its slice, the last
// slice to finish (atomic counter) adds the slice sums in slice order, so the
// result does not depend on which block finished last (deterministic).
constexpr int RATIO_SLICES = 8;
// 2^d for d <= 0 (0 below the normal range: such terms are 2^-1022 below the
// largest and vanish in its rounding)
__device__ __forceinline__ double pow2le0(int d) {
    return d < -1022 ? 0.0 : __longlong_as_double((long long)(1023 + d) << 52);
}
// sum_r num_r and sum_r den_r of branch b, pattern c: with per-category
// exponents (a.Y) each category's terms are first brought to the largest
// exponent of the pattern (exact powers of two; a term 2^-1000 below the
// largest underflows to 0, far below rounding)
__device__ __forceinline__ void ratio_terms(const CodonArgs &a, int b, int c, double &num, double &den) {
    const double2 *nd = reinterpret_cast<const double2 *>(a.numden);
    num = 0.0;
    den = 0.0;
    if (!a.Y) {
        for (int r = 0; r < a.R; ++r) {
            const double2 v = __ldcg(nd + ((size_t)b * a.R + r) * a.Cpad + c);
            num += v.x;
            den += v.y;
        }
        return;
    }
    int ym = INT_MIN;
    for (int r = 0; r < a.R; ++r) ym = max(ym, __ldcg(a.Y + ((size_t)b * a.R + r) * a.Cpad + c));
    for (int r = 0; r < a.R; ++r) {
        const double2 v = __ldcg(nd + ((size_t)b * a.R + r) * a.Cpad + c);
        const double f = pow2le0(__ldcg(a.Y + ((size_t)b * a.R + r) * a.Cpad + c) - ym);
        num = fma(v.x, f, num);
        den = fma(v.y, f, den);
    }
}
// sum_r Lpart_r of pattern c relative to 2^Em (Em = the root's exponent;
// per category with a.Y: the largest of them)
__device__ __forceinline__ double root_likelihood(const CodonArgs &a, int c, int &Em) {
    const int root = 2 * a.N - 2;
    double L = 0.0;
    if (!a.Y) {
        for (int r = 0; r < a.R; ++r) L += __ldcg(a.Lpart + (size_t)r * a.Cpad + c);
        Em = __ldcg(a.E + (size_t)(root - a.N) * a.Cpad + c);
        return L;
    }
    Em = INT_MIN;
    for (int r = 0; r < a.R; ++r) Em = max(Em, __ldcg(a.E + ((size_t)(root - a.N) * a.R + r) * a.Cpad + c));
    for (int r = 0; r < a.R; ++r)
        L = fma(__ldcg(a.Lpart + (size_t)r * a.Cpad + c),
                pow2le0(__ldcg(a.E + ((size_t)(root - a.N) * a.R + r) * a.Cpad + c) - Em), L);
    return L;
}
__global__ void __launch_bounds__(256) codon_ratio_kernel(const CodonArgs a, double *out, double *slice_part,
                                                          int *slice_cnt) {
    __shared__ double sh[256];
    __shared__ bool last;
    asm volatile("griddepcontrol.wait;" ::: "memory");      // (PDL launch behind the last pre level)
    const int b = blockIdx.x, B = 2 * a.N - 2;
    const int ns = gridDim.y, per = (a.C + ns - 1) / ns;
    const int c0 = blockIdx.y * per, c1 = min(a.C, c0 + per);
    double acc = 0.0;
    for (int c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
        const double wc = a.pat_w[c];
        if (b < B) {
            double num, den;
            ratio_terms(a, b, c, num, den);
            if (wc != 0.0) acc += wc * (num / den);
        } else {
            int Em;
            const double L = root_likelihood(a, c, Em);
            if (!(L > 0.0) || !isfinite(L)) atomicMin(a.status, c);
            acc += wc * (log(L) + (double)Em * 0.69314718055994530942);
        }
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        slice_part[(size_t)b * ns + blockIdx.y] = sh[0];
        __threadfence();
        last = atomicAdd(slice_cnt + b, 1) == ns - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double t = 0.0;
        for (int k = 0; k < ns; ++k) t += __ldcg(slice_part + (size_t)b * ns + k);
        out[b < B ? 1 + b : 0] = t;
    }
}

template <int SP>
constexpr size_t pre_smem() { return (size_t)(4 * T * SP + 3 * (SP / 8) * T + 3 * T) * 8 + 2 * T * 4; }

// ---------------------------------------------------------------------------
// Dataflow ("flow") schedule: the post-order and pre-order items of every
// level in ONE persistent launch.  Work items are (task, category r, chunk of
// TCH tiles), task = entry of the level table (post levels by height, then pre
// levels by depth), chunk fastest; CTAs take items in that (topological) order
// from a global counter, wait until the item's inputs are complete, run it and
// publish completion:
//   post (k, r, chunk)  needs u of internal children, all R categories
//                       (rpost[child][chunk] == R: the children's fmax are final);
//   pre  (k, r, chunk)  needs q_k, all R categories (rpre[k][chunk] == R); at
//                       the root, u of both children instead.  pre(k)
//                       publishes q of its internal children as soon as their
//                       q GEMMs are stored, before its Eq. 8 terms.
// An item only waits on items taken earlier by running CTAs, so the schedule
// cannot deadlock; a node starts as soon as ITS inputs exist (not when its
// whole level is done), and no level pays a launch + tail.  Cross-item data
// is read through L2 only (cp.async.cg, ld.cg) after an acquire by thread 0
// and a CTA barrier; results are published by a CTA barrier, a device fence
// and an atomic increment by thread 0.
// ---------------------------------------------------------------------------

template <int SP>
constexpr size_t flow_smem() {
    return (post_smem<SP>() + 16) > pre_smem<SP>() ? (post_smem<SP>() + 16) : pre_smem<SP>();
}
__device__ __forceinline__ void wait_count(const int *p, int v) {
    int x;
    for (long long spin = 0;; ++spin) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
        if (x >= v) return;
        if (spin > (1ll << 27)) __trap();     // a schedule bug must fail loudly, not hang the GPU
#ifndef PG_FLOW_SLEEP
#define PG_FLOW_SLEEP 40
#endif
        if (PG_FLOW_SLEEP > 0) __nanosleep(PG_FLOW_SLEEP);
    }
}
template <int SP>
__global__ void __launch_bounds__(codon_threads<SP>(), codon_ctas_per_sm<SP>()) codon_flow_kernel(const CodonArgs a, const FlowArgs f) {
    CODON_GEO;
    extern __shared__ __align__(16) unsigned char smem_c[];
    __shared__ int s_item;
    int4 *tab = reinterpret_cast<int4 *>(smem_c + post_smem<SP>());
    const int per_task = a.R * f.nch, per_post = per_task * f.phalf;
    const int npre = f.ntask - f.npost;
    const int npost_items = f.npost * per_post;
    const int nitems = npost_items + (npre + (f.defer ? npre : 0)) * per_task;
    const int post_full = a.R * f.phalf;                   // completed post items per (node, chunk)
    const int root = 2 * a.N - 2;
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(f.ctr, 1);
        __syncthreads();
        const int item = s_item;
        if (item >= nitems) return;
        int vtask, r, ch, half = 0;
        if (item < npost_items) {
            vtask = item / per_post;
            const int rem = item - vtask * per_post;
            r = rem / (f.nch * f.phalf);
            const int rem2 = rem - r * f.nch * f.phalf;
            ch = rem2 / f.phalf;
            half = rem2 - ch * f.phalf;
        } else {
            const int i2 = item - npost_items;
            vtask = f.npost + i2 / per_task;
            const int rem = i2 - (vtask - f.npost) * per_task;
            r = rem / f.nch;
            ch = rem - r * f.nch;
        }
        const bool grad_item = vtask >= f.ntask;            // deferred Eq. 8 item of pre task vtask - npre
        const int task = grad_item ? vtask - npre : vtask;
        const int4 e = a.lev4[task];
        const int t0 = ch * f.tch, t1 = min(a.ntiles, t0 + f.tch);
        const bool post = task < f.npost;
        unsigned long long t_take = 0;
        if (f.trace && threadIdx.x == 0) t_take = gtimer();
        {   // B operands depend only on A1, not on earlier items: pull this
            // warp's fragments into L1 while thread 0 waits for the inputs
            const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
            auto pf = [&](const double *Bg) {
                const double *Bw = Bg + w * KT * 32 + lane;
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) asm volatile("prefetch.global.L1 [%0];" ::"l"(Bw + kt * 32));
            };
            if (post) {
                if (e.x != root) pf(a.PBpost + ((size_t)e.x * a.R + r) * MAT);
            } else {
                if (e.y >= a.N) pf(a.PBpre + ((size_t)e.y * a.R + r) * MAT);
                if (e.z >= a.N) pf(a.PBpre + ((size_t)e.z * a.R + r) * MAT);
            }
        }
        if (threadIdx.x == 0) {
            if (post || e.x == root) {
                if (e.y >= a.N) wait_count(f.rpost + (size_t)(e.y - a.N) * f.nch + ch, post_full);
                if (e.z >= a.N) wait_count(f.rpost + (size_t)(e.z - a.N) * f.nch + ch, post_full);
            } else {
                wait_count(f.rpre + (size_t)(e.x - a.N) * f.nch + ch, a.R);
            }
            if (post) tab[0] = e;
            if (f.trace) {
                unsigned smid;
                asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
                f.trace[TRW * (size_t)item] = smid;
                f.trace[TRW * (size_t)item + 1] = t_take;
                f.trace[TRW * (size_t)item + 2] = gtimer();
            }
        }
        __syncthreads();
        if (post && f.phalf == 2) {                   // one 16-pattern half of tile t0 (tch == 1)
            const int b = (r * a.ntiles + t0) * 2 + half;
            post_range<SP, 2, false>(a, tab, b, b + 1, smem_c, f.trace ? f.trace + TRW * (size_t)item + 4 : nullptr);
        } else if (post) {
            post_range<SP, 4, false>(a, tab, r * a.ntiles + t0, r * a.ntiles + t1, smem_c,
                          f.trace ? f.trace + TRW * (size_t)item + 4 : nullptr);
        } else {
            // q of the chunk is published inside the last tile, after its
            // q GEMMs and before its Eq. 8 terms (earlier tiles are complete)
            for (int tile = t0; tile < t1; ++tile) {
                pre_tile<SP>(a, e, r, tile, smem_c, f.trace ? f.trace + TRW * (size_t)item + 4 : nullptr,
                         (tile == t1 - 1 && !grad_item) ? &f : nullptr, ch,
                         grad_item ? 2 : (f.defer ? 1 : 0));
                __syncthreads();
            }
        }
        __syncthreads();
        if (f.trace && threadIdx.x == 0) f.trace[TRW * (size_t)item + 7] = gtimer();
        if (threadIdx.x == 0) {
            __threadfence();
            if (post) atomicAdd(f.rpost + (size_t)(e.x - a.N) * f.nch + ch, 1);
            if (f.trace) f.trace[TRW * (size_t)item + 3] = gtimer();
        }
    }
}

// ---------------------------------------------------------------------------
// Tips given as partial vectors (MMM hidden states, ambiguity codes; P:613-614
// generalised, R6): u_tip = P_tip p_tip, once per evaluation, as a
// GEMM per (tile, tip, category) on the tensor path -- afterwards these tips
// are read like internal u tiles (post: child tiles; pre: Q u by GEMM).
// ---------------------------------------------------------------------------
constexpr int TIPU_TILES = 4;            // tiles per CTA (B fragments loaded once)
template <int SP>
__global__ void __launch_bounds__(codon_threads<SP>(), 1) codon_tipu_kernel(const CodonArgs a) {
    CODON_GEO;
    extern __shared__ __align__(16) unsigned char smem_c[];
    const int tip = blockIdx.y, r = blockIdx.z;
    if (!a.tip_is_partial[tip]) return;
    const int t0 = blockIdx.x * TIPU_TILES, t1 = min(a.ntiles, t0 + TIPU_TILES);
    if (a.tip_masked[tip]) return;                 // codon_tipmask_kernel
    double *buf[2] = {reinterpret_cast<double *>(smem_c), reinterpret_cast<double *>(smem_c) + TILE};
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // tip partials are stored in A-fragment order per tile (pg_set_tip_partials)
    auto issue = [&](int tile, double *dst) {
        const double *src = a.tip_partials + ((size_t)tip * a.Cpad + (size_t)tile * T) * SP;
#pragma unroll
        for (int j = 0; j < TILE / 2 / NT; ++j) cp_async16(dst + 2 * (threadIdx.x + j * NT), src + 2 * (threadIdx.x + j * NT));
        cp_async_commit();
    };
    issue(t0, buf[0]);
    double b[SP / 4], acc[4][2];
    load_bfrag<SP>(b, a.PBpost + ((size_t)tip * a.R + r) * MAT, w, lane);
    for (int tile = t0; tile < t1; ++tile) {
        const int s = (tile - t0) & 1;
        if (tile + 1 < t1) {
            issue(tile + 1, buf[s ^ 1]);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        gemm_tile<SP>(acc, buf[s], b, lane);
        double *out = a.utip + (((size_t)tip * a.R + r) * a.ntiles + tile) * TILE;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int m = mt * 8 + (lane >> 2), n = w * 8 + 2 * (lane & 3);
            *reinterpret_cast<double2 *>(out + apos<SP>(m, n)) = make_double2(acc[mt][0], acc[mt][1]);
        }
        __syncthreads();                     // buf[s] is refilled two tiles later
    }
}
// Mask tips (0/1 partials with <= 4 ones, e.g. the hidden copies of an
// observed codon): u[s] = sum over the pattern's mask states t of P[s][t] =
// P'[t][s], contiguous rows of P' -- gathers, no GEMM; one CTA per (tile, tip,
// category), light registers so many CTAs share an SM.
template <int SP>
__global__ void __launch_bounds__(256) codon_tipmask_kernel(const CodonArgs a) {
    constexpr int TILE = T * SP;
    constexpr size_t MAT = (size_t)SP * SP;
    const int tile = blockIdx.x, tip = blockIdx.y, r = blockIdx.z;
    if (!a.tip_masked[tip]) return;
    const double *PT = a.PT + ((size_t)tip * a.R + r) * MAT;
    double *out = a.utip + (((size_t)tip * a.R + r) * a.ntiles + tile) * TILE;
    const uint8_t *mk = a.tip_mask + ((size_t)tip * a.Cpad + (size_t)tile * T) * 4;
#pragma unroll 4
    for (int i2 = threadIdx.x; i2 < TILE / 2; i2 += blockDim.x) {
        int m, k;
        apos_inv<SP>(2 * i2, m, k);
        const uchar4 ids = __ldg(reinterpret_cast<const uchar4 *>(mk + 4 * m));
        const uint8_t id4[4] = {ids.x, ids.y, ids.z, ids.w};
        double2 u = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (id4[j] != 255) {
                const double2 v = __ldg(reinterpret_cast<const double2 *>(PT + (size_t)id4[j] * SP + k));
                u.x += v.x;
                u.y += v.y;
            }
        reinterpret_cast<double2 *>(out)[i2] = u;
    }
}
template <int SP>
constexpr size_t tipu_smem() { return (size_t)2 * T * SP * 8; }

// ---------------------------------------------------------------------------
// A1 for this path: per (branch, category) P = (V diag(e)) V^{-1} and
// D = gamma Q P = (V diag(gamma lambda e)) V^{-1} (Eq. 1; Eq. 8's factor),
// e = exp(gamma b lambda), as two 64^3 products on the FP64 tensor path
// (V pre-arranged as A fragments, V^{-1} as B fragments at set_eigen); the
// results are written as PBpost, PBpre, P', D', P 1.
// ---------------------------------------------------------------------------
constexpr int PMAT_P_DONE = 1, PMAT_D_DONE = 256;         // pready increments per (branch, r): P CTA, D CTA
template <int SP>
__global__ void __launch_bounds__(256) codon_pmat_kernel(const double *__restrict__ VA,
                                                         const double *__restrict__ ViB,
                                                         const double *__restrict__ M0,
                                                         const double *__restrict__ Qd,
                                                         const double *__restrict__ lam,
                                                         const double *__restrict__ rates,
                                                         const double *__restrict__ bl, int S, int R, int N,
                                                         int tip_partials, double *PBpost, double *PBpre, double *PT,
                                                         double *DT, double *PONE, int *pready) {
    CODON_GEO;
    // programmatic dependent launch: the flow kernel may start now; it reads
    // this CTA's outputs only after pready[branch][r] is published below
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    extern __shared__ __align__(16) unsigned char smem_p[];
    double *Ps = reinterpret_cast<double *>(smem_p);     // [SP][SP+1]: P or D
    double *e = Ps + SP * (SP + 1);                      // [SP]
    // SP = 64: V's A fragments staged in shared memory once (all copies in
    // flight together; ncu: L2 loads inside the DMMA loop were the top stall);
    // SP = 128 reads them from L2 (no room next to the 132 KB output buffer)
    constexpr bool STAGE_V = SP == 64;
    double *Vs = e + 2 * SP;
    const int br = blockIdx.x, r = br % R, b = br / R;
    // blockIdx.y = 0: P (every branch), 1: D (tips only).  What each branch's
    // consumers read: internal branches the B fragments of P' (post, u_k =
    // p P') and P (pre, q_c = x_c P); tips the rows of P' (gathers), P 1
    // (missing data) and D' (Eq. 8 numerators); partial tips also P'-fragments
    // (codon_tipu_kernel).  Nothing else is formed or written.
    const int pass = blockIdx.y;
    const bool tip = b < N;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (pass == 0 || tip) {
        if constexpr (STAGE_V) {
            for (int i = threadIdx.x; i < (int)MAT / 2; i += blockDim.x) cp_async16(Vs + 2 * i, VA + 2 * i);
            cp_async_commit();
        }
        const double g = rates[r], t = g * bl[b];
        // P = M0 + V diag(e - 1) V^-1, D = gamma (Q + V diag(lambda (e - 1)) V^-1)
        // (M0 = V V^-1, Q formed once on the host; R15b)
        for (int k = threadIdx.x; k < SP; k += blockDim.x) {
            const double em1 = k < S ? expm1(lam[k] * t) : 0.0;
            e[k] = pass ? (k < S ? g * lam[k] * em1 : 0.0) : em1;
        }
        if constexpr (STAGE_V) cp_async_wait<0>();
        __syncthreads();
        const size_t base = (size_t)br * MAT;
        const double *Vsrc = STAGE_V ? Vs : VA;
        // Warp w computes column strips 8 cs .. 8 cs + 7, cs = w, w + nw, ...
#pragma unroll 1
        for (int cs = w; cs < NW; cs += nw) {
            double bfr[KT];
            load_bfrag<SP>(bfr, ViB, cs, lane);
#pragma unroll 1
            for (int h = 0; h < SP / 32; ++h) {      // rows 32h .. 32h+31
                double ap[4][2];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) ap[mt][0] = ap[mt][1] = 0.0;
                const double *A = Vsrc + h * TILE + lane;
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) {
                    const double ek = e[kt * 4 + (lane & 3)];
#pragma unroll
                    for (int mt = 0; mt < 4; ++mt) {
                        const double v = STAGE_V ? A[(mt * KT + kt) * 32] : __ldg(A + (mt * KT + kt) * 32);
                        dmma(ap[mt], v * ek, bfr[kt]);
                    }
                }
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) {
                    const int m = h * 32 + mt * 8 + (lane >> 2), n = cs * 8 + 2 * (lane & 3);
                    const double2 z = *reinterpret_cast<const double2 *>((pass ? Qd : M0) + m * SP + n);
                    const double zs = pass ? g : 1.0;
                    Ps[m * (SP + 1) + n] = fma(zs, z.x, ap[mt][0]);
                    Ps[m * (SP + 1) + n + 1] = fma(zs, z.y, ap[mt][1]);
                }
            }
        }
        __syncthreads();
        const bool frag_post = !tip || tip_partials, frag_pre = !tip;
        for (int idx = threadIdx.x; idx < (int)MAT; idx += blockDim.x) {
            const int row = idx / SP, col = idx % SP;
            if (pass == 0) {
                const int ln = idx & 31, kt = (idx >> 5) & (KT - 1), nt = idx / (32 * KT);
                const int kk = kt * 4 + (ln & 3), nn = nt * 8 + (ln >> 2);
                if (frag_post) PBpost[base + idx] = Ps[nn * (SP + 1) + kk];    // B[k=t][n=s] = P[s][t]
                if (frag_pre) PBpre[base + idx] = Ps[kk * (SP + 1) + nn];      // B[k=s][n=t] = P[s][t]
                if (tip) PT[base + idx] = Ps[col * (SP + 1) + row];            // P'[t][s] = P[s][t]
            } else {
                DT[base + idx] = Ps[col * (SP + 1) + row];                     // D'
            }
        }
        if (pass == 0 && tip)
            for (int s2 = threadIdx.x; s2 < SP; s2 += blockDim.x) {
                double acc = 0.0;
                for (int u = 0; u < SP; ++u) acc += Ps[s2 * (SP + 1) + u];
                PONE[(size_t)br * SP + s2] = acc;
            }
        __syncthreads();
    }
    if (pready && threadIdx.x == 0) {                    // publish (release): P and D CTAs per (branch, r)
        __threadfence();
        atomicAdd(pready + br, pass ? PMAT_D_DONE : PMAT_P_DONE);
    }
}
template <int SP>
constexpr size_t pmat_smem() { return ((size_t)SP * (SP + 1) + 2 * SP + (SP == 64 ? (size_t)SP * SP : 0)) * 8; }

}  // namespace codon
}  // namespace pg
