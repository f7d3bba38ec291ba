// traverse_big.cuh -- state spaces of 129..254 states padded to SP = 256
// (the paper's "S = 256 model with over 20,000 branch
// lengths"), fp64 on the FP64 tensor path, transpose-free.
//
// The paper stores every transition matrix AND its transpose (a separate
// matrixTranspose kernel; ~10 GB at S = 256 and 20,000 branches).
// Here each (branch, category) keeps ONE matrix, W = P' (row-major, 512 KB),
// and every product reads it in the orientation it needs, fragment by
// fragment, straight from L2:
//   post   u_k = p P_k'      (Eq. 2)   C = A W,    B[k][n] = W[k][n]
//   pre    q_c = x P_c       (Eq. 4)   C = A W',   B[k][n] = W[n][k]
//   grad   Q u               (Eq. 8)   C = A Q',   B[k][n] = Q[n][k]
//   tips   u_tip[s] = P[s][state] = W[state][s]: a contiguous ROW of W;
//          masked partial tips (hidden copies of an observed state) sum <= 4
//          rows of W; missing data u = P 1.
// A tile is 32 patterns x 256 states (64 KB, fragment order apos<256>, the
// layout of traverse_codon.cuh); a CTA of 16 warps computes one tile's
// [32 x 256] x [256 x 256] product, warp w owning output columns 16w..16w+15,
// with the B fragments of the next k-step loaded while the current one runs.
// Level-by-level launches (post levels by height, pre levels by depth), one
// CTA per (tile, node, category); rescaling, Eq. 3 and the ratio kernel are
// those of the codon path (traverse_codon.cuh).
#pragma once
#include "traverse_codon.cuh"

namespace pg {
namespace big {

using codon::CodonArgs;
using codon::T;
constexpr int SP = 256, KT = SP / 4, NWB = 16, NTB = NWB * 32, TILE = T * SP;
constexpr size_t MAT = (size_t)SP * SP;

__device__ __forceinline__ int ap(int m, int k) { return codon::apos<SP>(m, k); }

// acc (mt 4, nt 2 = columns 16w + 8j + ..) = A (32 x 256, smem fragment order;
// with A2: A o A2 formed in the loads) times B (256 x 256) from global:
// TRANS = false: B[k][n] = Bg[k][n]; TRANS = true: B[k][n] = Bg[n][k].
template <bool TRANS, bool PROD>
__device__ __forceinline__ void gemm256(double (&acc)[4][2][2], const double *As, const double *A2,
                                        const double *__restrict__ Bg, int w, int lane) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[mt][j][0] = acc[mt][j][1] = 0.0;
    auto bload = [&](int kt, int j) {
        const int k = kt * 4 + (lane & 3), n = (2 * w + j) * 8 + (lane >> 2);
        return __ldg(TRANS ? Bg + (size_t)n * SP + k : Bg + (size_t)k * SP + n);
    };
    double b0[2] = {bload(0, 0), bload(0, 1)}, b1[2] = {bload(1, 0), bload(1, 1)};
#pragma unroll 4
    for (int kt = 0; kt < KT; ++kt) {
        double bn[2] = {0.0, 0.0};
        if (kt + 2 < KT) { bn[0] = bload(kt + 2, 0); bn[1] = bload(kt + 2, 1); }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int p = (mt * KT + kt) * 32 + lane;
            const double av = PROD ? As[p] * A2[p] : As[p];
            codon::dmma(acc[mt][0], av, b0[0]);
            codon::dmma(acc[mt][1], av, b0[1]);
        }
        b0[0] = b1[0]; b0[1] = b1[1];
        b1[0] = bn[0]; b1[1] = bn[1];
    }
}

// child tile (category r, tile) into dst: internal u (HBM), masked partial
// tip (utip, formed by big_tipmask_kernel), state tip (rows of W by state)
__device__ void load_child256(double *dst, const CodonArgs &a, int child, int r, int tile, int *stbuf) {
    if (child >= a.N) {
        const double *src = a.u + (((size_t)(child - a.N) * a.R + r) * a.ntiles + tile) * TILE;
        for (int i = threadIdx.x; i < TILE / 2; i += NTB) cp_async16(dst + 2 * i, src + 2 * i);
        return;
    }
    const size_t br = (size_t)child * a.R + r;
    if (a.tip_is_partial[child]) {
        const double *src = a.utip + ((br * a.ntiles + tile) * TILE);
        for (int i = threadIdx.x; i < TILE / 2; i += NTB) cp_async16(dst + 2 * i, src + 2 * i);
        return;
    }
    const double *W = a.PT + br * MAT, *ONE = a.PONE + br * SP;
    for (int i = threadIdx.x; i < TILE / 2; i += NTB) {
        int m, k;
        codon::apos_inv<SP>(2 * i, m, k);
        const int s = stbuf[m];
        cp_async16(dst + 2 * i, s < a.S ? W + (size_t)s * SP + k : ONE + k);
    }
}

__device__ __forceinline__ void stage_states(int *stbuf, const CodonArgs &a, int child, int tile) {
    if (threadIdx.x < T) stbuf[threadIdx.x] = child < a.N ? a.tip_states[(size_t)child * a.Cpad + tile * T + threadIdx.x] : 0;
}

// scaled store of a [32 x 256] product (rows times f2[m]) in fragment order,
// with the IEEE-exponent max of every row into mx[m]
__device__ __forceinline__ void store_tile(double *out, int *mx, const double (&acc)[4][2][2], const double *f2, int w,
                                           int lane) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        const int m = mt * 8 + (lane >> 2);
        int f = 0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int n = (2 * w + j) * 8 + 2 * (lane & 3);
            const double c0 = acc[mt][j][0] * f2[m], c1 = acc[mt][j][1] * f2[m];
            *reinterpret_cast<double2 *>(out + ap(m, n)) = make_double2(c0, c1);
            f = max(f, max(__double2hiint(c0) >> 20, __double2hiint(c1) >> 20));
        }
        f = max(f, __shfl_xor_sync(0xffffffffu, f, 1));
        f = max(f, __shfl_xor_sync(0xffffffffu, f, 2));
        if ((lane & 3) == 0) atomicMax(mx + m, f);
    }
}

constexpr size_t post_smem() { return (size_t)2 * TILE * 8 + 4 * T * 8; }
constexpr size_t pre_smem() { return (size_t)3 * TILE * 8 + (size_t)3 * NWB * T * 8 + 4 * T * 8 + 2 * T * 4; }

// post-order level: one CTA per (tile, node of the level, category)
__global__ void __launch_bounds__(NTB, 1) big_post_kernel(const CodonArgs a, int level_off) {
    extern __shared__ __align__(16) unsigned char smem_b[];
    double *As = reinterpret_cast<double *>(smem_b), *Bs = As + TILE;
    double *f2 = Bs + TILE;                                   // [T] children's row scales
    int *sta = reinterpret_cast<int *>(f2 + T), *stb = sta + T;
    const int tile = blockIdx.x, r = blockIdx.z;
    const int4 e = a.lev4[level_off + blockIdx.y];
    const int k = e.x, ca = e.y, cb = e.z;
    const int root = 2 * a.N - 2, pat0 = tile * T;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    stage_states(sta, a, ca, tile);
    stage_states(stb, a, cb, tile);
    __syncthreads();
    load_child256(As, a, ca, r, tile, sta);
    load_child256(Bs, a, cb, r, tile, stb);
    cp_async_commit();
    const bool doE = r == 0 && threadIdx.x < T;
    int Ea = 0, Eb = 0, fa = 0, fb = 0;
    if (threadIdx.x < T) {
        const int m = threadIdx.x;
        if (ca >= a.N) fa = __ldcg(a.fmax + (size_t)(ca - a.N) * a.Cpad + pat0 + m);
        if (cb >= a.N) fb = __ldcg(a.fmax + (size_t)(cb - a.N) * a.Cpad + pat0 + m);
        if (doE && ca >= a.N) Ea = __ldcg(a.E + (size_t)(ca - a.N) * a.Cpad + pat0 + m);
        if (doE && cb >= a.N) Eb = __ldcg(a.E + (size_t)(cb - a.N) * a.Cpad + pat0 + m);
        f2[m] = (ca >= a.N ? codon::pow2neg(codon::lazy_exp(fa)) : 1.0) *
                (cb >= a.N ? codon::pow2neg(codon::lazy_exp(fb)) : 1.0);
    }
    cp_async_wait<0>();
    __syncthreads();
    if (doE) {
        const int m = threadIdx.x;
        a.E[(size_t)(k - a.N) * a.Cpad + pat0 + m] =
            Ea + Eb + (ca >= a.N ? codon::lazy_exp(fa) : 0) + (cb >= a.N ? codon::lazy_exp(fb) : 0);
    }
    if (k == root) {                                          // Eq. 3 terms
        const int m = threadIdx.x >> 4, j = threadIdx.x & 15;
        double sum = 0.0;
        for (int kk = j; kk < SP; kk += 16) {
            const int p = ap(m, kk);
            sum = fma(a.pi[kk], As[p] * Bs[p], sum);
        }
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (j == 0) a.Lpart[(size_t)r * a.Cpad + pat0 + m] = a.cat_w[r] * sum * f2[m];
        return;
    }
    for (int i = threadIdx.x; i < TILE / 2; i += NTB) {       // p = u_a o u_b in place
        double2 *pa = reinterpret_cast<double2 *>(As) + i;
        const double2 tb = reinterpret_cast<const double2 *>(Bs)[i];
        double2 v = *pa;
        v.x *= tb.x;
        v.y *= tb.y;
        *pa = v;
    }
    __syncthreads();
    double acc[4][2][2];
    gemm256<false, false>(acc, As, nullptr, a.PT + ((size_t)k * a.R + r) * MAT, w, lane);
    store_tile(a.u + (((size_t)(k - a.N) * a.R + r) * a.ntiles + tile) * TILE,
               a.fmax + (size_t)(k - a.N) * a.Cpad + pat0, acc, f2, w, lane);
}

// pre-order level: one CTA per (tile, parent of the level, category)
__global__ void __launch_bounds__(NTB, 1) big_pre_kernel(const CodonArgs a, int level_off) {
    extern __shared__ __align__(16) unsigned char smem_b[];
    double *Qs = reinterpret_cast<double *>(smem_b), *Ua = Qs + TILE, *Ub = Ua + TILE;
    double *part = Ub + TILE;                                 // [3][NWB][T]
    double *sc = part + 3 * NWB * T;                          // [4][T]: q_k, u_a, u_b scales, x row scale
    int *sta = reinterpret_cast<int *>(sc + 4 * T), *stb = sta + T;
    const int tile = blockIdx.x, r = blockIdx.z;
    const int4 e = a.lev4[level_off + blockIdx.y];
    const int k = e.x, ch[2] = {e.y, e.z};
    const int root = 2 * a.N - 2, pat0 = tile * T;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    stage_states(sta, a, ch[0], tile);
    stage_states(stb, a, ch[1], tile);
    if (threadIdx.x < T) {
        const int m = threadIdx.x;
        sc[m] = k == root ? 1.0 : codon::pow2neg(codon::lazy_exp(__ldcg(a.qmax + (size_t)(k - a.N) * a.Cpad + pat0 + m)));
        for (int c = 0; c < 2; ++c)
            sc[(1 + c) * T + m] = ch[c] >= a.N
                                      ? codon::pow2neg(codon::lazy_exp(__ldcg(a.fmax + (size_t)(ch[c] - a.N) * a.Cpad + pat0 + m)))
                                      : 1.0;
    }
    __syncthreads();
    if (k == root) {
        for (int idx = threadIdx.x; idx < TILE; idx += NTB) Qs[idx] = a.pi[((idx >> 5) & (KT - 1)) * 4 + (idx & 3)];
    } else {
        const double *src = a.q + (((size_t)(k - a.N) * a.R + r) * a.ntiles + tile) * TILE;
        for (int i = threadIdx.x; i < TILE / 2; i += NTB) cp_async16(Qs + 2 * i, src + 2 * i);
    }
    load_child256(Ua, a, ch[0], r, tile, sta);
    load_child256(Ub, a, ch[1], r, tile, stb);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    double *Us[2] = {Ua, Ub};
    // q_c = (q_k o u_sib) P_c for internal children (Eq. 4); rows scaled by
    // the q_k and sibling exponents
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
        const int node = ch[c];
        if (node < a.N) continue;
        double acc[4][2][2];
        gemm256<true, true>(acc, Qs, Us[1 - c], a.PT + ((size_t)node * a.R + r) * MAT, w, lane);
        double *f2 = sc + 3 * T;
        __syncthreads();                                      // previous child's store read f2
        if (threadIdx.x < T) f2[threadIdx.x] = sc[threadIdx.x] * sc[(2 - c) * T + threadIdx.x];
        __syncthreads();
        store_tile(a.q + (((size_t)(node - a.N) * a.R + r) * a.ntiles + tile) * TILE,
                   a.qmax + (size_t)(node - a.N) * a.Cpad + pat0, acc, f2, w, lane);
    }
    // Eq. 8 terms: num_c = x_c'(Q u_c), den = x_c'u_c (same for both children,
    // Eq. 5); tiles unscaled (factors cancel in the ratio over categories)
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
        double acc[4][2][2];
        gemm256<true, false>(acc, Us[c], nullptr, a.QB, w, lane);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const int m = mt * 8 + (lane >> 2);
            double sn = 0.0, sd = 0.0;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int n = (2 * w + j) * 8 + 2 * (lane & 3);
                const int p = ap(m, n);
                const double2 q2 = *reinterpret_cast<const double2 *>(Qs + p);
                const double2 o2 = *reinterpret_cast<const double2 *>(Us[1 - c] + p);
                const double x0 = q2.x * o2.x, x1 = q2.y * o2.y;
                sn += x0 * acc[mt][j][0] + x1 * acc[mt][j][1];
                if (c == 0) {
                    const double2 u2 = *reinterpret_cast<const double2 *>(Us[0] + p);
                    sd += x0 * u2.x + x1 * u2.y;
                }
            }
            sn += __shfl_xor_sync(0xffffffffu, sn, 1);
            sn += __shfl_xor_sync(0xffffffffu, sn, 2);
            sd += __shfl_xor_sync(0xffffffffu, sd, 1);
            sd += __shfl_xor_sync(0xffffffffu, sd, 2);
            if ((lane & 3) == 0) {
                part[(c * NWB + w) * T + m] = sn;
                if (c == 0) part[(2 * NWB + w) * T + m] = sd;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < T) {                                    // fixed-order sums over the warps
        const int m = threadIdx.x;
        double sd = 0.0, sn0 = 0.0, sn1 = 0.0;
        for (int ww = 0; ww < NWB; ++ww) {
            sn0 += part[ww * T + m];
            sn1 += part[(NWB + ww) * T + m];
            sd += part[(2 * NWB + ww) * T + m];
        }
        const double wr = a.cat_w[r], gr = a.cat_g[r];
        double2 *nd = reinterpret_cast<double2 *>(a.numden);
        nd[((size_t)ch[0] * a.R + r) * a.Cpad + pat0 + m] = make_double2(gr * wr * sn0, wr * sd);
        nd[((size_t)ch[1] * a.R + r) * a.Cpad + pat0 + m] = make_double2(gr * wr * sn1, wr * sd);
    }
}

// u of masked partial tips (0/1 partials with <= 4 ones: hidden copies of an
// observed state): u[m][s] = sum over the mask states t of P[s][t] = W[t][s],
// rows of W; one CTA per (tile, tip, category)
__global__ void __launch_bounds__(256) big_tipmask_kernel(const CodonArgs a) {
    const int tile = blockIdx.x, tip = blockIdx.y, r = blockIdx.z;
    if (!a.tip_is_partial[tip]) return;
    const double *W = a.PT + ((size_t)tip * a.R + r) * MAT;
    double *out = a.utip + (((size_t)tip * a.R + r) * a.ntiles + tile) * TILE;
    const uint8_t *mk = a.tip_mask + ((size_t)tip * a.Cpad + (size_t)tile * T) * 4;
    for (int i2 = threadIdx.x; i2 < TILE / 2; i2 += blockDim.x) {
        int m, kk;
        codon::apos_inv<SP>(2 * i2, m, kk);
        const uchar4 ids = __ldg(reinterpret_cast<const uchar4 *>(mk + 4 * m));
        const uint8_t id4[4] = {ids.x, ids.y, ids.z, ids.w};
        double2 u = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (id4[j] != 255) {
                const double2 v = __ldg(reinterpret_cast<const double2 *>(W + (size_t)id4[j] * SP + kk));
                u.x += v.x;
                u.y += v.y;
            }
        reinterpret_cast<double2 *>(out)[i2] = u;
    }
}

// A1: W = P' = M0' + (V^-1)' diag(expm1(gamma_r b_i lambda)) V' for every
// (branch, category) -- one 256^3 DMMA product per matrix, CTA = 32 rows of W
// (blockIdx.y: 8 row blocks), 8 warps x 32 columns; the A operand (V^-1)'
// and the B operand V' are pre-arranged in fragment order at pg_set_eigen
// (ViTA: [mt 64][kt 64][32], VTB: [nt 32][kt 64][32]).  P 1 (missing-data
// tips) = M0 1 + V diag(e - 1) (V^-1 1) by row block 0.
__global__ void __launch_bounds__(256) big_pmat_kernel(const double *__restrict__ ViTA, const double *__restrict__ VTB,
                                                       const double *__restrict__ M0, const double *__restrict__ M0one,
                                                       const double *__restrict__ V, const double *__restrict__ Vione,
                                                       const double *__restrict__ lam, const double *__restrict__ rates,
                                                       const double *__restrict__ bl, int S, int R, double *W,
                                                       double *PONE) {
    __shared__ double em1[SP];
    const int br = blockIdx.x, r = br % R, b = br / R, rb = blockIdx.y;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double t = rates[r] * bl[b];
    for (int k = threadIdx.x; k < SP; k += blockDim.x) em1[k] = k < S ? expm1(lam[k] * t) : 0.0;
    __syncthreads();
    double acc[4][4][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[mt][j][0] = acc[mt][j][1] = 0.0;
    const double *A = ViTA + (size_t)rb * 4 * KT * 32 + lane;        // rows 32 rb .. 32 rb + 31
#pragma unroll 2
    for (int kt = 0; kt < KT; ++kt) {
        const double ek = em1[kt * 4 + (lane & 3)];
        double bv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = __ldg(VTB + ((size_t)(4 * w + j) * KT + kt) * 32 + lane);
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
            const double av = __ldg(A + (mt * KT + kt) * 32) * ek;
#pragma unroll
            for (int j = 0; j < 4; ++j) codon::dmma(acc[mt][j], av, bv[j]);
        }
    }
    double *Wm = W + (size_t)br * MAT;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
        const int row = rb * 32 + mt * 8 + (lane >> 2);           // t
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = (4 * w + j) * 8 + 2 * (lane & 3);     // s
            // W[t][s] = P[s][t] = M0[s][t] + ...
            const double m0a = M0[(size_t)col * SP + row], m0b = M0[(size_t)(col + 1) * SP + row];
            *reinterpret_cast<double2 *>(Wm + (size_t)row * SP + col) = make_double2(acc[mt][j][0] + m0a, acc[mt][j][1] + m0b);
        }
    }
    if (rb == 0)
        for (int s = threadIdx.x; s < SP; s += blockDim.x) {
            double acc1 = 0.0;
            if (s < S)
                for (int k = 0; k < S; ++k) acc1 += V[(size_t)s * S + k] * em1[k] * Vione[k];
            PONE[(size_t)br * SP + s] = acc1 + M0one[s];
        }
}

}  // namespace big
}  // namespace pg
