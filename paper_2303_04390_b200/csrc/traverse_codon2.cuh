// traverse_codon2.cuh -- codon path (fp64, S > 16 padded to SP = 64 / 128),
// one-launch dataflow schedule, warp-specialised with TMA staging.
//
// Same work items, data layout (fragment order, traverse_codon.cuh) and
// dependency counters as codon_flow_kernel; what changes is how a CTA runs
// them.  A CTA is NW consumer warps (warp w owns output columns 8w..8w+7 of
// every [32 x SP] x [SP x SP] product) plus ONE PRODUCER warp, joined by an
// NST-stage shared-memory ring (mbarriers "full" / "empty"):
//   producer  claims the next item (global counter, topological order),
//             prefetches the item's B operands (P, Q fragments) into L1,
//             waits (acquire) until the item's inputs are published, then
//             stages them: the partial-likelihood TILES (u of internal
//             children, q of the parent, u of partial tips) with TMA tensor
//             loads (cp.async.bulk.tensor, SASS UTMALDG; 16 KB per tile, one
//             instruction), state-tip tiles as row gathers of P' (cp.async,
//             completion tracked by the same mbarrier), and the per-pattern
//             rescaling exponents and tip states;
//   consumers wait on "full", run the item's GEMMs on the FP64 tensor path
//             (mma.sync m8n8k4 f64, SASS DMMA), store results, publish
//             completion (fence + atomic counter) and release the stage.
// While the consumers compute item i, the producer is already waiting for /
// loading item i+1 (and i+2 with three stages), so dependency waits and tile
// loads leave the tensor pipe's critical path.
//   post item (node k, category r, tile): p = u_a o u_b formed in place,
//             u_k = p P_k' (Eq. 2), rows scaled by the children's exponents;
//             at the root the Eq. 3 terms P(gamma_r) pi' p.
//   pre item  (parent k, category r, tile): q_c = (q_k o u_sib) P_c (Eq. 4)
//             for internal children -- the A operand formed on the fly --
//             published before the Eq. 8 terms num_c = x_c'(Q u_c),
//             den = x_c'u_c (Eq. 6-8; state tips: rows of D').
// Paper: Eq. 2, Eq. 3, Eq. 4, Eq. 6-8
// P:274-365; Alg. 1/2's prefetch of partials into shared memory P:385-389,
// P:633-634 (here: TMA).
#pragma once
#include <cuda.h>

#include "traverse_codon.cuh"

namespace pg {
namespace codon {

struct TmaMaps {
    CUtensorMap u;      // u    as [rows][256] doubles, one tile = TILE/256 rows
    CUtensorMap q;      // q    (same geometry)
    CUtensorMap utip;   // utip (same geometry; partial tips)
};

__device__ __forceinline__ void tma_load_tile(uint32_t dst, const CUtensorMap *map, int row, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(row), "r"(bar)
        : "memory");
}
// arrive on `bar` (one of its expected arrivals) when this thread's prior
// cp.async copies have landed
__device__ __forceinline__ void cp_async_mbar_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void prefetch_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }
// mbarrier phase wait with a suspend-time hint: the waiting warp sleeps until
// the phase completes (or the hint expires) instead of re-issuing try_wait
// (ncu: 21 % of the flow kernel's issued instructions were the try_wait loop)
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAITS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAITS_%=;\n}\n" ::"r"(bar),
        "r"(parity), "r"(1000000u)
        : "memory");
}

// Poll a completion counter (acquire) until >= v.  A stall longer than
// ~20 s (a schedule bug, or a neighbour that never lets a CTA run) is
// reported through status[1] instead of trapping, and the wait gives up so
// the launch terminates; pg_check_status / pg_compute turn it into an error.
__device__ __forceinline__ void wait_count2(const int *p, int v, int *status, int mask = -1) {
    int x;
    const unsigned long long t0 = gtimer();
    for (unsigned it = 0;; ++it) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
        if ((x & mask) >= v) return;
        if ((it & 1023u) == 1023u && gtimer() - t0 > 20000000000ull) {
            atomicExch(status + 1, 1);
            return;
        }
        __nanosleep(32);
    }
}

// Per-stage metadata written by the producer (generic stores, ordered before
// its arrive on "full").
struct alignas(16) Meta2 {
    int item, task, r, tile;
    int4 lev;                 // {k, child a, child b, kinds}
    int cs, pad0, pad1, pad2; // pre items: -1 both children, else the one child of a split item
    int fa[T], fb[T];         // children's fmax (IEEE exponent fields), internal children
    int fq[T];                // qmax of the parent (pre, non-root)
    int Ea[T], Eb[T];         // children's cumulative exponents (this category)
    int Qe[T];                // cumulative exponent of q_k (pre, non-root; this category)
    uint8_t sa[T], sb[T];     // state codes of state-tip children
};

// NST = ring stages.  NST = 2: the producer claims and stages item i+1 while
// the consumers compute item i (throughput: full-size workloads).  NST = 1:
// an item is claimed only when the consumers are free, so a busy CTA never
// holds back an item another CTA could start (latency: pattern shards whose
// levels have fewer items than CTA slots), and three CTAs fit on an SM.
// RS = 2 splits every product's rows over twice the consumer warps (warp
// 8 h + w: output columns 8w..8w+7, row blocks 2h, 2h+1): half the DMMA chain
// per warp on the latency-bound shards (SP = 64 only: 16 + 1 warps)
template <int SP, int NST, int RS = 1> constexpr int flow2_ctas() { return RS == 2 ? 1 : SP == 64 ? (NST == 1 ? 3 : 2) : 1; }
// consumer warps + the producer warp + the publisher warp
template <int SP, int RS = 1> constexpr int flow2_threads() { return (SP / 8 * RS + 2) * 32; }
template <int SP> constexpr size_t flow2_stage() { return (size_t)3 * T * SP * 8 + ((sizeof(Meta2) + 127) / 128) * 128; }
template <int SP, int NST>
constexpr size_t flow2_smem() {
    return 128 + (size_t)NST * flow2_stage<SP>() + (size_t)NST * 3 * (SP / 8) * T * 8;   // barriers, ring, Eq. 8 partials per stage
}

// A1 -> flow overlap (programmatic dependent launch): the flow kernel may
// start while codon_pmat_kernel is still running; an item then also waits
// until the transition matrices it reads are published (pready[branch][r]:
// + PMAT_P_DONE by the branch's P CTA, + PMAT_D_DONE by its D CTA).  Post
// items read P of the node and of tip children; pre items P of the children
// and D of tip children.
__device__ __forceinline__ void wait_p(const FlowArgs &f, int node, int r, int R, int root, bool need_d, int *status) {
    if (f.pready && node != root) {
        const int *p = f.pready + (size_t)node * R + r;
        if (need_d) wait_count2(p, PMAT_P_DONE + PMAT_D_DONE, status);
        else wait_count2(p, PMAT_P_DONE, status, PMAT_D_DONE - 1);
    }
}

template <int SP, int NST, int RS = 1>
__global__ void __launch_bounds__(flow2_threads<SP, RS>(), (flow2_ctas<SP, NST, RS>()))
    codon_flow2_kernel(const CodonArgs a, const FlowArgs f, const __grid_constant__ TmaMaps tm) {
    CODON_GEO;
    constexpr int NWC = NW * RS, NTC = NWC * 32, MTW = 4 / RS;     // consumer warps / threads, row blocks per warp
    constexpr size_t STG = flow2_stage<SP>();
    constexpr int ROWS = TILE / 256;                       // tensor-map rows per tile
    constexpr unsigned TILE_B = (unsigned)TILE * 8u;
    extern __shared__ __align__(128) unsigned char smem2[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem2);
    uint64_t *empty = full + NST;
    uint64_t *ldb = full + 2 * NST;              // f.pprod: the stage's copies landed (producer-side p)
    uint64_t *pub = full + 3 * NST;              // f.pub: the consumer warps' outputs are issued
    uint64_t *done = full + 4 * NST;             // f.pub: a pre item's Eq. 8 partials are written
    unsigned char *ring = smem2 + 128;
    double *part0 = reinterpret_cast<double *>(ring + NST * STG);         // [NST][3][NW][T]
    auto partS = [&](int s) { return part0 + (size_t)s * 3 * NW * T; };
    const uint32_t full_u = smem_u32(full), empty_u = smem_u32(empty), ldb_u = smem_u32(ldb), pub_u = smem_u32(pub),
                   done_u = smem_u32(done);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int R = a.R, ntiles = a.ntiles, N = a.N;
    const int root = 2 * N - 2;
    // per-category exponents and completion counters: an item depends only on
    // its own category's inputs (round 1: on all R categories, through the
    // exponent shared across categories)
    auto fi = [&](int node, int r, int p) -> size_t { return ((size_t)(node - N) * R + r) * a.Cpad + p; };
    auto ci = [&](int node, int r, int t) -> size_t { return ((size_t)(node - N) * R + r) * ntiles + t; };
    // items: post (task, r, tile); pre (task, r, tile) for both children, or
    // with f.split, for a parent whose children are both internal, (task,
    // child, r, tile): one child each -- the two q GEMMs of the parent then
    // run on different CTAs (shorter pre-order chain links); f.task_off holds
    // the first item of every task
    const int npost_items = f.npost * R * ntiles;
    const int nitems = f.split ? f.task_off[f.ntask] : f.ntask * R * ntiles;
    auto tileA = [&](int s) { return reinterpret_cast<double *>(ring + s * STG); };
    auto meta = [&](int s) { return reinterpret_cast<Meta2 *>(ring + s * STG + 3 * (size_t)TILE * 8); };
    if (threadIdx.x == 0) {
        // full: lane 0's expect_tx arrive + the 32 lanes' cp.async arrives +
        // lane 0's final arrive (after the metadata stores)
        for (int i = 0; i < NST; ++i) {
            mbar_init(full + i, 34);
            mbar_init(empty + i, 1);
            mbar_init(ldb + i, 34);
            mbar_init(pub + i, NWC);
            mbar_init(done + i, NWC);
        }
        fence_mbar_init();
    }
    __syncthreads();

    // ================================ producer ================================
    if (warp == NWC) {
        uint32_t ldph = 0;                           // ldb phase bits per stage
        for (int g = 0;; ++g) {
            const int s = g % NST;
            if (g >= NST) mbar_wait_sleep(empty_u + 8u * s, (uint32_t)(g / NST + 1) & 1u);
            int item = 0;
            if (lane == 0) item = atomicAdd(f.ctr, 1);
            item = __shfl_sync(0xffffffffu, item, 0);
            Meta2 *m = meta(s);
            if (item >= nitems) {
                const uint32_t bar = full_u + 8u * s;
                if (lane == 0) m->item = -1;
                cp_async_mbar_arrive(bar);
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive_u32(bar);
                    mbar_arrive_u32(bar);
                }
                break;
            }
            unsigned long long *tr = f.trace ? f.trace + TRW * (size_t)item : nullptr;   // PG_FLOW_TRACE
            if (tr && lane == 0) {
                unsigned smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                tr[0] = smid;
                tr[1] = gtimer();
                tr[7] = blockIdx.x;
            }
            int task, cs = -1, rem;
            if (item < npost_items || !f.split) {
                task = item / (R * ntiles);
                rem = item - task * R * ntiles;
            } else {
                int lo = f.npost, hi = f.ntask - 1;      // last task starting at or before item
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (__ldg(f.task_off + mid) <= item) lo = mid;
                    else hi = mid - 1;
                }
                task = lo;
                const int rr = item - __ldg(f.task_off + task), per = R * ntiles;
                if (__ldg(f.task_off + task + 1) - __ldg(f.task_off + task) == 2 * per) {
                    cs = rr / per;
                    rem = rr - cs * per;
                } else {
                    rem = rr;
                }
            }
            const int r = rem / ntiles, tile = rem - r * ntiles;
            const int4 e = a.lev4[task];
            const int k = e.x, ca = e.y, cb = e.z, kinds = e.w;
            const bool post = task < f.npost;
            // f.pprod: a post item's copies complete on ldb; the producer then
            // forms p = u_a o u_b in place and completes "full" itself
            const bool pp = f.pprod && post && k != root;
            const uint32_t bar = (pp ? ldb_u : full_u) + 8u * s;
            if (lane == 0 && f.pready) {             // the item's P, P', D' rows written by A1
                if (post) {
                    wait_p(f, k, r, R, root, false, a.status);
                    if (ca < N) wait_p(f, ca, r, R, root, false, a.status);
                    if (cb < N) wait_p(f, cb, r, R, root, false, a.status);
                } else {
                    if (cs != 1) wait_p(f, ca, r, R, root, ca < N, a.status);
                    if (cs != 0) wait_p(f, cb, r, R, root, cb < N, a.status);
                }
            }
            __syncwarp();
            // ---- what does not depend on other items, before the wait:
            // B operands into this SM's L1, tip states, state-tip tile gathers
            // (rows of P' picked by state: u_tip[s] = P[s][state]; missing data:
            // P 1) with cp.async, the item header, q = pi at the root
            {
                auto pf = [&](const double *Bg) {
                    for (int i = lane; i < (int)MAT / 16; i += 32) prefetch_l1(Bg + 16 * i);
                };
                if (post) {
                    if (k != root) pf(a.PBpost + ((size_t)k * R + r) * MAT);
                } else {
                    if (ca >= N && cs != 1) pf(a.PBpre + ((size_t)ca * R + r) * MAT);
                    if (cb >= N && cs != 0) pf(a.PBpre + ((size_t)cb * R + r) * MAT);
                }
            }
            const int pat = tile * T + lane;
            const int kc[2] = {kinds & 3, (kinds >> 2) & 3};
            const int cc[2] = {ca, cb};
            int st2[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                st2[c] = (cc[c] < N && kc[c] == 1) ? a.tip_states[(size_t)cc[c] * a.Cpad + pat] : 0;
                (c ? m->sb : m->sa)[lane] = (uint8_t)st2[c];
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                if (cc[c] >= N || kc[c] != 1) continue;
                const size_t br = (size_t)cc[c] * R + r;
                const double *PT = a.PT + br * MAT, *ONE = a.PONE + br * SP;
                double *dst = tileA(s) + (size_t)c * TILE;
                for (int i2 = lane; i2 < TILE / 2; i2 += 32) {
                    int mm, kk;
                    apos_inv<SP>(2 * i2, mm, kk);
                    const int sv = __shfl_sync(0xffffffffu, st2[c], mm);
                    cp_async16(dst + 2 * i2, sv < a.S ? PT + (size_t)sv * SP + kk : ONE + kk);
                }
            }
            if (!post && k == root) {
                double *Qs = tileA(s) + 2 * (size_t)TILE;
                for (int idx = lane; idx < TILE; idx += 32) Qs[idx] = a.pi[((idx >> 5) & (KT - 1)) * 4 + (idx & 3)];
            }
            if (lane == 0) {
                m->item = item;
                m->task = task;
                m->r = r;
                m->tile = tile;
                m->lev = e;
                m->cs = cs;
            }
            // ---- inputs published by other items
            if (lane == 0) {
                if (post || k == root) {
                    if (ca >= N) wait_count2(f.rpost + ci(ca, r, tile), 1, a.status);
                    if (cb >= N) wait_count2(f.rpost + ci(cb, r, tile), 1, a.status);
                } else {
                    wait_count2(f.rpre + ci(k, r, tile), 1, a.status);
                }
                if (tr) tr[2] = gtimer();
                fence_proxy_async_global();          // published generic stores -> our async-proxy reads
                unsigned bytes = 0;
                for (int c = 0; c < 2; ++c)
                    if (cc[c] >= N || kc[c] == 2) bytes += TILE_B;
                if (!post && k != root) bytes += TILE_B;
                fence_proxy_async_smem();            // earlier generic accesses of this stage -> TMA writes
                mbar_arrive_expect_tx_u32(bar, bytes);
                const uint32_t st_u = smem_u32(tileA(s));
                for (int c = 0; c < 2; ++c) {
                    if (cc[c] >= N)
                        tma_load_tile(st_u + c * TILE_B, &tm.u, (int)((((size_t)(cc[c] - N) * R + r) * ntiles + tile) * ROWS), bar);
                    else if (kc[c] == 2)
                        tma_load_tile(st_u + c * TILE_B, &tm.utip, (int)((((size_t)cc[c] * R + r) * ntiles + tile) * ROWS), bar);
                }
                if (!post && k != root)
                    tma_load_tile(st_u + 2 * TILE_B, &tm.q, (int)((((size_t)(k - N) * R + r) * ntiles + tile) * ROWS), bar);
            }
            __syncwarp();
            // per-pattern rescaling exponents of the inputs (lane = pattern),
            // 4-byte cp.async into the stage's metadata
            if (ca >= N) cp_async4(&m->fa[lane], a.fmax + fi(ca, r, pat));
            else m->fa[lane] = 0;
            if (cb >= N) cp_async4(&m->fb[lane], a.fmax + fi(cb, r, pat));
            else m->fb[lane] = 0;
            // (a.Y: exponents reconciled over R > 1 categories in A6; the pre
            // items then also need q_k's and the children's cumulative ones)
            if (!post) {
                if (k != root) cp_async4(&m->fq[lane], a.qmax + fi(k, r, pat));
                else m->fq[lane] = 0;
                if (a.Y) {
                    if (k != root) cp_async4(&m->Qe[lane], a.EQ + fi(k, r, pat));
                    else m->Qe[lane] = 0;
                }
            }
            if (post || a.Y) {
                if (ca >= N) cp_async4(&m->Ea[lane], a.E + fi(ca, r, pat));
                else m->Ea[lane] = 0;
                if (cb >= N) cp_async4(&m->Eb[lane], a.E + fi(cb, r, pat));
                else m->Eb[lane] = 0;
            }
            // the stage is complete when the TMA bytes, every lane's cp.async
            // copies and lane 0's arrive below have all landed
            cp_async_mbar_arrive(bar);
            __syncwarp();
            if (lane == 0) mbar_arrive_u32(bar);
            if (pp) {
                mbar_wait_sleep(bar, (ldph >> s) & 1u);
                ldph ^= 1u << s;
                double2 *pa = reinterpret_cast<double2 *>(tileA(s));
                const double2 *pb = reinterpret_cast<const double2 *>(tileA(s) + TILE);
                for (int i2 = lane; i2 < TILE / 2; i2 += 32) {
                    double2 v = pa[i2];
                    const double2 tb = pb[i2];
                    v.x *= tb.x;
                    v.y *= tb.y;
                    pa[i2] = v;
                }
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], 34;\n" ::"r"(full_u + 8u * s) : "memory");
            }
        }
    }

    // Eq. 8 terms of a pre item -> numden: fixed-order sums over the column
    // warps' partials (pattern mm), weights w_r and gamma_r w_r (Eq. 8)
    auto finish_pre = [&](const Meta2 *m, const double *part, int mm) {
        const int r = m->r, cs = m->cs, ca = m->lev.y, cb = m->lev.z, kinds = m->lev.w;
        const int c0 = cs < 0 ? 0 : cs, c1 = cs < 0 ? 1 : cs;
        double sd = 0.0, sn0 = 0.0, sn1 = 0.0;
        for (int ww = 0; ww < NW; ++ww) {
            if (c0 == 0) sn0 += part[ww * T + mm];
            if (c1 == 1) sn1 += part[(NW + ww) * T + mm];
            sd += part[(2 * NW + ww) * T + mm];
        }
        const double wr = a.cat_w[r], gr = a.cat_g[r];
        double2 *nd = reinterpret_cast<double2 *>(a.numden);
        const bool qa = ca >= N || (kinds & 3) == 2, qb = cb >= N || ((kinds >> 2) & 3) == 2;
        const double s0 = qa ? gr * wr : wr, s1 = qb ? gr * wr : wr;
        const size_t pat = (size_t)m->tile * T + mm;
        if (c0 == 0) nd[((size_t)ca * R + r) * a.Cpad + pat] = make_double2(s0 * sn0, wr * sd);
        if (c1 == 1) nd[((size_t)cb * R + r) * a.Cpad + pat] = make_double2(s1 * sn1, wr * sd);
        // the terms' exponent: q_k's and both children's (tiles are unscaled)
        if (a.Y) {
            const int y = m->Qe[mm] + m->Ea[mm] + m->Eb[mm];
            if (c0 == 0) a.Y[((size_t)ca * R + r) * a.Cpad + pat] = y;
            if (c1 == 1) a.Y[((size_t)cb * R + r) * a.Cpad + pat] = y;
        }
    };

    // ================================ publisher ===============================
    // f.pub: completion flags are raised by this warp, so the consumer warps
    // never wait on the device-scope fence (its latency is ~1 us after a
    // tile's stores).  Per stage use, every consumer warp arrives on "pub"
    // once its outputs are issued (post: after the tile stores, which are also
    // the warp's last reads of the stage; pre: after the q stores).  Ordering:
    // each warp's stores -> __syncwarp -> mbarrier arrive (release.cta) ->
    // this warp's wait (acquire.cta) -> __threadfence -> flag atomic; the
    // reader acquires the flag at gpu scope (cumulativity of the PTX model,
    // as with the bar.sync + thread-0 fence it replaces).
    // A pre item's consumers then write their Eq. 8 partials and arrive on
    // "done"; this warp forms the fixed-order sums (lane = pattern), stores
    // numden and releases the stage -- the consumers go straight on to the
    // next item.
    if (warp == NWC + 1) {
        uint32_t dph = 0;                            // done phase bits per stage
        for (int g = 0; f.pub; ++g) {
            const int s = g % NST;
            mbar_wait_sleep(pub_u + 8u * s, (uint32_t)(g / NST) & 1u);
            const Meta2 *m = meta(s);
            const int item = m->item;
            if (item < 0) break;
            const int k = m->lev.x, ca = m->lev.y, cb = m->lev.z, tile = m->tile, cs = m->cs, r = m->r;
            const bool post = m->task < f.npost;
            unsigned long long *tr = (f.trace && lane == 0) ? f.trace + TRW * (size_t)item : nullptr;
            if (lane == 0) {
                if (post) {
                    mbar_arrive_u32(empty_u + 8u * s);   // fields read above: the stage is free
                    __threadfence();
                    atomicAdd(f.rpost + ci(k, r, tile), 1);
                } else {
                    const bool pa = cs != 1 && ca >= N, pb = cs != 0 && cb >= N;
                    if (pa || pb) {
                        __threadfence();
                        if (pa) atomicAdd(f.rpre + ci(ca, r, tile), 1);
                        if (pb) atomicAdd(f.rpre + ci(cb, r, tile), 1);
                    }
                }
                if (tr) tr[5] = gtimer();
            }
            if (!post) {
                mbar_wait_sleep(done_u + 8u * s, (dph >> s) & 1u);
                dph ^= 1u << s;
                finish_pre(m, partS(s), lane);
                __syncwarp();
                if (lane == 0) mbar_arrive_u32(empty_u + 8u * s);
                if (tr) tr[6] = gtimer();
            }
            __syncwarp();
        }
    }

    // ================================ consumers ===============================
    if (warp < NWC) {
        const int w = warp % NW, mt0 = (warp / NW) * MTW;              // column strip, first row block
        for (int g = 0;; ++g) {
            const int s = g % NST;
            mbar_wait_sleep(full_u + 8u * s, (uint32_t)(g / NST) & 1u);
            const Meta2 *m = meta(s);
            const int item = m->item;
            if (item < 0) {
                if (f.pub && lane == 0) mbar_arrive_u32(pub_u + 8u * s);   // the publisher sees the end too
                break;
            }
            const int r = m->r, tile = m->tile;
            const int k = m->lev.x, ca = m->lev.y, cb = m->lev.z, kinds = m->lev.w;
            const int pat0 = tile * T;
            unsigned long long *tr = (f.trace && threadIdx.x == 0) ? f.trace + TRW * (size_t)item : nullptr;
            if (tr) tr[3] = gtimer();
            double *As = tileA(s), *Bs = As + TILE, *Qs = As + 2 * (size_t)TILE;
            double *part = partS(s);
            const bool post = m->task < f.npost;
            if (post) {
                auto scA = [&](int mm) { return ca >= N ? pow2neg(lazy_exp(m->fa[mm])) : 1.0; };
                auto scB = [&](int mm) { return cb >= N ? pow2neg(lazy_exp(m->fb[mm])) : 1.0; };
                auto storeE = [&]() {
                    const int mm = threadIdx.x;
                    const int Ek = m->Ea[mm] + m->Eb[mm] + (ca >= N ? lazy_exp(m->fa[mm]) : 0) +
                                   (cb >= N ? lazy_exp(m->fb[mm]) : 0);
                    a.E[fi(k, r, pat0 + mm)] = Ek;
                };
                if (k == root) {
                    if (threadIdx.x < T) storeE();
                    // Eq. 3 terms: thread -> (pattern mm, states j, j+TPP, ...)
                    constexpr int TPP = NTC / T;
                    const int mm = threadIdx.x / TPP, j = threadIdx.x % TPP;
                    double sum = 0.0;
                    if (mm < T)
                        for (int kk = j; kk < SP; kk += TPP) {
                            const int p = apos<SP>(mm, kk);
                            sum = fma(a.pi[kk], As[p] * Bs[p], sum);
                        }
    #pragma unroll
                    for (int o = 1; o < TPP; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                    if (j == 0 && mm < T) a.Lpart[(size_t)r * a.Cpad + pat0 + mm] = a.cat_w[r] * sum * (scA(mm) * scB(mm));
                } else {
                    double bfr[KT];
                    load_bfrag<SP>(bfr, a.PBpost + ((size_t)k * R + r) * MAT, w, lane);
                    // p = u_a o u_b in place (one A operand for the GEMM), unless
                    // the producer formed it already
                    if (!f.pprod) {
                        for (int i2 = threadIdx.x; i2 < TILE / 2; i2 += NTC) {
                            double2 *pa = reinterpret_cast<double2 *>(As) + i2;
                            const double2 tb = reinterpret_cast<const double2 *>(Bs)[i2];
                            double2 v = *pa;
                            v.x *= tb.x;
                            v.y *= tb.y;
                            *pa = v;
                        }
                        consumer_sync(NTC);
                    }
                    double acc[MTW][2];
                    gemm_tile<SP, MTW>(acc, As + mt0 * KT * 32, bfr, lane);
                    if (tr) tr[4] = gtimer();
                    if (threadIdx.x < T) storeE();
                    double *out = a.u + (((size_t)(k - N) * R + r) * ntiles + tile) * TILE;
                    int *fm = a.fmax + fi(k, r, pat0);
    #pragma unroll
                    for (int ml = 0; ml < MTW; ++ml) {
                        const int mm = (mt0 + ml) * 8 + (lane >> 2), n = w * 8 + 2 * (lane & 3);
                        const double f2 = scA(mm) * scB(mm);
                        const double c0 = acc[ml][0] * f2, c1 = acc[ml][1] * f2;
                        *reinterpret_cast<double2 *>(out + apos<SP>(mm, n)) = make_double2(c0, c1);
                        int fx = max(__double2hiint(c0) >> 20, __double2hiint(c1) >> 20);
                        fx = max(fx, __shfl_xor_sync(0xffffffffu, fx, 1));
                        fx = max(fx, __shfl_xor_sync(0xffffffffu, fx, 2));
                        if ((lane & 3) == 0) atomicMax(fm + mm, fx);
                    }
                }
                fence_proxy_async_global();              // our generic stores -> later TMA reads (other CTAs)
                if (f.pub) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive_u32(pub_u + 8u * s);
                    if (tr) tr[6] = gtimer();
                    continue;
                }
                if (tr) tr[5] = gtimer();
                consumer_sync(NTC);                      // stage consumed, outputs issued
                if (threadIdx.x == 0) {
                    __threadfence();
                    atomicAdd(f.rpost + ci(k, r, tile), 1);
                    mbar_arrive_u32(empty_u + 8u * s);
                    if (tr) tr[6] = gtimer();
                }
                continue;
            }
            // ------------------------------- pre item ------------------------------
            const int cs = m->cs;                        // -1: both children, else the one child of a split item
            auto scQ = [&](int mm) { return k == root ? 1.0 : pow2neg(lazy_exp(m->fq[mm])); };
            auto scC = [&](int c, int mm) {
                return (c ? cb : ca) >= N ? pow2neg(lazy_exp(c ? m->fb[mm] : m->fa[mm])) : 1.0;
            };
            auto Uc = [&](int c) { return c ? Bs : As; };
            // cumulative exponent inside the stored q_c (row mm): q_k's plus the
            // sibling's u exponent, plus the factors applied to this product
            auto q_exp = [&](int c, int node, int mm) {
                const int fs = c ? m->fa[mm] : m->fb[mm], sib = c ? ca : cb;
                const int e = m->Qe[mm] + (c ? m->Ea[mm] : m->Eb[mm]) + (k == root ? 0 : lazy_exp(m->fq[mm])) +
                              (sib >= N ? lazy_exp(fs) : 0);
                a.EQ[fi(node, r, pat0 + mm)] = e;
            };
            // q_c = x_c P_c (Eq. 4) from the x_c tile Xs; rows scaled by the q_k
            // and sibling exponents
            auto q_gemm = [&](int c, const double *Xs) {
                const int node = c ? cb : ca;
                double bq[KT], acc[MTW][2];
                load_bfrag<SP>(bq, a.PBpre + ((size_t)node * R + r) * MAT, w, lane);
                gemm_tile<SP, MTW>(acc, Xs + mt0 * KT * 32, bq, lane);
                double *out = a.q + (((size_t)(node - N) * R + r) * ntiles + tile) * TILE;
                int *qm = a.qmax + fi(node, r, pat0);
                if (a.Y && threadIdx.x < T) q_exp(c, node, threadIdx.x);
    #pragma unroll
                for (int ml = 0; ml < MTW; ++ml) {
                    const int mm = (mt0 + ml) * 8 + (lane >> 2), n = w * 8 + 2 * (lane & 3);
                    const double f2 = scQ(mm) * scC(1 - c, mm);
                    const double c0 = acc[ml][0] * f2, c1 = acc[ml][1] * f2;
                    *reinterpret_cast<double2 *>(out + apos<SP>(mm, n)) = make_double2(c0, c1);
                    int fx = max(__double2hiint(c0) >> 20, __double2hiint(c1) >> 20);
                    fx = max(fx, __shfl_xor_sync(0xffffffffu, fx, 1));
                    fx = max(fx, __shfl_xor_sync(0xffffffffu, fx, 2));
                    if ((lane & 3) == 0) atomicMax(qm + mm, fx);
                }
            };
            auto publish_q = [&](bool pa, bool pb) {
                if (f.pub) {                             // every pre item arrives once
                    fence_proxy_async_global();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_u32(pub_u + 8u * s);
                    return;
                }
                if (!pa && !pb) return;
                fence_proxy_async_global();
                consumer_sync(NTC);
                if (threadIdx.x == 0) {
                    __threadfence();
                    if (pa) atomicAdd(f.rpre + ci(ca, r, tile), 1);
                    if (pb) atomicAdd(f.rpre + ci(cb, r, tile), 1);
                }
            };
            // Eq. 8 terms of child c: num_c = x_c'(Q u_c) (internal child or partial
            // tip: Q u on the tensor path; state tip: the D' row, which carries
            // gamma_r), with x_c at the output positions from xat(p); den = x_c'u_c
            // (the same for both children, q_k o u_a o u_b, Eq. 5).  Tiles are
            // unscaled: the factors cancel in the ratio over categories.
            auto eq8 = [&](int c, bool den, auto xat) {
                const int node = c ? cb : ca;
                const size_t br = (size_t)node * R + r;
                const int kind = (kinds >> (2 * c)) & 3;
                double acc[MTW][2];
                if (node >= N || kind == 2) {
                    double b[KT];
                    load_bfrag<SP>(b, a.QB, w, lane);
                    gemm_tile<SP, MTW>(acc, Uc(c) + mt0 * KT * 32, b, lane);
                } else {
                    const uint8_t *stc = c ? m->sb : m->sa;
    #pragma unroll
                    for (int ml = 0; ml < MTW; ++ml) {
                        const int mm = (mt0 + ml) * 8 + (lane >> 2), n = w * 8 + 2 * (lane & 3);
                        const int sv = stc[mm];
                        if (sv < a.S) {
                            const double2 v = __ldg(reinterpret_cast<const double2 *>(a.DT + br * MAT + (size_t)sv * SP + n));
                            acc[ml][0] = v.x;
                            acc[ml][1] = v.y;
                        } else {
                            acc[ml][0] = acc[ml][1] = 0.0;
                        }
                    }
                }
    #pragma unroll
                for (int ml = 0; ml < MTW; ++ml) {
                    const int mm = (mt0 + ml) * 8 + (lane >> 2), n = w * 8 + 2 * (lane & 3);
                    const int p = apos<SP>(mm, n);
                    const double2 x2 = xat(p);
                    double sn = x2.x * acc[ml][0] + x2.y * acc[ml][1];
                    sn += __shfl_xor_sync(0xffffffffu, sn, 1);
                    sn += __shfl_xor_sync(0xffffffffu, sn, 2);
                    if ((lane & 3) == 0) part[(c * NW + w) * T + mm] = sn;
                    if (den) {
                        const double2 u2 = *reinterpret_cast<const double2 *>(Uc(c) + p);
                        double sd = x2.x * u2.x + x2.y * u2.y;
                        sd += __shfl_xor_sync(0xffffffffu, sd, 1);
                        sd += __shfl_xor_sync(0xffffffffu, sd, 2);
                        if ((lane & 3) == 0) part[(2 * NW + w) * T + mm] = sd;
                    }
                }
            };
            if (cs >= 0) {
                // split item (latency): x_c = q_k o u_sib formed in place over q_k
                // (q_k is not needed again), q_c GEMM and publication first, then
                // child c's Eq. 8 terms from x_c and u_c
                const int c = cs;
                const double *Usib = Uc(1 - c);
                for (int i2 = threadIdx.x; i2 < TILE / 2; i2 += NTC) {
                    double2 *px = reinterpret_cast<double2 *>(Qs) + i2;
                    const double2 us = reinterpret_cast<const double2 *>(Usib)[i2];
                    double2 v = *px;
                    v.x *= us.x;
                    v.y *= us.y;
                    *px = v;
                }
                consumer_sync(NTC);
                if ((c ? cb : ca) >= N) q_gemm(c, Qs);
                if (tr) tr[4] = gtimer();
                publish_q(c == 0 && ca >= N, c == 1 && cb >= N);
                if (tr) tr[5] = gtimer();
                eq8(c, true, [&](int p) { return *reinterpret_cast<const double2 *>(Qs + p); });
            } else {
                // both children: q GEMMs first with x_c = q_k o u_sib formed in the
                // A-fragment loads (q_k, u_a, u_b are all needed again), published
                // before the Eq. 8 terms (measured faster than forming x in place
                // after the Eq. 8 GEMMs: yeast 1.155 -> 1.106 ms, the pre-order
                // chain link is shorter)
    #pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int node = c ? cb : ca;
                    if (node < N) continue;
                    double bq[KT], acc[MTW][2];
                    load_bfrag<SP>(bq, a.PBpre + ((size_t)node * R + r) * MAT, w, lane);
                    const double *Ub = Uc(1 - c);
    #pragma unroll
                    for (int ml = 0; ml < MTW; ++ml) acc[ml][0] = acc[ml][1] = 0.0;
    #pragma unroll
                    for (int kt = 0; kt < KT; ++kt)
    #pragma unroll
                        for (int ml = 0; ml < MTW; ++ml) {
                            const int p = ((mt0 + ml) * KT + kt) * 32 + lane;
                            dmma(acc[ml], Qs[p] * Ub[p], bq[kt]);
                        }
                    double *out = a.q + (((size_t)(node - N) * R + r) * ntiles + tile) * TILE;
                    int *qm = a.qmax + fi(node, r, pat0);
                    if (a.Y && threadIdx.x < T) q_exp(c, node, threadIdx.x);
    #pragma unroll
                    for (int ml = 0; ml < MTW; ++ml) {
                        const int mm = (mt0 + ml) * 8 + (lane >> 2), n = w * 8 + 2 * (lane & 3);
                        const double f2 = scQ(mm) * scC(1 - c, mm);
                        const double c0 = acc[ml][0] * f2, c1 = acc[ml][1] * f2;
                        *reinterpret_cast<double2 *>(out + apos<SP>(mm, n)) = make_double2(c0, c1);
                        int fx = max(__double2hiint(c0) >> 20, __double2hiint(c1) >> 20);
                        fx = max(fx, __shfl_xor_sync(0xffffffffu, fx, 1));
                        fx = max(fx, __shfl_xor_sync(0xffffffffu, fx, 2));
                        if ((lane & 3) == 0) atomicMax(qm + mm, fx);
                    }
                }
                if (tr) tr[4] = gtimer();
                publish_q(ca >= N, cb >= N);
                if (tr) tr[5] = gtimer();
                auto xq = [&](int c) {
                    return [&, c](int p) {
                        const double2 q2 = *reinterpret_cast<const double2 *>(Qs + p);
                        const double2 o2 = *reinterpret_cast<const double2 *>(Uc(1 - c) + p);
                        return make_double2(q2.x * o2.x, q2.y * o2.y);
                    };
                };
                eq8(0, true, xq(0));
                eq8(1, false, xq(1));
            }
            if (f.pub) {                                 // the publisher sums the partials and frees the stage
                __syncwarp();
                if (lane == 0) mbar_arrive_u32(done_u + 8u * s);
                continue;
            }
            consumer_sync(NTC);                          // stage and partials complete
            if (threadIdx.x < T) finish_pre(m, part, threadIdx.x);   // fixed-order sums over the warps
            consumer_sync(NTC);                          // partials read before the next item writes them
            if (threadIdx.x == 0) mbar_arrive_u32(empty_u + 8u * s);
            if (tr) tr[6] = gtimer();
        }
    }

    // ============================ A6 (fused, f.a6cnt) ==========================
    // After its last item every CTA counts itself finished; once all are, the
    // CTAs form [logL, g] (Eq. 3, Eq. 6-8) for rows b = blockIdx.x, +gridDim.x,
    // ... in place of codon_ratio_kernel, with its fixed summation order
    // (patterns strided over the threads, then a fixed tree): the result does
    // not depend on which CTA takes a row.
    if (f.a6cnt) {
        __shared__ double red[32];
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(f.a6cnt, 1);
            wait_count2(f.a6cnt, (int)gridDim.x, a.status);
            __threadfence();
        }
        __syncthreads();
        const int B = 2 * N - 2;
        for (int row = blockIdx.x; row <= B; row += gridDim.x) {
            double acc = 0.0;
            for (int c = threadIdx.x; c < a.C; c += blockDim.x) {
                const double wc = a.pat_w[c];
                if (row < B) {
                    double num, den;
                    ratio_terms(a, row, c, num, den);
                    if (wc != 0.0) acc += wc * (num / den);
                } else {
                    int Em;
                    const double L = root_likelihood(a, c, Em);
                    if (!(L > 0.0) || !isfinite(L)) atomicMin(a.status, c);
                    acc += wc * (log(L) + (double)Em * 0.69314718055994530942);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) red[warp] = acc;
            __syncthreads();
            if (threadIdx.x == 0) {
                double t = 0.0;
                for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) t += red[w2];
                f.out[row < B ? 1 + row : 0] = t;
            }
            __syncthreads();
        }
    }
}

}  // namespace codon
}  // namespace pg
