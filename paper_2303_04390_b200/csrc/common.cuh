// common.cuh -- device helpers shared by the phylograd kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>

#include "schedule.hpp"

namespace pg {

// Masks of coded partial tips on the S = 16 tensor path (n < 0: none).
struct MaskTable {
    int n = 0;
    uint16_t mask[16] = {};
};

// Arguments of one traversal launch (both kernel variants).
struct TravArgs {
    const Op4 *post;            // [N-1] post program (schedule.hpp)
    const Op4 *pre;             // [N-1] pre program
    const void *P;              // Real [B][R][SP][SP]   P[s][t] = Pr(child t | parent s)
    const void *PT;             // Real [B][R][SP][SP]   transposed copy (large-S kernel)
    const void *Q;              // Real [SP][SP]         generator (zero padded)
    const void *QT;             // Real [SP][SP]         transposed generator
    const void *pi;             // Real [SP]             root prior
    const double *cat_w;        // [R]  P(gamma_r)
    const double *cat_g;        // [R]  gamma_r
    const double *pat_w;        // [Cpad] pattern weights, 0 on padding
    const uint8_t *tip_states;  // [N][Cpad], code >= S = missing
    const void *tip_partials;   // Real [N][Cpad][SP] (tips flagged partial)
    void *u;                    // Real [N-2][R][Cpad][SP] branch-top post vectors
    double *grad_part;          // [B][n_tiles] per-tile gradient partial sums
    double *logl_part;          // [n_tiles] per-tile logL partial sums
    int *status;                // first zero-likelihood pattern (INT_MAX = none)
    int N, S, R, Cpad, C, n_tiles, depth, prefetch;
    int prog_smem_off;          // > 0: byte offset of the staged op programs in dynamic smem
    // grouped post-order staging (small-S kernel): per post
    // step a record [op][P_k][P_a][P_b] (A1 writes the matrices) and, per
    // CTA, the step's two tip-code windows; GPOST steps per ring stage, two
    // bulk copies per stage.  null: per-step copies.
    const unsigned char *rec_post;
    const unsigned char *rec_pre;     // per pre step [op][P_a][P_b] (grouped mode)
    const unsigned char *tipstream;   // [CTA][N-1][2][tipw]
    int tipw;
    // A6 fused into the traversal (co-resident grids): finished-CTA counter
    // (reset by A1) and the [logL, g] output; null: reduce_kernel
    int *a6cnt;
    double *out;
    long long *trace;           // PG_TRACE builds only: clock64 samples of CTA 0
};

// ---- optional phase timing (compiled in only with -DPG_TRACE) --------------
#ifdef PG_TRACE
#define PG_TSTAMP(slot, dep)                                                             \
    do {                                                                                 \
        long long _c;                                                                    \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(_c) : "r"(__double2hiint((double)(dep))) : "memory"); \
        if (a.trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0) a.trace[(slot)] = _c;  \
    } while (0)
#else
#define PG_TSTAMP(slot, dep) do { } while (0)
#endif

// ---- cp.async (LDGSTS) ----------------------------------------------------
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// ---- exact power-of-two rescaling (reading R4) --------
// exponent e with m = f * 2^e, f in [0.5, 1); 0 for m == 0.
__device__ __forceinline__ int exponent_of(double m) {
    int e;
    (void)frexp(m, &e);
    return m > 0.0 ? e : 0;
}
__device__ __forceinline__ int exponent_of(float m) {
    int e;
    (void)frexpf(m, &e);
    return m > 0.0f ? e : 0;
}
__device__ __forceinline__ double scale_pow2(double x, int k) { return ldexp(x, k); }
__device__ __forceinline__ float scale_pow2(float x, int k) { return ldexpf(x, k); }


}  // namespace pg

// m8n8k4 f64 MMA statements: plain asm (no side effects beyond the outputs),
// so the compiler may interleave independent products' DMMAs;
// -DPG_MMA_VOLATILE keeps them in program order
#ifdef PG_MMA_VOLATILE
#define PG_MMA_ASM asm volatile
#else
#define PG_MMA_ASM asm
#endif
namespace pg {
// ---- mbarrier + 1-D bulk copy (TMA engine, sm_90+) ------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy; bytes % 16 == 0, both addresses 16-B aligned
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
}  // namespace pg

namespace pg {
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// the same operations on precomputed shared-window addresses (no generic ->
// shared conversion in the loop)
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_u32(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_u32(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
}  // namespace pg
