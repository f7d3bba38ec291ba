// phylograd.cu -- C ABI (include/phylograd.h) and runtime: validation, device
// workspace layout, traversal planning, launch configuration and CUDA-graph
// capture of one evaluation:
//     memset(status) -> pmat_kernel (A1) -> traverse_*_kernel (A2-A5)
//                    -> reduce_kernel (A6)
// A7 (the cross-GPU allreduce) is the caller's, on the same stream, over the
// 2N-1 doubles pg_compute_device leaves in device memory.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/phylograd.h"
#include "aux_kernels.cuh"
#include "common.cuh"
#include "schedule.hpp"
#include "traverse_codon.cuh"
#include "traverse_codon2.cuh"
#include "traverse_big.cuh"
#include "traverse_tc.cuh"
#include "traverse_large.cuh"
#include "traverse_small.cuh"

using pg::Op4;

namespace {

constexpr size_t kAlign = 256;
size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

struct Layout {
    int SP = 0, variant = 0, Cpad = 0, n_tiles = 0, B = 0, tpl = 32, cat_stride = 0;
    bool mma = false;                   // small-S traversal on the FP64 tensor path (SP = 16, R = 1, fp64)
    size_t real = 8;
    size_t off_P, off_PT, off_M0, off_Q, off_QT, off_pi, off_V, off_Vi, off_lam, off_rates, off_cw,
        off_bl, off_patw, off_tips, off_tipp, off_u, off_gpart, off_lpart, off_out, off_status,
        off_post, off_pre, total;
    // codon (variant 2) extras
    size_t off_M0one = 0, off_PBpre = 0, off_DT = 0, off_PONE = 0, off_QB = 0, off_q = 0, off_E = 0, off_child = 0,
           off_levels = 0, off_lev4 = 0, off_EQ = 0, off_Y = 0, off_taskoff = 0, off_tipmode = 0, off_utip = 0, off_tipmask = 0, off_tipmasked = 0, off_VA = 0, off_ViB = 0, off_fmax = 0, off_qmax = 0, off_numden = 0, off_Lpart = 0,
           off_flow = 0, flow_bytes = 0, reset_bytes = 0;
    // time-tree parameterisation: parent/child_a/child_b [3][2N-1], heights, rate scalars, branch sets
    size_t off_tree = 0, off_h = 0, off_rho = 0, off_bset = 0;
};

int padded_states(int S) {
    if (S <= 4) return 4;
    if (S <= 8) return 8;
    if (S <= 16) return 16;
    if (S <= 32) return 32;
    if (S <= 64) return 64;
    if (S <= 128) return 128;          // S = 122: MMM of two codon models (NEXT-2)
    if (S <= 256) return 256;          // S = 256 class (NEXT-2): fp64 only
    return 0;
}

// ints of the flow schedules' completion counters {rpost, rpre}, per
// (internal node, category, tile)
static size_t flow_counter_ints(long long N, int R, int n_tiles) { return (size_t)2 * (N - 1) * R * n_tiles; }

int make_layout(const pg_config *c, Layout *L, std::string *err) {
    if (!c) { if (err) *err = "config is NULL"; return PG_ERR_ARG; }
    if (c->tips < 2 || c->patterns < 1 || c->states < 2 || c->categories < 1) {
        if (err) *err = "need tips >= 2, patterns >= 1, states >= 2, categories >= 1";
        return PG_ERR_ARG;
    }
    if (c->precision != PG_FP64 && c->precision != PG_FP32) {
        if (err) *err = "precision must be PG_FP64 or PG_FP32";
        return PG_ERR_ARG;
    }
    int SP = padded_states(c->states);
    if (!SP) { if (err) *err = "states > 256 are not supported by this build"; return PG_ERR_UNSUPPORTED; }
    // fp64 with S > 16: FP64 tensor-core path, states padded to 64 (codon),
    // 128 (S = 122, two-class codon MMM) or 256 (transpose-free level kernels,
    // traverse_big.cuh); fp32 S > 16: SIMT large-state kernel (S <= 128)
    const bool codon = SP > 16 && c->precision == PG_FP64;
    if (codon) SP = SP <= 64 ? 64 : SP <= 128 ? 128 : 256;
    if (SP == 256 && !codon) { if (err) *err = "states > 128 need PG_FP64"; return PG_ERR_UNSUPPORTED; }
    if (c->states > 254) { if (err) *err = "states > 254"; return PG_ERR_UNSUPPORTED; }
    const int R = c->categories;
    L->SP = SP;
    L->variant = SP <= 16 ? 0 : (codon ? (SP == 256 ? 3 : 2) : 1);
    // fp32, 16 < S <= 64, state tips: tcgen05 (kind::tf32, 3xTF32) level kernels
    // (traverse_tc.cuh); PG_NO_TC=1 keeps the SIMT kernel
    const char *ntc = getenv("PG_NO_TC");
    if (L->variant == 1 && SP <= 64 && c->states > 16 && !(c->flags & PG_FLAG_TIP_PARTIALS) && !(ntc && atoi(ntc))) {
        L->variant = 4;
        L->SP = SP = 64;
    }
    L->real = c->precision == PG_FP64 ? 8 : 4;
    if (L->variant == 0) {
        if (R > (SP == 16 ? 8 : 16)) {
            if (err) *err = "too many rate categories for this state count (max 16; 8 for S > 8)";
            return PG_ERR_UNSUPPORTED;
        }
        int Rp = 1;
        while (Rp < R) Rp <<= 1;
        L->tpl = 32 / (Rp * pg::small_lanes_per_vector(SP, Rp));   // patterns per warp tile (lane = pattern x category x state group)
    } else if (L->variant >= 2) {
        if (R > 16) { if (err) *err = "too many rate categories (max 16)"; return PG_ERR_UNSUPPORTED; }
        L->tpl = L->variant == 4 ? pg::tcp::TM : pg::codon::T;
    } else {
        if (R > (SP == 128 ? 8 : 16)) {
            if (err) *err = "too many rate categories (max 16; 8 for S > 64)";
            return PG_ERR_UNSUPPORTED;
        }
        L->tpl = (L->real == 8) ? pg::LargeCfg<double, 64>::tpl(R) : pg::LargeCfg<float, 64>::tpl(R);
        if (SP == 32) L->tpl = (L->real == 8) ? pg::LargeCfg<double, 32>::tpl(R) : pg::LargeCfg<float, 32>::tpl(R);
        if (SP == 128) L->tpl = (L->real == 8) ? pg::LargeCfg<double, 128>::tpl(R) : pg::LargeCfg<float, 128>::tpl(R);
    }
    const long long N = c->tips, C = c->patterns;
    L->Cpad = (int)((C + L->tpl - 1) / L->tpl * L->tpl);      // whole tiles (32; 128 for variant 4)
    if (L->Cpad % 32) L->Cpad = (L->Cpad + 31) / 32 * 32;
    L->n_tiles = L->Cpad / L->tpl;
    L->B = (int)(2 * N - 2);
    // small-S kernels read P with a padded category stride (SmallCfg::CS); the
    // tensor-core S = 16 variant keeps a three-layout record per branch
    L->mma = L->variant == 0 && pg::small_tc(SP, R, (int)L->real);
    L->cat_stride = L->mma ? (SP == 16 ? pg::MMA_REC / 8 : 2 * pg::MMA4_SLOT / 8 / R)   // per category (x R = record)
                  : L->variant == 4 ? (int)pg::tcp::BREC                                      // 4 TF32 B images
                           : SP * SP + ((L->variant == 0 && R > 1) ? pg::small_cat_pad(L->real, SP) / L->real : 0);
    const size_t mats = (size_t)L->B * R * L->cat_stride * L->real;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t at = o; o = align_up(o + bytes); return at; };
    L->off_P = take(mats);
    // variant 3 keeps ONE matrix per (branch, category), W = P' in off_P
    // (transpose-free, traverse_big.cuh); variants 1-2 keep P' beside it
    L->off_PT = take((L->variant == 1 || L->variant == 2) ? (size_t)L->B * R * SP * SP * L->real : 0);
    if (L->variant >= 2) {
        L->off_PBpre = take(L->variant == 2 ? mats : 0);
        L->off_DT = take(L->variant == 2 ? mats : 0);
        L->off_PONE = take((size_t)L->B * R * SP * 8);
        L->off_QB = take((size_t)SP * SP * 8);      // variant 3: Q row-major
        L->off_VA = take((size_t)SP * SP * 8);      // variant 3: (V^-1)' as A fragments
        L->off_ViB = take((size_t)SP * SP * 8);     // variant 3: V' as B fragments
        L->off_M0one = take((size_t)SP * 8 * 2);    // variant 3: M0 1 and V^-1 1
    }
    L->off_M0 = take((size_t)SP * SP * 8);     // V V^-1 (A1's identity term, host long double)
    L->off_Q = take((size_t)std::max(SP * SP, 32) * L->real);   // (S = 4 tensor-core variant: 32 fragment values)
    L->off_QT = take((size_t)SP * SP * L->real);
    L->off_pi = take((size_t)SP * L->real);
    L->off_V = take((size_t)c->states * c->states * 8);
    L->off_Vi = take((size_t)c->states * c->states * 8);
    L->off_lam = take((size_t)c->states * 8);
    L->off_rates = take((size_t)R * 8);
    L->off_cw = take((size_t)R * 8);
    L->off_bl = take((size_t)L->B * 8);
    L->off_patw = take((size_t)L->Cpad * 8);
    L->off_tips = take((size_t)N * L->Cpad);
    // (variant 3 takes partial tips only as 0/1 masks: no dense copy)
    L->off_tipp = take((c->flags & PG_FLAG_TIP_PARTIALS) && L->variant != 3 ? (size_t)N * L->Cpad * SP * L->real : 0);
    L->off_u = take((size_t)(N - 2) * R * L->Cpad * SP * L->real);
    L->off_gpart = take((size_t)L->B * L->n_tiles * 8);
    L->off_lpart = take((size_t)L->n_tiles * 8);
    L->off_out = take((size_t)(L->B + 1) * 8);
    L->off_status = take(sizeof(int) * 4);
    L->off_post = take((size_t)(N - 1) * sizeof(Op4));
    L->off_pre = take((size_t)(N - 1) * sizeof(Op4));
    L->off_tree = take((size_t)3 * (2 * N - 1) * 4);
    L->off_h = take((size_t)(2 * N - 1) * 8);
    L->off_rho = take((size_t)(2 * N - 2) * 8);
    L->off_bset = take((size_t)(2 * N - 2) * 4);     // zeroed at create: one set (strict clock)
    if (L->variant >= 2) {
        L->off_q = take((size_t)(N - 2) * R * L->Cpad * SP * (L->variant == 4 ? 4 : 8));
        // u = P p of partial tips (formed once per evaluation by codon_tipu_kernel)
        L->off_utip = take((c->flags & PG_FLAG_TIP_PARTIALS) ? (size_t)N * R * L->Cpad * SP * 8 : 0);
        // 0/1 mask partials with <= 4 ones (MMM hidden states): state lists, u by gathers
        L->off_tipmask = take((c->flags & PG_FLAG_TIP_PARTIALS) ? (size_t)N * L->Cpad * 4 : 0);
        L->off_tipmasked = take((size_t)N);
        // exponent arrays and completion counters sized per category: the
        // flow v2 kernel keeps them per (node, category) (its items depend
        // only on their own category); the other schedules use the first
        // [node][Cpad] / [node][chunk] part
        L->off_E = take((size_t)(N - 1) * R * L->Cpad * 4);
        L->off_EQ = take((size_t)(N - 2 > 0 ? N - 2 : 1) * R * L->Cpad * 4);
        L->off_Y = take((size_t)L->B * R * L->Cpad * 4);
        // fmax [N-1], qmax [N-2], then the flow schedule's counters
        // {item counter, rpost [N-1][<= ntiles], rpre [N-1][<= ntiles]}: one memset
        // {item counter, rpost, rpre, A1 done flags [B][R], ratio slice counters [B+1]}
        // + the fused A6's finished-CTA counter
        L->flow_bytes = ((size_t)32 + flow_counter_ints(N, R, L->n_tiles) + (size_t)L->B * R + (L->B + 1) + 32) * 4;
        L->reset_bytes = (size_t)(2 * N - 3) * R * L->Cpad * 4 + L->flow_bytes;
        L->off_fmax = take(L->reset_bytes);
        L->off_qmax = L->off_fmax + (size_t)(N - 1) * R * L->Cpad * 4;
        L->off_flow = L->off_qmax + (size_t)(N - 2) * R * L->Cpad * 4;
        L->off_numden = take((size_t)L->B * R * L->Cpad * 16);
        L->off_Lpart = take((size_t)R * L->Cpad * 8);
        L->off_child = take((size_t)2 * (2 * N - 1) * 4);
        L->off_levels = take((size_t)2 * (N - 1) * 4);
        L->off_lev4 = take((size_t)2 * (N - 1) * 16);
        L->off_taskoff = take((size_t)(2 * (N - 1) + 1) * 4);
        L->off_tipmode = take((size_t)N);
    }
    L->total = o;
    return PG_OK;
}

const char *code_name(int code) {
    switch (code) {
        case PG_OK: return "ok";
        case PG_ERR_ARG: return "invalid argument";
        case PG_ERR_DOMAIN: return "value outside its domain";
        case PG_ERR_TOPOLOGY: return "invalid tree topology";
        case PG_ERR_SEQUENCE: return "inputs not set before compute";
        case PG_ERR_ZERO_LIKELIHOOD: return "zero site likelihood";
        case PG_ERR_CUDA: return "CUDA error";
        case PG_ERR_UNSUPPORTED: return "unsupported configuration";
        case PG_ERR_MEMORY: return "out of memory";
        default: return "unknown error";
    }
}

}  // namespace

struct pg_instance {
    pg_config cfg{};
    Layout L{};
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    char *ws = nullptr;
    bool own_ws = false;
    int sm_count = 148;
    // host-side state
    std::vector<uint8_t> tips_h;        // [N][Cpad]
    std::vector<uint8_t> tip_is_partial, tip_set, tip_masked;
    // S = 16 tensor path: tip partials that are 0/1 masks (e.g. the hidden
    // copies of an observed nucleotide) -- per tip the pattern's mask as bits,
    // empty when the tip's partials are not all masks; mask_mode: every tip
    // is such a tip and there are <= 16 distinct masks (besides all-ones)
    std::vector<std::vector<uint16_t>> tip_mask16;
    bool mask_mode = false;
    pg::MaskTable mask_table{};
    bool have_ops = false, have_eigen = false, have_pi = false, have_rates = false,
         have_cw = false, have_bl = false, have_patw = false;
    pg::Plan plan;
    bool plan_dirty = true, tips_dirty = true, partial_modes_dirty = false;
    double *bl_pinned = nullptr, *out_pinned = nullptr;
    int *status_pinned = nullptr;
    bool bl_host_pending = false;
    double *clock_pinned = nullptr;     // [2N-1] heights then [2N-2] rate scalars
    bool clock_host_pending = false, have_heights = false;
    cudaEvent_t staged_ev = nullptr;    // recorded after the H2D copies that read the pinned staging buffers
    bool staged_pending = false;
    int n_sets = 1;
    // launch configuration
    int prefetch = 4, smem = 0, grid = 0, block = 0, tiles_per_cta = 1, prog_smem_off = 0;
    int flow_tch = 0;                   // codon: tiles per flow item (0 = level-by-level kernels)
    int flow_ver = 2;                   // codon flow kernel: 2 = warp-specialised TMA ring (codon_flow2_kernel), 1 = round-1 kernel
    int flow_nst = 2;                   // codon_flow2_kernel ring stages (1: latency, 2: throughput)
    int flow_pdl = 0;                   // A1 -> flow programmatic dependent launch (PG_FLOW_PDL=0/1 overrides)
    int flow_pub = 1;                   // flow v2: publisher warp (PG_FLOW_PUB)
    bool a6_fused = false;              // set per enqueue: the flow kernel also formed [logL, g]
    // small-S grouped post-order staging (library-owned buffers)
    bool grouped = false, tipstream_on = false, tipstream_dirty = true;
    bool small_coresident = false;      // small-S grid fits the GPU at once (fused A6 possible)
    int tipw = 0;
    unsigned char *rec_post = nullptr, *rec_pre = nullptr, *tipstream = nullptr;
    int *post_dst = nullptr;
    std::vector<int32_t> post_dst_h;
    size_t rec_cap = 0, ts_cap = 0, dst_cap = 0;
    int flow_pprod = 0;                 // flow v2: the producer forms p = u_a o u_b (PG_FLOW_PPROD)
    int split_items = 0;                // items of the split schedule (task offsets table)
    int flow_split = 0;                 // codon_flow2_kernel: one pre item per child (PG_FLOW_SPLIT=0/1 overrides)
    int flow_rs = 1;                    // codon_flow2_kernel: rows of a product split over 2x the warps (PG_FLOW_RS)
    pg::codon::TmaMaps tmaps{};         // TMA tensor maps of u, q, utip (codon_flow2_kernel)
    int flow_defer = 0;                 // codon flow: Eq. 8 items after all pre items (PG_FLOW_DEFER)
    int flow_half = 0;                  // codon flow: half-tile post items when tch == 1 (PG_FLOW_HALF)
    unsigned long long *flow_trace = nullptr;   // PG_FLOW_TRACE=<file>: per-item timestamps (diagnostics)
    size_t flow_trace_n = 0;
    cudaGraphExec_t gexec = nullptr;
    double *gexec_out = nullptr;
    bool timing = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    std::string err;
    long long *trace = nullptr;         // PG_TRACE builds: [2(N-1)][8] clock samples

    template <typename T> T *at(size_t off) { return reinterpret_cast<T *>(ws + off); }
    int fail(int code, const std::string &msg) { err = msg; return code; }
    int cuda_fail(cudaError_t e, const char *what) {
        err = std::string(what) + ": " + cudaGetErrorString(e);
        return PG_ERR_CUDA;
    }
};

#define CK(call, what)                                            \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return inst->cuda_fail(_e, what);  \
    } while (0)

// Every entry point that touches the GPU runs on the instance's device and
// restores the caller's current device on return (an instance is
// bound to one device; torch's current device must not change under it).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        int cur = -1;
        if (dev < 0 || cudaGetDevice(&cur) != cudaSuccess || cur == dev) return;
        if (cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    explicit DeviceGuard(const pg_instance *inst) : DeviceGuard(inst ? inst->cfg.device : -1) {}
    ~DeviceGuard() { if (prev >= 0) cudaSetDevice(prev); }
};

// Host staging buffers (bl_pinned, clock_pinned) are read by stream-ordered
// H2D copies that may still be queued when the caller sets new values
// (pg_compute_device returns without synchronising): wait for the copy that
// last read them before overwriting.
static int wait_staging(pg_instance *inst) {
    if (!inst->staged_pending) return PG_OK;
    CK(cudaEventSynchronize(inst->staged_ev), "staging buffer wait");
    inst->staged_pending = false;
    return PG_OK;
}
static int mark_staging(pg_instance *inst) {
    CK(cudaEventRecord(inst->staged_ev, inst->stream), "staging event");
    inst->staged_pending = true;
    return PG_OK;
}
static bool capturing(const pg_instance *inst) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(inst->stream, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone;
}

// Exported functions get C linkage from their declarations in phylograd.h.

int pg_version(void) { return 100; }

const char *pg_strerror(int code) { return code_name(code); }

const char *pg_last_error(const pg_instance *inst) { return inst ? inst->err.c_str() : "NULL instance"; }

int pg_workspace_bytes(const pg_config *cfg, size_t *bytes) {
    Layout L;
    int rc = make_layout(cfg, &L, nullptr);
    if (rc) return rc;
    if (!bytes) return PG_ERR_ARG;
    *bytes = L.total;
    return PG_OK;
}

int pg_plan_check(int32_t tips, const int32_t *ops, int32_t n_ops, int32_t *post_depth, int32_t *pre_depth) {
    pg::Plan p;
    std::string e;
    int rc = pg::build_plan(tips, ops, n_ops, &p, &e);
    if (rc) return rc;
    if (post_depth) *post_depth = p.post_depth;
    if (pre_depth) *pre_depth = p.pre_depth;
    return PG_OK;
}

int pg_create(const pg_config *cfg, void *cuda_stream, void *dev_workspace, size_t workspace_bytes,
              pg_instance **out) {
    if (!out) return PG_ERR_ARG;
    *out = nullptr;
    Layout L;
    std::string err;
    int rc = make_layout(cfg, &L, &err);
    if (rc) return rc;
    pg_instance *inst = new pg_instance();
    inst->cfg = *cfg;
    inst->L = L;
    auto bail = [&](int code) { pg_destroy(inst); return code; };
    DeviceGuard dg(cfg->device);         // restores the caller's current device on return
    int cur = -1;
    cudaError_t e = cudaGetDevice(&cur);
    if (e == cudaSuccess && cur != cfg->device) e = cudaErrorInvalidDevice;
    if (e != cudaSuccess) { inst->cuda_fail(e, "cudaSetDevice"); return bail(PG_ERR_CUDA); }
    int dev_sms = 0;
    if (cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, cfg->device) == cudaSuccess && dev_sms > 0)
        inst->sm_count = dev_sms;
    if (cuda_stream) {
        inst->stream = (cudaStream_t)cuda_stream;
    } else {
        if (cudaStreamCreateWithFlags(&inst->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(PG_ERR_CUDA);
        inst->own_stream = true;
    }
    if (dev_workspace) {
        if (workspace_bytes < L.total || ((uintptr_t)dev_workspace % kAlign) != 0) return bail(PG_ERR_MEMORY);
        inst->ws = (char *)dev_workspace;
    } else {
        if (cudaMalloc((void **)&inst->ws, L.total) != cudaSuccess) return bail(PG_ERR_MEMORY);
        inst->own_ws = true;
    }
    if (cudaMallocHost((void **)&inst->bl_pinned, sizeof(double) * L.B) != cudaSuccess ||
        cudaMallocHost((void **)&inst->out_pinned, sizeof(double) * (L.B + 1)) != cudaSuccess ||
        cudaMallocHost((void **)&inst->status_pinned, sizeof(int) * 4) != cudaSuccess ||
        cudaMallocHost((void **)&inst->clock_pinned, sizeof(double) * (2 * L.B + 1)) != cudaSuccess)
        return bail(PG_ERR_MEMORY);
    if (cudaEventCreateWithFlags(&inst->staged_ev, cudaEventDisableTiming) != cudaSuccess) return bail(PG_ERR_CUDA);
    const int N = cfg->tips;
    inst->tips_h.assign((size_t)N * L.Cpad, (uint8_t)cfg->states);   // all missing
    inst->tip_is_partial.assign(N, 0);
    inst->tip_masked.assign(N, 0);
    inst->tip_set.assign(N, 0);
    // zero padded weights, partials (all-ones for padding is set per tip), Q, pi, matrices
    if (cudaMemsetAsync(inst->ws, 0, L.total, inst->stream) != cudaSuccess) return bail(PG_ERR_CUDA);
    *out = inst;
    return PG_OK;
}

int pg_destroy(pg_instance *inst) {
    DeviceGuard dg(inst);
    if (!inst) return PG_OK;
    if (inst->stream) cudaStreamSynchronize(inst->stream);
    if (inst->gexec) cudaGraphExecDestroy(inst->gexec);
    for (auto &e : inst->ev) if (e) cudaEventDestroy(e);
    if (inst->staged_ev) cudaEventDestroy(inst->staged_ev);
    if (inst->own_ws && inst->ws) cudaFree(inst->ws);
    if (inst->flow_trace) cudaFree(inst->flow_trace);
    if (inst->rec_post) cudaFree(inst->rec_post);
    if (inst->tipstream) cudaFree(inst->tipstream);
    if (inst->post_dst) cudaFree(inst->post_dst);
    if (inst->bl_pinned) cudaFreeHost(inst->bl_pinned);
    if (inst->clock_pinned) cudaFreeHost(inst->clock_pinned);
    if (inst->out_pinned) cudaFreeHost(inst->out_pinned);
    if (inst->status_pinned) cudaFreeHost(inst->status_pinned);
    if (inst->own_stream && inst->stream) cudaStreamDestroy(inst->stream);
    delete inst;
    return PG_OK;
}

static bool finite_all(const double *p, size_t n) {
    for (size_t i = 0; i < n; ++i) if (!std::isfinite(p[i])) return false;
    return true;
}

// upload `n` doubles to a double buffer (synchronous w.r.t. the host copy)
static int upload_doubles(pg_instance *inst, size_t off, const double *src, size_t n) {
    CK(cudaMemcpyAsync(inst->ws + off, src, n * sizeof(double), cudaMemcpyHostToDevice, inst->stream), "upload");
    CK(cudaStreamSynchronize(inst->stream), "upload sync");
    return PG_OK;
}
// upload `n` doubles converted to the compute precision, zero padded to n_pad
static int upload_real(pg_instance *inst, size_t off, const std::vector<double> &v) {
    if (inst->L.real == 8) {
        CK(cudaMemcpyAsync(inst->ws + off, v.data(), v.size() * 8, cudaMemcpyHostToDevice, inst->stream), "upload");
    } else {
        std::vector<float> f(v.begin(), v.end());
        CK(cudaMemcpyAsync(inst->ws + off, f.data(), f.size() * 4, cudaMemcpyHostToDevice, inst->stream), "upload");
    }
    CK(cudaStreamSynchronize(inst->stream), "upload sync");
    return PG_OK;
}

int pg_set_tip_states(pg_instance *inst, int32_t tip, const int32_t *states) {
    if (!inst) return PG_ERR_ARG;
    const pg_config &c = inst->cfg;
    if (tip < 0 || tip >= c.tips || !states) return inst->fail(PG_ERR_ARG, "tip index out of range or NULL states");
    for (int i = 0; i < c.patterns; ++i)
        if (states[i] < 0 || states[i] > c.states)
            return inst->fail(PG_ERR_ARG, "tip state outside 0..S (S = missing) at pattern " + std::to_string(i));
    uint8_t *row = inst->tips_h.data() + (size_t)tip * inst->L.Cpad;
    for (int i = 0; i < c.patterns; ++i) row[i] = (uint8_t)states[i];
    if (inst->tip_is_partial[tip]) { inst->tip_is_partial[tip] = 0; inst->partial_modes_dirty = true; }
    inst->tip_set[tip] = 1;
    inst->tips_dirty = true;
    return PG_OK;
}

int pg_set_tip_partials(pg_instance *inst, int32_t tip, const double *partials) {
    DeviceGuard dg(inst);
    if (!inst) return PG_ERR_ARG;
    const pg_config &c = inst->cfg;
    if (!(c.flags & PG_FLAG_TIP_PARTIALS))
        return inst->fail(PG_ERR_UNSUPPORTED, "instance created without PG_FLAG_TIP_PARTIALS");
    if (tip < 0 || tip >= c.tips || !partials) return inst->fail(PG_ERR_ARG, "tip index out of range or NULL");
    const int S = c.states, SP = inst->L.SP, Cp = inst->L.Cpad;
    for (size_t i = 0; i < (size_t)c.patterns * S; ++i)
        if (!(partials[i] >= 0.0) || !std::isfinite(partials[i]))
            return inst->fail(PG_ERR_DOMAIN, "tip partials must be finite and >= 0");
    std::vector<double> v(inst->L.variant == 3 ? 0 : (size_t)Cp * SP, 0.0);
    const int KT = SP / 4;
    for (int p = 0; p < (inst->L.variant == 3 ? 0 : Cp); ++p)
        for (int s = 0; s < S; ++s) {
            const double x = p < c.patterns ? partials[(size_t)p * S + s] : 1.0;
            if (inst->L.variant == 2) {      // 32-pattern tiles in A-fragment order (codon_tipu_kernel)
                const int m = p & 31;
                v[(size_t)(p >> 5) * 32 * SP + ((((m >> 3) * KT + (s >> 2)) << 5) + ((m & 7) << 2) + (s & 3))] = x;
            } else {
                v[(size_t)p * SP + s] = x;
            }
        }
    int rc = inst->L.variant == 3 ? PG_OK : upload_real(inst, inst->L.off_tipp + (size_t)tip * Cp * SP * inst->L.real, v);
    if (rc) return rc;
    if (inst->L.variant == 0 && inst->L.mma && S <= 16) {
        std::vector<uint16_t> mk((size_t)c.patterns);
        bool ok = true;
        for (int p = 0; p < c.patterns && ok; ++p) {
            uint16_t b = 0;
            for (int s2 = 0; s2 < S && ok; ++s2) {
                const double x = partials[(size_t)p * S + s2];
                if (x == 1.0) b |= (uint16_t)(1u << s2);
                else if (x != 0.0) ok = false;
            }
            if (b == 0) ok = false;
            mk[p] = b;
        }
        if (inst->tip_mask16.size() != (size_t)c.tips) inst->tip_mask16.resize(c.tips);
        inst->tip_mask16[tip] = ok ? std::move(mk) : std::vector<uint16_t>();
        inst->partial_modes_dirty = true;
    }
    if (inst->L.variant >= 2) {
        // a 0/1 mask with 1..4 ones per pattern (e.g. the hidden copies of an
        // observed state): keep the state list so u = P p is a sum of <= 4
        // columns of P instead of a GEMM (codon_tipu_kernel)
        std::vector<uint8_t> idx((size_t)Cp * 4, 255);
        bool masked = true;
        for (int p = 0; p < c.patterns && masked; ++p) {
            int n = 0;
            for (int s = 0; s < S && masked; ++s) {
                const double x = partials[(size_t)p * S + s];
                if (x == 1.0) {
                    if (n == 4) masked = false;
                    else idx[(size_t)p * 4 + n++] = (uint8_t)s;
                } else if (x != 0.0) {
                    masked = false;
                }
            }
            if (n == 0) masked = false;
        }
        for (int p = c.patterns; p < Cp; ++p) idx[(size_t)p * 4] = 0;      // padding: weight 0, any finite u
        if (masked) {
            CK(cudaMemcpyAsync(inst->ws + inst->L.off_tipmask + (size_t)tip * Cp * 4, idx.data(), idx.size(),
                               cudaMemcpyHostToDevice, inst->stream), "tip mask upload");
            CK(cudaStreamSynchronize(inst->stream), "tip mask sync");
        }
        if (!masked && inst->L.variant == 3)
            return inst->fail(PG_ERR_UNSUPPORTED, "S > 128: tip partials must be 0/1 masks with 1..4 ones per pattern");
        if (inst->tip_masked[tip] != (uint8_t)masked) {
            inst->tip_masked[tip] = (uint8_t)masked;
            inst->partial_modes_dirty = true;
        }
    }
    if (!inst->tip_is_partial[tip]) { inst->tip_is_partial[tip] = 1; inst->partial_modes_dirty = true; }
    inst->tip_set[tip] = 1;
    return PG_OK;
}

int pg_set_pattern_weights(pg_instance *inst, const double *w) {
    DeviceGuard dg(inst);
    if (!inst || !w) return PG_ERR_ARG;
    const int C = inst->cfg.patterns;
    for (int i = 0; i < C; ++i)
        if (!(w[i] >= 0.0) || !std::isfinite(w[i])) return inst->fail(PG_ERR_DOMAIN, "pattern weights must be finite and >= 0");
    std::vector<double> v(inst->L.Cpad, 0.0);
    std::copy(w, w + C, v.begin());
    int rc = upload_doubles(inst, inst->L.off_patw, v.data(), v.size());
    if (rc) return rc;
    inst->have_patw = true;
    return PG_OK;
}

int pg_set_state_frequencies(pg_instance *inst, const double *pi) {
    DeviceGuard dg(inst);
    if (!inst || !pi) return PG_ERR_ARG;
    const int S = inst->cfg.states, SP = inst->L.SP;
    for (int s = 0; s < S; ++s)
        if (!(pi[s] >= 0.0) || !std::isfinite(pi[s])) return inst->fail(PG_ERR_DOMAIN, "pi must be finite and >= 0");
    std::vector<double> v(SP, 0.0);
    std::copy(pi, pi + S, v.begin());
    int rc = upload_real(inst, inst->L.off_pi, v);
    if (rc) return rc;
    inst->have_pi = true;
    return PG_OK;
}

int pg_set_eigen(pg_instance *inst, const double *evec, const double *ievec, const double *eval) {
    DeviceGuard dg(inst);
    if (!inst || !evec || !ievec || !eval) return PG_ERR_ARG;
    const int S = inst->cfg.states, SP = inst->L.SP;
    if (!finite_all(evec, (size_t)S * S) || !finite_all(ievec, (size_t)S * S) || !finite_all(eval, S))
        return inst->fail(PG_ERR_ARG, "eigensystem must be finite");
    int rc;
    if ((rc = upload_doubles(inst, inst->L.off_V, evec, (size_t)S * S))) return rc;
    if ((rc = upload_doubles(inst, inst->L.off_Vi, ievec, (size_t)S * S))) return rc;
    if ((rc = upload_doubles(inst, inst->L.off_lam, eval, S))) return rc;
    // Q = V diag(lambda) V^{-1} and M0 = V V^{-1} (host, long double sums,
    // rounded once), padded; and Q'.  A1 evaluates Eq. 1 as
    //   P = V diag(e) V^-1 = M0 + V diag(e - 1) V^-1,   e - 1 = expm1(gamma b lambda),
    //   D = gamma V diag(lambda e) V^-1 = gamma (Q + V diag(lambda (e - 1)) V^-1):
    // identical in exact arithmetic, but the summed terms are smaller by |gamma
    // b lambda| on short branches, so the cancellation that forms P's tiny
    // entries (multi-nucleotide codon changes) loses far less (R15b)
    std::vector<double> Q((size_t)SP * SP, 0.0), QT((size_t)SP * SP, 0.0), M0((size_t)SP * SP, 0.0);
    for (int s = 0; s < S; ++s)
        for (int t = 0; t < S; ++t) {
            long double acc = 0.0L, acc0 = 0.0L;
            for (int k = 0; k < S; ++k) {
                const long double vv = (long double)evec[s * S + k] * (long double)ievec[k * S + t];
                acc += vv * (long double)eval[k];
                acc0 += vv;
            }
            Q[(size_t)s * SP + t] = (double)acc;
            QT[(size_t)t * SP + s] = (double)acc;
            M0[(size_t)s * SP + t] = (double)acc0;
        }
    if ((rc = upload_doubles(inst, inst->L.off_M0, M0.data(), M0.size()))) return rc;
    if (inst->L.mma && SP == 4) {       // Q as the B operand of Q u (S = 4 variant: Q[n/2][k])
        std::vector<double> QB(32, 0.0);
        for (int l = 0; l < 32; ++l) QB[l] = Q[(size_t)((l >> 2) >> 1) * SP + (l & 3)];
        if ((rc = upload_real(inst, inst->L.off_Q, QB))) return rc;
    } else if (inst->L.mma) {           // Q as the B operand of Q u (S = 16 variant fragment order)
        std::vector<double> QB((size_t)SP * SP, 0.0);
        for (int idx = 0; idx < 256; ++idx) {
            const int f = idx >> 5, l = idx & 31, k = 4 * (f >> 1) + (l & 3), n = 8 * (f & 1) + (l >> 2);
            QB[idx] = Q[(size_t)pg::mma_sigma(n) * SP + k];
        }
        if ((rc = upload_real(inst, inst->L.off_Q, QB))) return rc;
    } else if ((rc = upload_real(inst, inst->L.off_Q, Q))) {
        return rc;
    }
    if ((rc = upload_real(inst, inst->L.off_QT, QT))) return rc;
    if (inst->L.variant == 4) {      // traverse_tc.cuh: Q' as the TF32 hi/lo B images of y = x Q
        std::vector<float> BQ(2 * (size_t)SP * SP, 0.f);
        for (int n = 0; n < SP; ++n)
            for (int kk = 0; kk < SP; ++kk) {
                const float v = (float)Q[(size_t)kk * SP + n], h = pg::tc::tf32_hi(v);   // image (n, k) = Q[k][n]
                const uint32_t off = pg::tc::kmajor_off(n, kk, SP) / 4;
                BQ[off] = h;
                BQ[(size_t)SP * SP + off] = v - h;
            }
        CK(cudaMemcpyAsync(inst->ws + inst->L.off_QB, BQ.data(), BQ.size() * 4, cudaMemcpyHostToDevice, inst->stream),
           "BQ upload");
        CK(cudaStreamSynchronize(inst->stream), "BQ sync");
    }
    if (inst->L.variant == 3) {      // traverse_big.cuh: Q row-major; A1 operands in fragment order
        const int KT = SP / 4;
        std::vector<double> ViTA((size_t)SP * SP, 0.0), VTB((size_t)SP * SP, 0.0), ones(2 * (size_t)SP, 0.0);
        for (int idx = 0; idx < SP * SP; ++idx) {
            const int lane = idx & 31, kt = (idx >> 5) & (KT - 1), mt = idx / (32 * KT);
            const int t = mt * 8 + (lane >> 2), k = kt * 4 + (lane & 3);          // A[t][k] = V^-1[k][t]
            ViTA[idx] = (t < S && k < S) ? ievec[(size_t)k * S + t] : 0.0;
            const int sn = mt * 8 + (lane >> 2);                                  // B[k][s] = V[s][k] (nt = mt)
            VTB[idx] = (sn < S && k < S) ? evec[(size_t)sn * S + k] : 0.0;
        }
        for (int r0 = 0; r0 < S; ++r0) {
            long double a = 0.0L, b = 0.0L;
            for (int t = 0; t < S; ++t) { a += M0[(size_t)r0 * SP + t]; b += ievec[(size_t)r0 * S + t]; }
            ones[r0] = (double)a;            // M0 1
            ones[SP + r0] = (double)b;       // V^-1 1
        }
        if ((rc = upload_doubles(inst, inst->L.off_QB, Q.data(), Q.size()))) return rc;
        if ((rc = upload_doubles(inst, inst->L.off_VA, ViTA.data(), ViTA.size()))) return rc;
        if ((rc = upload_doubles(inst, inst->L.off_ViB, VTB.data(), VTB.size()))) return rc;
        if ((rc = upload_doubles(inst, inst->L.off_M0one, ones.data(), ones.size()))) return rc;
    }
    if (inst->L.variant == 2 || inst->L.variant == 4) {      // (variant 4: V, V^-1 fragments for A1)
        std::vector<double> QB((size_t)SP * SP);
        const int KT = SP / 4;           // B fragments: [nt SP/8][kt SP/4][lane 32]
        for (int idx = 0; idx < SP * SP; ++idx) {
            const int lane = idx & 31, kt = (idx >> 5) & (KT - 1), nt = idx / (32 * KT);
            QB[idx] = Q[(size_t)(nt * 8 + (lane >> 2)) * SP + kt * 4 + (lane & 3)];
        }
        if (inst->L.variant == 2 && (rc = upload_doubles(inst, inst->L.off_QB, QB.data(), QB.size()))) return rc;
        // V as A fragments (element (m,k) at apos(m,k), 64 rows) and V^{-1} as B fragments
        std::vector<double> VA((size_t)SP * SP, 0.0), ViB((size_t)SP * SP, 0.0);
        for (int m = 0; m < S; ++m)
            for (int k = 0; k < S; ++k) {
                const int pos = (((m >> 3) * KT + (k >> 2)) << 5) + ((m & 7) << 2) + (k & 3);
                VA[pos] = evec[m * S + k];
            }
        for (int idx = 0; idx < SP * SP; ++idx) {
            const int lane = idx & 31, kt = (idx >> 5) & (KT - 1), nt = idx / (32 * KT);
            const int kk = kt * 4 + (lane & 3), nn = nt * 8 + (lane >> 2);
            ViB[idx] = (kk < S && nn < S) ? ievec[kk * S + nn] : 0.0;
        }
        if ((rc = upload_doubles(inst, inst->L.off_VA, VA.data(), VA.size()))) return rc;
        if ((rc = upload_doubles(inst, inst->L.off_ViB, ViB.data(), ViB.size()))) return rc;
    }
    inst->have_eigen = true;
    return PG_OK;
}

int pg_set_category_rates(pg_instance *inst, const double *rates) {
    DeviceGuard dg(inst);
    if (!inst || !rates) return PG_ERR_ARG;
    for (int r = 0; r < inst->cfg.categories; ++r)
        if (!(rates[r] > 0.0) || !std::isfinite(rates[r])) return inst->fail(PG_ERR_DOMAIN, "category rates must be > 0");
    int rc = upload_doubles(inst, inst->L.off_rates, rates, inst->cfg.categories);
    if (rc) return rc;
    inst->have_rates = true;
    return PG_OK;
}

int pg_set_category_weights(pg_instance *inst, const double *w) {
    DeviceGuard dg(inst);
    if (!inst || !w) return PG_ERR_ARG;
    for (int r = 0; r < inst->cfg.categories; ++r)
        if (!(w[r] >= 0.0) || !std::isfinite(w[r])) return inst->fail(PG_ERR_DOMAIN, "category weights must be >= 0");
    int rc = upload_doubles(inst, inst->L.off_cw, w, inst->cfg.categories);
    if (rc) return rc;
    inst->have_cw = true;
    return PG_OK;
}

int pg_set_operations(pg_instance *inst, const int32_t *ops, int32_t n_ops) {
    DeviceGuard dg(inst);
    if (!inst) return PG_ERR_ARG;
    pg::Plan p;
    std::string e;
    int rc = pg::build_plan(inst->cfg.tips, ops, n_ops, &p, &e);
    if (rc) return inst->fail(rc, e);
    inst->plan = std::move(p);
    inst->have_ops = true;
    inst->plan_dirty = true;
    // parent / children of every node for the time-tree parameterisation
    const int N = inst->cfg.tips, nn = 2 * N - 1;
    std::vector<int32_t> tree(3 * (size_t)nn, -1);
    for (int v = N; v < nn; ++v) {
        const int a = inst->plan.child_a[v], b = inst->plan.child_b[v];
        tree[nn + v] = a;
        tree[2 * nn + v] = b;
        tree[a] = v;
        tree[b] = v;
    }
    CK(cudaMemcpyAsync(inst->ws + inst->L.off_tree, tree.data(), tree.size() * 4, cudaMemcpyHostToDevice, inst->stream),
       "tree upload");
    CK(cudaStreamSynchronize(inst->stream), "tree upload sync");
    inst->have_heights = false;
    return PG_OK;
}

// ---- time-tree parameterisation (b_i = rho_i (h_parent(i) - h_i))
static int launch_clock_bl(pg_instance *inst, const double *h_src, const double *rho_src) {
    const Layout &L = inst->L;
    const int N = inst->cfg.tips;
    const int *parent = inst->at<int>(L.off_tree);
    double *h = inst->at<double>(L.off_h), *rho = inst->at<double>(L.off_rho), *bl = inst->at<double>(L.off_bl);
    pg::clock_bl_kernel<<<(2 * N - 1 + 255) / 256, 256, 0, inst->stream>>>(parent, h_src, rho_src, N, h, rho, bl);
    CK(cudaGetLastError(), "clock_bl launch");
    return PG_OK;
}

int pg_set_node_heights(pg_instance *inst, const double *heights, const double *rates) {
    DeviceGuard dg(inst);
    if (!inst || !heights) return PG_ERR_ARG;
    if (!inst->have_ops) return inst->fail(PG_ERR_SEQUENCE, "operations not set (node parents unknown)");
    const int N = inst->cfg.tips, B = inst->L.B;
    if (!finite_all(heights, 2 * N - 1)) return inst->fail(PG_ERR_DOMAIN, "node heights must be finite");
    for (int v = N; v < 2 * N - 1; ++v)
        for (int c : {inst->plan.child_a[v], inst->plan.child_b[v]})
            if (!(heights[v] >= heights[c]))
                return inst->fail(PG_ERR_DOMAIN, "node " + std::to_string(c) + " is above its parent " + std::to_string(v));
    if (rates)
        for (int i = 0; i < B; ++i)
            if (!(rates[i] >= 0.0) || !std::isfinite(rates[i]))
                return inst->fail(PG_ERR_DOMAIN, "rate scalar " + std::to_string(i) + " is negative or not finite");
    int rc = wait_staging(inst);
    if (rc) return rc;
    std::memcpy(inst->clock_pinned, heights, sizeof(double) * (2 * N - 1));
    for (int i = 0; i < B; ++i) inst->clock_pinned[2 * N - 1 + i] = rates ? rates[i] : 1.0;
    inst->clock_host_pending = true;
    inst->bl_host_pending = false;
    inst->have_bl = inst->have_heights = true;
    return PG_OK;
}

int pg_set_node_heights_device(pg_instance *inst, const double *d_heights, const double *d_rates) {
    DeviceGuard dg(inst);
    if (!inst || !d_heights) return PG_ERR_ARG;
    if (!inst->have_ops) return inst->fail(PG_ERR_SEQUENCE, "operations not set (node parents unknown)");
    int rc = launch_clock_bl(inst, d_heights, d_rates);
    if (rc) return rc;
    inst->clock_host_pending = inst->bl_host_pending = false;
    inst->have_bl = inst->have_heights = true;
    return PG_OK;
}

// host heights/rates staged by pg_set_node_heights -> device, then b (stream-ordered)
static int flush_clock_host(pg_instance *inst) {
    if (!inst->clock_host_pending) return PG_OK;
    const Layout &L = inst->L;
    const int N = inst->cfg.tips;
    CK(cudaMemcpyAsync(inst->ws + L.off_h, inst->clock_pinned, sizeof(double) * (2 * N - 1), cudaMemcpyHostToDevice,
                       inst->stream), "heights H2D");
    CK(cudaMemcpyAsync(inst->ws + L.off_rho, inst->clock_pinned + 2 * N - 1, sizeof(double) * L.B,
                       cudaMemcpyHostToDevice, inst->stream), "rates H2D");
    return launch_clock_bl(inst, inst->at<double>(L.off_h), inst->at<double>(L.off_rho));
}

int pg_set_branch_sets(pg_instance *inst, const int32_t *set_of_branch, int32_t n_sets) {
    DeviceGuard dg(inst);
    if (!inst || !set_of_branch) return PG_ERR_ARG;
    const int B = inst->L.B;
    if (n_sets < 1 || n_sets > B) return inst->fail(PG_ERR_ARG, "n_sets must be in 1..2N-2");
    for (int i = 0; i < B; ++i)
        if (set_of_branch[i] < -1 || set_of_branch[i] >= n_sets)
            return inst->fail(PG_ERR_ARG, "branch " + std::to_string(i) + ": set id out of range");
    CK(cudaMemcpyAsync(inst->ws + inst->L.off_bset, set_of_branch, sizeof(int32_t) * B, cudaMemcpyHostToDevice,
                       inst->stream), "branch sets upload");
    CK(cudaStreamSynchronize(inst->stream), "branch sets sync");
    inst->n_sets = n_sets;
    return PG_OK;
}

int pg_clock_gradient_device(pg_instance *inst, const double *d_out, double *d_grad_rates, double *d_grad_heights,
                             double *d_set_sums) {
    DeviceGuard dg(inst);
    if (!inst || !d_out) return PG_ERR_ARG;
    if (!inst->have_heights) return inst->fail(PG_ERR_SEQUENCE, "node heights not set");
    const Layout &L = inst->L;
    const int N = inst->cfg.tips;
    const int *tree = inst->at<int>(L.off_tree);
    const double *h = inst->at<double>(L.off_h), *rho = inst->at<double>(L.off_rho);
    if (d_grad_rates || d_grad_heights) {
        pg::clock_grad_kernel<<<(2 * N - 1 + 255) / 256, 256, 0, inst->stream>>>(
            tree, tree + (2 * N - 1), tree + 2 * (2 * N - 1), h, rho, N, d_out, d_grad_rates, d_grad_heights);
        CK(cudaGetLastError(), "clock_grad launch");
    }
    if (d_set_sums) {
        pg::clock_set_kernel<<<inst->n_sets, 256, 0, inst->stream>>>(tree, h, inst->at<int>(L.off_bset), N, d_out,
                                                                     d_set_sums);
        CK(cudaGetLastError(), "clock_set launch");
    }
    return PG_OK;
}

int pg_set_branch_lengths(pg_instance *inst, const double *b) {
    DeviceGuard dg(inst);
    if (!inst || !b) return PG_ERR_ARG;
    const int B = inst->L.B;
    for (int i = 0; i < B; ++i)
        if (!(b[i] >= 0.0) || !std::isfinite(b[i]))
            return inst->fail(PG_ERR_DOMAIN, "branch length " + std::to_string(i) + " is negative or not finite");
    int rc = wait_staging(inst);
    if (rc) return rc;
    std::memcpy(inst->bl_pinned, b, sizeof(double) * B);
    inst->bl_host_pending = true;
    inst->clock_host_pending = false;
    inst->have_bl = true;
    return PG_OK;
}

int pg_set_branch_lengths_device(pg_instance *inst, const double *d_b) {
    DeviceGuard dg(inst);
    if (!inst || !d_b) return PG_ERR_ARG;
    CK(cudaMemcpyAsync(inst->ws + inst->L.off_bl, d_b, sizeof(double) * inst->L.B, cudaMemcpyDeviceToDevice,
                       inst->stream), "branch lengths D2D");
    inst->bl_host_pending = inst->clock_host_pending = false;
    inst->have_bl = true;
    return PG_OK;
}

// -------------------------------------------------------------------------
// launch configuration
// -------------------------------------------------------------------------

template <typename Real, int SP, int RP, int TC = 0, bool GRP = false>
static void *small_kernel() { return (void *)pg::traverse_small_kernel<Real, SP, RP, TC, GRP>; }
template <typename Real, int SP>
static void *large_kernel() { return (void *)pg::traverse_large_kernel<Real, SP>; }
template <typename Real, int SP>
static void *pmat_fn() { return (void *)pg::pmat_kernel<Real, SP>; }

// kernels and launch geometry of the FP64 tensor-core path for SP = 64 / 128
struct CodonFns {
    void *post4, *post2, *pre, *pmat, *flow, *tipu, *tipmask, *flow2[2];     // flow2[NST - 1]
    int threads, ctas_per_sm, flow2_threads, flow2_ctas[2];
    size_t post_smem, pre_smem, pmat_smem, flow_smem, tipu_smem, flow2_smem[2];
    void *flow2rs;                      // NST = 2 with the rows split over 2x the consumer warps (SP = 64)
    int flow2rs_threads;
};
template <int SP>
static CodonFns codon_fns_t() {
    namespace c = pg::codon;
    return {(void *)c::codon_post_kernel<SP, 4>, (void *)c::codon_post_kernel<SP, 2>, (void *)c::codon_pre_kernel<SP>,
            (void *)c::codon_pmat_kernel<SP>, (void *)c::codon_flow_kernel<SP>,
            (void *)c::codon_tipu_kernel<SP>, (void *)c::codon_tipmask_kernel<SP>,
            {(void *)c::codon_flow2_kernel<SP, 1>, (void *)c::codon_flow2_kernel<SP, 2>},
            c::codon_threads<SP>(), c::codon_ctas_per_sm<SP>(), c::flow2_threads<SP>(),
            {c::flow2_ctas<SP, 1>(), c::flow2_ctas<SP, 2>()},
            c::post_smem<SP>(), c::pre_smem<SP>(), c::pmat_smem<SP>(), c::flow_smem<SP>(), c::tipu_smem<SP>(),
            {c::flow2_smem<SP, 1>(), c::flow2_smem<SP, 2>()},
            SP == 64 ? (void *)c::codon_flow2_kernel<64, 2, 2> : nullptr, c::flow2_threads<SP, 2>()};
}
static CodonFns codon_fns(int SP) { return SP == 128 ? codon_fns_t<128>() : codon_fns_t<64>(); }

static int pad_categories(int R) {
    int p = 1;
    while (p < R) p <<= 1;
    return p;
}

template <typename Real, int SP, bool GRP = false>
static void *small_by_rp(int RP) {
    switch (RP) {
        case 1: return small_kernel<Real, SP, 1, 0, GRP>();
        case 2: return small_kernel<Real, SP, 2, 0, GRP>();
        case 4: return small_kernel<Real, SP, 4, 0, GRP>();
        case 8: return small_kernel<Real, SP, 8, 0, GRP>();
        default: return small_kernel<Real, SP, 16, 0, GRP>();
    }
}

// grouped: the small-S kernel with grouped post-order staging (SP = 4)
static void *traverse_fn(const Layout &L, int R, bool grouped = false) {
    const bool d = L.real == 8;
    const int RP = pad_categories(R);
#ifdef PG_SMALL_MMA4
    if (L.mma) return L.SP == 16 ? small_kernel<double, 16, 1, 1>() : small_kernel<double, 4, 4, 1>();
#else
    if (L.mma) return grouped ? small_kernel<double, 16, 1, 1, true>() : small_kernel<double, 16, 1, 1>();
#endif
    switch (L.SP) {
        case 4:
            if (grouped) return d ? small_by_rp<double, 4, true>(RP) : small_by_rp<float, 4, true>(RP);
            return d ? small_by_rp<double, 4>(RP) : small_by_rp<float, 4>(RP);
        case 8: return d ? small_by_rp<double, 8>(RP) : small_by_rp<float, 8>(RP);
        case 16: return d ? small_by_rp<double, 16>(RP) : small_by_rp<float, 16>(RP);
        case 32: return d ? large_kernel<double, 32>() : large_kernel<float, 32>();
        case 64: return d ? large_kernel<double, 64>() : large_kernel<float, 64>();
        case 128: return d ? large_kernel<double, 128>() : large_kernel<float, 128>();
    }
    return nullptr;
}
static void *pmat_kernel_fn(const Layout &L) {
    const bool d = L.real == 8;
    switch (L.SP) {
        case 4: return d ? pmat_fn<double, 4>() : pmat_fn<float, 4>();
        case 8: return d ? pmat_fn<double, 8>() : pmat_fn<float, 8>();
        case 16: return d ? pmat_fn<double, 16>() : pmat_fn<float, 16>();
        case 32: return d ? pmat_fn<double, 32>() : pmat_fn<float, 32>();
        case 64: return d ? pmat_fn<double, 64>() : pmat_fn<float, 64>();
        case 128: return d ? pmat_fn<double, 128>() : pmat_fn<float, 128>();
    }
    return nullptr;
}

template <typename Real, int SP>
static size_t small_smem_t(int RP, int R, int K, int depth, int tipw) {
    switch (RP) {
        case 1: return pg::SmallCfg<Real, SP, 1>::smem(R, K, depth, tipw);
        case 2: return pg::SmallCfg<Real, SP, 2>::smem(R, K, depth, tipw);
        case 4: return pg::SmallCfg<Real, SP, 4>::smem(R, K, depth, tipw);
        case 8: return pg::SmallCfg<Real, SP, 8>::smem(R, K, depth, tipw);
        default: return pg::SmallCfg<Real, SP, 16>::smem(R, K, depth, tipw);
    }
}
// tipw > 0: grouped post-order staging (its ring may be larger than the
// per-step one)
static size_t small_smem(const Layout &L, int R, int K, int depth, int tipw = 0) {
    const bool d = L.real == 8;
    const int RP = pad_categories(R);
    if (L.mma) return L.SP == 16 ? pg::SmallCfg<double, 16, 1, 1>::smem(R, K, depth) : pg::SmallCfg<double, 4, 4, 1>::smem(R, K, depth);
    switch (L.SP) {
        case 4: return d ? small_smem_t<double, 4>(RP, R, K, depth, tipw) : small_smem_t<float, 4>(RP, R, K, depth, tipw);
        case 8: return d ? small_smem_t<double, 8>(RP, R, K, depth, tipw) : small_smem_t<float, 8>(RP, R, K, depth, tipw);
        default: return d ? small_smem_t<double, 16>(RP, R, K, depth, tipw) : small_smem_t<float, 16>(RP, R, K, depth, tipw);
    }
}
// tip-code window of a CTA of K tiles (bytes, whole 16-B units): the CTA's
// first pattern rounded down to 16 plus K tiles of patterns
static int small_tipw(const Layout &L, int K) { return (15 + K * L.tpl + 15) / 16 * 16; }
static size_t large_smem(const Layout &L, int R, int depth) {
    const size_t nvec = (size_t)L.tpl * R;
    const size_t vb = nvec * L.SP * L.real;
    return (5 + (size_t)depth) * vb + nvec * (4 * 8 + 2 * 4) + (size_t)L.tpl * 16;
}

// TMA tensor maps over the fragment-ordered tile arrays u, q, utip
// ([tiles][TILE] doubles viewed as rows of 256 doubles; one box = one tile)
static int make_tile_maps(pg_instance *inst) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return inst->fail(PG_ERR_CUDA, "cuTensorMapEncodeTiled is not available from the driver");
        encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const Layout &L = inst->L;
    const int N = inst->cfg.tips, R = inst->cfg.categories;
    const cuuint32_t rows = (cuuint32_t)(pg::codon::T * L.SP / 256);
    auto enc = [&](CUtensorMap *m, size_t off, size_t tiles) -> int {
        cuuint64_t dims[2] = {256, (cuuint64_t)std::max<size_t>(tiles, 1) * rows};
        cuuint64_t strides[1] = {256 * 8};
        cuuint32_t box[2] = {256, rows};
        cuuint32_t es[2] = {1, 1};
        CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, inst->ws + off, dims, strides, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return inst->fail(PG_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
        return PG_OK;
    };
    int rc;
    const size_t t_int = (size_t)std::max(N - 2, 0) * R * L.n_tiles;
    if ((rc = enc(&inst->tmaps.u, L.off_u, t_int))) return rc;
    if ((rc = enc(&inst->tmaps.q, L.off_q, t_int))) return rc;
    const bool tp = inst->cfg.flags & PG_FLAG_TIP_PARTIALS;
    return enc(&inst->tmaps.utip, tp ? L.off_utip : L.off_u, tp ? (size_t)N * R * L.n_tiles : t_int);
}

static int configure(pg_instance *inst) {
    const Layout &L = inst->L;
    const int R = inst->cfg.categories;
    const int depth = std::max(inst->plan.post_depth, inst->plan.pre_depth);
    void *fn = traverse_fn(L, R);
    inst->grid = L.n_tiles;
    if (L.variant == 0) {
        // CTA = K tile warps + 1 producer warp; K = tiles / SMs (one wave), at
        // most 9 (launch bounds) and within the shared-memory budget.
        int K = std::max(1, std::min(pg::small_max_consumers(L.SP, pad_categories(R)),
                                     (L.n_tiles + inst->sm_count - 1) / inst->sm_count));
        while (K > 1 && small_smem(L, R, K, depth) > 227 * 1024) --K;
        // fp32 S = 4: three CTAs of K = 3 per SM (three producers) beat one
        // CTA of K = 9 when all tiles still fit in one wave (dengue fp32
        // 1.293 -> 1.268 ms, scripts/gpu_smallk.sh)
        const char *ke = getenv("PG_SMALL_K");                      // experiments (ignored unless > 0)
        if (ke && atoi(ke) > 0)
            K = std::min(K, atoi(ke));
        else if (L.real == 4 && L.SP == 4 && K > 3 && 3 * (small_smem(L, R, 3, depth) + 1024) <= 228 * 1024 &&
                 (L.n_tiles + 2) / 3 <= 3 * inst->sm_count)
            K = 3;
        inst->tiles_per_cta = K;
        inst->block = 32 * (K + 1);
        inst->grid = (L.n_tiles + K - 1) / K;
        inst->prefetch = (L.SP <= 8) ? 4 : 2;
        inst->smem = (int)small_smem(L, R, K, depth);
        if (inst->smem > 227 * 1024) return inst->fail(PG_ERR_UNSUPPORTED, "traversal does not fit in shared memory");
        // grouped post-order staging: state tips only, the
        // SIMT kernel, library-owned memory, and when its ring fits
        {
            bool any_partial = false;
            for (int t = 0; t < inst->cfg.tips; ++t) any_partial |= inst->tip_is_partial[t] != 0;
            const char *ge = getenv("PG_GPOST");
            const int tw = small_tipw(L, K);
            // S = 4, state tips: records + grouped post stages; the S = 16
            // tensor path (MMM, partial tips): records only
            const bool grp4 = !L.mma && L.SP == 4 && !any_partial && small_smem(L, R, K, depth, tw) <= 227 * 1024;
            const bool rec16 = L.mma && L.SP == 16;
            inst->grouped = (grp4 || rec16) && !(ge && atoi(ge) == 0);
            inst->tipstream_on = inst->grouped && grp4;
            if (getenv("PG_DEBUG_PLAN"))
                fprintf(stderr, "[phylograd] small-S: K=%d grid=%d grouped=%d (partial=%d own_ws=%d smem=%zu)\n", K,
                        inst->grid, (int)inst->grouped, (int)any_partial, (int)inst->own_ws,
                        small_smem(L, R, K, depth, tw));
            if (inst->grouped) {
                inst->tipw = inst->tipstream_on ? tw : 0;
                if (inst->tipstream_on) inst->smem = (int)small_smem(L, R, K, depth, tw);
                const int N = inst->cfg.tips, B = L.B;
                const size_t ms = L.mma ? (size_t)pg::MMA_SLOT : (size_t)R * L.cat_stride * L.real;   // one slot
                const size_t recb = 16 + 3 * ms, recpb = 16 + 2 * ms;
                const size_t rec_need = (size_t)(N - 1) * (recb + recpb);
                const size_t ts_need = inst->tipstream_on ? (size_t)inst->grid * (N - 1) * 2 * tw : 1;
                if (inst->rec_cap < rec_need) {
                    if (inst->rec_post) cudaFree(inst->rec_post);
                    CK(cudaMalloc(&inst->rec_post, rec_need), "post records alloc");
                    inst->rec_cap = rec_need;
                }
                if (inst->ts_cap < ts_need) {
                    if (inst->tipstream) cudaFree(inst->tipstream);
                    CK(cudaMalloc(&inst->tipstream, ts_need), "tip stream alloc");
                    inst->ts_cap = ts_need;
                }
                if (inst->dst_cap < (size_t)2 * B) {
                    if (inst->post_dst) cudaFree(inst->post_dst);
                    CK(cudaMalloc(&inst->post_dst, sizeof(int) * 2 * B), "record map alloc");
                    inst->dst_cap = 2 * B;
                }
                inst->rec_pre = inst->rec_post + (size_t)(N - 1) * recb;
                // the records' op words (static per plan) and, per branch, the
                // record slot A1 writes its matrices into
                CK(cudaMemcpy2DAsync(inst->rec_post, recb, inst->plan.post.data(), sizeof(Op4), sizeof(Op4), N - 1,
                                     cudaMemcpyHostToDevice, inst->stream), "record ops upload");
                CK(cudaMemcpy2DAsync(inst->rec_pre, recpb, inst->plan.pre.data(), sizeof(Op4), sizeof(Op4), N - 1,
                                     cudaMemcpyHostToDevice, inst->stream), "record ops upload");
                // [post slot][pre slot] per branch: byte offset (S = 16 tensor
                // path: offset * 4 + which of the branch's three layouts the
                // slot's reader takes, as mat_src in traverse_small.cuh)
                std::vector<int32_t> dst(2 * B, -1);
                const int pbit = pg::kTipPartialBit;
                auto enc = [&](size_t off, int lay) { return L.mma ? (int)(off * 4 + lay) : (int)off; };
                auto tip_lay = [&](int code) { return (code & pbit) ? 0 : 2; };
                for (int m = 0; m < N - 1; ++m) {
                    const Op4 op = inst->plan.post[m];
                    if (op.x != 2 * N - 2) dst[op.x] = enc(m * recb + 16, 0);
                    if (op.y >= 0) dst[op.y & ~pbit] = enc(m * recb + 16 + ms, tip_lay(op.y));
                    if (op.z >= 0) dst[op.z & ~pbit] = enc(m * recb + 16 + 2 * ms, tip_lay(op.z));
                    const Op4 oq = inst->plan.pre[m];
                    const int ny = oq.y & ~pbit, nz = oq.z & ~pbit;
                    dst[B + ny] = enc(m * recpb + 16, ny >= N ? 1 : tip_lay(oq.y));
                    dst[B + nz] = enc(m * recpb + 16 + ms, nz >= N ? 1 : tip_lay(oq.z));
                }
                inst->post_dst_h = dst;
                CK(cudaMemcpyAsync(inst->post_dst, inst->post_dst_h.data(), sizeof(int) * 2 * B, cudaMemcpyHostToDevice,
                                   inst->stream), "record map upload");
                CK(cudaStreamSynchronize(inst->stream), "record upload sync");
                inst->tipstream_dirty = true;
            }
        }
        // stage both op programs in smem when they fit (producer/consumers never read ops from HBM)
        const int prog_bytes = 2 * (inst->cfg.tips - 1) * (int)sizeof(Op4);
        const int off = (inst->smem + 15) / 16 * 16;
        inst->prog_smem_off = 0;
#ifdef PG_NO_PROG_SMEM
        if (false) {
#else
        if (off + prog_bytes <= 227 * 1024) {
#endif
            inst->prog_smem_off = off;
            inst->smem = off + prog_bytes;
        }
    } else if (L.variant == 4) {
        inst->block = pg::tcp::TM;
        inst->prefetch = 0;
        inst->flow_tch = 0;
        inst->smem = (int)pg::tcp::pre_smem();
        CK(cudaFuncSetAttribute((void *)pg::tcp::tc_post_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pg::tcp::post_smem()), "smem attr");
        CK(cudaFuncSetAttribute((void *)pg::tcp::tc_pre_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pg::tcp::pre_smem()), "smem attr");
        CK(cudaFuncSetAttribute((void *)pg::tcp::tc_pmat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pg::tcp::pmat_smem()), "smem attr");
        return PG_OK;
    } else if (L.variant == 3) {
        inst->block = pg::big::NTB;
        inst->prefetch = 0;
        inst->flow_tch = 0;                    // level-by-level launches
        inst->smem = (int)pg::big::pre_smem();
        CK(cudaFuncSetAttribute((void *)pg::big::big_post_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pg::big::post_smem()), "smem attr");
        CK(cudaFuncSetAttribute((void *)pg::big::big_pre_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pg::big::pre_smem()), "smem attr");
        return PG_OK;
    } else if (L.variant == 2) {
        const CodonFns cf = codon_fns(L.SP);
        inst->block = cf.threads;
        inst->prefetch = 0;
        inst->smem = (int)cf.pre_smem;
        CK(cudaFuncSetAttribute(cf.pre, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cf.pre_smem), "smem attr");
        CK(cudaFuncSetAttribute(cf.pmat, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cf.pmat_smem), "smem attr");
        CK(cudaFuncSetAttribute(cf.flow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cf.flow_smem), "smem attr");
        CK(cudaFuncSetAttribute(cf.tipu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cf.tipu_smem), "smem attr");
        // flow schedule (default): chunks of TCH tiles per item, enough items
        // per node that a level of a few nodes still fills the 3 CTAs/SM
        const char *fe = getenv("PG_CODON_FLOW"), *te = getenv("PG_FLOW_TCH");
        inst->flow_ver = (fe && atoi(fe) == 1) ? 1 : 2;
        if (fe && atoi(fe) == 0) {
            inst->flow_tch = 0;
        } else if (inst->flow_ver == 2) {
            // warp-specialised TMA kernel: one tile per item (loads overlap compute)
            inst->flow_tch = 1;
            // ring depth 2 (claim-ahead) measured faster than 1 for every
            // workload, shards included (scripts/gpu_codon3.sh)
            const char *ne = getenv("PG_FLOW_NST"), *pe = getenv("PG_FLOW_PDL");
            inst->flow_nst = (ne && atoi(ne) >= 1 && atoi(ne) <= 2) ? atoi(ne) : 2;
            // PDL: on when a task's items do not fill the grid (latency-bound
            // shards: yeast x8 0.251 -> 0.239 ms); off at full size (1.175 -> 1.203)
            const bool latency = L.n_tiles * R < cf.flow2_ctas[inst->flow_nst - 1] * inst->sm_count;
            inst->flow_pdl = pe ? (atoi(pe) != 0) : latency;
            // one pre item per child in the latency regime (S = 122 x8 shard
            // 0.297 -> 0.206 ms, WNV x8 0.579 -> 0.462 ms; scripts/gpu_codon3.sh)
            const char *se = getenv("PG_FLOW_SPLIT");
            inst->flow_split = se ? (atoi(se) != 0) : latency;
            const char *ppe = getenv("PG_FLOW_PPROD");
            inst->flow_pprod = ppe ? (atoi(ppe) != 0) : 0;
            const char *pbe = getenv("PG_FLOW_PUB");
            inst->flow_pub = pbe ? (atoi(pbe) != 0) : 1;
            const char *re = getenv("PG_FLOW_RS");
            inst->flow_rs = (L.SP == 64 && inst->flow_nst == 2 && re && atoi(re) == 2) ? 2 : 1;
            if (cf.flow2rs)
                CK(cudaFuncSetAttribute(cf.flow2rs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cf.flow2_smem[1]),
                   "smem attr");
            for (int v = 0; v < 2; ++v)
                CK(cudaFuncSetAttribute(cf.flow2[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cf.flow2_smem[v]),
                   "smem attr");
            int rc = make_tile_maps(inst);
            if (rc) return rc;
        } else if (te && atoi(te) > 0) {
            inst->flow_tch = std::min(atoi(te), L.n_tiles);
        } else {
            // measured (profiles/r01/flow_sweep.jsonl): 2 tiles per item once a
            // node alone fills the CTA slots (WNV 2.47 -> 2.38 ms), else 1
            // (8-way shards: yeast 0.288 -> 0.261 ms, WNV 0.714 -> 0.702 ms)
            const int slots = cf.ctas_per_sm * inst->sm_count;
            inst->flow_tch = L.n_tiles * R >= slots ? 2 : 1;
        }
        if (inst->flow_tch == 0) {
            // level-by-level kernels: post levels stage their node table (16 B
            // per node) after the ring; size the attribute for the widest level
            const auto &po = inst->plan.post_off;
            int widest = 1;
            for (size_t i = 0; i + 1 < po.size(); ++i) widest = std::max(widest, po[i + 1] - po[i]);
            const size_t need = cf.post_smem + 16 * (size_t)widest;
            if (need > 227 * 1024)
                return inst->fail(PG_ERR_UNSUPPORTED, "a post-order level of " + std::to_string(widest) +
                                                          " nodes does not fit the level kernel's shared memory; "
                                                          "use the flow schedule (PG_CODON_FLOW unset)");
            for (void *fn : {cf.post4, cf.post2})
                CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need), "smem attr");
        }
        const char *de = getenv("PG_FLOW_DEFER");
        inst->flow_defer = de ? (atoi(de) != 0) : 0;
        const char *he = getenv("PG_FLOW_HALF");
        inst->flow_half = he ? (atoi(he) != 0) : 0;
        if (getenv("PG_FLOW_TRACE") && inst->flow_tch > 0) {    // diagnostics buffer (allocated before capture)
            const size_t items = 2 * inst->plan.level_nodes.size() * (size_t)R *     // x2: split pre items
                                 ((L.n_tiles + inst->flow_tch - 1) / inst->flow_tch);
            if (inst->flow_trace) cudaFree(inst->flow_trace);
            CK(cudaMalloc(&inst->flow_trace, sizeof(unsigned long long) * pg::codon::TRW * items), "trace alloc");
            CK(cudaMemset(inst->flow_trace, 0, sizeof(unsigned long long) * pg::codon::TRW * items), "trace clear");
            inst->flow_trace_n = items;
        }
        return PG_OK;
    } else {
        inst->block = L.tpl * R * (L.SP / 4);
        inst->prefetch = 0;
        inst->smem = (int)large_smem(L, R, depth);
        if (inst->smem > 227 * 1024) return inst->fail(PG_ERR_UNSUPPORTED, "traversal does not fit in shared memory");
    }
    if (L.variant == 0) fn = traverse_fn(L, R, inst->grouped);
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, inst->smem), "smem attr");
    if (L.variant == 0) {
        // A6 can be fused into the traversal only when the whole grid is
        // co-resident (its CTAs wait for each other at the end)
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, inst->block, inst->smem), "occupancy");
        inst->small_coresident = per_sm > 0 && inst->grid <= per_sm * inst->sm_count;
    }
    return PG_OK;
}

// S = 16 tensor path: when every tip's partials are 0/1 masks drawn from at
// most 16 distinct masks (besides all-ones), the tips become coded tips:
// code = mask index (all-ones: 16, missing), and A1 writes the column sums
// sum_{t in mask m} P[s][t] where the row-major layout keeps its columns --
// a tip's u = P p is then a gather (as for observed states) instead of a
// product, and the traversal copies one code byte per pattern instead of the
// partial vector
static void decide_mask_mode(pg_instance *inst) {
    const pg_config &c = inst->cfg;
    inst->mask_mode = false;
    if (!(inst->L.variant == 0 && inst->L.mma) || inst->tip_mask16.size() != (size_t)c.tips) return;
    if (getenv("PG_NO_MASK_TIPS")) return;
    const uint16_t all = (uint16_t)((1u << c.states) - 1u);
    pg::MaskTable mt{};
    std::vector<uint8_t> codes((size_t)c.tips * inst->L.Cpad, 16);
    for (int t = 0; t < c.tips; ++t) {
        if (!inst->tip_is_partial[t] || inst->tip_mask16[t].size() != (size_t)c.patterns) return;
        for (int p = 0; p < c.patterns; ++p) {
            const uint16_t b = inst->tip_mask16[t][p];
            int code = 16;
            if (b != all) {
                code = -1;
                for (int m = 0; m < mt.n; ++m)
                    if (mt.mask[m] == b) code = m;
                if (code < 0) {
                    if (mt.n == 16) return;          // too many distinct masks
                    mt.mask[mt.n] = b;
                    code = mt.n++;
                }
            }
            codes[(size_t)t * inst->L.Cpad + p] = (uint8_t)code;
        }
    }
    inst->mask_mode = true;
    inst->mask_table = mt;
    inst->tips_h = std::move(codes);
    inst->tips_dirty = true;
}

static int refresh_plan(pg_instance *inst) {
    if (!inst->plan_dirty && !inst->partial_modes_dirty) return PG_OK;
    decide_mask_mode(inst);
    if (inst->mask_mode) {
        // coded tips: no partial-tip bit in the programs
        const std::vector<uint8_t> none(inst->cfg.tips, 0);
        pg::encode_tip_modes(&inst->plan, none);
    } else {
        pg::encode_tip_modes(&inst->plan, inst->tip_is_partial);
    }
    const int N = inst->cfg.tips;
    CK(cudaMemcpyAsync(inst->ws + inst->L.off_post, inst->plan.post.data(), sizeof(Op4) * (N - 1),
                       cudaMemcpyHostToDevice, inst->stream), "plan upload");
    CK(cudaMemcpyAsync(inst->ws + inst->L.off_pre, inst->plan.pre.data(), sizeof(Op4) * (N - 1),
                       cudaMemcpyHostToDevice, inst->stream), "plan upload");
    if (inst->L.variant >= 2) {
        std::vector<int32_t> ch(2 * (2 * N - 1));
        for (int v = 0; v < 2 * N - 1; ++v) { ch[v] = inst->plan.child_a[v]; ch[2 * N - 1 + v] = inst->plan.child_b[v]; }
        CK(cudaMemcpyAsync(inst->ws + inst->L.off_child, ch.data(), ch.size() * 4, cudaMemcpyHostToDevice, inst->stream),
           "children upload");
        CK(cudaMemcpyAsync(inst->ws + inst->L.off_levels, inst->plan.level_nodes.data(), inst->plan.level_nodes.size() * 4,
                           cudaMemcpyHostToDevice, inst->stream), "levels upload");
        CK(cudaMemcpyAsync(inst->ws + inst->L.off_tipmode, inst->tip_is_partial.data(), N, cudaMemcpyHostToDevice,
                           inst->stream), "tip modes upload");
        CK(cudaMemcpyAsync(inst->ws + inst->L.off_tipmasked, inst->tip_masked.data(), N, cudaMemcpyHostToDevice,
                           inst->stream), "tip mask modes upload");
        // per level entry: {node, child a, child b, kinds}; kind 0 internal, 1 tip states, 2 tip partials
        auto kind = [&](int c) { return c >= N ? 0 : (inst->tip_is_partial[c] ? 2 : 1); };
        std::vector<int32_t> l4(4 * inst->plan.level_nodes.size());
        for (size_t i = 0; i < inst->plan.level_nodes.size(); ++i) {
            const int k = inst->plan.level_nodes[i], ca = inst->plan.child_a[k], cb = inst->plan.child_b[k];
            l4[4 * i] = k;
            l4[4 * i + 1] = ca;
            l4[4 * i + 2] = cb;
            l4[4 * i + 3] = kind(ca) | (kind(cb) << 2);
        }
        CK(cudaMemcpyAsync(inst->ws + inst->L.off_lev4, l4.data(), l4.size() * 4, cudaMemcpyHostToDevice, inst->stream),
           "level table upload");
        // flow v2 split schedule: first item of every task.  A pre task is
        // split into one item group per child only when BOTH children are
        // internal (two q GEMMs to run in parallel); a parent with a tip child
        // has at most one q GEMM, and a tip child's Eq. 8 terms are a row
        // gather, too little work for an item of its own
        const int per = inst->cfg.categories * inst->L.n_tiles;
        std::vector<int32_t> toff(inst->plan.level_nodes.size() + 1, 0);
        const int npost_tasks = inst->plan.post_off.back();
        for (size_t i = 0; i < inst->plan.level_nodes.size(); ++i) {
            const bool two = (int)i >= npost_tasks && l4[4 * i + 1] >= N && l4[4 * i + 2] >= N;
            toff[i + 1] = toff[i] + (two ? 2 : 1) * per;
        }
        inst->split_items = toff.back();
        CK(cudaMemcpyAsync(inst->ws + inst->L.off_taskoff, toff.data(), toff.size() * 4, cudaMemcpyHostToDevice,
                           inst->stream), "task offsets upload");
    }
    CK(cudaStreamSynchronize(inst->stream), "plan upload sync");
    int rc = configure(inst);
    if (rc) return rc;
    inst->plan_dirty = inst->partial_modes_dirty = false;
    if (inst->gexec) { cudaGraphExecDestroy(inst->gexec); inst->gexec = nullptr; }
    return PG_OK;
}

static pg::TravArgs trav_args(pg_instance *inst) {
    const Layout &L = inst->L;
    pg::TravArgs a{};
    a.post = inst->at<Op4>(L.off_post);
    a.pre = inst->at<Op4>(L.off_pre);
    a.P = inst->ws + L.off_P;
    a.PT = L.variant == 1 ? inst->ws + L.off_PT : nullptr;
    a.Q = inst->ws + L.off_Q;
    a.QT = inst->ws + L.off_QT;
    a.pi = inst->ws + L.off_pi;
    a.cat_w = inst->at<double>(L.off_cw);
    a.cat_g = inst->at<double>(L.off_rates);
    a.pat_w = inst->at<double>(L.off_patw);
    a.tip_states = inst->at<uint8_t>(L.off_tips);
    a.tip_partials = (inst->cfg.flags & PG_FLAG_TIP_PARTIALS) ? inst->ws + L.off_tipp : nullptr;
    a.u = inst->ws + L.off_u;
    a.grad_part = inst->at<double>(L.off_gpart);
    a.logl_part = inst->at<double>(L.off_lpart);
    a.status = inst->at<int>(L.off_status);
    a.N = inst->cfg.tips;
    a.S = inst->mask_mode ? inst->mask_table.n : inst->cfg.states;   // mask mode: codes < n are masks
    a.R = inst->cfg.categories;
    a.Cpad = L.Cpad;
    a.C = inst->cfg.patterns;
    a.n_tiles = L.n_tiles;
    a.depth = std::max(inst->plan.post_depth, inst->plan.pre_depth);
    a.prefetch = inst->prefetch;
    a.prog_smem_off = inst->prog_smem_off;
    a.trace = inst->trace;
    a.rec_post = inst->grouped ? inst->rec_post : nullptr;
    a.rec_pre = inst->grouped ? inst->rec_pre : nullptr;
    a.tipstream = inst->tipstream_on ? inst->tipstream : nullptr;
    a.tipw = inst->tipstream_on ? inst->tipw : 0;
    return a;
}

static pg::codon::CodonArgs codon_args(pg_instance *inst) {
    const Layout &L = inst->L;
    pg::codon::CodonArgs c{};
    const int N = inst->cfg.tips;
    c.child_a = inst->at<int>(L.off_child);
    c.child_b = c.child_a + (2 * N - 1);
    c.levels = inst->at<int>(L.off_levels);
    c.lev4 = reinterpret_cast<const int4 *>(inst->ws + L.off_lev4);
    c.PBpost = inst->at<double>(L.off_P);
    c.PBpre = inst->at<double>(L.off_PBpre);
    c.PT = inst->at<double>(L.variant == 3 ? L.off_P : L.off_PT);     // variant 3: W = P' (the only copy)
    c.DT = inst->at<double>(L.off_DT);
    c.PONE = inst->at<double>(L.off_PONE);
    c.QB = inst->at<double>(L.off_QB);
    c.pi = inst->at<double>(L.off_pi);
    c.cat_w = inst->at<double>(L.off_cw);
    c.cat_g = inst->at<double>(L.off_rates);
    c.pat_w = inst->at<double>(L.off_patw);
    c.tip_states = inst->at<uint8_t>(L.off_tips);
    c.tip_partials = (inst->cfg.flags & PG_FLAG_TIP_PARTIALS) ? inst->at<double>(L.off_tipp) : nullptr;
    c.tip_is_partial = inst->at<uint8_t>(L.off_tipmode);
    c.utip = (inst->cfg.flags & PG_FLAG_TIP_PARTIALS) ? inst->at<double>(L.off_utip) : nullptr;
    c.tip_mask = (inst->cfg.flags & PG_FLAG_TIP_PARTIALS) ? inst->at<uint8_t>(L.off_tipmask) : nullptr;
    c.tip_masked = inst->at<uint8_t>(L.off_tipmasked);
    c.u = inst->at<double>(L.off_u);
    c.q = inst->at<double>(L.off_q);
    c.E = inst->at<int>(L.off_E);
    c.fmax = inst->at<int>(L.off_fmax);
    c.qmax = inst->at<int>(L.off_qmax);
    c.numden = inst->at<double>(L.off_numden);
    // flow v2: per-category exponents (the ratio kernel reconciles them)
    if (L.variant == 2 && inst->flow_ver == 2 && inst->flow_tch > 0 && inst->cfg.categories > 1) {
        c.EQ = inst->at<int>(L.off_EQ);
        c.Y = inst->at<int>(L.off_Y);
    }
    c.Lpart = inst->at<double>(L.off_Lpart);
    c.grad_part = inst->at<double>(L.off_gpart);
    c.logl_part = inst->at<double>(L.off_lpart);
    c.status = inst->at<int>(L.off_status);
    c.N = N;
    c.S = inst->cfg.states;
    c.R = inst->cfg.categories;
    c.Cpad = L.Cpad;
    c.C = inst->cfg.patterns;
    c.ntiles = L.n_tiles;
    return c;
}

static pg::tcp::TcArgs tc_args(pg_instance *inst) {
    const Layout &L = inst->L;
    pg::tcp::TcArgs t{};
    t.c = codon_args(inst);
    t.B = inst->at<float>(L.off_P);
    t.BQ = inst->at<float>(L.off_QB);
    t.ONE = inst->at<float>(L.off_PONE);
    t.pi = inst->at<float>(L.off_pi);
    t.u = inst->at<float>(L.off_u);
    t.q = inst->at<float>(L.off_q);
    return t;
}

// enqueue one evaluation (no host sync) writing [logL, g] to d_out
static int enqueue_eval(pg_instance *inst, double *d_out) {
    const Layout &L = inst->L;
    inst->a6_fused = false;
    const int R = inst->cfg.categories;
    // variants 0 / 1: A1 resets the status words (pdl_trigger_and_reset)
    if (L.variant >= 2) {
        CK(cudaMemsetAsync(inst->at<int>(L.off_status), 0x7f, sizeof(int), inst->stream), "status reset");
        CK(cudaMemsetAsync(inst->at<int>(L.off_status) + 1, 0, sizeof(int), inst->stream), "stall flag reset");
    }
    int *status_w = inst->at<int>(L.off_status);
    // small-S traversal and A6 launched with programmatic stream
    // serialization (setup overlaps the previous kernel; griddepcontrol.wait
    // before the dependent reads); not with timing events in between
    const bool pdl_small = L.variant == 0 && !inst->timing && !getenv("PG_NO_SMALL_PDL");
    // A6 inside the traversal (no reduce launch) when its grid is co-resident;
    // not under the per-kernel timing pass, which times A6 on its own
    const char *fse = getenv("PG_SMALL_FUSED_A6");
    // (measured slower than the separate launch: dengue 1.216 vs 1.246 ms, MMM
    // 0.1159 vs 0.1174 ms -- the last CTA's wait, then one CTA per row; off
    // unless PG_SMALL_FUSED_A6=1)
    const bool fuse_small_a6 = L.variant == 0 && !L.mma && !inst->timing && inst->small_coresident && fse && atoi(fse) != 0;
    if (inst->timing) CK(cudaEventRecordWithFlags(inst->ev[0], inst->stream, cudaEventRecordExternal), "event");
    const double *V = inst->at<double>(L.off_V), *Vi = inst->at<double>(L.off_Vi),
                 *lam = inst->at<double>(L.off_lam), *rates = inst->at<double>(L.off_rates),
                 *bl = inst->at<double>(L.off_bl);
    int S = inst->cfg.states;
    if (L.variant == 4) {
        CK(cudaMemsetAsync(inst->ws + L.off_fmax, 0, L.reset_bytes, inst->stream), "fmax/counters reset");
        const double *M0 = inst->at<double>(L.off_M0);
        const double *VA = inst->at<double>(L.off_VA), *ViB = inst->at<double>(L.off_ViB);
        float *Bm = inst->at<float>(L.off_P), *ONE = inst->at<float>(L.off_PONE);
        void *args[] = {&VA, &ViB, &M0, &lam, &rates, &bl, &S, (void *)&R, &Bm, &ONE};
        CK(cudaLaunchKernel((void *)pg::tcp::tc_pmat_kernel, dim3(L.B * R), dim3(256), args, pg::tcp::pmat_smem(),
                            inst->stream), "tc pmat launch");
    } else if (L.variant == 3) {
        // A1: W = P' per (branch, category), 8 row blocks each; masked tips' u
        CK(cudaMemsetAsync(inst->ws + L.off_fmax, 0, L.reset_bytes, inst->stream), "fmax/counters reset");
        const double *ViTA = inst->at<double>(L.off_VA), *VTB = inst->at<double>(L.off_ViB);
        const double *M0 = inst->at<double>(L.off_M0), *M0one = inst->at<double>(L.off_M0one),
                     *Vione = M0one + L.SP;
        double *W = inst->at<double>(L.off_P), *PONE = inst->at<double>(L.off_PONE);
        void *args[] = {&ViTA, &VTB, &M0, &M0one, &V, &Vione, &lam, &rates, &bl, &S, (void *)&R, &W, &PONE};
        CK(cudaLaunchKernel((void *)pg::big::big_pmat_kernel, dim3(L.B * R, 8), dim3(256), args, 0, inst->stream),
           "big pmat launch");
        if (inst->cfg.flags & PG_FLAG_TIP_PARTIALS) {
            pg::codon::CodonArgs c = codon_args(inst);
            void *targs[] = {&c};
            CK(cudaLaunchKernel((void *)pg::big::big_tipmask_kernel, dim3(L.n_tiles, inst->cfg.tips, R), dim3(256),
                                targs, 0, inst->stream), "big tip-mask launch");
        }
    } else if (L.variant == 2) {
        double *PBpost = inst->at<double>(L.off_P), *PBpre = inst->at<double>(L.off_PBpre),
               *PT = inst->at<double>(L.off_PT), *DT = inst->at<double>(L.off_DT), *PONE = inst->at<double>(L.off_PONE);
        const double *VA = inst->at<double>(L.off_VA), *ViB = inst->at<double>(L.off_ViB);
        const double *M0 = inst->at<double>(L.off_M0), *Qd = inst->at<double>(L.off_Q);
        // per-evaluation counters (rescaling maxima, flow counters, A1 flags)
        CK(cudaMemsetAsync(inst->ws + L.off_fmax, 0, L.reset_bytes, inst->stream), "fmax/flow reset");
        int *pready = inst->at<int>(L.off_flow) + 32 + flow_counter_ints(inst->cfg.tips, R, L.n_tiles);
        int Nt = inst->cfg.tips, tipp = (inst->cfg.flags & PG_FLAG_TIP_PARTIALS) ? 1 : 0;
        void *args[] = {&VA, &ViB, &M0, &Qd, &lam, &rates, &bl, &S, (void *)&R, &Nt, &tipp, &PBpost, &PBpre, &PT, &DT, &PONE, &pready};
        const CodonFns cf = codon_fns(L.SP);
        CK(cudaLaunchKernel(cf.pmat, dim3(L.B * R, 2), dim3(256), args, cf.pmat_smem, inst->stream), "codon pmat launch");
        if (inst->cfg.flags & PG_FLAG_TIP_PARTIALS) {     // u = P p of partial tips (A2's tip step)
            pg::codon::CodonArgs c = codon_args(inst);
            void *targs[] = {&c};
            CK(cudaLaunchKernel(cf.tipu, dim3((L.n_tiles + pg::codon::TIPU_TILES - 1) / pg::codon::TIPU_TILES,
                                              inst->cfg.tips, R),
                                dim3(cf.threads), targs, cf.tipu_smem, inst->stream), "codon tip-partials launch");
            CK(cudaLaunchKernel(cf.tipmask, dim3(L.n_tiles, inst->cfg.tips, R), dim3(256), targs, 0, inst->stream),
               "codon tip-mask launch");
        }
    } else {
        void *fn = pmat_kernel_fn(L);
        void *P = inst->ws + L.off_P;
        void *PT = L.variant == 1 ? inst->ws + L.off_PT : nullptr;
        int cs = L.cat_stride;
        const double *M0 = inst->at<double>(L.off_M0);
        if (L.mma) {
            int rec = cs * R;                            // doubles per branch record
            pg::MaskTable mt = inst->mask_table;
            if (!inst->mask_mode) mt.n = -1;            // the plain row-major layout
            unsigned char *recp = inst->grouped ? inst->rec_post : nullptr, *recq = inst->grouped ? inst->rec_pre : nullptr;
            const int *pdst = inst->post_dst, *qdst = inst->grouped ? inst->post_dst + L.B : nullptr;
            void *args16[] = {&V, &Vi, &M0, &lam, &rates, &bl, &S, &rec, &P, &status_w, &mt, &recp, &pdst, &recq, &qdst};
            if (L.SP == 16)
                CK(cudaLaunchKernel((void *)pg::pmat16_mma_kernel, dim3(L.B), dim3(256), args16, 0, inst->stream),
                   "pmat16 launch");
            else
                CK(cudaLaunchKernel((void *)pg::pmat4_mma_kernel, dim3(L.B), dim3(128), args16, 0, inst->stream),
                   "pmat4 launch");
        } else {
            unsigned char *recp = (L.variant == 0 && inst->grouped) ? inst->rec_post : nullptr;
            const int *pdst = inst->post_dst;
            unsigned char *recq = recp ? inst->rec_pre : nullptr;
            const int *qdst = recp ? inst->post_dst + L.B : nullptr;
            void *args[] = {&V, &Vi, &M0, &lam, &rates, &bl, &S, (void *)&R, &cs, &P, &PT, &status_w, &recp, &pdst,
                            &recq, &qdst};
            CK(cudaLaunchKernel(fn, dim3(L.B * R), dim3(std::min(256, L.SP * L.SP)), args, 0, inst->stream),
               "pmat launch");
        }
    }
    if (inst->timing) CK(cudaEventRecordWithFlags(inst->ev[1], inst->stream, cudaEventRecordExternal), "event");
    if (L.variant == 4) {
        pg::tcp::TcArgs t = tc_args(inst);
        const auto &pl = inst->plan;
        // every level launched with programmatic stream serialization: its
        // CTAs set up (TMEM, barriers, tip states) while the previous level's
        // last CTAs run, then griddepcontrol.wait (not with timing events)
        const bool pdl = !inst->timing && !getenv("PG_NO_TC_PDL");
        auto lvl = [&](void *fn, int off, int cnt, size_t smem) -> cudaError_t {
            void *args[] = {&t, &off};
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(L.n_tiles, cnt, R);
            lc.blockDim = dim3(pg::tcp::TM);
            lc.dynamicSmemBytes = smem;
            lc.stream = inst->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            lc.attrs = at;
            lc.numAttrs = pdl ? 1 : 0;
            return cudaLaunchKernelExC(&lc, fn, args);
        };
        for (size_t i = 0; i + 1 < pl.post_off.size(); ++i) {
            int off = pl.post_off[i], cnt = pl.post_off[i + 1] - off;
            CK(lvl((void *)pg::tcp::tc_post_kernel, off, cnt, pg::tcp::post_smem()), "tc post launch");
        }
        for (size_t i = 0; i + 1 < pl.pre_off.size(); ++i) {
            int off = pl.pre_off[i], cnt = pl.pre_off[i + 1] - off;
            CK(lvl((void *)pg::tcp::tc_pre_kernel, off, cnt, pg::tcp::pre_smem()), "tc pre launch");
        }
    } else if (L.variant == 3) {
        pg::codon::CodonArgs c = codon_args(inst);
        const auto &pl = inst->plan;
        for (size_t i = 0; i + 1 < pl.post_off.size(); ++i) {
            int off = pl.post_off[i], cnt = pl.post_off[i + 1] - off;
            void *args[] = {&c, &off};
            CK(cudaLaunchKernel((void *)pg::big::big_post_kernel, dim3(L.n_tiles, cnt, R), dim3(pg::big::NTB), args,
                                pg::big::post_smem(), inst->stream), "big post launch");
        }
        for (size_t i = 0; i + 1 < pl.pre_off.size(); ++i) {
            int off = pl.pre_off[i], cnt = pl.pre_off[i + 1] - off;
            void *args[] = {&c, &off};
            CK(cudaLaunchKernel((void *)pg::big::big_pre_kernel, dim3(L.n_tiles, cnt, R), dim3(pg::big::NTB), args,
                                pg::big::pre_smem(), inst->stream), "big pre launch");
        }
    } else if (L.variant == 2) {
        pg::codon::CodonArgs c = codon_args(inst);
        const CodonFns cf = codon_fns(L.SP);
        const auto &pl = inst->plan;
        const int N = inst->cfg.tips;
        if (inst->flow_tch > 0) {
            pg::codon::FlowArgs f{};
            f.ctr = inst->at<int>(L.off_flow);
            f.tch = inst->flow_tch;
            f.nch = (L.n_tiles + f.tch - 1) / f.tch;
            f.rpost = f.ctr + 32;
            // flow v2: per (node, category, tile); v1: per (node, chunk)
            f.rpre = f.rpost + (size_t)(N - 1) * f.nch * (inst->flow_ver == 2 ? R : 1);
            f.npost = pl.post_off.back();
            f.ntask = (int)pl.level_nodes.size();
            f.defer = inst->flow_defer;
            f.phalf = (inst->flow_half && f.tch == 1) ? 2 : 1;
            const int npre = f.ntask - f.npost;
            const int items = f.npost * R * f.nch * f.phalf + (npre + (f.defer ? npre : 0)) * R * f.nch;
            f.trace = inst->flow_trace_n >= (size_t)items ? inst->flow_trace : nullptr;
            if (inst->flow_ver == 2)
                f.trace = inst->flow_trace_n >= (size_t)(f.npost + 2 * (f.ntask - f.npost)) * R * L.n_tiles ? inst->flow_trace
                                                                                                          : nullptr;
            if (inst->flow_ver == 2) {
                f.split = inst->flow_split;
                f.task_off = inst->at<int>(L.off_taskoff);
                f.pprod = inst->flow_pprod;
                f.pub = inst->flow_pub;
                // A6 at the end of the flow launch (no ratio kernel) when a
                // row's patterns are few (<= 2 per thread: pattern shards;
                // yeast 8-way 0.2232 -> 0.2215 ms, WNV 8-way 0.4947 -> 0.4872
                // ms; at full size the sliced ratio kernel is faster: yeast
                // 1.093 vs 1.107 ms); not under the per-kernel timing pass
                const char *fa6 = getenv("PG_FUSED_A6");
                const bool fuse = fa6 ? atoi(fa6) != 0 : inst->cfg.patterns <= 2 * (int)cf.flow2_threads;
                if (fuse && !inst->timing) {
                    f.a6cnt = inst->at<int>(L.off_flow) + 32 + flow_counter_ints(N, R, L.n_tiles) + (size_t)L.B * R + (L.B + 1);
                    f.out = d_out;
                    inst->a6_fused = true;
                }
                const int items2 = f.split ? inst->split_items : f.ntask * R * L.n_tiles;
                const int v = inst->flow_nst - 1;
                // programmatic dependent launch right behind A1 (no partial-tip
                // kernels or timing events in between): items wait on pready
                const bool pdl = inst->flow_pdl && !inst->timing && !(inst->cfg.flags & PG_FLAG_TIP_PARTIALS);
                f.pready = pdl ? inst->at<int>(L.off_flow) + 32 + flow_counter_ints(N, R, L.n_tiles) : nullptr;
                void *args2[] = {&c, &f, &inst->tmaps};
                cudaLaunchConfig_t lc{};
                const bool rs = inst->flow_rs == 2;
                lc.gridDim = dim3(std::min(items2, (rs ? 1 : cf.flow2_ctas[v]) * inst->sm_count));
                lc.blockDim = dim3(rs ? cf.flow2rs_threads : cf.flow2_threads);
                lc.dynamicSmemBytes = cf.flow2_smem[v];
                lc.stream = inst->stream;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                lc.attrs = at;
                lc.numAttrs = pdl ? 1 : 0;
                CK(cudaLaunchKernelExC(&lc, rs ? cf.flow2rs : cf.flow2[v], args2), "codon flow2 launch");
            } else {
                void *args[] = {&c, &f};
                CK(cudaLaunchKernel(cf.flow, dim3(std::min(items, cf.ctas_per_sm * inst->sm_count)),
                                    dim3(cf.threads), args, cf.flow_smem, inst->stream),
                   "codon flow launch");
            }
        }
        for (size_t i = 0; inst->flow_tch == 0 && i + 1 < pl.post_off.size(); ++i) {
            int off = pl.post_off[i], cnt = pl.post_off[i + 1] - off;
            // persistent: 3 CTAs per SM walk the level's items; narrow levels
            // (fewer full-tile items than ~2 waves) use half-tile items
            const bool narrow = L.n_tiles * cnt * R < 2 * cf.ctas_per_sm * inst->sm_count;
            const int items = L.n_tiles * cnt * R * (narrow ? 2 : 1);
            void *fn = narrow ? cf.post2 : cf.post4;
            void *args[] = {&c, &off, &cnt};
            CK(cudaLaunchKernel(fn, dim3(std::min(items, cf.ctas_per_sm * inst->sm_count)), dim3(cf.threads), args,
                                cf.post_smem + 16 * (size_t)cnt, inst->stream),
               "codon post launch");
        }
        for (size_t i = 0; inst->flow_tch == 0 && i + 1 < pl.pre_off.size(); ++i) {
            int off = pl.pre_off[i], cnt = pl.pre_off[i + 1] - off;
            void *args[] = {&c, &off};
            CK(cudaLaunchKernel(cf.pre, dim3(L.n_tiles, cnt, R), dim3(cf.threads), args, cf.pre_smem, inst->stream),
               "codon pre launch");
        }
    } else {
        pg::TravArgs a = trav_args(inst);
        if (fuse_small_a6) {
            a.a6cnt = status_w + 2;                  // reset by A1 (pdl_trigger_and_reset)
            a.out = d_out;
        }
        void *args[] = {&a};
        if (pdl_small) {
            cudaLaunchConfig_t lc{};
            lc.gridDim = dim3(inst->grid);
            lc.blockDim = dim3(inst->block);
            lc.dynamicSmemBytes = inst->smem;
            lc.stream = inst->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            CK(cudaLaunchKernelExC(&lc, traverse_fn(L, inst->cfg.categories, inst->grouped), args), "traverse launch");
        } else {
            CK(cudaLaunchKernel(traverse_fn(L, inst->cfg.categories, inst->grouped), dim3(inst->grid), dim3(inst->block), args,
                                inst->smem, inst->stream),
               "traverse launch");
        }
    }
    if (inst->timing) CK(cudaEventRecordWithFlags(inst->ev[2], inst->stream, cudaEventRecordExternal), "event");
    if (inst->a6_fused || fuse_small_a6) {
        // A6 ran inside the flow kernel / the small-S traversal
    } else if (L.variant >= 2) {
        pg::codon::CodonArgs c = codon_args(inst);
        int *cnt = inst->at<int>(L.off_flow) + 32 + flow_counter_ints(inst->cfg.tips, R, L.n_tiles) + (size_t)L.B * R;
        double *sp = inst->at<double>(L.off_gpart);      // [B+1][slices] <= [B][n_tiles] + [n_tiles] (codon path)
        const int ns = std::min(pg::codon::RATIO_SLICES, L.n_tiles);
        void *args[] = {&c, &d_out, &sp, &cnt};
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(L.B + 1, ns);
        lc.blockDim = dim3(256);
        lc.stream = inst->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = (L.variant == 4 && !inst->timing && !getenv("PG_NO_TC_PDL")) ? 1 : 0;
        CK(cudaLaunchKernelExC(&lc, (void *)pg::codon::codon_ratio_kernel, args), "codon ratio launch");
    } else {
        const double *gp = inst->at<double>(L.off_gpart), *lp = inst->at<double>(L.off_lpart);
        int B = L.B, nt = L.n_tiles;
        void *args[] = {&gp, &lp, &B, &nt, &d_out};
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(L.B + 1);
        lc.blockDim = dim3(256);
        lc.stream = inst->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = pdl_small ? 1 : 0;
        CK(cudaLaunchKernelExC(&lc, (void *)pg::reduce_kernel, args), "reduce launch");
    }
    if (inst->timing) CK(cudaEventRecordWithFlags(inst->ev[3], inst->stream, cudaEventRecordExternal), "event");
    return PG_OK;
}

static int prepare(pg_instance *inst, bool captured = false) {
    if (!inst->have_ops) return inst->fail(PG_ERR_SEQUENCE, "operations not set");
    if (!inst->have_eigen) return inst->fail(PG_ERR_SEQUENCE, "eigensystem not set");
    if (!inst->have_pi) return inst->fail(PG_ERR_SEQUENCE, "state frequencies not set");
    if (!inst->have_rates || !inst->have_cw) return inst->fail(PG_ERR_SEQUENCE, "category rates/weights not set");
    if (!inst->have_patw) return inst->fail(PG_ERR_SEQUENCE, "pattern weights not set");
    if (!inst->have_bl) return inst->fail(PG_ERR_SEQUENCE, "branch lengths not set");
    for (int t = 0; t < inst->cfg.tips; ++t)
        if (!inst->tip_set[t]) return inst->fail(PG_ERR_SEQUENCE, "tip " + std::to_string(t) + " has no data");
    if (captured) {
        // inside the caller's stream capture nothing may synchronise: the
        // plan, launch configuration and tip data must already be on the device
        if (inst->plan_dirty || inst->partial_modes_dirty || inst->tips_dirty || (inst->tipstream_on && inst->tipstream_dirty))
            return inst->fail(PG_ERR_SEQUENCE, "pending uploads (operations, tips or launch plan): run one evaluation "
                                               "outside stream capture before capturing pg_compute_device");
        return PG_OK;
    }
    int rc = refresh_plan(inst);
    if (rc) return rc;
    if (inst->tips_dirty) {
        CK(cudaMemcpyAsync(inst->ws + inst->L.off_tips, inst->tips_h.data(), inst->tips_h.size(),
                           cudaMemcpyHostToDevice, inst->stream), "tips upload");
        CK(cudaStreamSynchronize(inst->stream), "tips sync");
        inst->tips_dirty = false;
        inst->tipstream_dirty = true;
    }
    if (inst->tipstream_on && inst->tipstream_dirty) {
        // per CTA and post step, the tip-code windows of the step's tip
        // children (static while tips and plan are unchanged)
        const Layout &L = inst->L;
        const int N = inst->cfg.tips, K = inst->tiles_per_cta;
        const uint8_t *tips = inst->at<uint8_t>(L.off_tips);
        const Op4 *post = inst->at<Op4>(L.off_post);
        pg::tipstream_kernel<<<dim3(N - 1, inst->grid), 128, 0, inst->stream>>>(post, tips, inst->tipstream, N, L.Cpad,
                                                                              K * L.tpl, inst->tipw);
        CK(cudaGetLastError(), "tip stream launch");
        CK(cudaStreamSynchronize(inst->stream), "tip stream sync");
        inst->tipstream_dirty = false;
    }
    return PG_OK;
}

// one evaluation via a cached CUDA graph (captured per output pointer); when
// the caller is itself capturing the stream, the kernels are enqueued into
// the caller's graph instead (a caller can then capture [branch lengths,
// evaluation, allreduce] as one graph)
static int launch_eval(pg_instance *inst, double *d_out, bool captured = false) {
    if (captured) return enqueue_eval(inst, d_out);
    if (!inst->gexec || inst->gexec_out != d_out) {
        if (inst->gexec) { cudaGraphExecDestroy(inst->gexec); inst->gexec = nullptr; }
#ifdef PG_TRACE
        if (!inst->trace) {   // allocation is illegal inside stream capture
            cudaMalloc((void **)&inst->trace, sizeof(long long) * 16 * 2 * (size_t)inst->cfg.tips);
            cudaMemset(inst->trace, 0, sizeof(long long) * 16 * 2 * (size_t)inst->cfg.tips);
        }
#endif
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(inst->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
        int rc = enqueue_eval(inst, d_out);
        cudaError_t e2 = cudaStreamEndCapture(inst->stream, &g);
        if (rc) return rc;
        if (e2 != cudaSuccess) return inst->cuda_fail(e2, "end capture");
        cudaError_t e3 = cudaGraphInstantiate(&inst->gexec, g, 0);
        cudaGraphDestroy(g);
        if (e3 != cudaSuccess) return inst->cuda_fail(e3, "graph instantiate");
        inst->gexec_out = d_out;
    }
    CK(cudaGraphLaunch(inst->gexec, inst->stream), "graph launch");
    return PG_OK;
}

int pg_compute_device(pg_instance *inst, double *d_out) {
    if (!inst || !d_out) return PG_ERR_ARG;
    DeviceGuard dg(inst);
    const bool cap = capturing(inst);
    int rc = prepare(inst, cap);
    if (rc) return rc;
    // host-staged inputs: stream-ordered copies from the pinned buffers.  In a
    // caller's capture they become memcpy nodes that re-read the buffers at
    // every replay (the pending flags are left as they are)
    const bool staged = inst->bl_host_pending || inst->clock_host_pending;
    if (inst->bl_host_pending) {
        CK(cudaMemcpyAsync(inst->ws + inst->L.off_bl, inst->bl_pinned, sizeof(double) * inst->L.B,
                           cudaMemcpyHostToDevice, inst->stream), "branch lengths H2D");
        if (!cap) inst->bl_host_pending = false;
    }
    if ((rc = flush_clock_host(inst))) return rc;
    if (!cap) {
        inst->clock_host_pending = false;
        if (staged && (rc = mark_staging(inst))) return rc;
    }
    return launch_eval(inst, d_out, cap);
}

int pg_compute(pg_instance *inst, double *log_likelihood, double *gradient) {
    DeviceGuard dg(inst);
    if (!inst || !log_likelihood) return PG_ERR_ARG;
    if (capturing(inst)) return inst->fail(PG_ERR_SEQUENCE, "pg_compute synchronises: use pg_compute_device under stream capture");
    int rc = prepare(inst);
    if (rc) return rc;
    const Layout &L = inst->L;
    if (inst->bl_host_pending) {
        CK(cudaMemcpyAsync(inst->ws + L.off_bl, inst->bl_pinned, sizeof(double) * L.B, cudaMemcpyHostToDevice,
                           inst->stream), "branch lengths H2D");
        // host branch lengths stay "pending": every pg_compute re-uploads them
    }
    if ((rc = flush_clock_host(inst))) return rc;      // likewise host heights / rate scalars
    double *d_out = inst->at<double>(L.off_out);
    if ((rc = launch_eval(inst, d_out))) return rc;
    CK(cudaMemcpyAsync(inst->out_pinned, d_out, sizeof(double) * (L.B + 1), cudaMemcpyDeviceToHost, inst->stream),
       "result D2H");
    CK(cudaMemcpyAsync(inst->status_pinned, inst->at<int>(L.off_status), 2 * sizeof(int), cudaMemcpyDeviceToHost,
                       inst->stream), "status D2H");
    CK(cudaStreamSynchronize(inst->stream), "compute sync");
    inst->staged_pending = false;
    if (inst->status_pinned[1]) return inst->fail(PG_ERR_CUDA, "codon flow schedule stalled (> 20 s waiting for an input)");
    const int zp = inst->status_pinned[0];
    if (zp != 0x7f7f7f7f) {
        *log_likelihood = -INFINITY;
        return inst->fail(PG_ERR_ZERO_LIKELIHOOD, "site likelihood is zero at pattern " + std::to_string(zp));
    }
    *log_likelihood = inst->out_pinned[0];
    if (gradient) std::memcpy(gradient, inst->out_pinned + 1, sizeof(double) * L.B);
    if (inst->flow_trace) {                          // diagnostics: dump the last evaluation's item trace
        std::vector<unsigned long long> h(pg::codon::TRW * inst->flow_trace_n);
        CK(cudaMemcpy(h.data(), inst->flow_trace, h.size() * 8, cudaMemcpyDeviceToHost), "trace D2H");
        if (FILE *fp = fopen(getenv("PG_FLOW_TRACE"), "wb")) {
            fwrite(h.data(), 8, h.size(), fp);
            fclose(fp);
        }
    }
    return PG_OK;
}

int pg_hmc_leapfrog(pg_instance *inst, double *d_theta, double *d_p, const double *d_inv_mass, double eps,
                    int32_t n_steps, double *d_out, double *d_grad_theta) {
    DeviceGuard dg(inst);
    if (!inst) return PG_ERR_ARG;
    if (!d_theta || !d_p || !d_out || n_steps < 0 || !std::isfinite(eps))
        return inst->fail(PG_ERR_ARG, "NULL pointer, n_steps < 0 or non-finite eps");
    const int B = inst->L.B;
    double *bl = inst->at<double>(inst->L.off_bl);
    // the branch lengths now come from theta: drop pending host uploads
    inst->bl_host_pending = inst->clock_host_pending = false;
    inst->have_bl = true;
    const bool cap = capturing(inst);
    int rc = prepare(inst, cap);
    if (rc) return rc;
    const dim3 grid((B + 127) / 128), block(128);
    auto drift = [&](double e) -> int {
        pg::hmc_drift_kernel<<<grid, block, 0, inst->stream>>>(d_theta, d_p, d_inv_mass, e, bl, B);
        CK(cudaGetLastError(), "hmc drift launch");
        return PG_OK;
    };
    auto kick = [&](double coef) -> int {
        pg::hmc_kick_kernel<<<grid, block, 0, inst->stream>>>(bl, d_out, coef, d_p, d_grad_theta, B);
        CK(cudaGetLastError(), "hmc kick launch");
        return PG_OK;
    };
    if ((rc = drift(0.0)) || (rc = launch_eval(inst, d_out, cap)) || (rc = kick(n_steps > 0 ? 0.5 * eps : 0.0))) return rc;
    for (int s = 0; s < n_steps; ++s) {
        if ((rc = drift(eps)) || (rc = launch_eval(inst, d_out, cap))) return rc;
        if ((rc = kick(s + 1 < n_steps ? eps : 0.5 * eps))) return rc;
    }
    return PG_OK;
}

int pg_check_status(pg_instance *inst, int32_t *zero_pattern) {
    DeviceGuard dg(inst);
    if (!inst) return PG_ERR_ARG;
    int v = 0;
    CK(cudaMemcpyAsync(inst->status_pinned, inst->at<int>(inst->L.off_status), 2 * sizeof(int), cudaMemcpyDeviceToHost,
                       inst->stream), "status D2H");
    CK(cudaStreamSynchronize(inst->stream), "status sync");
    if (inst->status_pinned[1]) return inst->fail(PG_ERR_CUDA, "codon flow schedule stalled (> 20 s waiting for an input)");
    v = inst->status_pinned[0];
    const bool bad = v != 0x7f7f7f7f;
    if (zero_pattern) *zero_pattern = bad ? v : -1;
    if (bad) return inst->fail(PG_ERR_ZERO_LIKELIHOOD, "site likelihood is zero at pattern " + std::to_string(v));
    return PG_OK;
}

int pg_set_kernel_timing(pg_instance *inst, int enable) {
    DeviceGuard dg(inst);
    if (!inst) return PG_ERR_ARG;
    if (enable && !inst->ev[0])
        for (auto &e : inst->ev) CK(cudaEventCreate(&e), "event create");
    if ((bool)enable != inst->timing && inst->gexec) {
        cudaGraphExecDestroy(inst->gexec);
        inst->gexec = nullptr;
    }
    inst->timing = enable != 0;
    return PG_OK;
}

int pg_get_kernel_times(pg_instance *inst, float *ms) {
    DeviceGuard dg(inst);
    if (!inst || !ms) return PG_ERR_ARG;
    if (!inst->timing) return inst->fail(PG_ERR_SEQUENCE, "kernel timing is not enabled");
    CK(cudaEventSynchronize(inst->ev[3]), "event sync");
    for (int k = 0; k < 3; ++k) CK(cudaEventElapsedTime(&ms[k], inst->ev[k], inst->ev[k + 1]), "elapsed");
    return PG_OK;
}

#ifdef PG_TRACE
// trace builds only: copy the clock64 samples of the last evaluation
extern "C" int pg_trace_copy(pg_instance *inst, long long *host, int n) {
    if (!inst || !inst->trace) return PG_ERR_SEQUENCE;
    cudaStreamSynchronize(inst->stream);
    cudaMemcpy(host, inst->trace, sizeof(long long) * n, cudaMemcpyDeviceToHost);
    return PG_OK;
}
#endif

int pg_kernels_per_eval(const pg_instance *inst, int32_t *n) {
    if (!inst || !n) return PG_ERR_ARG;
    *n = 3;   // pmat, traverse, reduce
    if (inst->L.variant == 4)   // pmat + one launch per post level + per pre level + ratio
        *n = 2 + (int32_t)(inst->plan.post_off.size() - 1) + (int32_t)(inst->plan.pre_off.size() - 1);
    else if (inst->L.variant == 3)   // pmat + [masked tips] + one launch per post level + per pre level + ratio
        *n = 2 + ((inst->cfg.flags & PG_FLAG_TIP_PARTIALS) ? 1 : 0) + (int32_t)(inst->plan.post_off.size() - 1) +
             (int32_t)(inst->plan.pre_off.size() - 1);
    else if (inst->L.variant == 2)   // pmat + (one flow launch | one launch per post level + per pre level) + reduce
        *n = 2 + ((inst->cfg.flags & PG_FLAG_TIP_PARTIALS) ? 2 : 0) +
             (inst->flow_tch > 0 ? 1 : (int32_t)(inst->plan.post_off.size() - 1) + (int32_t)(inst->plan.pre_off.size() - 1));
    return PG_OK;
}

int pg_get_plan_info(const pg_instance *inst, pg_plan_info *info) {
    if (!inst || !info) return PG_ERR_ARG;
    info->post_depth = inst->plan.post_depth;
    info->pre_depth = inst->plan.pre_depth;
    info->grid = inst->grid;
    info->block = inst->block;
    info->smem_bytes = inst->smem;
    info->prefetch_depth = inst->prefetch;
    info->padded_patterns = inst->L.Cpad;
    info->kernel_variant = inst->L.variant;
    info->flow_tiles = inst->flow_tch;
    info->flow_version = inst->L.variant == 2 && inst->flow_tch > 0 ? inst->flow_ver : 0;
    info->flow_stages = info->flow_version == 2 ? inst->flow_nst : 0;
    info->flow_pdl = info->flow_version == 2 && inst->flow_pdl && !inst->timing &&
                     !(inst->cfg.flags & PG_FLAG_TIP_PARTIALS);
    if (inst->L.variant == 2 && inst->flow_tch > 0) {
        const int nch = (inst->L.n_tiles + inst->flow_tch - 1) / inst->flow_tch;
        const CodonFns cf = codon_fns(inst->L.SP);
        const int v = inst->flow_nst - 1;
        const int slots = inst->flow_ver == 2 ? cf.flow2_ctas[v] * inst->sm_count : cf.ctas_per_sm * inst->sm_count;
        info->grid = std::min((int)inst->plan.level_nodes.size() * inst->cfg.categories * nch, slots);
        info->smem_bytes = (int)(inst->flow_ver == 2 ? cf.flow2_smem[v] : cf.flow_smem);
        info->block = inst->flow_ver == 2 ? cf.flow2_threads : cf.threads;
    }
    return PG_OK;
}
