// Level-batched control for the small-S design choice (VERDICT r01
// weak #3): a lower-bound proxy of a level-by-level dengue evaluation -- one
// launch per tree level (post by height, pre by depth), every (node, pattern,
// category) vector read from / written to HBM (SURVEY §8(d)'s B_min traffic:
// u written once and read twice, q written and read once), the same S = 4
// matvecs, Eq. 8 terms reduced per warp -- but no rescaling and no exact
// ratio bookkeeping, so a real level-batched implementation can only be
// slower.  Not part of the library; timed with CUDA events around a CUDA
// graph of all launches, L2 flushed between replays.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o level_proxy scripts/level_proxy.cu
//   ./level_proxy levels.bin
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

struct Ent { int k, a, b; };

__device__ __forceinline__ double4 ld4(const double *p) {
    const double2 x = __ldcs(reinterpret_cast<const double2 *>(p)), y = __ldcs(reinterpret_cast<const double2 *>(p) + 1);
    return make_double4(x.x, x.y, y.x, y.y);
}
__device__ __forceinline__ void st4(double *p, double4 v) {
    __stcs(reinterpret_cast<double2 *>(p), make_double2(v.x, v.y));
    __stcs(reinterpret_cast<double2 *>(p) + 1, make_double2(v.z, v.w));
}

__device__ __forceinline__ void child_vec(double (&v)[4], int child, int N, int C, int R, int c, int r,
                                          const double *__restrict__ u, const signed char *__restrict__ tips,
                                          const double *__restrict__ P) {
    if (child >= N) {
        double4 t = ld4(u + ((((size_t)(child - N) * C + c) * R + r) * 4));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
        const int s = tips[(size_t)child * C + c];
        const double *M = P + ((size_t)child * R + r) * 16;
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = s < 4 ? M[i * 4 + s] : (M[i * 4] + M[i * 4 + 1]) + (M[i * 4 + 2] + M[i * 4 + 3]);
    }
}

__global__ void post_level(const Ent *__restrict__ ent, int cnt, int N, int C, int R, double *__restrict__ u,
                           const signed char *__restrict__ tips, const double *__restrict__ P, double *__restrict__ L) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t per = (size_t)C * R;
    if (idx >= cnt * per) return;
    const Ent e = ent[idx / per];
    const int rem = (int)(idx % per), c = rem / R, r = rem % R;
    double ua[4], ub[4], p[4];
    child_vec(ua, e.a, N, C, R, c, r, u, tips, P);
    child_vec(ub, e.b, N, C, R, c, r, u, tips, P);
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = ua[i] * ub[i];
    if (e.k == 2 * N - 2) {                       // root: Eq. 3 terms
        L[idx % per] = 0.25 * (p[0] + p[1] + p[2] + p[3]);
        return;
    }
    const double *M = P + ((size_t)e.k * R + r) * 16;
    double o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = M[i * 4] * p[0] + M[i * 4 + 1] * p[1] + M[i * 4 + 2] * p[2] + M[i * 4 + 3] * p[3];
    st4(u + ((((size_t)(e.k - N) * C + c) * R + r) * 4), make_double4(o[0], o[1], o[2], o[3]));
}

__global__ void pre_level(const Ent *__restrict__ ent, int cnt, int N, int C, int R, const double *__restrict__ u,
                          double *__restrict__ q, const signed char *__restrict__ tips, const double *__restrict__ P,
                          const double *__restrict__ Q, double *__restrict__ grad) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t per = (size_t)C * R;
    const bool live = idx < cnt * per;
    const Ent e = ent[live ? idx / per : 0];
    const int rem = (int)(idx % per), c = rem / R, r = rem % R;
    double qk[4], ua[4], ub[4];
    double na = 0.0, nb = 0.0;
    if (live) {
        if (e.k == 2 * N - 2) {
            qk[0] = qk[1] = qk[2] = qk[3] = 0.25;
        } else {
            double4 t = ld4(q + ((((size_t)(e.k - N) * C + c) * R + r) * 4));
            qk[0] = t.x; qk[1] = t.y; qk[2] = t.z; qk[3] = t.w;
        }
        child_vec(ua, e.a, N, C, R, c, r, u, tips, P);
        child_vec(ub, e.b, N, C, R, c, r, u, tips, P);
        double xa[4], xb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { xa[i] = qk[i] * ub[i]; xb[i] = qk[i] * ua[i]; }
        double den = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double qa = Q[i * 4] * ua[0] + Q[i * 4 + 1] * ua[1] + Q[i * 4 + 2] * ua[2] + Q[i * 4 + 3] * ua[3];
            const double qb = Q[i * 4] * ub[0] + Q[i * 4 + 1] * ub[1] + Q[i * 4 + 2] * ub[2] + Q[i * 4 + 3] * ub[3];
            na += xa[i] * qa;
            nb += xb[i] * qb;
            den += xa[i] * ua[i];
        }
        na /= den;
        nb /= den;
        for (int ch = 0; ch < 2; ++ch) {          // q_c = P_c' x_c for internal children
            const int cn = ch ? e.b : e.a;
            if (cn < N) continue;
            const double *M = P + ((size_t)cn * R + r) * 16;
            const double *x = ch ? xb : xa;
            double o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = M[j] * x[0] + M[4 + j] * x[1] + M[8 + j] * x[2] + M[12 + j] * x[3];
            st4(q + ((((size_t)(cn - N) * C + c) * R + r) * 4), make_double4(o[0], o[1], o[2], o[3]));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        na += __shfl_xor_sync(0xffffffffu, na, o);
        nb += __shfl_xor_sync(0xffffffffu, nb, o);
    }
    if (live && (threadIdx.x & 31) == 0) {       // per-warp partials, summed later (no atomics)
        const size_t wi = idx >> 5;
        grad[2 * wi] = na;
        grad[2 * wi + 1] = nb;
    }
}

int main(int argc, char **argv) {
    FILE *fp = fopen(argv[1], "rb");
    int hdr[5];
    fread(hdr, 4, 5, fp);
    const int N = hdr[0], C = hdr[1], R = hdr[2], npl = hdr[3], nql = hdr[4];
    std::vector<std::vector<Ent>> post(npl), pre(nql);
    for (auto *lv : {&post, &pre})
        for (auto &l : *lv) {
            int cnt;
            fread(&cnt, 4, 1, fp);
            l.resize(cnt);
            fread(l.data(), sizeof(Ent), cnt, fp);
        }
    std::vector<signed char> tips((size_t)N * C);
    fread(tips.data(), 1, tips.size(), fp);
    fclose(fp);
    const int B = 2 * N - 2;
    double *u, *q, *P, *Q, *grad, *L, *flush;
    signed char *dt;
    const size_t V = (size_t)C * R * 4 * 8;
    CK(cudaMalloc(&u, V * (N - 1)));
    CK(cudaMalloc(&q, V * (N - 1)));
    CK(cudaMalloc(&P, (size_t)B * R * 16 * 8));
    CK(cudaMalloc(&Q, 16 * 8));
    size_t maxw = 0;                               // per-warp partial slots of the widest pre level
    for (auto &l : pre) maxw = std::max(maxw, l.size() * (size_t)C * R / 32 + 1);
    CK(cudaMalloc(&grad, 2 * maxw * 8));
    CK(cudaMalloc(&L, (size_t)C * R * 8));
    CK(cudaMalloc(&flush, 256u << 20));
    CK(cudaMalloc(&dt, tips.size()));
    CK(cudaMemcpy(dt, tips.data(), tips.size(), cudaMemcpyHostToDevice));
    std::vector<double> hp((size_t)B * R * 16);
    for (size_t i = 0; i < hp.size(); ++i) hp[i] = ((i % 16) % 5 == 0) ? 0.9 : 0.033;
    CK(cudaMemcpy(P, hp.data(), hp.size() * 8, cudaMemcpyHostToDevice));
    double hq[16];
    for (int i = 0; i < 16; ++i) hq[i] = (i % 5 == 0) ? -0.75 : 0.25;
    CK(cudaMemcpy(Q, hq, sizeof(hq), cudaMemcpyHostToDevice));
    std::vector<Ent *> dpost(npl), dpre(nql);
    for (int i = 0; i < npl; ++i) { CK(cudaMalloc(&dpost[i], post[i].size() * sizeof(Ent))); CK(cudaMemcpy(dpost[i], post[i].data(), post[i].size() * sizeof(Ent), cudaMemcpyHostToDevice)); }
    for (int i = 0; i < nql; ++i) { CK(cudaMalloc(&dpre[i], pre[i].size() * sizeof(Ent))); CK(cudaMemcpy(dpre[i], pre[i].data(), pre[i].size() * sizeof(Ent), cudaMemcpyHostToDevice)); }
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
    const int T = 256;
    for (int i = 0; i < npl; ++i) {
        const size_t n = post[i].size() * (size_t)C * R;
        post_level<<<(unsigned)((n + T - 1) / T), T, 0, st>>>(dpost[i], (int)post[i].size(), N, C, R, u, dt, P, L);
    }
    for (int i = 0; i < nql; ++i) {
        const size_t n = pre[i].size() * (size_t)C * R;
        pre_level<<<(unsigned)((n + T - 1) / T), T, 0, st>>>(dpre[i], (int)pre[i].size(), N, C, R, u, q, dt, P, Q, grad);
    }
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int i = 0; i < 5; ++i) CK(cudaGraphLaunch(ge, st));
    const int K = 200;
    double tot = 0.0;
    std::vector<float> ms(K);
    for (int i = 0; i < K; ++i) {
        CK(cudaMemsetAsync(flush, i & 0xff, 256u << 20, st));
        CK(cudaEventRecord(e0, st));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms[i], e0, e1));
        tot += ms[i];
    }
    const double mean = tot / K;
    const double bmin = 5.0 * (N - 2) * (double)V + 2.0 * N * C + 8.0 * (N - 1) * C;
    printf("{\"proxy\": \"level-batched dengue lower bound\", \"launches\": %d, \"ms_per_eval\": %.4f, "
           "\"b_min_bytes\": %.0f, \"achieved_gbs\": %.1f}\n", npl + nql, mean, bmin, bmin / (mean * 1e-3) / 1e9);
    return 0;
}
