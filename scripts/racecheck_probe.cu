// racecheck_probe.cu -- is compute-sanitizer racecheck able to follow an
// mbarrier-synchronised 1-D bulk-copy (TMA engine) ring?  A textbook
// producer/consumer ring (the pattern of traverse_small_kernel): producer
// warp waits "empty", fences the async proxy, arms "full" with expect_tx and
// issues cp.async.bulk; consumer warps wait "full", read the stage with
// ld.shared, and arrive on "empty".  The result is checked on the host.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -o racecheck_probe scripts/racecheck_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2303_04390_b200/csrc/common.cuh"

constexpr int D = 4, CONS = 4, CHUNK = 1024, STEPS = 64;

__global__ void ring(const double *src, double *out) {
    __shared__ __align__(128) double stage[D][CHUNK / 8];
    __shared__ __align__(8) uint64_t full[D], empty[D];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < D; ++i) { pg::mbar_init(&full[i], 1); pg::mbar_init(&empty[i], CONS); }
        pg::fence_mbar_init();
    }
    __syncthreads();
    if (warp == CONS) {                       // producer
        for (int t = 0; t < STEPS; ++t) {
            const int s = t % D;
            if (t >= D) pg::mbar_wait(&empty[s], (uint32_t)((t / D + 1) & 1));
            if (lane == 0) {
                pg::fence_proxy_async_smem();
                pg::mbar_arrive_expect_tx(&full[s], CHUNK);
                pg::bulk_g2s(stage[s], src + (size_t)t * (CHUNK / 8), CHUNK, &full[s]);
            }
            __syncwarp();
        }
        return;
    }
    double acc = 0.0;
    for (int t = 0; t < STEPS; ++t) {
        const int s = t % D;
        pg::mbar_wait(&full[s], (uint32_t)((t / D) & 1));
        for (int i = lane; i < CHUNK / 8; i += 32) acc += stage[s][i];
        __syncwarp();
        if (lane == 0) pg::mbar_arrive(&empty[s]);
    }
    out[threadIdx.x] = acc;
}

// the same ring with the producer's 32 lanes filling a stage by cp.async
// (LDGSTS) and arriving through cp.async.mbarrier.arrive.noinc (the flow2
// kernel's tip gathers)
__global__ void ring_cpasync(const double *src, double *out) {
    __shared__ __align__(128) double stage[D][CHUNK / 8];
    __shared__ __align__(8) uint64_t full[D], empty[D];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < D; ++i) { pg::mbar_init(&full[i], 32); pg::mbar_init(&empty[i], CONS); }
        pg::fence_mbar_init();
    }
    __syncthreads();
    if (warp == CONS) {
        for (int t = 0; t < STEPS; ++t) {
            const int s = t % D;
            if (t >= D) pg::mbar_wait(&empty[s], (uint32_t)((t / D + 1) & 1));
            for (int i = lane; i < CHUNK / 16; i += 32)
                pg::cp_async16(&stage[s][2 * i], src + (size_t)t * (CHUNK / 8) + 2 * i);
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(pg::smem_u32(&full[s])) : "memory");
        }
        return;
    }
    double acc = 0.0;
    for (int t = 0; t < STEPS; ++t) {
        const int s = t % D;
        pg::mbar_wait(&full[s], (uint32_t)((t / D) & 1));
        for (int i = lane; i < CHUNK / 8; i += 32) acc += stage[s][i];
        __syncwarp();
        if (lane == 0) pg::mbar_arrive(&empty[s]);
    }
    out[threadIdx.x] = acc;
}

int main() {
    const int n = STEPS * CHUNK / 8;
    double *h = new double[n], *src, *out;
    for (int i = 0; i < n; ++i) h[i] = 1.0;
    cudaMalloc(&src, n * 8);
    cudaMalloc(&out, 32 * CONS * 8);
    cudaMemcpy(src, h, n * 8, cudaMemcpyHostToDevice);
    bool all = true;
    for (int v = 0; v < 2; ++v) {
        cudaMemset(out, 0, 32 * CONS * 8);
        if (v == 0) ring<<<1, 32 * (CONS + 1)>>>(src, out);
        else ring_cpasync<<<1, 32 * (CONS + 1)>>>(src, out);
        double o[32 * CONS];
        cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
        bool ok = cudaGetLastError() == cudaSuccess;
        for (int i = 0; i < 32 * CONS; ++i) ok = ok && o[i] == STEPS * 4.0;
        printf("racecheck_probe: %s ring result %s\n", v ? "cp.async + mbarrier" : "bulk-copy + mbarrier",
               ok ? "correct" : "WRONG");
        all = all && ok;
    }
    return all ? 0 : 1;
}
