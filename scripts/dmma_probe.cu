// dmma_probe.cu -- how fast can the codon GEMM inner loop run on this B200?
// Variants of a [32 x 64] x [64 x 8]-per-warp DMMA loop (the codon kernels'
// shape): accumulators per warp, A from registers or shared memory, CTAs/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_probe scripts/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int MT, bool SMEM_A>
__global__ void gemm_probe(double *out, int iters) {
    extern __shared__ double As[];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < MT * 16 * 32; i += blockDim.x) As[i] = 1e-3 * (i & 63);
    __syncthreads();
    double b[16];
#pragma unroll
    for (int kt = 0; kt < 16; ++kt) b[kt] = 1e-3 * (kt + lane);
    double acc[MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kt = 0; kt < 16; ++kt)
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const double av = SMEM_A ? As[(m * 16 + kt) * 32 + lane] : 1e-3 * (m + kt);
                dmma(acc[m], av, b[kt]);
            }
    }
    double s = 0;
#pragma unroll
    for (int m = 0; m < MT; ++m) s += acc[m][0] + acc[m][1];
    if (s == 12345.678) out[0] = s;
}

template <int MT, bool SMEM_A>
void run(const char *name, int ctas_per_sm, int warps, int sms, double *out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int smem = MT * 16 * 32 * 8;
    cudaFuncSetAttribute(gemm_probe<MT, SMEM_A>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 400;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        gemm_probe<MT, SMEM_A><<<sms * ctas_per_sm, warps * 32, smem>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double flops = 2.0 * 256 * 16 * MT * (double)iters * sms * ctas_per_sm * warps;
    printf("%-28s ctas/SM %d warps %2d: %6.2f TF/s\n", name, ctas_per_sm, warps, flops / best / 1e9);
}

int main() {
    double *out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int c : {1, 2, 3, 4}) {
        run<4, false>("4 acc, A regs", c, 8, sms, out);
        run<4, true>("4 acc, A smem", c, 8, sms, out);
        run<8, true>("8 acc, A smem", c, 8, sms, out);
        run<2, true>("2 acc, A smem", c, 8, sms, out);
    }
    return 0;
}
