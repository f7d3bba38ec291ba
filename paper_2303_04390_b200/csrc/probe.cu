// probe.cu -- measurement helper for bench.py (not part of the hot path or
// of the C ABI in include/phylograd.h): the FP64 roofline denominators of
// the codon path, measured on the GPU the bench runs on, inside the bench
// run (MEASURED_PEAKS.json has no FP64 entry).
//   * DMMA: mma.sync.aligned.m8n8k4.f64 (SASS DMMA.8x8x4), 8 independent
//     accumulators per warp, 4 CTAs of 8 warps per SM;
//   * DFMA: 16 independent fma chains per thread.
// Each kernel is repeated until ~`ms_target` ms have elapsed; the best
// single-launch rate is returned (TFLOP/s).
#include <cuda_runtime.h>

namespace {

__global__ void probe_dfma(double *out, int iters) {
    double a[16];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    double s = 0;
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 12345.678) out[0] = s;
}

__global__ void probe_dmma(double *out, int iters) {
    double acc[8][2];
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    const double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[i][0]), "+d"(acc[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[0] = s;
}

}  // namespace

extern "C" int pgprobe_fp64_peak(int device, float ms_target, double *dmma_tflops, double *dfma_tflops,
                                 int *launches) {
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double *out = nullptr;
    if (cudaMalloc(&out, 8) != cudaSuccess) return 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 4, threads = 256, iters = 20000;
    const double fl_dfma = 2.0 * 16 * (double)iters * blocks * threads;
    const double fl_dmma = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
    float best[2] = {1e30f, 1e30f}, spent = 0.f;
    int n = 0;
    while (n < 4 || spent < ms_target) {
        for (int k = 0; k < 2; ++k) {
            cudaEventRecord(e0);
            if (k == 0) probe_dmma<<<blocks, threads>>>(out, iters);
            else probe_dfma<<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            best[k] = ms < best[k] ? ms : best[k];
            spent += ms;
            ++n;
        }
        if (n > 400) break;
    }
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return 3;
    *dmma_tflops = fl_dmma / best[0] / 1e9;
    *dfma_tflops = fl_dfma / best[1] / 1e9;
    if (launches) *launches = n;
    return 0;
}
