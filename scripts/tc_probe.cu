// tc_probe.cu -- validates the tcgen05 building block of the fp32 codon path
// (traverse_tc.cuh): C[128 x 64] = A[128 x 64] B[64 x 64] on the 5th-gen
// tensor cores, kind::tf32, A and B K-major in the SWIZZLE_NONE canonical
// layout (8-row x 16-byte core matrices), D in TMEM, read back with
// tcgen05.ld 32x32b.x64 (thread = row); 1xTF32 and 3xTF32 (hi/lo split)
// against an fp64 host product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tc_probe scripts/tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#include "../paper_2303_04390_b200/csrc/tc_common.cuh"

using namespace pg::tc;

__global__ void probe(const float *A, const float *B, float *C, int split) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float *Ahi = reinterpret_cast<float *>(sm), *Alo = Ahi + 128 * 64, *Bhi = Alo + 128 * 64, *Blo = Bhi + 64 * 64;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;
    // operands into the canonical layout, hi/lo split
    for (int i = tid; i < 128 * 64; i += blockDim.x) {
        const int m = i / 64, k = i % 64;
        const float v = A[i], h = tf32_hi(v);
        Ahi[kmajor_off(m, k, 64) / 4] = h;
        Alo[kmajor_off(m, k, 64) / 4] = v - h;
    }
    for (int i = tid; i < 64 * 64; i += blockDim.x) {
        const int k = i / 64, n = i % 64;                       // B[k][n] row-major input; K-major image [n][k]
        const float v = B[i], h = tf32_hi(v);
        Bhi[kmajor_off(n, k, 64) / 4] = h;
        Blo[kmajor_off(n, k, 64) / 4] = v - h;
    }
    if (warp == 0) tmem_alloc<64>(&tmem_base);
    if (tid == 0) { pg::mbar_init(&bar, 1); pg::fence_mbar_init(); }
    fence_async_smem();                                         // generic smem writes -> tensor core reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t d = tmem_base;
    if (tid == 0) {
        const uint32_t idesc = idesc_tf32(128, 64);
        const uint32_t a0 = pg::smem_u32(Ahi), a1 = pg::smem_u32(Alo), b0 = pg::smem_u32(Bhi), b1 = pg::smem_u32(Blo);
        int first = 1;
        for (int kk = 0; kk < 8; ++kk) {
            mma_tf32(d, sdesc(a0 + 256 * kk, 128, 2048), sdesc(b0 + 256 * kk, 128, 2048), idesc, !first);
            first = 0;
            if (split) {
                mma_tf32(d, sdesc(a0 + 256 * kk, 128, 2048), sdesc(b1 + 256 * kk, 128, 2048), idesc, 1);
                mma_tf32(d, sdesc(a1 + 256 * kk, 128, 2048), sdesc(b0 + 256 * kk, 128, 2048), idesc, 1);
            }
        }
        mma_commit(&bar);
    }
    pg::mbar_wait(&bar, 0);
    tc_fence_after();
    float r[64];
    tmem_ld64(d + ((uint32_t)(32 * warp) << 16), r);
    const int m = 32 * warp + (tid & 31);
    for (int n = 0; n < 64; ++n) C[m * 64 + n] = r[n];
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_free<64>(d);
}

int main() {
    std::mt19937 g(7);
    std::uniform_real_distribution<float> U(0.f, 1.f);
    std::vector<float> A(128 * 64), B(64 * 64), C(128 * 64);
    for (auto &x : A) x = U(g);
    for (auto &x : B) x = U(g) * 1e-3f;
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const int smem = (2 * 128 * 64 + 2 * 64 * 64) * 4;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int rc = 0;
    for (int split = 0; split < 2; ++split) {
        cudaMemset(dC, 0, C.size() * 4);
        probe<<<1, 128, smem>>>(dA, dB, dC, split);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        double maxrel = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 64; ++n) {
                double ref = 0;
                for (int k = 0; k < 64; ++k) ref += (double)A[m * 64 + k] * B[k * 64 + n];
                maxrel = fmax(maxrel, fabs(C[m * 64 + n] - ref) / fabs(ref));
            }
        printf("tc_probe %s: max rel err %.3e\n", split ? "3xTF32" : "1xTF32", maxrel);
        if (maxrel > (split ? 1e-5 : 5e-3)) rc = 1;
    }
    printf("tc_probe %s\n", rc ? "FAILED" : "ok");
    return rc;
}
