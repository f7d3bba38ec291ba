// aux_kernels.cuh -- transition matrices (A1) and the site/branch reduction (A6).
#pragma once
#include "common.cuh"

namespace pg {

// A1 -- Eq. 1: P^{(r)}(b_i) = V diag(exp(gamma_r b_i lambda)) V^{-1}
// for every branch i and category r, in the compute precision, zero padded to
// SP x SP (category blocks `cs` Reals apart).  One CTA per (branch, category): the S exponentials go to shared
// memory, then every thread forms entries of P and (optionally) P'.  Padded
// rows/columns are exactly 0.  The work is ~2% of an evaluation.
template <typename Real, int SP>
__global__ void __launch_bounds__(256) pmat_kernel(const double *__restrict__ V,
                                                   const double *__restrict__ Vi,
                                                   const double *__restrict__ lam,
                                                   const double *__restrict__ rates,
                                                   const double *__restrict__ bl, int S, int R,
                                                   int cs, Real *__restrict__ P, Real *__restrict__ PT) {
    __shared__ double e[SP];
    const int br = blockIdx.x;          // branch * R + r
    const int r = br % R, b = br / R;
    const double t = rates[r] * bl[b];
    for (int k = threadIdx.x; k < SP; k += blockDim.x) e[k] = k < S ? exp(lam[k] * t) : 0.0;
    __syncthreads();
    Real *Pm = P + (size_t)br * cs;     // cs = category stride (>= SP*SP, zero padded)
    Real *PTm = PT ? PT + (size_t)br * SP * SP : nullptr;
    for (int idx = threadIdx.x; idx < SP * SP; idx += blockDim.x) {
        const int s = idx / SP, u = idx % SP;
        double acc = 0.0;
        if (s < S && u < S)
            for (int k = 0; k < S; ++k) acc += V[s * S + k] * e[k] * Vi[k * S + u];
        Pm[idx] = (Real)acc;
        if (PTm) PTm[u * SP + s] = (Real)acc;
    }
}

// A6 -- Eq. 6 column sum, deterministic: block b < B sums the
// per-tile gradient partials of branch b, block B the per-tile logL partials,
// in a fixed order (strided serial sums, then a fixed smem tree).  No atomics,
// so fp64 results are bitwise reproducible run to run.
__global__ void __launch_bounds__(256) reduce_kernel(const double *__restrict__ grad_part,
                                                     const double *__restrict__ logl_part,
                                                     int B, int n_tiles, double *__restrict__ out) {
    __shared__ double sh[256];
    const int b = blockIdx.x;
    const double *src = (b < B) ? grad_part + (size_t)b * n_tiles : logl_part;
    double acc = 0.0;
    for (int i = threadIdx.x; i < n_tiles; i += blockDim.x) acc += src[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[b < B ? 1 + b : 0] = sh[0];
}

}  // namespace pg
