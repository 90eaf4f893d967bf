// sweep.cu -- the on-device error-vs-T experiment (Fig. 5; Eq. (20) at
// PAPER.md:254-256): after each checkpoint T_j of a Monte Carlo realisation, fold the new
// samples' partial sums into running (P', Z) planes, form S = P'/Z + mu (Alg. 1, readings
// R4 / R12) and reduce sum_c sum_i (B_c(i) - S_c(i))^2 against the exact filter B, all in one
// pass over the image.
#include <cuda_runtime.h>

#include "internal.h"

namespace bfvec {
namespace {

__global__ void mse_accum_kernel(const float *__restrict__ pz, int groups, int D, int d, long long npix,
                                 MuArg mu, float *__restrict__ run, int first, const float *__restrict__ ref,
                                 double *__restrict__ out) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double err = 0.0;
    if (e < npix) {
        const long long gstride = (long long)(D + 1) * npix;
        float z = first ? 0.f : run[(long long)d * npix + e];
        for (int g = 0; g < groups; ++g) z += pz[g * gstride + (long long)D * npix + e];
        run[(long long)d * npix + e] = z;
        const float rz = 1.0f / z;
        for (int c = 0; c < d; ++c) {
            float p = first ? 0.f : run[(long long)c * npix + e];
            for (int g = 0; g < groups; ++g) p += pz[g * gstride + (long long)c * npix + e];
            run[(long long)c * npix + e] = p;
            const double diff = (double)ref[(long long)c * npix + e] - (double)(p * rz + mu.v[c]);
            err += diff * diff;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
    __shared__ double part[32];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) part[w] = err;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += part[i];
        atomicAdd(out, s);
    }
}

// one (pixel block, realisation) per CTA: fold realisation r's partial planes into its running sums,
// S_r = P'_r / Z_r + mu, and add sum_c (ref - S_r)^2 to out[r]
__global__ void mse_accum_batch_kernel(const float *__restrict__ pz, int D, int d, long long npix, MuArg mu,
                                       float *__restrict__ run, int first, const float *__restrict__ ref,
                                       double *__restrict__ out) {
    const int r = blockIdx.y;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const float *pr = pz + (long long)r * (D + 1) * npix;
    float *rr = run + (long long)r * (d + 1) * npix;
    double err = 0.0;
    if (e < npix) {
        const float z = (first ? 0.f : rr[(long long)d * npix + e]) + pr[(long long)D * npix + e];
        rr[(long long)d * npix + e] = z;
        const float rz = 1.0f / z;
        for (int c = 0; c < d; ++c) {
            const float p = (first ? 0.f : rr[(long long)c * npix + e]) + pr[(long long)c * npix + e];
            rr[(long long)c * npix + e] = p;
            const double diff = (double)ref[(long long)c * npix + e] - (double)(p * rz + mu.v[c]);
            err += diff * diff;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) err += __shfl_xor_sync(0xffffffffu, err, o);
    __shared__ double part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = err;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += part[i];
        atomicAdd(out + r, s);
    }
}

}  // namespace

cudaError_t launch_mse_accum_batch(const float *pz, int nr, int D, int d, long long npix, const float *mu,
                                   float *run, int first, const float *ref, double *out, cudaStream_t s) {
    MuArg m;
    for (int c = 0; c < kMaxD; ++c) m.v[c] = mu[c];
    const int threads = 256;
    dim3 grid((unsigned)((npix + threads - 1) / threads), (unsigned)nr);
    mse_accum_batch_kernel<<<grid, threads, 0, s>>>(pz, D, d, npix, m, run, first, ref, out);
    return cudaGetLastError();
}

cudaError_t launch_mse_accum(const float *pz, int groups, int D, int d, long long npix, const float *mu,
                             float *run, int first, const float *ref, double *out, cudaStream_t s) {
    MuArg m;
    for (int c = 0; c < kMaxD; ++c) m.v[c] = mu[c];
    const int threads = 256;
    mse_accum_kernel<<<(unsigned)((npix + threads - 1) / threads), threads, 0, s>>>(pz, groups, D, d, npix, m, run,
                                                                                    first, ref, out);
    return cudaGetLastError();
}

}  // namespace bfvec
