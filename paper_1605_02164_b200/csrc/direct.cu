// direct.cu -- the exact bilateral filter, Eq. (2)-(3), on the
// square window [-r, r]^2 with half-sample reflection (reading R1).
// Accuracy reference for the MC path (PSNR), not part of the MC hot path.
//
// phi(f_j - f_i) = exp(-(f_j - f_i)^T C^-1 (f_j - f_i) / 2) = exp2(-|u_j - u_i|^2)
// with u = sqrt(log2(e)/2) diag(alpha) Q^T f (Eq. (4)), so a
// pair costs d FSUB + d FFMA + one MUFU.EX2 + (d+1) FFMA.
#include <cuda_runtime.h>

#include "internal.h"

namespace bfvec {
namespace {

__device__ __forceinline__ int reflect_idx(int i, int n) {
    if ((unsigned)i < (unsigned)n) return i;
    int p = 2 * n;
    i %= p;
    if (i < 0) i += p;
    return i < n ? i : p - 1 - i;
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct RotArgs {
    float A[kMaxD * kMaxD];
};

// U (d, H, W) = A f, A = sqrt(log2(e)/2) diag(alpha) Q^T
__global__ void rotate_kernel(const float *__restrict__ f, int d, long long npix,
                              const __grid_constant__ RotArgs ra, float *__restrict__ U) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= npix) return;
    float fv[kMaxD];
    for (int c = 0; c < d; ++c) fv[c] = f[(long long)c * npix + e];
    for (int k = 0; k < d; ++k) {
        float u = 0.f;
        for (int c = 0; c < d; ++c) u = fmaf(ra.A[k * d + c], fv[c], u);
        U[(long long)k * npix + e] = u;
    }
}

struct DirectArgs {
    float w[kMaxR + 1];
};

template <int D>
__global__ void __launch_bounds__(256) direct_kernel(const float *__restrict__ f,
                                                     const float *__restrict__ U, int H, int W, int r,
                                                     const __grid_constant__ DirectArgs da,
                                                     float *__restrict__ out) {
    __shared__ float sw[kMaxR + 1];
    for (int i = threadIdx.x; i <= r; i += blockDim.x) sw[i] = da.w[i];
    __syncthreads();
    const int x = blockIdx.x * 32 + (threadIdx.x & 31);
    const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (x >= W || y >= H) return;
    const long long npix = (long long)H * W;
    float ui[D];
#pragma unroll
    for (int c = 0; c < D; ++c) ui[c] = U[(long long)c * npix + (long long)y * W + x];
    float num[D];
#pragma unroll
    for (int c = 0; c < D; ++c) num[c] = 0.f;
    float den = 0.f;
    for (int jy = -r; jy <= r; ++jy) {
        const int yy = reflect_idx(y - jy, H);
        const float wy = sw[jy < 0 ? -jy : jy];
        const long long rowoff = (long long)yy * W;
        for (int jx = -r; jx <= r; ++jx) {
            const int xx = reflect_idx(x - jx, W);
            const long long o = rowoff + xx;
            float q = 0.f;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const float du = __ldg(U + (long long)c * npix + o) - ui[c];
                q = fmaf(du, du, q);
            }
            const float wt = wy * sw[jx < 0 ? -jx : jx] * ex2_approx(-q);
            den += wt;
#pragma unroll
            for (int c = 0; c < D; ++c) num[c] = fmaf(wt, __ldg(f + (long long)c * npix + o), num[c]);
        }
    }
    const float rd = 1.0f / den;
#pragma unroll
    for (int c = 0; c < D; ++c) out[(long long)c * npix + (long long)y * W + x] = num[c] * rd;
}

}  // namespace

cudaError_t launch_direct(const float *f, int d, int H, int W, int r, const float *w, const float *A,
                          float *U, float *out, cudaStream_t s) {
    const long long npix = (long long)H * W;
    RotArgs ra{};
    for (int i = 0; i < d * d; ++i) ra.A[i] = A[i];
    rotate_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, s>>>(f, d, npix, ra, U);
    DirectArgs da{};
    for (int i = 0; i <= r; ++i) da.w[i] = w[i];
    dim3 grid((W + 31) / 32, (H + 7) / 8);
    switch (d) {
#define BFV_D(DD) \
    case DD: direct_kernel<DD><<<grid, 256, 0, s>>>(f, U, H, W, r, da, out); break;
        BFV_D(1) BFV_D(2) BFV_D(3) BFV_D(4) BFV_D(5) BFV_D(6) BFV_D(7) BFV_D(8)
#undef BFV_D
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace bfvec
