// pad.cu -- prepares the input of the fused kernel's TMA loads: a reflect-padded,
// centred, pixel-interleaved copy of the (slab of the) image.
//   fpad[yp][xp][0..DP) = f(rho_H(row_begin + yp) - slab_row0, rho_W(xp - R))[c] - mu_c  (c < d)
//                         0                                                          (d <= c < DP)
// rho = half-sample reflection about the FULL image (reading R1); TMA has no
// reflect mode, so the boundary is baked in here. Centring by mu is the exact
// invariance S[f - mu] + mu = S[f] (reading R12). One pass over f: HBM-bound.
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

template <int DP>
__global__ void pad_kernel(const float *__restrict__ f, long long plane, int d, int H, int W, int slab_row0,
                           int slab_rows, int row_begin, int Hp, int Wp, int R, PadMu mu,
                           float *__restrict__ fpad) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)Hp * Wp) return;
    const int yp = (int)(e / Wp), xp = (int)(e - (long long)yp * Wp);
    const int y = min(max(reflect_idx(row_begin + yp, H) - slab_row0, 0), slab_rows - 1);
    const int x = reflect_idx(xp - R, W);
    const float *src = f + (long long)y * W + x;
    float v[DP];
#pragma unroll
    for (int c = 0; c < DP; ++c) v[c] = (c < d) ? __ldg(src + c * plane) - mu.v[c] : 0.f;
    float4 *dst = reinterpret_cast<float4 *>(fpad + e * DP);
#pragma unroll
    for (int c = 0; c < DP; c += 4) dst[c / 4] = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
}

}  // namespace

cudaError_t launch_pad(const float *f, long long plane, int d, int H, int W, int slab_row0, int slab_rows,
                       int row_begin, int Hp, int Wp, int R, int DP, const float *mu, float *fpad,
                       cudaStream_t s) {
    PadMu m{};
    for (int c = 0; c < kMaxD; ++c) m.v[c] = mu[c];
    const long long n = (long long)Hp * Wp;
    const int threads = 256;
    const unsigned blocks = (unsigned)((n + threads - 1) / threads);
    if (DP == 4)
        pad_kernel<4><<<blocks, threads, 0, s>>>(f, plane, d, H, W, slab_row0, slab_rows, row_begin, Hp, Wp, R, m, fpad);
    else
        pad_kernel<8><<<blocks, threads, 0, s>>>(f, plane, d, H, W, slab_row0, slab_rows, row_begin, Hp, Wp, R, m, fpad);
    return cudaGetLastError();
}

}  // namespace bfvec
