// color.cu -- sRGB <-> CIE-Lab (D65) around the filter: PAPER.md:305-308 ("we first performed a
// color transformation from the RGB to the CIE-Lab space, performed the filtering in the CIE-Lab
// space, and then transformed back"). Reading R18 fixes the standard: sRGB transfer of
// IEC 61966-2-1, the RGB -> XYZ matrix derived from the sRGB primaries and the D65 white point,
// CIE 1976 L*a*b* relative to that white. Planar (3, npix) fp32, one thread per pixel.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"

namespace bfvec {
namespace {

struct ColorArgs {
    float m[9];      // linear RGB -> XYZ (row-major)
    float mi[9];     // XYZ -> linear RGB
    float wn[3];     // 1 / white (Xn, Yn, Zn)
    float w[3];      // white
};

constexpr float kDelta = 6.0f / 29.0f;

__device__ __forceinline__ float to_lin(float v) {
    const float c = v * (1.0f / 255.0f);
    return c <= 0.04045f ? c * (1.0f / 12.92f) : powf((c + 0.055f) * (1.0f / 1.055f), 2.4f);
}
__device__ __forceinline__ float from_lin(float c) {
    const float s = c <= 0.0031308f ? 12.92f * c : 1.055f * copysignf(powf(fabsf(c), 1.0f / 2.4f), c) - 0.055f;
    return 255.0f * s;
}
__device__ __forceinline__ float lab_f(float t) {
    return t > kDelta * kDelta * kDelta ? cbrtf(t) : t * (1.0f / (3.0f * kDelta * kDelta)) + 4.0f / 29.0f;
}
__device__ __forceinline__ float lab_finv(float t) {
    return t > kDelta ? t * t * t : 3.0f * kDelta * kDelta * (t - 4.0f / 29.0f);
}

__global__ void srgb_to_lab_kernel(const float *__restrict__ in, float *__restrict__ out, long long n,
                                   const __grid_constant__ ColorArgs c) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float r = to_lin(in[i]), g = to_lin(in[n + i]), b = to_lin(in[2 * n + i]);
    float f[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) f[k] = lab_f((c.m[3 * k] * r + c.m[3 * k + 1] * g + c.m[3 * k + 2] * b) * c.wn[k]);
    out[i] = 116.0f * f[1] - 16.0f;
    out[n + i] = 500.0f * (f[0] - f[1]);
    out[2 * n + i] = 200.0f * (f[1] - f[2]);
}

__global__ void lab_to_srgb_kernel(const float *__restrict__ in, float *__restrict__ out, long long n,
                                   const __grid_constant__ ColorArgs c) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float fy = (in[i] + 16.0f) * (1.0f / 116.0f);
    const float xyz[3] = {c.w[0] * lab_finv(fy + in[n + i] * (1.0f / 500.0f)), c.w[1] * lab_finv(fy),
                          c.w[2] * lab_finv(fy - in[2 * n + i] * (1.0f / 200.0f))};
#pragma unroll
    for (int k = 0; k < 3; ++k)
        out[k * n + i] = from_lin(c.mi[3 * k] * xyz[0] + c.mi[3 * k + 1] * xyz[1] + c.mi[3 * k + 2] * xyz[2]);
}

// 3x3 inverse by the adjugate (fp64)
void inv3(const double *a, double *o) {
    const double det = a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
                       a[2] * (a[3] * a[7] - a[4] * a[6]);
    o[0] = (a[4] * a[8] - a[5] * a[7]) / det;
    o[1] = (a[2] * a[7] - a[1] * a[8]) / det;
    o[2] = (a[1] * a[5] - a[2] * a[4]) / det;
    o[3] = (a[5] * a[6] - a[3] * a[8]) / det;
    o[4] = (a[0] * a[8] - a[2] * a[6]) / det;
    o[5] = (a[2] * a[3] - a[0] * a[5]) / det;
    o[6] = (a[3] * a[7] - a[4] * a[6]) / det;
    o[7] = (a[1] * a[6] - a[0] * a[7]) / det;
    o[8] = (a[0] * a[4] - a[1] * a[3]) / det;
}

ColorArgs color_args() {
    // chromaticities of the sRGB primaries and of D65; XYZ at Y = 1 is (x/y, 1, (1-x-y)/y)
    const double prim[3][2] = {{0.64, 0.33}, {0.30, 0.60}, {0.15, 0.06}};
    const double wx = 0.3127, wy = 0.3290;
    const double W[3] = {wx / wy, 1.0, (1.0 - wx - wy) / wy};
    double P[9], Pi[9], S[3], M[9], Mi[9];
    for (int j = 0; j < 3; ++j) {
        P[0 * 3 + j] = prim[j][0] / prim[j][1];
        P[1 * 3 + j] = 1.0;
        P[2 * 3 + j] = (1.0 - prim[j][0] - prim[j][1]) / prim[j][1];
    }
    inv3(P, Pi);
    for (int j = 0; j < 3; ++j) S[j] = Pi[3 * j] * W[0] + Pi[3 * j + 1] * W[1] + Pi[3 * j + 2] * W[2];
    for (int r = 0; r < 3; ++r)
        for (int j = 0; j < 3; ++j) M[3 * r + j] = P[3 * r + j] * S[j];
    inv3(M, Mi);
    ColorArgs c;
    for (int i = 0; i < 9; ++i) { c.m[i] = (float)M[i]; c.mi[i] = (float)Mi[i]; }
    for (int k = 0; k < 3; ++k) { c.w[k] = (float)W[k]; c.wn[k] = (float)(1.0 / W[k]); }
    return c;
}

}  // namespace

cudaError_t launch_srgb_to_lab(const float *in, float *out, long long npix, cudaStream_t s) {
    if (npix <= 0) return cudaSuccess;
    const int threads = 256;
    srgb_to_lab_kernel<<<(unsigned)((npix + threads - 1) / threads), threads, 0, s>>>(in, out, npix, color_args());
    return cudaGetLastError();
}

cudaError_t launch_lab_to_srgb(const float *in, float *out, long long npix, cudaStream_t s) {
    if (npix <= 0) return cudaSuccess;
    const int threads = 256;
    lab_to_srgb_kernel<<<(unsigned)((npix + threads - 1) / threads), threads, 0, s>>>(in, out, npix, color_args());
    return cudaGetLastError();
}

}  // namespace bfvec
