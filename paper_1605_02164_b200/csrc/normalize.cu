// normalize.cu -- epilogues of the MCSF path.
//   normalize_groups : Alg. 1 L231 S_c = P_c / Z with the real-part
//                      convention (reading R4), summing the per-sample-group
//                      partials in a fixed order (deterministic), undoing the
//                      centring (S[f] = S[f - mu] + mu, reading R12), float4 stores.
//   finalize_partial : raw, uncentred (P_c, Z) sums for sample sharding.
//   normalize_raw    : S_c = P_c / Z from raw sums (after the NCCL reduction).
// All three record the small-Z diagnostics (reading R5): min Z/M and
// #{Z/M < z_floor}.
#include <cuda_runtime.h>

#include "internal.h"

namespace bfvec {
namespace {

__device__ __forceinline__ unsigned int ordered(float v) {
    const unsigned int u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ void record_diag(unsigned long long *diag, float zm, float z_floor, bool valid) {
    const unsigned int key = valid ? ordered(zm) : 0xFFFFFFFFu;
    unsigned int mn = key;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    const unsigned int small = __ballot_sync(0xffffffffu, valid && zm < z_floor);
    if ((threadIdx.x & 31) == 0) {
        if (mn != 0xFFFFFFFFu) atomicMin(reinterpret_cast<unsigned int *>(diag), mn);
        if (small) atomicAdd(diag + 1, (unsigned long long)__popc(small));
    }
}

template <int VEC>
__global__ void normalize_groups_kernel(const float *__restrict__ pz, int groups, int D, int d,
                                        long long npix, const float *__restrict__ mu_dev,
                                        float mu0, float mu1, float mu2, float mu3, float mu4,
                                        float mu5, float mu6, float mu7, float *__restrict__ out,
                                        unsigned long long *diag, float inv_m, float z_floor, int W,
                                        const int *__restrict__ strip_slots) {
    const float mu[8] = {mu0, mu1, mu2, mu3, mu4, mu5, mu6, mu7};
    (void)mu_dev;
    const long long e = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * VEC;
    const bool valid = e < npix;
    const long long gstride = (long long)(D + 1) * npix;
    // persistent schedule: the slots written for this pixel's 32-column strip (a VEC group never
    // straddles strips: VEC = 4 needs W % 4 == 0)
    if (strip_slots && valid) groups = strip_slots[(int)(e % W) >> 5];
    float z[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) z[v] = 0.f;
    if (valid) {
        for (int g = 0; g < groups; ++g) {
            const float *p = pz + g * gstride + (long long)D * npix + e;
            if (VEC == 4) {
                const float4 q = *reinterpret_cast<const float4 *>(p);
                z[0] += q.x; z[VEC > 1 ? 1 : 0] += q.y; z[VEC > 2 ? 2 : 0] += q.z; z[VEC > 3 ? 3 : 0] += q.w;
            } else {
                z[0] += p[0];
            }
        }
    }
    float zmin = 3.4e38f;
#pragma unroll
    for (int v = 0; v < VEC; ++v) zmin = fminf(zmin, z[v] * inv_m);
    // per-pixel small-Z counting: count each of the VEC pixels
    int nsmall = 0;
#pragma unroll
    for (int v = 0; v < VEC; ++v) nsmall += (valid && z[v] * inv_m < z_floor) ? 1 : 0;
    {
        const unsigned int key = valid ? ordered(zmin) : 0xFFFFFFFFu;
        unsigned int mn = key;
        int cnt = nsmall;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
        if ((threadIdx.x & 31) == 0) {
            if (mn != 0xFFFFFFFFu) atomicMin(reinterpret_cast<unsigned int *>(diag), mn);
            if (cnt) atomicAdd(diag + 1, (unsigned long long)cnt);
        }
    }
    if (!valid) return;
    float rz[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) rz[v] = 1.0f / z[v];
    for (int c = 0; c < d; ++c) {
        float p[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) p[v] = 0.f;
        for (int g = 0; g < groups; ++g) {
            const float *src = pz + g * gstride + (long long)c * npix + e;
            if (VEC == 4) {
                const float4 q = *reinterpret_cast<const float4 *>(src);
                p[0] += q.x; p[VEC > 1 ? 1 : 0] += q.y; p[VEC > 2 ? 2 : 0] += q.z; p[VEC > 3 ? 3 : 0] += q.w;
            } else {
                p[0] += src[0];
            }
        }
        float *dst = out + (long long)c * npix + e;
        if (VEC == 4) {
            *reinterpret_cast<float4 *>(dst) =
                make_float4(p[0] * rz[0] + mu[c], p[VEC > 1 ? 1 : 0] * rz[VEC > 1 ? 1 : 0] + mu[c],
                            p[VEC > 2 ? 2 : 0] * rz[VEC > 2 ? 2 : 0] + mu[c],
                            p[VEC > 3 ? 3 : 0] * rz[VEC > 3 ? 3 : 0] + mu[c]);
        } else {
            dst[0] = p[0] * rz[0] + mu[c];
        }
    }
}

__global__ void finalize_partial_kernel(const float *__restrict__ pz, int groups, int D, int d,
                                        int rows, int W, float mu0, float mu1, float mu2,
                                        float mu3, float mu4, float mu5, float mu6, float mu7,
                                        int rpb, float *__restrict__ PZ,
                                        const int *__restrict__ strip_slots) {
    const float mu[8] = {mu0, mu1, mu2, mu3, mu4, mu5, mu6, mu7};
    const long long npix = (long long)rows * W;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= npix) return;
    if (strip_slots) groups = strip_slots[(int)(e % W) >> 5];   // persistent schedule
    const long long gstride = (long long)(D + 1) * npix;
    float z = 0.f;
    for (int g = 0; g < groups; ++g) z += pz[g * gstride + (long long)D * npix + e];
    const int y = (int)(e / W), x = (int)(e - (long long)y * W);
    const int b = y / rpb;
    const int brows = min(rpb, rows - b * rpb);
    float *base = PZ + (long long)b * rpb * (d + 1) * W;
    const long long inrow = (long long)(y - b * rpb) * W + x;
    for (int c = 0; c < d; ++c) {
        float p = 0.f;
        for (int g = 0; g < groups; ++g) p += pz[g * gstride + (long long)c * npix + e];
        base[(long long)c * brows * W + inrow] = fmaf(mu[c], z, p);      // P = P' + mu Z
    }
    base[(long long)d * brows * W + inrow] = z;
}

__global__ void normalize_raw_kernel(const float *__restrict__ PZ, int d, long long npix,
                                     float *__restrict__ out, unsigned long long *diag,
                                     float inv_m, float z_floor) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = e < npix;
    const float z = valid ? PZ[(long long)d * npix + e] : 1.f;
    record_diag(diag, z * inv_m, z_floor, valid);
    if (!valid) return;
    const float rz = 1.0f / z;
    for (int c = 0; c < d; ++c) out[(long long)c * npix + e] = PZ[(long long)c * npix + e] * rz;
}

__global__ void diag_reset_kernel(unsigned long long *diag) {
    reinterpret_cast<unsigned int *>(diag)[0] = 0xFFFFFFFFu;
    reinterpret_cast<unsigned int *>(diag)[1] = 0u;
    diag[1] = 0ULL;
}

}  // namespace

cudaError_t launch_normalize_groups(const float *pz, int groups, int D, int d, int rows, int W,
                                    const float *mu, float *out, float *diag, float inv_m,
                                    float z_floor, cudaStream_t s, const int *strip_slots) {
    const long long npix = (long long)rows * W;
    const int threads = 256;
    auto dg = reinterpret_cast<unsigned long long *>(diag);
    // float4 path only when every row starts 16-byte aligned in both buffers (out is the caller's
    // pointer: a view may start anywhere; the scalar path serves the rest)
    const bool vec_ok = W % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                        (reinterpret_cast<uintptr_t>(pz) & 15) == 0;
    if (vec_ok) {
        const long long n = npix / 4;
        normalize_groups_kernel<4><<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(
            pz, groups, D, d, npix, nullptr, mu[0], mu[1], mu[2], mu[3], mu[4], mu[5], mu[6], mu[7],
            out, dg, inv_m, z_floor, W, strip_slots);
    } else {
        normalize_groups_kernel<1><<<(unsigned)((npix + threads - 1) / threads), threads, 0, s>>>(
            pz, groups, D, d, npix, nullptr, mu[0], mu[1], mu[2], mu[3], mu[4], mu[5], mu[6], mu[7],
            out, dg, inv_m, z_floor, W, strip_slots);
    }
    return cudaGetLastError();
}

cudaError_t launch_finalize_partial(const float *pz, int groups, int D, int d, int rows, int W,
                                    const float *mu, int rows_per_band, float *PZ, cudaStream_t s,
                                    const int *strip_slots) {
    const long long npix = (long long)rows * W;
    const int threads = 256;
    finalize_partial_kernel<<<(unsigned)((npix + threads - 1) / threads), threads, 0, s>>>(
        pz, groups, D, d, rows, W, mu[0], mu[1], mu[2], mu[3], mu[4], mu[5], mu[6], mu[7],
        rows_per_band, PZ, strip_slots);
    return cudaGetLastError();
}

cudaError_t launch_normalize_raw(const float *PZ, int d, int rows, int W, float *out, float *diag,
                                 float inv_m, float z_floor, cudaStream_t s) {
    const long long npix = (long long)rows * W;
    const int threads = 256;
    normalize_raw_kernel<<<(unsigned)((npix + threads - 1) / threads), threads, 0, s>>>(
        PZ, d, npix, out, reinterpret_cast<unsigned long long *>(diag), inv_m, z_floor);
    return cudaGetLastError();
}

cudaError_t launch_diag_reset(float *diag, cudaStream_t s) {
    diag_reset_kernel<<<1, 1, 0, s>>>(reinterpret_cast<unsigned long long *>(diag));
    return cudaGetLastError();
}

}  // namespace bfvec
