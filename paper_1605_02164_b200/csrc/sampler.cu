// sampler.cu -- device frequency sampler (Prop. 2; Eq. (13)-(14),
// PAPER.md:144-163; Alg. 1 L221 hoisted out of the sample loop).
//
// Generator (reading R9): Philox4x64-10 (Salmon et al., SC'11), key (seed, 0);
// stream word w = lane w % 4 of the block with counter (w / 4 + 1, 0, 0, 0).
// Draw (k, c) uses word k*d + c:  X = popcount(word & (2^N - 1)) ~ B(N, 1/2),
// Y = N - 2X, and the frequency t_k = Q (Y_k o gamma), gamma = alpha / sqrt(N)
// (reading R7), accumulated in fp64 and rounded once to fp32.
#include <cuda_runtime.h>

#include "internal.h"

namespace bfvec {
namespace {

constexpr uint64_t kM0 = 0xD2E7470EE14C6C93ULL;
constexpr uint64_t kM1 = 0xCA5A826395121157ULL;
constexpr uint64_t kW0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kW1 = 0xBB67AE8584CAA73BULL;

__host__ __device__ inline void mulhilo(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
#ifdef __CUDA_ARCH__
    *lo = a * b;
    *hi = __umul64hi(a, b);
#else
    unsigned __int128 p = (unsigned __int128)a * b;
    *lo = (uint64_t)p;
    *hi = (uint64_t)(p >> 64);
#endif
}

__host__ __device__ inline void philox_block(const uint64_t ctr_in[4], const uint64_t key_in[2],
                                             uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += kW0; k1 += kW1; }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo(kM0, c0, &hi0, &lo0);
        mulhilo(kM1, c2, &hi1, &lo1);
        const uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// one thread per sample k: d words, popcounts, t_k = Q (Y o gamma)
__global__ void sampler_kernel(int M, int d, int N, uint64_t seed, const double *__restrict__ Q,
                               const double *__restrict__ gamma, int32_t *__restrict__ X,
                               float *__restrict__ t) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= M) return;
    const uint64_t mask = (N >= 64) ? ~0ULL : ((1ULL << N) - 1ULL);
    const uint64_t key[2] = {seed, 0ULL};
    double yg[kMaxD];
    uint64_t blk[4];
    long long cur = -1;
    for (int c = 0; c < d; ++c) {
        const long long w = (long long)k * d + c;
        const long long b = w >> 2;
        if (b != cur) {
            const uint64_t ctr[4] = {(uint64_t)b + 1ULL, 0ULL, 0ULL, 0ULL};
            philox_block(ctr, key, blk);
            cur = b;
        }
        const int x = __popcll(blk[w & 3] & mask);
        X[(long long)k * d + c] = x;
        yg[c] = (double)(N - 2 * x) * gamma[c];
    }
    for (int r = 0; r < d; ++r) {
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc = fma(Q[r * d + c], yg[c], acc);
        t[(long long)k * d + r] = (float)acc;
    }
}

}  // namespace

cudaError_t launch_sampler(int M, int d, int N, uint64_t seed, const double *dQ,
                           const double *dgamma, int32_t *dX, float *dt, cudaStream_t s) {
    const int threads = 128;
    sampler_kernel<<<(M + threads - 1) / threads, threads, 0, s>>>(M, d, N, seed, dQ, dgamma, dX, dt);
    return cudaGetLastError();
}

void philox4x64_10_host(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
    philox_block(ctr, key, out);
}

}  // namespace bfvec
