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

// ---------------------------------------------------------------------------------------------
// Stratified draws (option "sampler" = 1, reading R17; the paper's future work "improving the
// Monte Carlo integration"): per dimension c a Latin-hypercube stratification of
// the binomial CDF -- sample k takes stratum pi_c(k) of M equal strata of [0, 1), where pi_c is
// the rank of word (k d + c) of key (seed, 1) among the M words of dimension c (ties by k), and
//   u = (pi_c(k) + (word (k d + c) of key (seed, 2) >> 11) 2^-53) / M,
//   X = min { n < N : u < cum(n) 2^-N } (else N),  cum(n) = sum_{m <= n} C(N, m),
// all in IEEE fp64 with explicit rounding (the oracle repeats the same operations).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t philox_word(uint64_t seed, uint64_t kw, long long w) {
    const uint64_t ctr[4] = {(uint64_t)(w >> 2) + 1ULL, 0ULL, 0ULL, 0ULL};
    const uint64_t key[2] = {seed, kw};
    uint64_t blk[4];
    philox_block(ctr, key, blk);
    return blk[w & 3];
}

__global__ void strat_keys_kernel(long long n, uint64_t seed, uint64_t *__restrict__ keys) {
    const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (w < n) keys[w] = philox_word(seed, 1ULL, w);
}

__global__ void strat_sampler_kernel(int M, int d, int N, uint64_t seed, const uint64_t *__restrict__ keys,
                                     CumTable cum, const double *__restrict__ Q,
                                     const double *__restrict__ gamma, int32_t *__restrict__ X,
                                     float *__restrict__ t) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= M) return;
    double yg[kMaxD];
    const double scale = ldexp(1.0, -N);
    for (int c = 0; c < d; ++c) {
        const uint64_t mine = keys[(long long)k * d + c];
        long long rank = 0;
        for (int j = 0; j < M; ++j) {
            const uint64_t o = keys[(long long)j * d + c];
            rank += (o < mine || (o == mine && j < k)) ? 1 : 0;
        }
        const uint64_t v = philox_word(seed, 2ULL, (long long)k * d + c);
        const double u = __ddiv_rn(__dadd_rn((double)rank, __dmul_rn((double)(v >> 11), 0x1p-53)), (double)M);
        int x = N;
        for (int n = 0; n < N; ++n)
            if (u < __dmul_rn(__ull2double_rn(cum.v[n]), scale)) { x = n; break; }
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

cudaError_t launch_sampler_stratified(int M, int d, int N, uint64_t seed, const double *dQ, const double *dgamma,
                                      uint64_t *dkeys, int32_t *dX, float *dt, cudaStream_t s) {
    // cum(n) = sum_{m <= n} C(N, m), exact in 128-bit integers (cum(n) < 2^64 for n < N <= 64)
    CumTable cum;
    unsigned __int128 c = 1, acc = 0;
    for (int n = 0; n <= 64; ++n) {
        if (n <= N) {
            acc += c;
            cum.v[n] = (n < N) ? (uint64_t)acc : ~0ULL;
            c = c * (unsigned __int128)(N - n) / (unsigned __int128)(n + 1);
        } else {
            cum.v[n] = ~0ULL;
        }
    }
    const long long n = (long long)M * d;
    const int threads = 128;
    strat_keys_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(n, seed, dkeys);
    strat_sampler_kernel<<<(M + threads - 1) / threads, threads, 0, s>>>(M, d, N, seed, dkeys, cum, dQ, dgamma, dX,
                                                                         dt);
    return cudaGetLastError();
}

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
