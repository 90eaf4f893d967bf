// tc_probe.cu -- standalone check of the tcgen05 pieces the tensor-core recursive pass 2 uses:
// A (M = 128 x K = 8, fp32 bits read as tf32) written to TMEM with tcgen05.st, B (N x K = 8) in
// shared memory in the K-major no-swizzle canonical layout (core matrices of 8 rows x 16 B, LBO =
// K-adjacent core-matrix stride, SBO = N-adjacent), D = A B^T by tcgen05.mma.kind::tf32 (A from
// TMEM), committed to an mbarrier, read back with tcgen05.ld. Test infrastructure only (not linked
// into libbfvec): nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC tc_probe.cu
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// A [128][KS*8] (row-major fp32), B [N][KS*8] (row-major fp32), D [128][N]; one CTA of 128 threads
__global__ void __launch_bounds__(128, 1) probe_kernel(const float *A, const float *B, float *D, int N, int KS) {
    __shared__ __align__(1024) float bs[64 * 40];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase_s;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int K = KS * 8;
    // B in the canonical layout: element (n, k) at ((n / 8) * (K / 4) + k / 4) * 32 + (n % 8) * 4 + k % 4 floats
    for (int e = tid; e < N * K; e += 128) {
        const int n = e / K, k = e % K;
        bs[((n / 8) * (K / 4) + k / 4) * 32 + (n % 8) * 4 + (k % 4)] = B[e];
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tbase_s)), "n"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tbase_s;
    const uint32_t ta = tbase + 128;   // A at columns [128, 128 + K)
    // A rows to TMEM: thread = row, 8 columns per store
    for (int ks = 0; ks < KS; ++ks) {
        uint32_t v[8];
        for (int j = 0; j < 8; ++j) v[j] = __float_as_uint(A[tid * K + ks * 8 + j]);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         ta + ((uint32_t)(warp * 32) << 16) + ks * 8),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        for (int ks = 0; ks < KS; ++ks) {
            const uint32_t start = sa(bs) + ks * 2 * 128;   // k-step = 2 core matrices along K
            const uint64_t lbo = 128, sbo = (uint64_t)(K / 4) * 128;
            const uint64_t desc = (uint64_t)((start >> 4) & 0x3FFF) | ((lbo >> 4) << 16) | ((sbo >> 4) << 32) |
                                  (1ull << 46);
            const uint32_t acc = ks > 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tbase),
                "r"(ta + ks * 8), "l"(desc), "r"(idesc), "r"(acc)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar))
                     : "memory");
    }
    {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], 0;\n\t"
                         "selp.b32 %0, 1, 0, q;\n\t}"
                         : "=r"(done)
                         : "r"(sa(&bar))
                         : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tbase + ((uint32_t)(warp * 32) << 16) + c0)
                     : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 8; ++j) D[tid * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(256) : "memory");
}

extern "C" int tc_probe(const float *A, const float *B, float *D, int N, int KS) {
    probe_kernel<<<1, 128>>>(A, B, D, N, KS);
    cudaError_t e = cudaDeviceSynchronize();
    return (int)e;
}
