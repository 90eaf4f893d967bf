// tmem_test.cu -- validates the TMEM usage the v4 fused kernel relies on:
//  * tcgen05.alloc / relinquish / dealloc (one warp)
//  * tcgen05.st.32x32b.x16 from warp w lands in lanes 32*(w%4)+laneid
//  * producer warp (quarter q) stores, mbarrier handoff with tcgen05 fences,
//    consumer warp of the same quarter loads (.32x32b.x16 / .x32) and checks
//  * 8x8 float2 shuffle transpose inside groups of 8 lanes
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tmem_kernel(int *err, float *dump) {
    __shared__ uint32_t taddr_s;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(saddr(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(&bar)), "r"(128));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = taddr_s;
    // ---- producers: warps 0..3 (quarter q = warp); each thread builds an 8x8 float2 block row
    if (warp < 4) {
        const int q = warp;
        const int r = lane & 7, cg = lane >> 3;
        float2 A[8];
        for (int o = 0; o < 8; ++o)              // value(row r, col cg*8+o) for pair q
            A[o] = make_float2(1000.f * q + 32.f * r + (cg * 8 + o), -(1000.f * q + 32.f * r + (cg * 8 + o)));
        // transpose within groups of 8 lanes: lane (cg, o') ends with rows 0..7 of col cg*8+o'
#pragma unroll
        for (int s = 4; s >= 1; s >>= 1) {
            const bool upper = (r & s) != 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if ((i & s) == 0) {
                    float2 send = upper ? A[i] : A[i + s];
                    float2 recv;
                    recv.x = __shfl_xor_sync(0xffffffffu, send.x, s);
                    recv.y = __shfl_xor_sync(0xffffffffu, send.y, s);
                    if (upper) A[i] = recv; else A[i + s] = recv;
                }
            }
        }
        // lane x = cg*8 + r now holds rows 0..7 of column x: store 16 columns at col offset 16*q2
        uint32_t v[16];
        for (int i = 0; i < 8; ++i) { v[2 * i] = __float_as_uint(A[i].x); v[2 * i + 1] = __float_as_uint(A[i].y); }
        const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + 32;   // column 32
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                       "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&bar)));
    } else {
        // ---- consumers: warps 4..7, quarter q = warp % 4
        const int q = warp & 3;
        uint32_t done = 0;
        do {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(saddr(&bar)));
        } while (!done);
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint32_t v[16];
        const uint32_t ta = tbase + ((uint32_t)(32 * q) << 16) + 32;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(ta));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        const int x = lane;   // column
        for (int rr = 0; rr < 8; ++rr) {
            const float ex = 1000.f * q + 32.f * rr + x;
            const float gx = __uint_as_float(v[2 * rr]), gy = __uint_as_float(v[2 * rr + 1]);
            if (gx != ex || gy != -ex) atomicAdd(err, 1);
            dump[(q * 32 + x) * 16 + 2 * rr] = gx;
            dump[(q * 32 + x) * 16 + 2 * rr + 1] = gy;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tbase));
}

int main() {
    int *err; float *dump;
    cudaMalloc(&err, 4); cudaMemset(err, 0, 4);
    cudaMalloc(&dump, 128 * 16 * 4);
    tmem_kernel<<<148, 256>>>(err, dump);
    cudaError_t e = cudaDeviceSynchronize();
    int h = -1;
    cudaMemcpy(&h, err, 4, cudaMemcpyDeviceToHost);
    float d[8];
    cudaMemcpy(d, dump + (1 * 32 + 5) * 16, 32, cudaMemcpyDeviceToHost);
    printf("cuda: %s  mismatches: %d  sample q1 x5: %.0f %.0f %.0f %.0f\n", cudaGetErrorString(e), h, d[0], d[1], d[2], d[3]);
    return (e == cudaSuccess && h == 0) ? 0 : 1;
}
