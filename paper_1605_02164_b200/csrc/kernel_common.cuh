// kernel_common.cuh -- device helpers shared by the fused-kernel variants
// (mcsf_fused.cuh: shared-memory ring, mcsf_tmem.cuh: tensor-memory ring).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include <atomic>
#include <utility>

#include "internal.h"

namespace bfvec {
namespace {

constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }
// stride (in float2) of a `modcs` row: >= n, == 2 (mod 4) so the H-pass LDS.128
// of 8 consecutive rows hit 8 distinct 4-bank groups.
constexpr int cs_stride(int n) {
    int s = round_up(n, 2);
    while (s % 4 != 2) s += 2;
    return s;
}
// stride (in floats) of a `modf` row: >= n, == 2 (mod 4): LDS.64 of 16 consecutive rows
// hit 16 distinct 2-bank groups (an odd multiple of 2 is a bijection mod 32).
constexpr int f_stride(int n) { return cs_stride(n); }

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t saddr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Wait for the phase with the given parity to complete. try_wait with a suspend-time hint parks the
// warp in hardware until the phase completes (or the hint expires) instead of re-issuing the probe
// in a loop: the spinning modulation / consumer warps no longer take issue slots from the FIR warps
// (BRA was 13-18 % of the fused kernels' PC samples). -DBFVEC_MBAR_SPIN restores the
// plain probe loop for A/B measurements.
//
// Checked build (-DBFVEC_CHECKED, tools/checked_build.sh; the stand-in for compute-sanitizer, which
// this pool does not run): every wait has a watchdog -- a phase that does not complete within
// ~2^24 probes of <= 1 us (seconds) is a protocol deadlock: the kernel prints the barrier and
// traps instead of hanging the GPU. BF_CHECK(cond) traps with the failed condition.
#ifdef BFVEC_CHECKED
constexpr uint32_t kMbarSuspendNs = 1000;
#define BF_CHECK(cond)                                                                                     \
    do {                                                                                                   \
        if (!(cond)) {                                                                                     \
            printf("BF_CHECK failed: %s (%s:%d) block (%d,%d,%d) thread %d\n", #cond, __FILE__, __LINE__,    \
                   blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x);                                       \
            __trap();                                                                                      \
        }                                                                                                  \
    } while (0)
#else
constexpr uint32_t kMbarSuspendNs = 0x989680;   // 10 ms upper bound; the phase completion wakes the warp
#define BF_CHECK(cond) \
    do {               \
    } while (0)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
#ifdef BFVEC_CHECKED
    uint32_t probes = 0;
#endif
    do {
#ifdef BFVEC_CHECKED
        if (++probes == (1u << 24)) {
            printf("mbar_wait watchdog: barrier %p parity %u never completed (block (%d,%d,%d) thread %d)\n",
                   (void *)bar, parity, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x);
            __trap();
        }
#endif
#ifdef BFVEC_MBAR_SPIN
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(saddr(bar)), "r"(parity)
            : "memory");
#else
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(saddr(bar)), "r"(parity), "r"(kMbarSuspendNs)
            : "memory");
#endif
    } while (!done);
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(saddr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(saddr(bar))
        : "memory");
}

template <class F, int... Js>
__device__ __forceinline__ void static_for_impl(F &&f, std::integer_sequence<int, Js...>) {
    (f(std::integral_constant<int, Js>{}), ...);
}
// compile-time loop: f(std::integral_constant<int, j>) for j = 0..N-1, always fully
// expanded (NVVM's unroller gives up on the larger FIR bodies, which would turn the
// taps into runtime constant loads)
template <int N, class F>
__device__ __forceinline__ void static_for(F &&f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

__device__ __forceinline__ float2 ffma2(float w, float2 v, float2 acc) {
    return __ffma2_rn(make_float2(w, w), v, acc);
}

// Opt a kernel into `bytes` of dynamic shared memory once per device (the attribute is per
// function and per device; one process may drive several devices through the C ABI).
template <class K>
cudaError_t ensure_smem_attr(K kernel, size_t bytes, std::atomic<uint64_t> &done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
template <int N>
__device__ __forceinline__ void named_sync(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(N) : "memory");
}

}  // namespace
}  // namespace bfvec
