// peaks.cu -- microbenchmarks of the pipes the MCSF kernel is bound by:
// FP32 FFMA (register and uniform/constant operand), packed FFMA2 (fma.rn.f32x2),
// MUFU sin/cos, LDS.128. Prints lane-ops per SM clock and per second.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_ffma(float *out, float a, float b, long long *cyc) {
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma_reg(float *out, float a, float b, long long *cyc) {
    float x[16], y[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { x[i] = threadIdx.x * 1e-3f + i; y[i] = a + i * 1e-4f; }
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], y[i], x[(i + 1) & 15]);
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ffma2(float *out, float a, float b, long long *cyc) {
    unsigned long long x[8];
    float2 ab = make_float2(a, a), bb = make_float2(b, b);
    unsigned long long A = *reinterpret_cast<unsigned long long *>(&ab);
    unsigned long long B = *reinterpret_cast<unsigned long long *>(&bb);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float2 v = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        x[i] = *reinterpret_cast<unsigned long long *>(&v);
    }
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(A), "l"(B));
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2 *>(&x[i]); s += v.x + v.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_mufu(float *out, float a, float b, long long *cyc) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    long long t0 = clock64();
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = __sinf(x[i]) + __cosf(x[i]) * a;
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_lds(float *out, float a, float b, long long *cyc) {
    __shared__ float4 sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(i, a, b, 1);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    int idx = threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float4 v = sm[(idx + i * 32) & 2047];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        idx += 256;
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef void (*kern)(float *, float, float, long long *);

void run(const char *name, kern k, double ops_per_thread, int sms) {
    const int threads = 1024, blocks = sms * 2;
    float *out;
    long long *cyc;
    cudaMalloc(&out, sizeof(float) * threads * blocks);
    cudaMalloc(&cyc, sizeof(long long) * blocks);
    k<<<blocks, threads>>>(out, 0.999f, 0.001f, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(out, 0.999f, 0.001f, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long hc[1024];
    cudaMemcpy(hc, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    double cmax = 0;
    for (int i = 0; i < blocks; ++i) cmax = hc[i] > cmax ? hc[i] : cmax;
    const double total = ops_per_thread * threads * blocks;
    // 2 blocks of 1024 threads per SM run concurrently (64 warps): per-SM ops / cycles
    printf("%-28s %8.1f lane-ops/clk/SM   %8.2f T lane-op/s   (%.3f ms, clk %.0f MHz)\n", name,
           ops_per_thread * threads * 2 / cmax, total / (ms * 1e-3) / 1e12, ms, cmax / (ms * 1e3));
    cudaFree(out); cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs: %d\n", sms);
    run("FFMA (imm/const operand)", k_ffma, 16.0 * ITERS, sms);
    run("FFMA (3 registers)", k_ffma_reg, 16.0 * ITERS, sms);
    run("FFMA2 f32x2 (lane-FMA)", k_ffma2, 16.0 * ITERS, sms);
    run("MUFU sin+cos (ops)", k_mufu, 16.0 * ITERS / 4, sms);
    run("LDS.128 (floats)", k_lds, 32.0 * ITERS / 4, sms);
    return 0;
}
