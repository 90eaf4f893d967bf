// mcsf_fused.cu -- the fused Monte Carlo shiftable-filter kernel for sm_100a (v2).
//
// One CTA owns a strip of TX = 32 output columns x tile_rows output rows and a
// group of samples. For every sample k (Alg. 1) it streams
// the strip top to bottom in chunks of KB output rows. Per sub-step of SH rows:
//
//   TMA       cp.async.bulk.tensor box (DP floats x WIN pixels x SH rows) of the
//             reflect-padded, centred, pixel-interleaved copy of f (pad.cu) ->
//             shared `fbuf`, completion on an mbarrier. The next box is issued
//             as soon as `fbuf` is consumed, so it lands during the H-pass.
//   modulate  (Alg. 1, Eq. (16))
//             theta = t_k . (f - mu) (d FFMA), (c, s) = sincos(theta) on the SFU;
//             (c, s) pairs -> `modcs`, centred f -> `modf`, and (c, s) of the
//             strip's own columns -> the ring `ring` (needed again at accumulate).
//   H-pass    (Alg. 1; "bulk of the computation")
//             (2R+1)-tap FIR along x on (cos, sin) channel PAIRS with packed
//             FFMA2 (taps = uniform-register scalars), G-pairs formed on the fly
//             as (c, s) * f_q with FMUL2 -> `hb` (KB + 2R rows).
//   V-pass + accumulate (Alg. 1, Eq. (18)-(19))
//             (2R+1)-tap FIR along y over `hb` (FFMA2), then
//             Z += c blur(c) + s blur(s),  P'_q += c blur(c f'_q) + s blur(s f'_q)
//             (= Re[conj(H) blur], reading R4), read-modify-write of the CTA's
//             L2-resident partial tile.
//
// H_k and G_k never touch HBM. Separability is exact for the square window
// (omega(j) = w(j_y) w(j_x)). Boundary: reflection (reading R1),
// baked into the padded copy.
#include <cuda.h>
#include <cuda_runtime.h>

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

template <int D_, int R_, int NT_, int KB_, int SH_>
struct Cfg {
    static constexpr int D = D_;
    static constexpr int R = R_;
    static constexpr int NT = NT_;
    static constexpr int KB = KB_;           // output rows per chunk (multiple of 8)
    static constexpr int SH = SH_;           // rows per TMA box / H-pass sub-step
    static constexpr int TX = kTX;
    static constexpr int NP = D + 1;         // (cos, sin) channel pairs: Z, P_0..P_{D-1}
    static constexpr int DP = (D <= 4) ? 4 : 8;   // floats per padded pixel
    static constexpr int WIN = TX + 2 * R;   // haloed columns
    static constexpr int MS = cs_stride(WIN);
    static constexpr int MSF = f_stride(WIN);
    static constexpr int HROWS = KB + 2 * R;
    static constexpr int RING = KB + R;
    static constexpr int NIN = 8 + 2 * R;    // H-pass inputs per 8 outputs
    // shared-memory carve-up (bytes, 128-aligned regions)
    static constexpr int SZ_F = SH * WIN * DP * 4;
    static constexpr int SZ_CS = SH * MS * 8;
    static constexpr int SZ_MF = D * SH * MSF * 4;
    static constexpr int SZ_HB = NP * HROWS * TX * 8;
    static constexpr int SZ_RING = RING * TX * 8;
    static constexpr int OFF_F = 0;
    static constexpr int OFF_CS = round_up(OFF_F + SZ_F, 128);
    static constexpr int OFF_MF = round_up(OFF_CS + SZ_CS, 128);
    static constexpr int OFF_HB = round_up(OFF_MF + SZ_MF, 128);
    static constexpr int OFF_RING = round_up(OFF_HB + SZ_HB, 128);
    static constexpr int OFF_BAR = round_up(OFF_RING + SZ_RING, 128);
    static constexpr size_t SMEM = OFF_BAR + 16;
    static constexpr uint32_t TMA_BYTES = SZ_F;
    static_assert(KB % 8 == 0, "KB must be a multiple of 8");
    static_assert(SH == 8 || SH == 16, "SH must be 8 or 16");
    static_assert(NT == NP * SH * 4, "one H-pass item (pair, row, 8 columns) per thread");
    static_assert(SMEM <= 232448, "shared memory budget");
    static_assert(WIN <= 256, "TMA box dimension");
};

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
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(saddr(bar)), "r"(parity)
            : "memory");
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

__device__ __forceinline__ float2 ffma2(float w, float2 v, float2 acc) {
    return __ffma2_rn(make_float2(w, w), v, acc);
}

// ---------------------------------------------------------------------------
// stages
// ---------------------------------------------------------------------------
// modulate n rows of fbuf (tile-frame rows u0 .. u0+n-1) -> modcs, modf, ring
template <class C>
__device__ __forceinline__ void modulate(const float *fbuf, float2 *modcs, float *modf, float2 *ring,
                                         const float (&tk)[C::D], int u0, int n) {
    for (int it = threadIdx.x; it < C::SH * C::WIN; it += C::NT) {
        const int row = it / C::WIN;
        const int j = it - row * C::WIN;
        if (row >= n) continue;
        const float *px = fbuf + (row * C::WIN + j) * C::DP;
        float fv[C::D];
#pragma unroll
        for (int c4 = 0; c4 < C::DP; c4 += 4) {
            const float4 q = *reinterpret_cast<const float4 *>(px + c4);
            if (c4 + 0 < C::D) fv[c4 + 0] = q.x;
            if (c4 + 1 < C::D) fv[c4 + 1] = q.y;
            if (c4 + 2 < C::D) fv[c4 + 2] = q.z;
            if (c4 + 3 < C::D) fv[c4 + 3] = q.w;
        }
        float th = 0.f;
#pragma unroll
        for (int c = 0; c < C::D; ++c) th = fmaf(tk[c], fv[c], th);
        float s, c;
        __sincosf(th, &s, &c);
        const float2 cs = make_float2(c, s);
        modcs[row * C::MS + j] = cs;
#pragma unroll
        for (int q = 0; q < C::D; ++q) modf[(q * C::SH + row) * C::MSF + j] = fv[q];
        if (j >= C::R && j < C::R + C::TX) ring[((u0 + row) % C::RING) * C::TX + (j - C::R)] = cs;
    }
}

// horizontal FIR of one item (pair p, row, 8-column group cg); HAS_F: pair is (c, s) * f_q
template <class C, bool HAS_F>
__device__ __forceinline__ void hpass_item(const FusedArgs &a, const float2 *csrow, const float *frow,
                                           float2 *dst) {
    float2 acc[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
    for (int jj = 0; jj < C::NIN / 2; ++jj) {
        const float4 c2 = *reinterpret_cast<const float4 *>(csrow + 2 * jj);
        float2 v[2] = {make_float2(c2.x, c2.y), make_float2(c2.z, c2.w)};
        if (HAS_F) {
            const float2 f2 = *reinterpret_cast<const float2 *>(frow + 2 * jj);
            v[0] = __fmul2_rn(v[0], make_float2(f2.x, f2.x));
            v[1] = __fmul2_rn(v[1], make_float2(f2.y, f2.y));
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = 2 * jj + e;
#pragma unroll
            for (int o = 0; o < 8; ++o) {
                const int m = j - o - C::R;          // tap offset, compile-time
                if (m >= -C::R && m <= C::R) acc[o] = ffma2(a.w[m < 0 ? -m : m], v[e], acc[o]);
            }
        }
    }
#pragma unroll
    for (int o = 0; o < 8; o += 2)
        *reinterpret_cast<float4 *>(dst + o) = make_float4(acc[o].x, acc[o].y, acc[o + 1].x, acc[o + 1].y);
}

template <class C>
__device__ __forceinline__ void hpass(const FusedArgs &a, const float2 *modcs, const float *modf, float2 *hb,
                                      int hb_row0, int n) {
    const int it = threadIdx.x;                      // exactly one item per thread
    const int row = it % C::SH;
    const int cg = (it / C::SH) & 3;
    const int p = it / (4 * C::SH);                  // warp-uniform
    if (row >= n) return;
    const float2 *csrow = modcs + row * C::MS + cg * 8;
    float2 *dst = hb + (p * C::HROWS + hb_row0 + row) * C::TX + cg * 8;
    if (p == 0) {
        hpass_item<C, false>(a, csrow, nullptr, dst);
    } else {
        const float *frow = modf + ((p - 1) * C::SH + row) * C::MSF + cg * 8;
        hpass_item<C, true>(a, csrow, frow, dst);
    }
}

template <class C>
__global__ void __launch_bounds__(C::NT, 1) mcsf_fused_kernel(const __grid_constant__ FusedArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *fbuf = reinterpret_cast<float *>(smem + C::OFF_F);
    float2 *modcs = reinterpret_cast<float2 *>(smem + C::OFF_CS);
    float *modf = reinterpret_cast<float *>(smem + C::OFF_MF);
    float2 *hb = reinterpret_cast<float2 *>(smem + C::OFF_HB);
    float2 *ring = reinterpret_cast<float2 *>(smem + C::OFF_RING);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * C::TX;
    const int ty0 = a.out_row0 + blockIdx.y * a.tile_rows;
    const int ty1 = min(ty0 + a.tile_rows, a.out_row0 + a.out_rows);
    const int g = blockIdx.z;
    const int ns = a.k1 - a.k0;
    const int gk0 = a.k0 + (int)((long long)ns * g / a.groups);
    const int gk1 = a.k0 + (int)((long long)ns * (g + 1) / a.groups);
    const long long plane_out = (long long)a.out_rows * a.W;
    float *pzg = a.pz + (long long)g * (C::D + 1) * plane_out;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    constexpr int NWARP = C::NT / 32;
    const int x = x0 + lane;
    // padded-copy row of tile-frame row u = 0 (image row ty0 - R): pad row 0 is image row out_row0 - R
    const int prow0 = ty0 - a.out_row0;

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.tmap)) : "memory");
        mbar_init(bar, 1);
    }
    __syncthreads();
    uint32_t parity = 0;
    if (tid == 0 && gk0 < gk1) tma_load_3d(fbuf, &a.tmap, bar, 0, x0, prow0, C::TMA_BYTES);

    for (int k = gk0; k < gk1; ++k) {
        float tk[C::D];
#pragma unroll
        for (int c = 0; c < C::D; ++c) tk[c] = (c < a.d) ? __ldg(a.t + (long long)k * a.d + c) : 0.f;
        const bool first_k = (k == gk0);

        for (int cy = ty0; cy < ty1; cy += C::KB) {
            const bool first_c = (cy == ty0);
            if (!first_c) {
                // keep the last 2R blurred rows: hb rows [KB, KB+2R) -> [0, 2R), in rounds of
                // KB rows (source and destination of one round never overlap)
                for (int r0 = 0; r0 < 2 * C::R; r0 += C::KB) {
                    const int nr = min(C::KB, 2 * C::R - r0);
                    const int n4 = C::NP * nr * (C::TX / 2);
                    for (int it = tid; it < n4; it += C::NT) {
                        const int c4 = it % (C::TX / 2);
                        const int rr = (it / (C::TX / 2)) % nr;
                        const int p = it / ((C::TX / 2) * nr);
                        float4 *base = reinterpret_cast<float4 *>(hb + p * C::HROWS * C::TX);
                        base[(r0 + rr) * (C::TX / 2) + c4] = base[(r0 + rr + C::KB) * (C::TX / 2) + c4];
                    }
                    __syncthreads();
                }
            }
            const int u_begin = first_c ? 0 : (cy - ty0) + 2 * C::R;   // tile-frame row of the first new row
            const int n_new = first_c ? C::HROWS : C::KB;
            const int hb_dst0 = first_c ? 0 : 2 * C::R;
            for (int s0 = 0; s0 < n_new; s0 += C::SH) {
                const int n = min(C::SH, n_new - s0);
                mbar_wait(bar, parity);
                parity ^= 1u;
                modulate<C>(fbuf, modcs, modf, ring, tk, u_begin + s0, n);
                __syncthreads();
                if (tid == 0) {
                    // issue the next box (mirrors the loop structure exactly)
                    int nu = -1;
                    if (s0 + C::SH < n_new) nu = u_begin + s0 + C::SH;
                    else if (cy + C::KB < ty1) nu = (cy + C::KB - ty0) + 2 * C::R;
                    else if (k + 1 < gk1) nu = 0;
                    if (nu >= 0) tma_load_3d(fbuf, &a.tmap, bar, 0, x0, prow0 + nu, C::TMA_BYTES);
                }
                hpass<C>(a, modcs, modf, hb, hb_dst0 + s0, n);
                __syncthreads();
            }

            // vertical FIR + accumulate: warp item = (pair p, 8-row group rg), lane = column
            constexpr int WITEMS = C::NP * (C::KB / 8);
            const bool xok = x < a.W;
            for (int wi = warp; wi < WITEMS; wi += NWARP) {
                const int p = wi % C::NP;           // 0 -> Z, 1 + q -> P'_q
                const int rg = wi / C::NP;
                const int plane = (p == 0) ? C::D : p - 1;
                float *dst = pzg + plane * plane_out + (long long)(cy + rg * 8 - a.out_row0) * a.W + x;
                float old[8];
#pragma unroll
                for (int o = 0; o < 8; ++o) {
                    const bool ok = xok && (cy + rg * 8 + o < ty1);
                    old[o] = (!first_k && ok) ? dst[(long long)o * a.W] : 0.f;
                }
                const float2 *col = hb + (p * C::HROWS + rg * 8) * C::TX + lane;
                float2 acc[8];
#pragma unroll
                for (int o = 0; o < 8; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < 8 + 2 * C::R; ++j) {
                    const float2 v = col[j * C::TX];
#pragma unroll
                    for (int o = 0; o < 8; ++o) {
                        const int m = j - o - C::R;
                        if (m >= -C::R && m <= C::R) acc[o] = ffma2(a.w[m < 0 ? -m : m], v, acc[o]);
                    }
                }
                int slot = (cy - ty0 + C::R + rg * 8) % C::RING;
#pragma unroll
                for (int o = 0; o < 8; ++o) {
                    if (xok && cy + rg * 8 + o < ty1) {
                        const float2 cs = ring[slot * C::TX + lane];
                        dst[(long long)o * a.W] = fmaf(cs.x, acc[o].x, fmaf(cs.y, acc[o].y, old[o]));
                    }
                    slot = (slot + 1 == C::RING) ? 0 : slot + 1;
                }
            }
            __syncthreads();
        }
    }
}

template <class C>
cudaError_t launch_cfg(const FusedArgs &a, dim3 grid, cudaStream_t s) {
    auto k = mcsf_fused_kernel<C>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k<<<grid, C::NT, C::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <class C>
void fill_info(KernelInfo *info) {
    info->D = C::D;
    info->R = C::R;
    info->threads = C::NT;
    info->kb = C::KB;
    info->sh = C::SH;
    info->dp = C::DP;
    info->win = C::WIN;
    info->smem = C::SMEM;
    info->regs = 0;
    info->occupancy = 0;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, mcsf_fused_kernel<C>) == cudaSuccess) info->regs = fa.numRegs;
    if (cudaFuncSetAttribute(mcsf_fused_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)C::SMEM) == cudaSuccess) {
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mcsf_fused_kernel<C>, C::NT, C::SMEM) ==
            cudaSuccess)
            info->occupancy = occ;
    }
    cudaGetLastError();
}

// ---------------------------------------------------------------------------
// instance table: (D, R) -> Cfg<D, R, NT, KB, SH>. A plan with radius r uses the
// smallest compiled R >= r (taps beyond r are zero); d uses the smallest D >= d.
// NT = (D+1) * SH * 4 (one H-pass item per thread).
// ---------------------------------------------------------------------------
#define BFV_INSTANCES(X)                                                                      \
    X(1, 2, 128, 32, 16) X(1, 6, 128, 32, 16) X(1, 15, 128, 32, 16) X(1, 32, 128, 32, 16)    \
    X(1, 64, 128, 32, 16)                                                                     \
    X(2, 6, 192, 32, 16) X(2, 15, 192, 32, 16) X(2, 32, 192, 32, 16) X(2, 64, 192, 32, 16)    \
    X(3, 2, 256, 32, 16) X(3, 4, 256, 32, 16) X(3, 6, 256, 32, 16) X(3, 10, 256, 32, 16)      \
    X(3, 15, 256, 32, 16) X(3, 24, 256, 32, 16) X(3, 30, 256, 32, 16) X(3, 48, 256, 32, 16)   \
    X(3, 64, 128, 16, 8)                                                                     \
    X(4, 6, 160, 32, 8) X(4, 15, 160, 32, 8) X(4, 32, 160, 32, 8) X(4, 48, 160, 16, 8)        \
    X(8, 6, 288, 16, 8) X(8, 15, 288, 16, 8) X(8, 24, 288, 16, 8)

}  // namespace

bool fused_select(int d, int r, KernelInfo *info) {
    int bestD = 1 << 30, bestR = 1 << 30;
#define BFV_PICK(D_, R_, NT_, KB_, SH_)                                        \
    if (D_ >= d && R_ >= r && (D_ < bestD || (D_ == bestD && R_ < bestR))) { \
        bestD = D_; bestR = R_;                                              \
    }
    BFV_INSTANCES(BFV_PICK)
#undef BFV_PICK
    if (bestD == (1 << 30)) return false;
#define BFV_FILL(D_, R_, NT_, KB_, SH_) \
    if (D_ == bestD && R_ == bestR) fill_info<Cfg<D_, R_, NT_, KB_, SH_>>(info);
    BFV_INSTANCES(BFV_FILL)
#undef BFV_FILL
    return true;
}

cudaError_t fused_launch(const KernelInfo &info, const FusedArgs &a, dim3 grid, cudaStream_t s) {
#define BFV_LAUNCH(D_, R_, NT_, KB_, SH_) \
    if (info.D == D_ && info.R == R_) return launch_cfg<Cfg<D_, R_, NT_, KB_, SH_>>(a, grid, s);
    BFV_INSTANCES(BFV_LAUNCH)
#undef BFV_LAUNCH
    return cudaErrorInvalidValue;
}

}  // namespace bfvec
