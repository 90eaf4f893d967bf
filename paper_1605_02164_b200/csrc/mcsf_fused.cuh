// mcsf_fused.cuh -- the fused Monte Carlo shiftable-filter kernel for sm_100a (v3,
// warp-specialised).
//
// One CTA owns a strip of TX = 32 output columns x tile_rows output rows and a
// group of samples. For every sample k (Alg. 1) it streams
// the strip top to bottom in chunks of KB output rows. Two warp groups run
// concurrently and hand chunks over through full/empty mbarriers:
//
// PRODUCER warps (NA threads), per sub-step of SH rows:
//   TMA       cp.async.bulk.tensor box (DP floats x WIN pixels x SH rows) of the
//             reflect-padded, centred, pixel-interleaved copy of f (pad.cu) ->
//             shared `fbuf` (mbarrier completion); the next box is issued as soon
//             as `fbuf` is consumed, so it lands during the H-pass.
//   modulate  (Alg. 1, Eq. (16))
//             theta = t_k . (f - mu) (d FFMA), (c, s) = sincos(theta) on the SFU;
//             (c, s) pairs -> `modcs`, centred f -> `modf`, (c, s) of the strip's own
//             columns -> the ring `csring` (needed again at accumulate).
//   H-pass    (Alg. 1; "bulk of the computation")
//             (2R+1)-tap FIR along x on (cos, sin) channel PAIRS with packed FFMA2
//             (taps = uniform-register scalars); G-pairs formed on the fly as
//             (c, s) * f_q with FMUL2 -> ring `hb` of HROWS = 2 KB + 2R rows.
// CONSUMER warps (one per pair), per chunk:
//   V-pass + accumulate (Alg. 1, Eq. (18)-(19))
//             (2R+1)-tap FIR along y over `hb` (FFMA2), then
//             Z += c blur(c) + s blur(s),  P'_q += c blur(c f'_q) + s blur(s f'_q)
//             (= Re[conj(H) blur], reading R4), read-modify-write of the CTA's
//             partial tile.
// The producer runs one chunk ahead of the consumers, so the SFU/LDS-heavy
// modulation and the barriers of one group overlap FFMA2 work of the other.
//
// H_k and G_k never touch HBM. Separability is exact for the square window
// (omega(j) = w(j_y) w(j_x)). Boundary: reflection (reading R1),
// baked into the padded copy. Row bookkeeping: the g-th row the producer emits
// in this CTA (counting across samples) lives in hb slot g % HROWS and csring
// slot g % RING; sample s (0-based in the CTA) starts at g0 = s * (nchunks*KB + 2R).
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernel_common.cuh"

namespace bfvec {
namespace {

template <int D_, int R_, int NA_, int KB_, int SH_>
struct Cfg {
    static constexpr int D = D_;
    static constexpr int R = R_;
    static constexpr int KB = KB_;           // output rows per chunk = V-pass rows per consumer warp
    static constexpr int SH = SH_;           // rows per TMA box / H-pass sub-step
    static constexpr int TX = kTX;
    static constexpr int NP = D + 1;         // (cos, sin) channel pairs: Z, P_0..P_{D-1}
    static constexpr int NA = NA_;           // producer threads
    static constexpr int NB = NP * 32;       // consumer threads: one warp per pair
    static constexpr int NT = NA + NB;
    static constexpr int DP = (D <= 4) ? 4 : 8;   // floats per padded pixel
    static constexpr int WIN = TX + 2 * R;   // haloed columns
    static constexpr int MS = cs_stride(WIN);
    static constexpr int MSF = f_stride(WIN);
    static constexpr int HROWS = 2 * KB + 2 * R;   // producer may run one chunk ahead
    static constexpr int RING = 2 * KB + R;
    static constexpr int NIN = 8 + 2 * R;    // H-pass inputs per 8 outputs
    static constexpr int HITEMS = NP * SH * 4;     // H-pass items (pair, row, 8-column group)
    // PM (pre-modulated, d = 8): the modulation writes every pair's G = (c f_q, s f_q) once, so the
    // H-pass reads one float2 per tap input instead of (c, s) and f and an FMUL2 (the kernel is
    // shared-memory-bandwidth bound at nine pairs, profiles/r01_v3_fused_c4_ncu.md)
    static constexpr bool PM = (D == 8);
    // shared-memory carve-up (bytes, 128-aligned regions)
    static constexpr int SZ_F = SH * WIN * DP * 4;
    static constexpr int SZ_CS = PM ? NP * SH * MS * 8 : SH * MS * 8;
    static constexpr int SZ_MF = PM ? 0 : D * SH * MSF * 4;
    static constexpr int SZ_HB = NP * HROWS * TX * 8;
    static constexpr int SZ_RING = RING * TX * 8;
    static constexpr int OFF_F = 0;
    static constexpr int OFF_CS = round_up(OFF_F + SZ_F, 128);
    static constexpr int OFF_MF = round_up(OFF_CS + SZ_CS, 128);
    static constexpr int OFF_HB = round_up(OFF_MF + SZ_MF, 128);
    static constexpr int OFF_RING = round_up(OFF_HB + SZ_HB, 128);
    static constexpr int SZ_ONES = round_up(WIN + 8, 32) * 4;   // pair 0 (Z) has no f factor
    static constexpr int OFF_ONES = round_up(OFF_RING + SZ_RING, 128);
    static constexpr int OFF_BAR = round_up(OFF_ONES + SZ_ONES, 128);
    static constexpr size_t SMEM = OFF_BAR + 5 * 8;       // tma, full[2], empty[2]
    static constexpr uint32_t TMA_BYTES = SZ_F;
    // CTAs per SM the smem footprint allows (capped at 2); used as __launch_bounds__ minBlocks
    static constexpr int MINB = (NT <= 256 && 2 * (SMEM + 1024) <= 233472) ? 2 : 1;
    static_assert(SH == 8 || SH == 16, "SH must be 8 or 16");
    static_assert(NA % 32 == 0 && HITEMS % NA == 0, "H-pass items split evenly over producer warps");
    static_assert(SMEM <= 232448, "shared memory budget");
    static_assert(WIN <= 256, "TMA box dimension");
};

// ---------------------------------------------------------------------------
// producer stages
// ---------------------------------------------------------------------------
// modulate n rows of fbuf; row `row` is emitted row g0 + row
template <class C>
__device__ __forceinline__ void modulate(int ta, const float *fbuf, float2 *modcs, float *modf, float2 *csring,
                                         const float (&tk)[C::D], int g0, int n) {
    // fixed trip count, fully unrolled: the per-pixel LDS -> FFMA -> MUFU -> STS chains of
    // all of a thread's pixels interleave instead of running back to back
    constexpr int PER = (C::SH * C::WIN + C::NA - 1) / C::NA;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int it = ta + i * C::NA;
        const int row = it / C::WIN;
        const int j = it - row * C::WIN;
        if (it >= C::SH * C::WIN || row >= n) continue;
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
        if constexpr (C::PM) {
            modcs[row * C::MS + j] = cs;                                  // pair 0: Z
#pragma unroll
            for (int q = 0; q < C::D; ++q)
                modcs[((q + 1) * C::SH + row) * C::MS + j] = __fmul2_rn(cs, make_float2(fv[q], fv[q]));
        } else {
            modcs[row * C::MS + j] = cs;
#pragma unroll
            for (int q = 0; q < C::D; ++q) modf[(q * C::SH + row) * C::MSF + j] = fv[q];
        }
        if (j >= C::R && j < C::R + C::TX) csring[((g0 + row) % C::RING) * C::TX + (j - C::R)] = cs;
    }
}

// horizontal FIR of one item (pair p, row, 8-column group cg): the input pair is
// (c, s) * f_q (f = 1 for the Z pair), one code path for every pair (I-cache)
template <class C>
__device__ __forceinline__ void hpass_item(const FusedArgs &a, const float2 *csrow, const float *frow,
                                           float2 *dst) {
    float2 acc[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) acc[o] = make_float2(0.f, 0.f);
    static_for<C::NIN / 2>([&](auto JJ) {
        constexpr int jj = decltype(JJ)::value;
        const float4 c2 = *reinterpret_cast<const float4 *>(csrow + 2 * jj);
        float2 v[2] = {make_float2(c2.x, c2.y), make_float2(c2.z, c2.w)};
        if constexpr (!C::PM) {
            const float2 f2 = *reinterpret_cast<const float2 *>(frow + 2 * jj);
            v[0] = __fmul2_rn(v[0], make_float2(f2.x, f2.x));
            v[1] = __fmul2_rn(v[1], make_float2(f2.y, f2.y));
        }
        static_for<2>([&](auto E) {
            constexpr int e = decltype(E)::value;
            constexpr int j = 2 * jj + e;
            static_for<8>([&](auto O) {
                constexpr int o = decltype(O)::value;
                constexpr int m = j - o - C::R;              // tap offset
                if constexpr (m >= -C::R && m <= C::R) acc[o] = ffma2(a.w[m < 0 ? -m : m], v[e], acc[o]);
            });
        });
    });
#pragma unroll
    for (int o = 0; o < 8; o += 2)
        *reinterpret_cast<float4 *>(dst + o) = make_float4(acc[o].x, acc[o].y, acc[o + 1].x, acc[o + 1].y);
}

// all H-pass items of one sub-step; row `row` is emitted row g0 + row
template <class C>
__device__ __forceinline__ void hpass(int ta, const FusedArgs &a, const float2 *modcs, const float *modf,
                                      const float *ones, float2 *hb, int g0, int n) {
#pragma unroll 1
    for (int it = ta; it < C::HITEMS; it += C::NA) {
        const int row = it % C::SH;
        const int cg = (it / C::SH) & 3;
        const int p = it / (4 * C::SH);              // warp-uniform
        if (row >= n) continue;
        const float2 *csrow = modcs + ((C::PM ? p * C::SH : 0) + row) * C::MS + cg * 8;
        float2 *dst = hb + (p * C::HROWS + (g0 + row) % C::HROWS) * C::TX + cg * 8;
        const float *frow = (C::PM || p == 0) ? ones + cg * 8 : modf + ((p - 1) * C::SH + row) * C::MSF + cg * 8;
        hpass_item<C>(a, csrow, frow, dst);
    }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <class C>
__global__ void __launch_bounds__(C::NT, C::MINB) mcsf_fused_kernel(const __grid_constant__ FusedArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *fbuf = reinterpret_cast<float *>(smem + C::OFF_F);
    float2 *modcs = reinterpret_cast<float2 *>(smem + C::OFF_CS);
    float *modf = reinterpret_cast<float *>(smem + C::OFF_MF);
    float2 *hb = reinterpret_cast<float2 *>(smem + C::OFF_HB);
    float2 *csring = reinterpret_cast<float2 *>(smem + C::OFF_RING);
    float *ones = reinterpret_cast<float *>(smem + C::OFF_ONES);
    uint64_t *tma_bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *full = tma_bar + 1;            // [2] producer -> consumers: chunk rows ready
    uint64_t *empty = tma_bar + 3;           // [2] consumers -> producer: chunk consumed

    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * C::TX;
    const int img = a.tiles_per_img ? (int)blockIdx.y / a.tiles_per_img : 0;     // image of the batch
    const int tile = a.tiles_per_img ? (int)blockIdx.y % a.tiles_per_img : (int)blockIdx.y;
    const int ty0 = a.out_row0 + tile * a.tile_rows;
    const int ty1 = min(ty0 + a.tile_rows, a.out_row0 + a.out_rows);
    const int g = blockIdx.z;
    const int ns = a.k1 - a.k0;
    // sample range of group g: a slice of [k0, k1), or -- realisation batching (gstride > 0,
    // bf_vec_mse_sweep) -- the same [k0, k1) of realisation g's draws at t rows g * gstride + k
    const int gk0 = a.gstride ? a.k0 + g * a.gstride : a.k0 + (int)((long long)ns * g / a.groups);
    const int gk1 = a.gstride ? a.k1 + g * a.gstride : a.k0 + (int)((long long)ns * (g + 1) / a.groups);
    const int nchunks = (ty1 - ty0 + C::KB - 1) / C::KB;
    const int rows_per_sample = nchunks * C::KB + 2 * C::R;
    // padded-copy row of tile-frame row u = 0 (image row ty0 - R): pad row 0 is image row out_row0 - R
    const int prow0 = img * a.img_prows + (ty0 - a.out_row0);

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.tmap)) : "memory");
        mbar_init(tma_bar, 1);
        mbar_init(&full[0], C::NA);
        mbar_init(&full[1], C::NA);
        mbar_init(&empty[0], C::NB);
        mbar_init(&empty[1], C::NB);
    }
    for (int i = tid; i < C::SZ_ONES / 4; i += C::NT) ones[i] = 1.f;
    __syncthreads();
    if (gk0 >= gk1) return;

    if (tid < C::NA) {
        // ============================ PRODUCER ============================
        const int ta = tid;
        uint32_t tparity = 0;
        if (ta == 0) tma_load_3d(fbuf, &a.tmap, tma_bar, 0, x0, prow0, C::TMA_BYTES);
        int q = 0;                                      // chunk index across samples
        for (int k = gk0; k < gk1; ++k) {
            float tk[C::D];
#pragma unroll
            for (int c = 0; c < C::D; ++c) tk[c] = (c < a.d) ? __ldg(a.t + (long long)k * a.d + c) : 0.f;
            const int gs = (k - gk0) * rows_per_sample;   // emitted-row index of tile-frame row 0
            for (int ci = 0; ci < nchunks; ++ci, ++q) {
                const bool first_c = (ci == 0);
                // ring slots this chunk overwrites must have been consumed
                if (first_c) {
                    if (q >= 1) mbar_wait(&empty[(q - 1) & 1], ((q - 1) >> 1) & 1);
                } else if (q >= 2) {
                    mbar_wait(&empty[q & 1], ((q - 2) >> 1) & 1);
                }
                const int u_begin = first_c ? 0 : ci * C::KB + 2 * C::R;
                const int n_new = first_c ? C::KB + 2 * C::R : C::KB;
                for (int s0 = 0; s0 < n_new; s0 += C::SH) {
                    const int n = min(C::SH, n_new - s0);
                    mbar_wait(tma_bar, tparity);
                    tparity ^= 1u;
                    modulate<C>(ta, fbuf, modcs, modf, csring, tk, gs + u_begin + s0, n);
                    named_sync<C::NA>(1);
                    if (ta == 0) {
                        // issue the next box (mirrors the loop structure exactly)
                        int nu = -1;
                        if (s0 + C::SH < n_new) nu = u_begin + s0 + C::SH;
                        else if (ci + 1 < nchunks) nu = (ci + 1) * C::KB + 2 * C::R;
                        else if (k + 1 < gk1) nu = 0;
                        if (nu >= 0) tma_load_3d(fbuf, &a.tmap, tma_bar, 0, x0, prow0 + nu, C::TMA_BYTES);
                    }
                    hpass<C>(ta, a, modcs, modf, ones, hb, gs + u_begin + s0, n);
                    if (s0 + C::SH >= n_new) mbar_arrive(&full[q & 1]);   // this thread's rows are written
                    named_sync<C::NA>(1);
                }
            }
        }
    } else {
        // ============================ CONSUMERS ===========================
        const int tb = tid - C::NA;
        const int p = tb >> 5;                          // pair: 0 -> Z, 1 + q -> P'_q
        const int lane = tb & 31;
        const int x = x0 + lane;
        const bool xok = x < a.W;
        const long long plane_out = (long long)a.out_rows * a.W;
        const int plane = (p == 0) ? C::D : p - 1;
        float *pzp = a.pz + img * a.img_pz + ((long long)g * (C::D + 1) + plane) * plane_out + x;
        int q = 0;
        for (int k = gk0; k < gk1; ++k) {
            const bool first_k = (k == gk0);
            const int gs = (k - gk0) * rows_per_sample;
            for (int ci = 0; ci < nchunks; ++ci, ++q) {
                const int cy = ty0 + ci * C::KB;
                float *dst = pzp + (long long)(cy - a.out_row0) * a.W;
                float old[C::KB];
#pragma unroll
                for (int o = 0; o < C::KB; ++o) {
                    const bool ok = xok && (cy + o < ty1);
                    old[o] = (!first_k && ok) ? dst[(long long)o * a.W] : 0.f;
                }
                mbar_wait(&full[q & 1], (q >> 1) & 1);
                // window: emitted rows gs + ci*KB + j, j in [0, KB + 2R); slots wrap at most once
                const int b = (gs + ci * C::KB) % C::HROWS;
                const float2 *col0 = hb + (p * C::HROWS + b) * C::TX + lane;
                const float2 *col1 = col0 - C::HROWS * C::TX;
                const int jw = C::HROWS - b;             // first j that wraps
                float2 acc[C::KB];
#pragma unroll
                for (int o = 0; o < C::KB; ++o) acc[o] = make_float2(0.f, 0.f);
                static_for<C::KB + 2 * C::R>([&](auto J) {
                    constexpr int j = decltype(J)::value;
                    const float2 v = (j < jw ? col0 : col1)[j * C::TX];
                    static_for<C::KB>([&](auto O) {
                        constexpr int o = decltype(O)::value;
                        constexpr int m = j - o - C::R;          // tap offset
                        if constexpr (m >= -C::R && m <= C::R) acc[o] = ffma2(a.w[m < 0 ? -m : m], v, acc[o]);
                    });
                });
                int slot = (gs + ci * C::KB + C::R) % C::RING;
                float2 cs[C::KB];
#pragma unroll
                for (int o = 0; o < C::KB; ++o) {
                    cs[o] = csring[slot * C::TX + lane];
                    slot = (slot + 1 == C::RING) ? 0 : slot + 1;
                }
                mbar_arrive(&empty[q & 1]);              // hb / csring reads of this chunk are done
#pragma unroll
                for (int o = 0; o < C::KB; ++o)
                    if (xok && cy + o < ty1) dst[(long long)o * a.W] = fmaf(cs[o].x, acc[o].x, fmaf(cs[o].y, acc[o].y, old[o]));
            }
        }
    }
}

template <class C>
cudaError_t launch_cfg(const FusedArgs &a, dim3 grid, cudaStream_t s) {
    auto k = mcsf_fused_kernel<C>;
    static std::atomic<uint64_t> attr{0};
    const cudaError_t e = ensure_smem_attr(k, C::SMEM, attr);
    if (e != cudaSuccess) return e;
    k<<<grid, C::NT, C::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <class C>
void fill_info(KernelInfo *info) {
    info->sp = 1;
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

}  // namespace
}  // namespace bfvec
