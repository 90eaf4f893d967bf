// mcsf_tmem.cuh -- the fused Monte Carlo shiftable-filter kernel, v4: the
// horizontally-blurred row ring lives in TENSOR MEMORY (d <= 3, r <= 48).
//
// Same dataflow as v3 (mcsf_fused.cuh): producer warps stage f by TMA, modulate
// (Alg. 1), run the horizontal FIR (Alg. 1) ; consumer warps run the
// vertical FIR and accumulate Re[conj(H) blur] (Alg. 1, Eq. (18)-(19)).
// What changes, B200-specific:
//
//  * hb ring -> TMEM. Pair p owns TMEM lane quarter p; lane 32p + x holds column x
//    of the strip; TMEM column 2*slot + {0,1} holds the (cos, sin) parts of ring row
//    `slot`. The producer transposes each 8x8 block of H-pass outputs with warp
//    shuffles (lane = column) and writes it with tcgen05.st.32x32b; the consumer warp
//    of quarter p reads its column with tcgen05.ld.32x32b (16 rows per load). Handoff:
//    tcgen05.wait::st / fence::before_thread_sync -> mbarrier -> fence::after_thread_sync.
//  * the ~128 KB of shared memory this frees holds the modulated G-pairs
//    (c f_q, s f_q) written ONCE per pixel by the modulation (no FMUL2 in the H-pass),
//    double-buffered so the producer needs a single barrier per sub-step.
//
// Row bookkeeping as in v3: the g-th row the producer emits in this CTA (counting
// across samples) lives in ring slot g % HROWS and (c, s) ring slot g % RING.
#pragma once
#include "kernel_common.cuh"

namespace bfvec {
namespace {

template <int D_, int R_, int KB_, int CW_ = 1>
struct CfgT {
    static constexpr int D = D_;
    static constexpr int R = R_;
    static constexpr int KB = KB_;           // output rows per chunk (= consumer rows); multiple of 16
    static constexpr int SH = 16;            // rows per TMA box / modulation / H-pass sub-step
    static constexpr int TX = kTX;
    static constexpr int NP = D + 1;         // (cos, sin) pairs: Z, P_0..P_{D-1}; one TMEM quarter each
    static constexpr int NA = 256;           // producer threads: warp w -> pair w % 4, rows 8*(w / 4) .. +8
    static constexpr int CW = CW_;           // consumer warps per pair: warp 8 + w -> pair w & 3,
    static constexpr int OR = KB / CW_;      //   output rows OR (w >> 2) .. +OR of every chunk
    static constexpr int NB = 128 * CW_;     // consumer threads
    static constexpr int NT = NA + NB;
    static constexpr int DP = 4;
    static constexpr int WIN = TX + 2 * R;
    static constexpr int MS = cs_stride(WIN);     // float2 stride of a G-pair row
    // aligned production: the first chunk of a sample emits A = round16(KB + 2R) rows, every
    // later chunk the next aligned 16-row block (at most 15 rows more than it strictly needs)
    static constexpr int A = round_up(KB + 2 * R, 16);
    static constexpr int HROWS = A + KB;          // ring rows: producer one chunk ahead
    static constexpr int RING = A + KB - R;       // (c, s) ring rows
    static constexpr int NIN = 8 + 2 * R;
    static constexpr int TCOLS = (2 * HROWS <= 32) ? 32 : (2 * HROWS <= 64) ? 64 : (2 * HROWS <= 128) ? 128
                               : (2 * HROWS <= 256) ? 256 : 512;
    static constexpr int SZ_F = SH * WIN * DP * 4;
    static constexpr int SZ_G = NP * SH * MS * 8;        // one buffer of G-pairs
    static constexpr int SZ_RING = RING * TX * 8;
    static constexpr int OFF_F = 0;
    static constexpr int OFF_G = round_up(OFF_F + SZ_F, 128);
    static constexpr int OFF_RING = round_up(OFF_G + 2 * SZ_G, 128);
    static constexpr int SZ_TP = (NA / 32) * TX * 9 * 8;      // per producer warp: 32 columns x 9 float2
    static constexpr int OFF_TP = round_up(OFF_RING + SZ_RING, 128);
    static constexpr int OFF_BAR = round_up(OFF_TP + SZ_TP, 128);
    static constexpr size_t SMEM = OFF_BAR + 5 * 8 + 8;  // tma, full[2], empty[2], tmem address
    static constexpr uint32_t TMA_BYTES = SZ_F;
    static constexpr int MINB = 1;
    static_assert(D >= 1 && D <= 3, "one TMEM lane quarter per pair");
    static_assert(KB == 16, "one aligned 16-row block per chunk");
    static_assert(CW_ == 1 || CW_ == 2, "one or two consumer warps per pair");
    static_assert(2 * HROWS <= 512, "TMEM columns");
    static_assert(SMEM <= 232448, "shared memory budget");
    static_assert(WIN <= 256, "TMA box dimension");
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float2 (&v)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "f"(v[0].x), "f"(v[0].y), "f"(v[1].x), "f"(v[1].y), "f"(v[2].x), "f"(v[2].y), "f"(v[3].x), "f"(v[3].y),
        "f"(v[4].x), "f"(v[4].y), "f"(v[5].x), "f"(v[5].y), "f"(v[6].x), "f"(v[6].y), "f"(v[7].x), "f"(v[7].y)
        : "memory");
}

// wait for every outstanding tcgen05.ld of this thread, then tie the destination registers
// to the wait so no use of them can be scheduled above it
__device__ __forceinline__ void tmem_wait_ld(float2 (&v)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("" : "+f"(v[i].x), "+f"(v[i].y));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float2 (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[1].x), "=f"(v[1].y), "=f"(v[2].x), "=f"(v[2].y), "=f"(v[3].x),
          "=f"(v[3].y), "=f"(v[4].x), "=f"(v[4].y), "=f"(v[5].x), "=f"(v[5].y), "=f"(v[6].x), "=f"(v[6].y),
          "=f"(v[7].x), "=f"(v[7].y), "=f"(v[8].x), "=f"(v[8].y), "=f"(v[9].x), "=f"(v[9].y), "=f"(v[10].x),
          "=f"(v[10].y), "=f"(v[11].x), "=f"(v[11].y), "=f"(v[12].x), "=f"(v[12].y), "=f"(v[13].x),
          "=f"(v[13].y), "=f"(v[14].x), "=f"(v[14].y), "=f"(v[15].x), "=f"(v[15].y)
        : "r"(taddr)
        : "memory");
}

// modulation of n rows of fbuf into the G-pair buffer; row `row` is emitted row g0 + row
template <class C>
__device__ __forceinline__ void modulate_g(int ta, const float *fbuf, float2 *gbuf, float2 *csring,
                                           const float (&tk)[C::D], int g0, int n) {
    constexpr int PER = (C::SH * C::WIN + C::NA - 1) / C::NA;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int it = ta + i * C::NA;
        const int row = it / C::WIN;
        const int j = it - row * C::WIN;
        if (it >= C::SH * C::WIN || row >= n) continue;
        const float4 q = *reinterpret_cast<const float4 *>(fbuf + (row * C::WIN + j) * C::DP);
        const float fv[4] = {q.x, q.y, q.z, q.w};
        float th = 0.f;
#pragma unroll
        for (int c = 0; c < C::D; ++c) th = fmaf(tk[c], fv[c], th);
        float s, c;
        __sincosf(th, &s, &c);
        const float2 cs = make_float2(c, s);
        float2 *dst = gbuf + row * C::MS + j;
        dst[0] = cs;                                              // Z pair: (c, s)
#pragma unroll
        for (int p = 1; p < C::NP; ++p)
            dst[p * C::SH * C::MS] = __fmul2_rn(make_float2(c, s), make_float2(fv[p - 1], fv[p - 1]));
        if (j >= C::R && j < C::R + C::TX) csring[((g0 + row) % C::RING) * C::TX + (j - C::R)] = cs;
    }
}

template <class C>
__global__ void __launch_bounds__(C::NT, 1) mcsf_tmem_kernel(const __grid_constant__ FusedArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *fbuf = reinterpret_cast<float *>(smem + C::OFF_F);
    float2 *gbuf = reinterpret_cast<float2 *>(smem + C::OFF_G);
    float2 *csring = reinterpret_cast<float2 *>(smem + C::OFF_RING);
    float2 *tpose = reinterpret_cast<float2 *>(smem + C::OFF_TP);
    uint64_t *tma_bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *full = tma_bar + 1;
    uint64_t *empty = tma_bar + 3;
    uint32_t *taddr_s = reinterpret_cast<uint32_t *>(tma_bar + 5);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
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
    const int rows_per_sample = C::A + (nchunks - 1) * C::KB;   // multiple of 16
    const int prow0 = img * a.img_prows + (ty0 - a.out_row0);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(taddr_s)),
                     "n"(C::TCOLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.tmap)) : "memory");
        mbar_init(tma_bar, 1);
        mbar_init(&full[0], C::NA);
        mbar_init(&full[1], C::NA);
        mbar_init(&empty[0], C::NB);
        mbar_init(&empty[1], C::NB);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *taddr_s;

    if (gk0 < gk1) {
        if (tid < C::NA) {
            // ============================ PRODUCER ============================
            const int ta = tid;
            const int p = warp & 3;                          // pair == TMEM quarter
            const int rh = warp >> 2;                        // rows 8*rh .. 8*rh+7 of a sub-step
            const int r8 = lane & 7, cg = lane >> 3;         // item: row r8, columns 8cg .. 8cg+7
            const uint32_t tq = tbase + ((uint32_t)(32 * p) << 16);
            uint32_t tparity = 0;
            int buf = 0;
            if (ta == 0) tma_load_3d(fbuf, &a.tmap, tma_bar, 0, x0, prow0, C::TMA_BYTES);
            int q = 0;
            for (int k = gk0; k < gk1; ++k) {
                float tk[C::D];
#pragma unroll
                for (int c = 0; c < C::D; ++c) tk[c] = (c < a.d) ? __ldg(a.t + (long long)k * a.d + c) : 0.f;
                const int gs = (k - gk0) * rows_per_sample;
                for (int ci = 0; ci < nchunks; ++ci, ++q) {
                    const bool first_c = (ci == 0);
                    if (first_c) {
                        if (q >= 1) mbar_wait(&empty[(q - 1) & 1], ((q - 1) >> 1) & 1);
                    } else if (q >= 2) {
                        mbar_wait(&empty[q & 1], ((q - 2) >> 1) & 1);
                    }
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const int u_begin = first_c ? 0 : C::A + (ci - 1) * C::KB;
                    const int n_new = first_c ? C::A : C::KB;   // whole 16-row sub-steps
                    for (int s0 = 0; s0 < n_new; s0 += C::SH, buf ^= 1) {
                        const int n = C::SH;
                        const int gsub = gs + u_begin + s0;  // emitted-row index of sub-step row 0
                        float2 *gb = gbuf + buf * (C::NP * C::SH * C::MS);
                        mbar_wait(tma_bar, tparity);
                        tparity ^= 1u;
                        modulate_g<C>(ta, fbuf, gb, csring, tk, gsub, n);
                        named_sync<C::NA>(1);   // G-pairs complete; fbuf free; previous H-pass done
                        if (ta == 0) {
                            int nu = -1;
                            if (s0 + C::SH < n_new) nu = u_begin + s0 + C::SH;
                            else if (ci + 1 < nchunks) nu = C::A + ci * C::KB;
                            else if (k + 1 < gk1) nu = 0;
                            if (nu >= 0) tma_load_3d(fbuf, &a.tmap, tma_bar, 0, x0, prow0 + nu, C::TMA_BYTES);
                        }
                        if (p < C::NP) {
                            // horizontal FIR: 8 outputs (row 8rh + r8, columns 8cg .. 8cg+7)
                            const float2 *in = gb + (p * C::SH + 8 * rh + r8) * C::MS + cg * 8;
                            float2 acc[8];
#pragma unroll
                            for (int o = 0; o < 8; ++o) acc[o] = make_float2(0.f, 0.f);
                            static_for<C::NIN / 2>([&](auto JJ) {
                                constexpr int jj = decltype(JJ)::value;
                                const float4 v2 = *reinterpret_cast<const float4 *>(in + 2 * jj);
                                const float2 v[2] = {make_float2(v2.x, v2.y), make_float2(v2.z, v2.w)};
                                static_for<2>([&](auto E) {
                                    constexpr int e = decltype(E)::value;
                                    constexpr int j = 2 * jj + e;
                                    static_for<8>([&](auto O) {
                                        constexpr int o = decltype(O)::value;
                                        constexpr int m = j - o - C::R;
                                        if constexpr (m >= -C::R && m <= C::R)
                                            acc[o] = ffma2(a.w[m < 0 ? -m : m], v[e], acc[o]);
                                    });
                                });
                            });
                            // transpose through this warp's shared-memory tile: lane (r8, cg) holds
                            // row r8 of columns 8cg..8cg+7; lane x needs rows 0..7 of column x
                            // (stride 9 float2 per column: conflict-free both ways)
                            float2 *tt = tpose + warp * (C::TX * 9);
#pragma unroll
                            for (int o = 0; o < 8; ++o) tt[(8 * cg + o) * 9 + r8] = acc[o];
                            __syncwarp();
#pragma unroll
                            for (int o = 0; o < 8; ++o) acc[o] = tt[lane * 9 + o];
                            __syncwarp();
                            const int slot = (gsub + 8 * rh) % C::HROWS;   // 8 consecutive slots, no wrap
                            tmem_st16(tq + 2 * slot, acc);
                        }
                        if (s0 + C::SH >= n_new) {
                            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                            mbar_arrive(&full[q & 1]);
                        }
                    }
                }
            }
        } else {
            // ============================ CONSUMERS ===========================
            // warp 8 + w: pair p = w & 3 (TMEM quarter p = warp % 4); part h = w >> 2 owns
            // output rows OR h .. OR h + OR - 1 of every chunk
            const int p = warp & 3;
            const int h = (warp - C::NA / 32) >> 2;
            const uint32_t tq = tbase + ((uint32_t)(32 * p) << 16);
            const int x = x0 + lane;
            const bool active = p < C::NP;
            const bool xok = x < a.W;
            const long long plane_out = (long long)a.out_rows * a.W;
            const int plane = (p == 0) ? C::D : p - 1;
            float *pzp = a.pz + img * a.img_pz + ((long long)g * (C::D + 1) + plane) * plane_out + x;
            auto body = [&](auto HH) {
                constexpr int OR = C::OR;
                constexpr int H0 = OR * decltype(HH)::value;       // first output row of this part
                constexpr int JB0 = H0 / 16;                       // first 16-row TMEM block read
                constexpr int JB1 = (H0 + OR - 1 + 2 * C::R) / 16 + 1;  // one past the last block read
                int q = 0;
                for (int k = gk0; k < gk1; ++k) {
                    const bool first_k = (k == gk0);
                    const int gs = (k - gk0) * rows_per_sample;
                    for (int ci = 0; ci < nchunks; ++ci, ++q) {
                        const int cy = ty0 + ci * C::KB + H0;
                        float *dst = pzp + (long long)(cy - a.out_row0) * a.W;
                        // prefetch the old partial sums before waiting (their L2 latency overlaps
                        // the wait and the FIR; 16 registers, no spill at <= 168)
                        float old[OR];
#pragma unroll
                        for (int o = 0; o < OR; ++o) {
                            const bool ok = active && xok && (cy + o < ty1);
                            old[o] = (!first_k && ok) ? dst[(long long)o * a.W] : 0.f;
                        }
                        mbar_wait(&full[q & 1], (q >> 1) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        float2 acc[OR];
#pragma unroll
                        for (int o = 0; o < OR; ++o) acc[o] = make_float2(0.f, 0.f);
                        const int b0 = (gs + ci * C::KB) % C::HROWS;   // multiple of 16
                        float2 v[2][16];
                        auto slot_of = [&](int bj) {
                            const int slot = b0 + 16 * bj;
                            return slot >= C::HROWS ? slot - C::HROWS : slot;
                        };
                        tmem_ld32(tq + 2 * slot_of(JB0), v[JB0 & 1]);
                        tmem_wait_ld(v[JB0 & 1]);
                        // block bj is in registers; the load of block bj + 1 overlaps its FFMA2s
                        static_for<JB1 - JB0>([&](auto B) {
                            constexpr int bj = JB0 + decltype(B)::value;
                            if constexpr (bj + 1 < JB1) tmem_ld32(tq + 2 * slot_of(bj + 1), v[(bj + 1) & 1]);
                            static_for<16>([&](auto JJ) {
                                constexpr int j = 16 * bj + decltype(JJ)::value;
                                static_for<OR>([&](auto O) {
                                    constexpr int o = H0 + decltype(O)::value;
                                    constexpr int m = j - o - C::R;
                                    if constexpr (m >= -C::R && m <= C::R)
                                        acc[o - H0] = ffma2(a.w[m < 0 ? -m : m], v[bj & 1][decltype(JJ)::value],
                                                            acc[o - H0]);
                                });
                            });
                            if constexpr (bj + 1 < JB1) tmem_wait_ld(v[(bj + 1) & 1]);
                        });
                        int slot = (gs + ci * C::KB + H0 + C::R) % C::RING;
                        float2 cs[OR];
#pragma unroll
                        for (int o = 0; o < OR; ++o) {
                            cs[o] = csring[slot * C::TX + lane];
                            slot = (slot + 1 == C::RING) ? 0 : slot + 1;
                        }
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        mbar_arrive(&empty[q & 1]);
                        if (active && xok) {
                            // Re[conj(H) blur] into the partial tile (each element is updated by
                            // this thread only, in sample order)
#pragma unroll
                            for (int o = 0; o < OR; ++o)
                                if (cy + o < ty1) {
                                    dst[(long long)o * a.W] = fmaf(cs[o].x, acc[o].x, fmaf(cs[o].y, acc[o].y, old[o]));
                                }
                        }
                    }
                }
            };
            if constexpr (C::CW == 1) {
                body(std::integral_constant<int, 0>{});
            } else {
                if (h == 0) body(std::integral_constant<int, 0>{});
                else body(std::integral_constant<int, 1>{});
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::TCOLS) : "memory");
}

template <class C>
cudaError_t launch_tmem(const FusedArgs &a, dim3 grid, cudaStream_t s) {
    auto k = mcsf_tmem_kernel<C>;
    static std::atomic<uint64_t> attr{0};
    const cudaError_t e = ensure_smem_attr(k, C::SMEM, attr);
    if (e != cudaSuccess) return e;
    k<<<grid, C::NT, C::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <class C>
void fill_info_tmem(KernelInfo *info) {
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
    if (cudaFuncGetAttributes(&fa, mcsf_tmem_kernel<C>) == cudaSuccess) info->regs = fa.numRegs;
    if (cudaFuncSetAttribute(mcsf_tmem_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) ==
        cudaSuccess) {
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mcsf_tmem_kernel<C>, C::NT, C::SMEM) == cudaSuccess)
            info->occupancy = occ;
    }
    cudaGetLastError();
}

}  // namespace
}  // namespace bfvec
