// mcsf_tmem8.cuh -- the tensor-memory-ring kernel for 8-channel images (variant 8; d = 5 .. 8).
//
// The TMEM kernels give every (cos, sin) pair of planes a TMEM lane quarter, i.e. an SM
// sub-partition (a warp reaches only the quarter warp_id % 4). Eight channels have nine pairs:
// Z, P_0 .. P_7 (Alg. 1, G_t = H_t f), which do not spread evenly over four
// quarters. So one filter call is two launches of this kernel, each filling all four quarters:
//   KIND 3: the eight pairs {Z, P_0 .. P_6}, two per quarter (TMEM column blocks 0 and 1), one
//           producer and one consumer warp per pair, one modulation per pixel for all eight,
//   KIND 2: pair P_7 of FOUR samples per pass (quarter q <- sample k + q); the four quarters'
//           Re[conj(H) blur] (Alg. 1) are summed through shared memory before the one
//           read-modify-write of the P_7 partial plane.
// 9/8 of a four-pair pass per sample in total, all quarters busy; the phase t_k . f (Alg. 1)
// needs all eight channels in both launches. (KIND 0 / 1 -- {Z, P_0 .. P_2} and {P_3 .. P_6} in two
// launches -- were the first version: the 8-channel modulation, done twice per pixel, bound them.)
//
// Otherwise the dataflow of v4 (mcsf_tmem.cuh): producer warps stage f by TMA (8 floats per
// padded pixel), modulate into G-pairs in shared memory, run the horizontal FIR with FFMA2
// (Alg. 1) and hand rows to the TMEM ring (transpose through a per-warp tile, tcgen05.st);
// consumer warps read 16-row TMEM blocks (tcgen05.ld), run the vertical FIR and accumulate. Row
// bookkeeping as in v4.
#pragma once
#include "mcsf_tmem.cuh"

namespace bfvec {
namespace {

template <int R_, int KIND_, int CW_ = 2>
struct CfgT8 {
    static constexpr int D = 8;              // channels of the phase; partial planes 0..7 = P, 8 = Z
    static constexpr int R = R_;
    static constexpr int KIND = KIND_;
    static constexpr int KB = 16;
    static constexpr int SH = 16;
    static constexpr int TX = kTX;
    // KIND 3: the eight pairs {Z, P_0 .. P_6} in ONE launch, two per TMEM quarter (column blocks
    // 0 and 1), one modulation per pixel for all eight; slots 0..3 otherwise
    static constexpr int NQ = (KIND_ == 3) ? 8 : 4;
    static constexpr int NS = (KIND_ == 2) ? 4 : 1;   // samples per pass
    static constexpr int NA = 256;           // producers: warp w -> slot w & 3, rows 8 (w >> 2) .. +8
                                             //   (KIND 3: slot w, both 8-row halves)
    static constexpr int CW = (KIND_ == 3) ? 1 : CW_;
    static constexpr int OR = KB / CW;
    static constexpr int NB = 256;           // consumers: (slot, half) pairs, KIND 3: one warp per slot
    static constexpr int GB = (KIND_ == 3) ? 1 : 2;   // G-pair buffers (KIND 3: one, it is 8 pairs wide)
    static constexpr int NT = NA + NB;
    static constexpr int DP = 8;
    static constexpr int WIN = TX + 2 * R;
    static constexpr int MS = cs_stride(WIN);
    static constexpr int A = round_up(KB + 2 * R, 16);
    static constexpr int HROWS = A + KB;
    static constexpr int RING = A + KB - R;
    static constexpr int NIN = 8 + 2 * R;
    static constexpr int QCOLS = (NQ / 4) * 2 * HROWS;   // TMEM columns per quarter
    static constexpr int TCOLS = (QCOLS <= 32) ? 32 : (QCOLS <= 64) ? 64 : (QCOLS <= 128) ? 128
                               : (QCOLS <= 256) ? 256 : 512;
    static constexpr int SZ_F = SH * WIN * DP * 4;
    static constexpr int SZ_G = NQ * SH * MS * 8;
    static constexpr int SZ_RING = RING * TX * 8;
    static constexpr int SZ_RED = (KIND_ == 2) ? 2 * NQ * KB * TX * 4 : 0;
    static constexpr int OFF_F = 0;
    static constexpr int OFF_G = round_up(OFF_F + SZ_F, 128);
    static constexpr int OFF_RING = round_up(OFF_G + GB * SZ_G, 128);
    static constexpr int SZ_TP = (NA / 32) * TX * 9 * 8;
    static constexpr int OFF_TP = round_up(OFF_RING + NS * SZ_RING, 128);
    static constexpr int OFF_RED = round_up(OFF_TP + SZ_TP, 128);
    static constexpr int OFF_BAR = round_up(OFF_RED + SZ_RED, 128);
    static constexpr size_t SMEM = OFF_BAR + 5 * 8 + 8;
    static constexpr uint32_t TMA_BYTES = SZ_F;
    // slot q: channel of its G pair (-1: Z), partial plane, sample offset within the pass
    static constexpr int ch(int q) { return (KIND_ == 0 || KIND_ == 3) ? q - 1 : KIND_ == 1 ? q + 3 : 7; }
    static constexpr int plane(int q) {
        return (KIND_ == 0 || KIND_ == 3) ? (q == 0 ? 8 : q - 1) : KIND_ == 1 ? q + 3 : 7;
    }
    // TMEM column offset of slot q's ring within its quarter
    static constexpr int qcol(int q) { return (q >> 2) * 2 * HROWS; }
    static constexpr int soff(int q) { return KIND_ == 2 ? q : 0; }
    static_assert(KB == 16, "one aligned 16-row block per chunk");
    static_assert(CW_ == 1 || CW_ == 2, "one or two consumer warps per slot");
    static_assert(QCOLS <= 512, "TMEM columns");
    static_assert(SMEM <= 232448, "shared memory budget");
    static_assert(WIN <= 256, "TMA box dimension");
};

// modulation of n rows of fbuf into the slots' G-pairs; row `row` is emitted row g0 + row
template <class C>
__device__ __forceinline__ void modulate8(int ta, const float *fbuf, float2 *gbuf, float2 *rings,
                                          const float (&tk)[C::NS][C::D], const bool (&act)[C::NS], int g0, int n) {
    constexpr int PER = (C::SH * C::WIN + C::NA - 1) / C::NA;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int it = ta + i * C::NA;
        const int row = it / C::WIN;
        const int j = it - row * C::WIN;
        if (it >= C::SH * C::WIN || row >= n) continue;
        const float4 q0 = *reinterpret_cast<const float4 *>(fbuf + (row * C::WIN + j) * C::DP);
        const float4 q1 = *reinterpret_cast<const float4 *>(fbuf + (row * C::WIN + j) * C::DP + 4);
        const float fv[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
        float th[C::NS];
        if constexpr (C::NS % 2 == 0) {   // two samples' phases per FFMA2
#pragma unroll
            for (int v = 0; v < C::NS / 2; ++v) {
                float2 t2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int c = 0; c < C::D; ++c)
                    t2 = __ffma2_rn(make_float2(tk[2 * v][c], tk[2 * v + 1][c]), make_float2(fv[c], fv[c]), t2);
                th[2 * v] = t2.x;
                th[2 * v + 1] = t2.y;
            }
        } else {   // one sample: two channels per FFMA2
#pragma unroll
            for (int u = 0; u < C::NS; ++u) {
                float2 t2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int c = 0; c < C::D; c += 2)
                    t2 = __ffma2_rn(make_float2(tk[u][c], tk[u][c + 1]), make_float2(fv[c], fv[c + 1]), t2);
                th[u] = t2.x + t2.y;
            }
        }
        float2 cs[C::NS];
#pragma unroll
        for (int u = 0; u < C::NS; ++u) {
            float s, c;
            __sincosf(th[u], &s, &c);
            cs[u] = act[u] ? make_float2(c, s) : make_float2(0.f, 0.f);   // inactive sample: no contribution
        }
        float2 *dst = gbuf + row * C::MS + j;
        static_for<C::NQ>([&](auto Q) {
            constexpr int q = decltype(Q)::value;
            constexpr int c = C::ch(q);
            const float2 h = cs[C::soff(q)];
            dst[q * C::SH * C::MS] = (c < 0) ? h : __fmul2_rn(h, make_float2(fv[c < 0 ? 0 : c], fv[c < 0 ? 0 : c]));
        });
        if (j >= C::R && j < C::R + C::TX) {
            const int rs = ((g0 + row) % C::RING) * C::TX + (j - C::R);
#pragma unroll
            for (int u = 0; u < C::NS; ++u) rings[u * C::RING * C::TX + rs] = cs[u];
        }
    }
}

template <class C>
__global__ void __launch_bounds__(C::NT, 1) mcsf_tmem8_kernel(const __grid_constant__ FusedArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *fbuf = reinterpret_cast<float *>(smem + C::OFF_F);
    float2 *gbuf = reinterpret_cast<float2 *>(smem + C::OFF_G);
    float2 *rings = reinterpret_cast<float2 *>(smem + C::OFF_RING);
    float2 *tpose = reinterpret_cast<float2 *>(smem + C::OFF_TP);
    float *red = reinterpret_cast<float *>(smem + C::OFF_RED);
    uint64_t *tma_bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *full = tma_bar + 1;
    uint64_t *empty = tma_bar + 3;
    uint32_t *taddr_s = reinterpret_cast<uint32_t *>(tma_bar + 5);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int x0 = blockIdx.x * C::TX;
    const int img = a.tiles_per_img ? (int)blockIdx.y / a.tiles_per_img : 0;
    const int tile = a.tiles_per_img ? (int)blockIdx.y % a.tiles_per_img : (int)blockIdx.y;
    const int ty0 = a.out_row0 + tile * a.tile_rows;
    const int ty1 = min(ty0 + a.tile_rows, a.out_row0 + a.out_rows);
    const int g = blockIdx.z;
    const int ns = a.k1 - a.k0;
    const int gk0 = a.gstride ? a.k0 + g * a.gstride : a.k0 + (int)((long long)ns * g / a.groups);
    const int gk1 = a.gstride ? a.k1 + g * a.gstride : a.k0 + (int)((long long)ns * (g + 1) / a.groups);
    const int nchunks = (ty1 - ty0 + C::KB - 1) / C::KB;
    const int rows_per_pass = C::A + (nchunks - 1) * C::KB;
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
    // let the next launch of the call start on SMs this one frees (its CTAs only begin once every
    // CTA of this grid has started; it writes other planes)
    if (C::KIND != 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (gk0 < gk1) {
        if (tid < C::NA) {
            // ============================ PRODUCER ============================
            const int ta = tid;
            const int p = (C::KIND == 3) ? warp : (warp & 3);   // slot; TMEM quarter p & 3
            const int r8 = lane & 7, cg = lane >> 3;
            const uint32_t tq = tbase + ((uint32_t)(32 * (p & 3)) << 16) + (uint32_t)C::qcol(p);
            uint32_t tparity = 0;
            int buf = 0, it = 0;
            if (ta == 0) tma_load_3d(fbuf, &a.tmap, tma_bar, 0, x0, prow0, C::TMA_BYTES);
            int q = 0;
            for (int k = gk0, pass = 0; k < gk1; k += C::NS, ++pass) {
                float tk[C::NS][C::D];
                bool act[C::NS];
#pragma unroll
                for (int u = 0; u < C::NS; ++u) {
                    act[u] = k + u < gk1;
#pragma unroll
                    for (int c = 0; c < C::D; ++c)
                        tk[u][c] = (act[u] && c < a.d) ? __ldg(a.t + (long long)(k + u) * a.d + c) : 0.f;
                }
                const int gs = pass * rows_per_pass;
                for (int ci = 0; ci < nchunks; ++ci, ++q) {
                    const bool first_c = (ci == 0);
                    if (first_c) {
                        if (q >= 1) mbar_wait(&empty[(q - 1) & 1], ((q - 1) >> 1) & 1);
                    } else if (q >= 2) {
                        mbar_wait(&empty[q & 1], ((q - 2) >> 1) & 1);
                    }
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const int u_begin = first_c ? 0 : C::A + (ci - 1) * C::KB;
                    const int n_new = first_c ? C::A : C::KB;
                    for (int s0 = 0; s0 < n_new; s0 += C::SH, buf ^= 1, ++it) {
                        const int gsub = gs + u_begin + s0;
                        float2 *gb = gbuf + (C::GB == 2 ? buf : 0) * (C::NQ * C::SH * C::MS);
                        if (C::GB == 1 && it > 0) named_sync<C::NA>(1);   // one G buffer: previous H-pass done
                        mbar_wait(tma_bar, tparity);
                        tparity ^= 1u;
                        modulate8<C>(ta, fbuf, gb, rings, tk, act, gsub, C::SH);
                        named_sync<C::NA>(1);   // G-pairs complete; fbuf free; previous H-pass done
                        if (ta == 0) {
                            int nu = -1;
                            if (s0 + C::SH < n_new) nu = u_begin + s0 + C::SH;
                            else if (ci + 1 < nchunks) nu = C::A + ci * C::KB;
                            else if (k + C::NS < gk1) nu = 0;
                            if (nu >= 0) tma_load_3d(fbuf, &a.tmap, tma_bar, 0, x0, prow0 + nu, C::TMA_BYTES);
                        }
                        // horizontal FIR: 8 outputs (row 8 rh + r8, columns 8 cg .. 8 cg + 7) of slot p
                        constexpr int NRH = (C::KIND == 3) ? 2 : 1;
#pragma unroll 1
                        for (int rr = 0; rr < NRH; ++rr) {
                        const int rh = (C::KIND == 3) ? rr : (warp >> 2);
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
                        float2 *tt = tpose + warp * (C::TX * 9);
#pragma unroll
                        for (int o = 0; o < 8; ++o) tt[(8 * cg + o) * 9 + r8] = acc[o];
                        __syncwarp();
#pragma unroll
                        for (int o = 0; o < 8; ++o) acc[o] = tt[lane * 9 + o];
                        __syncwarp();
                        const int slot = (gsub + 8 * rh) % C::HROWS;
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
            // warp NA/32 + w: slot p = w & 3 (TMEM quarter p = warp % 4); part h = w >> 2 owns output
            // rows OR h .. OR h + OR - 1 of every chunk
            const int wi = warp - C::NA / 32;
            const int p = (C::KIND == 3) ? wi : (warp & 3);   // slot; TMEM quarter warp % 4 == p & 3
            const int h = (C::KIND == 3) ? 0 : (wi >> 2);
            const uint32_t tq = tbase + ((uint32_t)(32 * (p & 3)) << 16) + (uint32_t)C::qcol(p);
            const int x = x0 + lane;
            const bool xok = x < a.W;
            const long long plane_out = (long long)a.out_rows * a.W;
            float *pzb = a.pz + img * a.img_pz + (long long)g * (C::D + 1) * plane_out + x;
            const long long pl = C::plane(p);   // this slot's partial plane (KIND 2: P_7 for every slot)
            auto body = [&](auto HH) {
                constexpr int OR = C::OR;
                constexpr int H0 = OR * decltype(HH)::value;
                constexpr int JB0 = H0 / 16;
                constexpr int JB1 = (H0 + OR - 1 + 2 * C::R) / 16 + 1;
                // KIND 2: rows of the chunk this warp reduces over the four slots and writes
                constexpr int RW = C::KB / (C::NB / 32);
                const int rr0 = wi * RW;
                // the old partial sums this thread read-modify-writes in chunk (first, cy), loaded one
                // chunk ahead so their latency overlaps the previous chunk's FIR
                constexpr int NO = (C::KIND == 2) ? RW : OR;
                const int orow = (C::KIND == 2) ? rr0 : H0;
                const long long opl = (C::KIND == 2) ? 7 : pl;
                auto load_old = [&](float (&o_)[NO], int cy, bool first) {
#pragma unroll
                    for (int o = 0; o < NO; ++o) {
                        const bool ok = xok && (cy + orow + o < ty1);
                        o_[o] = (!first && ok) ? pzb[opl * plane_out + (long long)(cy + orow + o - a.out_row0) * a.W]
                                               : 0.f;
                    }
                };
                float old[NO];
                load_old(old, ty0, true);
                int q = 0;
                for (int k = gk0, pass = 0; k < gk1; k += C::NS, ++pass) {
                    const int gs = pass * rows_per_pass;
                    for (int ci = 0; ci < nchunks; ++ci, ++q) {
                        const int cy = ty0 + ci * C::KB;
                        mbar_wait(&full[q & 1], (q >> 1) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        float2 acc[OR];
#pragma unroll
                        for (int o = 0; o < OR; ++o) acc[o] = make_float2(0.f, 0.f);
                        const int b0 = (gs + ci * C::KB) % C::HROWS;
                        float2 v[2][16];
                        auto slot_of = [&](int bj) {
                            const int slot = b0 + 16 * bj;
                            return slot >= C::HROWS ? slot - C::HROWS : slot;
                        };
                        tmem_ld32(tq + 2 * slot_of(JB0), v[JB0 & 1]);
                        tmem_wait_ld(v[JB0 & 1]);
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
                        const float2 *myring = rings + (C::KIND == 2 ? p : 0) * C::RING * C::TX;
                        int slot = (gs + ci * C::KB + H0 + C::R) % C::RING;
                        float2 cs[OR];
#pragma unroll
                        for (int o = 0; o < OR; ++o) {
                            cs[o] = myring[slot * C::TX + lane];
                            slot = (slot + 1 == C::RING) ? 0 : slot + 1;
                        }
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        mbar_arrive(&empty[q & 1]);
                        if constexpr (C::KIND == 2) {
                            // four samples of P_7 (one per quarter): sum through shared memory, then one RMW
                            float *rb = red + (q & 1) * (C::NQ * C::KB * C::TX);
#pragma unroll
                            for (int o = 0; o < OR; ++o)
                                rb[(p * C::KB + H0 + o) * C::TX + lane] = fmaf(cs[o].x, acc[o].x, cs[o].y * acc[o].y);
                            named_sync<C::NB>(2);
                            if (xok) {
#pragma unroll
                                for (int o = 0; o < RW; ++o) {
                                    const int row = rr0 + o;
                                    if (cy + row < ty1) {
                                        float sum = old[o];
#pragma unroll
                                        for (int s = 0; s < C::NQ; ++s) sum += rb[(s * C::KB + row) * C::TX + lane];
                                        pzb[7 * plane_out + (long long)(cy + row - a.out_row0) * a.W] = sum;
                                    }
                                }
                            }
                        } else {
                            if (xok) {
                                float *dst = pzb + pl * plane_out + (long long)(cy + H0 - a.out_row0) * a.W;
#pragma unroll
                                for (int o = 0; o < OR; ++o)
                                    if (cy + H0 + o < ty1)
                                        dst[(long long)o * a.W] = fmaf(cs[o].x, acc[o].x, fmaf(cs[o].y, acc[o].y, old[o]));
                            }
                        }
                        // next chunk: the next 16 rows of this pass, or the first rows of the next pass
                        if (ci + 1 < nchunks) load_old(old, cy + C::KB, k == gk0);   // first pass: initialise
                        else if (k + C::NS < gk1) load_old(old, ty0, false);
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
    // launches 1 and 2 start early (programmatic stream serialisation) to fill the previous
    // launch's last wave; they touch other partial planes, but a grid may only COMPLETE after its
    // predecessor, so whatever follows on the stream (normalise) sees all three launches done
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <class C>
cudaError_t launch_tmem8_one(const FusedArgs &a, dim3 grid, cudaStream_t s) {
    auto k = mcsf_tmem8_kernel<C>;
    static std::atomic<uint64_t> attr{0};
    const cudaError_t e = ensure_smem_attr(k, C::SMEM, attr);
    if (e != cudaSuccess) return e;
    if (C::KIND == 0 || C::KIND == 3) {   // the call's first launch
        k<<<grid, C::NT, C::SMEM, s>>>(a);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(C::NT);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, a);
}

// the launches of one filter call (disjoint partial planes of the same groups): KIND 3 (Z, P_0 .. P_6)
// then KIND 2 (P_7); KIND 0 / 1 split the eight pairs over two launches instead (the first version)
template <int R>
cudaError_t launch_tmem8(const FusedArgs &a, dim3 grid, cudaStream_t s) {
    cudaError_t e = launch_tmem8_one<CfgT8<R, 3>>(a, grid, s);
    if (e == cudaSuccess) e = launch_tmem8_one<CfgT8<R, 2>>(a, grid, s);
    return e;
}

template <int R>
void fill_info_tmem8(KernelInfo *info) {
    using C = CfgT8<R, 2>;
    info->sp = 1;
    info->D = 8;
    info->R = R;
    info->threads = C::NT;
    info->kb = C::KB;
    info->sh = C::SH;
    info->dp = C::DP;
    info->win = C::WIN;
    info->smem = C::SMEM;
    info->regs = 0;
    info->occupancy = 0;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, mcsf_tmem8_kernel<C>) == cudaSuccess) info->regs = fa.numRegs;
    if (cudaFuncSetAttribute(mcsf_tmem8_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) ==
        cudaSuccess) {
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mcsf_tmem8_kernel<C>, C::NT, C::SMEM) == cudaSuccess)
            info->occupancy = occ;
    }
    cudaGetLastError();
}

}  // namespace
}  // namespace bfvec
