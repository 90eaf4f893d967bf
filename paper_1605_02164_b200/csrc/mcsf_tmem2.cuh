// mcsf_tmem2.cuh -- fused MCSF kernel v5 (variant 4): the tensor-memory row ring of v4
// (mcsf_tmem.cuh), with TWO Monte Carlo samples per pass over a strip.
//
// Why: in v4 every sample re-streams the strip, re-loads f by TMA, hands every 16-row chunk
// between the producer and consumer warp groups through one mbarrier round trip, and reads,
// updates and writes the partial-sum tile once per sample. Pairing samples k and k+1 halves
// all three per unit of FIR work: one TMA box of f feeds both modulations (Alg. 1),
// one full/empty handoff covers both samples' rows, and the consumer folds both samples'
// Re[conj(H) blur] (Eq. (18)-(19), Alg. 1) into one read-modify-write of the tile.
//
//  * TMEM: 512 columns = two rings of 2*HROWS columns, ring s for the pass's sample s.
//  * producer warp w (8 warps): pair p = w & 3, sample slot s = w >> 2; sub-steps of SH = 8
//    rows, so one warp's 8 H-pass outputs per thread cover the whole sub-step of its sample.
//  * modulation: one f element feeds both samples' (c f, s f) pairs (2 sincos per pixel).
//  * consumer warp p (4 warps): for each chunk, the vertical FIR of ring 0 then ring 1 with the
//    same (looped, not duplicated) code; a pass with one sample (odd tail) skips slot 1.
// Row bookkeeping is v4's with "sample" replaced by "pass".
#pragma once
#include "mcsf_tmem.cuh"

namespace bfvec {
namespace {

template <int D_, int R_, int CW_ = 1, int MW_ = 0, bool BOX_ = false>
struct CfgT2 {
    static constexpr int D = D_;
    static constexpr int R = R_;
    static constexpr int KB = 16;            // output rows per chunk
    static constexpr int SH = 8;             // rows per TMA box / sub-step
    static constexpr int SP = 2;             // samples per pass
    static constexpr int TX = kTX;
    static constexpr int NP = D + 1;
    static constexpr int NA = 256;           // producers: warp w -> pair w & 3, sample slot w >> 2
    static constexpr int CW = CW_;           // consumer warps per pair: warp 8 + w -> pair w & 3,
    static constexpr int OR = KB / CW_;      //   output rows OR (w >> 2) .. + OR of every chunk
    static constexpr int NB = 128 * CW_;
    static constexpr int MW = MW_;           // dedicated modulation warps (0: the producers modulate)
    static constexpr bool BOX = BOX_;        // box taps (all equal, window exactly R): running sums
    static constexpr int NM = 32 * MW_;
    static constexpr int NT = NA + NB + NM;
    static constexpr int DP = 4;
    static constexpr int WIN = TX + 2 * R;
    static constexpr int MS = cs_stride(WIN);
    static constexpr int A = round_up(KB + 2 * R, 16);
    // Pass overlap: the ring holds HROWS = min(2A, what TMEM holds: 512 columns / (2 SP)) >= A + KB
    // rows. The first SPLIT = HROWS - A rows of a pass's A-row fill land in slots the previous
    // pass's last chunk no longer reads, so the producers write them while the consumers still
    // read that chunk (waiting only for chunk q-2, as every chunk does), and wait for the last
    // chunk only before the rest. R <= 24: SPLIT >= A, the whole fill overlaps (OV); R = 30: 48 of
    // 80 rows; R = 48: 16 of 112.
    static constexpr int HCAP = 512 / (2 * SP) / 16 * 16;
    static constexpr int HROWS = (2 * A <= HCAP) ? 2 * A : (A + KB > HCAP ? A + KB : HCAP);
    static constexpr int SPLIT = HROWS - A;
    static constexpr bool OV = SPLIT >= A;
    static constexpr int RING = HROWS - R + (MW_ > 0 ? 2 * SH : 0);   // modulators run <= 2 sub-steps ahead
    static constexpr int NIN = 8 + 2 * R;
    static constexpr int RCOLS = 2 * HROWS;                 // TMEM columns per ring
    static constexpr int TCOLS = (SP * RCOLS <= 32) ? 32 : (SP * RCOLS <= 64) ? 64 : (SP * RCOLS <= 128) ? 128
                               : (SP * RCOLS <= 256) ? 256 : 512;
    static constexpr int SZ_F = SH * WIN * DP * 4;
    static constexpr int SZ_G = NP * SH * MS * 8;           // one (buffer, slot) of G-pairs
    static constexpr int SZ_RING = RING * TX * 8;           // one slot's (c, s) ring
    static constexpr int OFF_F = 0;
    static constexpr int OFF_G = round_up(OFF_F + SZ_F, 128);
    static constexpr int OFF_RING = round_up(OFF_G + 2 * SP * SZ_G, 128);
    static constexpr int SZ_TP = (NA / 32) * TX * 9 * 8;      // per producer warp: 32 columns x 9 float2
    static constexpr int OFF_TP = round_up(OFF_RING + SP * SZ_RING, 128);
    static constexpr int OFF_BAR = round_up(OFF_TP + SZ_TP, 128);
#ifdef BFVEC_CHECKED
    // checked build: row tags of every ring slot (TMEM ring per (sample, pair), (c, s) ring per
    // sample) and the sub-step id held by each G buffer -- the consumers verify that every slot
    // they read still holds the row they expect, before and after reading it
    static constexpr int OFF_TAG = OFF_BAR + 128;
    static constexpr int NTAG = SP * 4 * HROWS + SP * RING + 2;
    static constexpr size_t SMEM = OFF_TAG + 4 * NTAG;
#else
    static constexpr size_t SMEM = OFF_BAR + 9 * 8 + 8;    // tma, full[2], empty[2], gfull[2], gempty[2]
#endif
    static constexpr uint32_t TMA_BYTES = SZ_F;
    static_assert(D >= 1 && D <= 3, "one TMEM lane quarter per pair");
    static_assert(CW_ == 1 || CW_ == 2, "one or two consumer warps per pair");
    static_assert(MW_ == 0 || MW_ == 4, "no or four modulation warps");
    static_assert(SP * RCOLS <= 512, "two rings in TMEM");
    static_assert(SPLIT % SH == 0 && SPLIT >= KB, "fill split on a sub-step boundary");
    static_assert(SMEM <= 232448, "shared memory budget");
    static_assert(WIN <= 256, "TMA box dimension");
};

// TMEM load of LR ring rows (2 LR columns) into LR float2, and the matching wait
__device__ __forceinline__ void tmem_ld16c(uint32_t taddr, float2 (&v)[8]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[1].x), "=f"(v[1].y), "=f"(v[2].x), "=f"(v[2].y), "=f"(v[3].x),
          "=f"(v[3].y), "=f"(v[4].x), "=f"(v[4].y), "=f"(v[5].x), "=f"(v[5].y), "=f"(v[6].x), "=f"(v[6].y),
          "=f"(v[7].x), "=f"(v[7].y)
        : "r"(taddr)
        : "memory");
}
template <int LR>
__device__ __forceinline__ void tmem_ld_rows(uint32_t taddr, float2 (&v)[LR]) {
    if constexpr (LR == 16) tmem_ld32(taddr, v);
    else tmem_ld16c(taddr, v);
}
template <int LR>
__device__ __forceinline__ void tmem_wait_rows(float2 (&v)[LR]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < LR; ++i) asm volatile("" : "+f"(v[i].x), "+f"(v[i].y));
}

// One FIR input v = x[J] (J = compile-time index into the item's input window) for NOUT consecutive
// outputs: out[o] = sum_{m=-R..R} w[|m|] x[o + R + m].
//  * general taps: every output the input reaches gets one FFMA2;
//  * box taps (BOX, "box ... filter", reading R15; all weights w = 1/(2R+1)): a running
//    sum -- out[0] takes x[0..2R], then out[o] = out[o-1] + w x[o+2R] - w x[o-1] -- so NOUT outputs
//    cost 2R+1 + 2(NOUT-1) FFMA2 instead of NOUT (2R+1); x[0..NOUT-2] are kept for the subtraction.
template <class C, int NOUT, int J>
__device__ __forceinline__ void fir_input(const FusedArgs &a, float2 (&acc)[NOUT], float2 (&early)[NOUT], float2 v) {
    if constexpr (C::BOX) {
        const float w = a.w[0];
        if constexpr (J <= 2 * C::R) acc[0] = ffma2(w, v, acc[0]);
        if constexpr (J < NOUT - 1) early[J] = v;
        if constexpr (J > 2 * C::R && J - 2 * C::R < NOUT) {
            constexpr int o = J - 2 * C::R;
            acc[o] = ffma2(-w, early[o - 1], ffma2(w, v, acc[o - 1]));
        }
    } else {
        (void)early;
        static_for<NOUT>([&](auto O) {
            constexpr int o = decltype(O)::value;
            constexpr int m = J - o - C::R;
            if constexpr (m >= -C::R && m <= C::R) acc[o] = ffma2(a.w[m < 0 ? -m : m], v, acc[o]);
        });
    }
}

__device__ __forceinline__ float2 add2(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 shfl_xor2(float2 v, int m) {
    return make_float2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
__device__ __forceinline__ float2 shfl_up2(float2 v, int d) {
    return make_float2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}

// Box H-pass as a running sum shared by the four lanes of a row (lanes r8 + 8 cg, cg = 0..3):
// S(c) = sum_{j=c}^{c+2R} x[j] for the strip's 32 columns c. S(0) is summed cooperatively (each lane
// a quarter of the 2R+1 inputs, two xor-shuffles), every lane forms its 8 deltas
// D(c) = x[c+2R] - x[c-1], an inclusive prefix of them, and the exclusive scan of the lanes' delta
// totals over cg (two shuffle-ups); out(c) = w S(c). ~(2R+1)/4 + 16 loads and ~50 paired adds per
// thread, independent of R apart from the base quarter, instead of 8 (2R+1) FFMA2.
template <class C>
__device__ __forceinline__ void box_hpass(const FusedArgs &a, const float2 *row, int cg, float2 (&acc)[8]) {
    constexpr int NW = 2 * C::R + 1;
    constexpr int QW = (NW + 3) / 4;
    const float w = a.w[0];
    float2 s0 = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < QW; ++i) {
        const int j = cg * QW + i;
        if (j < NW) s0 = add2(s0, row[j]);
    }
    s0 = add2(s0, shfl_xor2(s0, 8));
    s0 = add2(s0, shfl_xor2(s0, 16));
    float2 pre[8];
    float2 run = make_float2(0.f, 0.f);
#pragma unroll
    for (int o = 0; o < 8; ++o) {
        const int c = 8 * cg + o;
        if (c > 0) run = add2(run, sub2(row[c + 2 * C::R], row[c - 1]));
        pre[o] = run;
    }
    // exclusive scan of the lane totals over cg
    const float2 tot = run;
    float2 inc = tot;
    float2 up = shfl_up2(inc, 8);
    if (cg >= 1) inc = add2(inc, up);
    up = shfl_up2(inc, 16);
    if (cg >= 2) inc = add2(inc, up);
    const float2 base = add2(s0, sub2(inc, tot));
#pragma unroll
    for (int o = 0; o < 8; ++o) acc[o] = make_float2(w * (base.x + pre[o].x), w * (base.y + pre[o].y));
}

// modulation of one SH-row sub-step for the pass's samples (np of them) into G[buf][s]
template <class C, int NTH>
__device__ __forceinline__ void modulate2(int ta, const float *fbuf, float2 *gb0, float2 *gb1, float2 *cs0,
                                          float2 *cs1, const float (&tk)[2][C::D], int g0, int np,
                                          int *cstag = nullptr) {
    (void)cstag;
    constexpr int PER = (C::SH * C::WIN + NTH - 1) / NTH;
    const int base = g0 % C::RING;   // ring row of the sub-step's row 0 (one modulo per call)
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int it = ta + i * NTH;
        const int row = it / C::WIN;
        const int j = it - row * C::WIN;
        if (it >= C::SH * C::WIN) continue;
        const float4 q = *reinterpret_cast<const float4 *>(fbuf + (row * C::WIN + j) * C::DP);
        const float fv[4] = {q.x, q.y, q.z, q.w};
        const bool inner = j >= C::R && j < C::R + C::TX;
        const int rr = base + row;   // row < SH <= RING: at most one wrap
        const int rs = (rr >= C::RING ? rr - C::RING : rr) * C::TX + (j - C::R);
#pragma unroll
        float2 th2 = make_float2(0.f, 0.f);   // both samples' phases, one FFMA2 per channel
#pragma unroll
        for (int c = 0; c < C::D; ++c) th2 = __ffma2_rn(make_float2(tk[0][c], tk[1][c]), make_float2(fv[c], fv[c]), th2);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            if (s >= np) break;
            const float th = s == 0 ? th2.x : th2.y;
            float sn, cn;
            __sincosf(th, &sn, &cn);
            float2 *dst = (s == 0 ? gb0 : gb1) + row * C::MS + j;
            dst[0] = make_float2(cn, sn);
#pragma unroll
            for (int p = 1; p < C::NP; ++p)
                dst[p * C::SH * C::MS] = __fmul2_rn(make_float2(cn, sn), make_float2(fv[p - 1], fv[p - 1]));
            if (inner) (s == 0 ? cs0 : cs1)[rs] = make_float2(cn, sn);
#ifdef BFVEC_CHECKED
            if (j == C::R) cstag[s * C::RING + (g0 + row) % C::RING] = g0 + row;
#endif
        }
    }
}

// One pass over (part of) a strip: what every warp role needs to walk the same sequence of passes.
struct PassDesc {
    int x0;        // first column of the strip
    int k, np;     // first sample (row of the t table) and samples in this pass (<= SP)
    int cb, nch;   // first chunk of the tile and chunks in this pass
    int prow;      // padded (tensor-map) row of H-row 0 of this pass
    int ty0, ty1;  // output rows of the tile (image coordinates)
    int slot, img; // partial-sum slot (sample group) and image of the batch
    int ip;        // pass index within the item
    int cb0;       // first chunk of the item's first pass
    bool last;     // last pass of the item
};

// The pass sequence of one CTA: either the classic (strip, tile, group) of blockIdx -- passes of SP
// samples over the whole tile -- or the items of the persistent schedule (FusedArgs::items).
template <class C>
struct PassIter {
    const FusedArgs &a;
    // classic
    int x0, img, ty0, ty1, gk0, gk1, nch, prow0, g;
    // persistent
    int it, it_end, x, ub, ue, p, pe;
    int pass;
    __device__ explicit PassIter(const FusedArgs &a_) : a(a_) {
        if (a.items) {
            it = a.item_off[blockIdx.x];
            it_end = a.item_off[blockIdx.x + 1];
            load_item();
        } else {
            x0 = blockIdx.x * C::TX;
            img = a.tiles_per_img ? (int)blockIdx.y / a.tiles_per_img : 0;     // image of the batch
            const int tile = a.tiles_per_img ? (int)blockIdx.y % a.tiles_per_img : (int)blockIdx.y;
            ty0 = a.out_row0 + tile * a.tile_rows;
            ty1 = min(ty0 + a.tile_rows, a.out_row0 + a.out_rows);
            g = blockIdx.z;
            const int ns = a.k1 - a.k0;
            // sample range of group g: a slice of [k0, k1), or -- realisation batching (gstride > 0,
            // bf_vec_mse_sweep) -- the same [k0, k1) of realisation g's draws at t rows g * gstride + k
            gk0 = a.gstride ? a.k0 + g * a.gstride : a.k0 + (int)((long long)ns * g / a.groups);
            gk1 = a.gstride ? a.k1 + g * a.gstride : a.k0 + (int)((long long)ns * (g + 1) / a.groups);
            nch = (ty1 - ty0 + C::KB - 1) / C::KB;
            prow0 = img * a.img_prows + (ty0 - a.out_row0);
            pass = 0;
        }
    }
    __device__ void load_item() {
        if (it >= it_end) return;
        const int4 e = a.items[it];
        x = e.x;
        ub = e.y;
        ue = e.z;
        p = ub / a.nch_full;
        pe = (ue - 1) / a.nch_full;
        pass = 0;
    }
    __device__ bool valid() const { return a.items ? it < it_end : gk0 + pass * C::SP < gk1; }
    __device__ PassDesc get() const {
        PassDesc d;
        if (a.items) {
            const int nf = a.nch_full;
            d.x0 = x * C::TX;
            d.k = a.k0 + p * C::SP;
            d.np = min(C::SP, a.k1 - d.k);
            d.cb = (pass == 0) ? ub % nf : 0;
            const int ce = (p == pe) ? (ue - 1) % nf + 1 : nf;
            d.nch = ce - d.cb;
            d.prow = d.cb * C::KB;
            d.ty0 = a.out_row0;
            d.ty1 = a.out_row0 + a.out_rows;
            d.slot = a.items[it].w;
            d.img = 0;
            d.ip = pass;
            d.cb0 = ub % nf;
            d.last = p == pe;
        } else {
            d.x0 = x0;
            d.k = gk0 + pass * C::SP;
            d.np = min(C::SP, gk1 - d.k);
            d.cb = 0;
            d.nch = nch;
            d.prow = prow0;
            d.ty0 = ty0;
            d.ty1 = ty1;
            d.slot = g;
            d.img = img;
            d.ip = pass;
            d.cb0 = 0;
            d.last = d.k + C::SP >= gk1;
        }
        return d;
    }
    __device__ void advance() {
        ++pass;
        if (a.items && p++ == pe) {
            ++it;
            load_item();
        }
    }
};

// H-rows a pass streams: the first chunk's A (its 2R-row halo) and KB per further chunk
template <class C>
__device__ __forceinline__ int pass_rows(const PassDesc &d) {
    return C::A + (d.nch - 1) * C::KB;
}

template <class C>
__global__ void __launch_bounds__(C::NT, 1) mcsf_tmem2_kernel(const __grid_constant__ FusedArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *fbuf = reinterpret_cast<float *>(smem + C::OFF_F);
    float2 *gbase = reinterpret_cast<float2 *>(smem + C::OFF_G);
    float2 *csbase = reinterpret_cast<float2 *>(smem + C::OFF_RING);
    float2 *tpose = reinterpret_cast<float2 *>(smem + C::OFF_TP);
    uint64_t *tma_bar = reinterpret_cast<uint64_t *>(smem + C::OFF_BAR);
    uint64_t *full = tma_bar + 1;
    uint64_t *empty = tma_bar + 3;
    uint64_t *gfull = tma_bar + 5;    // modulators -> H-pass producers, per G buffer
    uint64_t *gempty = tma_bar + 7;   // H-pass producers -> modulators
    uint32_t *taddr_s = reinterpret_cast<uint32_t *>(tma_bar + 9);
#ifdef BFVEC_CHECKED
    int *ttag = reinterpret_cast<int *>(smem + C::OFF_TAG);          // [SP][4][HROWS]
    int *cstag = ttag + C::SP * 4 * C::HROWS;                         // [SP][RING]
    int *gtag = cstag + C::SP * C::RING;                              // [2]
    for (int i = threadIdx.x; i < C::NTAG; i += C::NT) ttag[i] = -1;
#else
    int *cstag = nullptr;
#endif
    constexpr int GSZ = C::NP * C::SH * C::MS;     // float2 per (buffer, slot)
    constexpr int CSZ = C::RING * C::TX;           // float2 per slot's (c, s) ring

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

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
        mbar_init(&gfull[0], C::NM > 0 ? C::NM : 1);
        mbar_init(&gfull[1], C::NM > 0 ? C::NM : 1);
        mbar_init(&gempty[0], C::NA);
        mbar_init(&gempty[1], C::NA);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *taddr_s;

    const PassIter<C> pit(a);   // this CTA's passes (every role walks the same sequence)
    if (pit.valid()) {
        if (tid < C::NA) {
            // ============================ PRODUCER ============================
            const int ta = tid;
            const int p = warp & 3;                          // pair == TMEM quarter
            const int sw = warp >> 2;                        // sample slot of this warp's H-pass
            const int r8 = lane & 7, cg = lane >> 3;         // item: row r8, columns 8cg .. 8cg+7
            const uint32_t tq = tbase + ((uint32_t)(32 * p) << 16) + (uint32_t)(sw * C::RCOLS);
            uint32_t tparity = 0;
            int buf = 0, it = 0;
            PassIter<C> pi = pit;
            if (C::MW == 0 && ta == 0) {
                const PassDesc d0 = pi.get();
                tma_load_3d(fbuf, &a.tmap, tma_bar, 0, d0.x0, d0.prow, C::TMA_BYTES);
            }
            int q = 0, gs = 0;   // chunk counter, H-row counter at the start of the pass
            for (; pi.valid(); pi.advance()) {
                const PassDesc pd = pi.get();
                const int np = pd.np, k = pd.k, nchunks = pd.nch;
                float tk[2][C::D];
#pragma unroll
                for (int s = 0; s < 2; ++s)
#pragma unroll
                    for (int c = 0; c < C::D; ++c)
                        tk[s][c] = (c < a.d && s < np) ? __ldg(a.t + (long long)(k + s) * a.d + c) : 0.f;
                for (int ci = 0; ci < nchunks; ++ci, ++q) {
                    const bool first_c = (ci == 0);
                    if (q >= 2) mbar_wait(&empty[q & 1], ((q - 2) >> 1) & 1);   // consumers' chunk q-2 done
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const int u_begin = first_c ? 0 : C::A + (ci - 1) * C::KB;
                    const int n_new = first_c ? C::A : C::KB;
                    for (int s0 = 0; s0 < n_new; s0 += C::SH, buf ^= 1, ++it) {
                        if (!C::OV && first_c && s0 == C::SPLIT && q >= 1) {
                            // the rest of the fill reuses the slots of the previous pass's last chunk
                            mbar_wait(&empty[(q - 1) & 1], ((q - 1) >> 1) & 1);
                            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        }
                        const int gsub = gs + u_begin + s0;
                        float2 *gb0 = gbase + (2 * buf + 0) * GSZ;
                        float2 *gb1 = gbase + (2 * buf + 1) * GSZ;
                        if constexpr (C::MW == 0) {
                            mbar_wait(tma_bar, tparity);
                            tparity ^= 1u;
                            modulate2<C, C::NA>(ta, fbuf, gb0, gb1, csbase, csbase + CSZ, tk, gsub, np, cstag);
                            named_sync<C::NA>(1);   // G-pairs complete; fbuf free; previous H-pass done
                            if (ta == 0) {
                                int nu = -1;
                                if (s0 + C::SH < n_new) nu = u_begin + s0 + C::SH;
                                else if (ci + 1 < nchunks) nu = C::A + ci * C::KB;
                                if (nu >= 0) {
                                    tma_load_3d(fbuf, &a.tmap, tma_bar, 0, pd.x0, pd.prow + nu, C::TMA_BYTES);
                                } else {   // first box of the next pass, if any
                                    PassIter<C> nx = pi;
                                    nx.advance();
                                    if (nx.valid()) {
                                        const PassDesc nd = nx.get();
                                        tma_load_3d(fbuf, &a.tmap, tma_bar, 0, nd.x0, nd.prow, C::TMA_BYTES);
                                    }
                                }
                            }
                        } else {
                            mbar_wait(&gfull[buf], (it >> 1) & 1);   // the modulators filled G[buf]
#ifdef BFVEC_CHECKED
                            BF_CHECK(gtag[buf] == it);
#endif
                        }
                        if (p < C::NP && sw < np) {
                            // horizontal FIR: 8 outputs (row r8, columns 8cg .. 8cg+7) of sample sw
                            const float2 *in = (sw == 0 ? gb0 : gb1) + (p * C::SH + r8) * C::MS + cg * 8;
                            float2 acc[8], early[8];
#pragma unroll
                            for (int o = 0; o < 8; ++o) acc[o] = make_float2(0.f, 0.f);
                            if constexpr (C::BOX) {
                                box_hpass<C>(a, in - cg * 8, cg, acc);
                            } else {
                                static_for<C::NIN / 2>([&](auto JJ) {
                                    constexpr int jj = decltype(JJ)::value;
                                    const float4 v2 = *reinterpret_cast<const float4 *>(in + 2 * jj);
                                    fir_input<C, 8, 2 * jj>(a, acc, early, make_float2(v2.x, v2.y));
                                    fir_input<C, 8, 2 * jj + 1>(a, acc, early, make_float2(v2.z, v2.w));
                                });
                            }
#ifdef BFVEC_CHECKED
                            if constexpr (C::MW > 0) BF_CHECK(gtag[buf] == it);   // not refilled while read
#endif
                            if constexpr (C::MW > 0) mbar_arrive(&gempty[buf]);   // G[buf] read
                            // transpose through this warp's shared-memory tile: lane (r8, cg) holds
                            // row r8 of columns 8cg..8cg+7; lane x needs rows 0..7 of column x.
                            // Stride 9 float2 per column: both directions are bank-conflict free.
                            float2 *tt = tpose + warp * (C::TX * 9);
#pragma unroll
                            for (int o = 0; o < 8; ++o) tt[(8 * cg + o) * 9 + r8] = acc[o];
                            __syncwarp();
#pragma unroll
                            for (int o = 0; o < 8; ++o) acc[o] = tt[lane * 9 + o];
                            __syncwarp();
                            const int slot = gsub % C::HROWS;   // 8 consecutive slots, no wrap
                            BF_CHECK(slot + 8 <= C::HROWS);
                            tmem_st16(tq + 2 * slot, acc);
#ifdef BFVEC_CHECKED
                            if (lane < 8) ttag[(sw * 4 + p) * C::HROWS + slot + lane] = gsub + lane;
#endif
                        } else if constexpr (C::MW > 0) {
                            mbar_arrive(&gempty[buf]);
                        }
                        if (s0 + C::SH >= n_new) {
                            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                            mbar_arrive(&full[q & 1]);
                        }
                    }
                }
                gs += pass_rows<C>(pd);
            }
        } else if (tid >= C::NA + C::NB) {
            // ============================ MODULATORS (MW > 0) =================
            // Alg. 1 L222-226 for both samples of a pass, one SH-row sub-step at a time, into the
            // double-buffered G-pairs; they also own the TMA of f. They run up to two sub-steps
            // ahead of the H-pass (gfull / gempty), which the (c, s) ring's 2 SH extra rows absorb.
            if constexpr (C::MW > 0) {
                const int tm = tid - C::NA - C::NB;
                uint32_t tparity = 0;
                int buf = 0, it = 0;
                PassIter<C> pi = pit;
                if (tm == 0) {
                    const PassDesc d0 = pi.get();
                    tma_load_3d(fbuf, &a.tmap, tma_bar, 0, d0.x0, d0.prow, C::TMA_BYTES);
                }
                int gs = 0;
                for (; pi.valid(); pi.advance()) {
                    const PassDesc pd = pi.get();
                    const int np = pd.np, k = pd.k, nchunks = pd.nch;
                    float tk[2][C::D];
#pragma unroll
                    for (int s = 0; s < 2; ++s)
#pragma unroll
                        for (int c = 0; c < C::D; ++c)
                            tk[s][c] = (c < a.d && s < np) ? __ldg(a.t + (long long)(k + s) * a.d + c) : 0.f;
                    for (int ci = 0; ci < nchunks; ++ci) {
                        const bool first_c = (ci == 0);
                        const int u_begin = first_c ? 0 : C::A + (ci - 1) * C::KB;
                        const int n_new = first_c ? C::A : C::KB;
                        for (int s0 = 0; s0 < n_new; s0 += C::SH, buf ^= 1, ++it) {
                            const int gsub = gs + u_begin + s0;
                            if (it >= 2) mbar_wait(&gempty[buf], ((it - 2) >> 1) & 1);
                            mbar_wait(tma_bar, tparity);
                            tparity ^= 1u;
                            modulate2<C, C::NM>(tm, fbuf, gbase + (2 * buf) * GSZ, gbase + (2 * buf + 1) * GSZ, csbase,
                                                csbase + CSZ, tk, gsub, np, cstag);
                            named_sync<C::NM>(2);   // fbuf consumed by every modulator
#ifdef BFVEC_CHECKED
                            if (tm == 0) gtag[buf] = it;
#endif
                            if (tm == 0) {
                                int nu = -1;
                                if (s0 + C::SH < n_new) nu = u_begin + s0 + C::SH;
                                else if (ci + 1 < nchunks) nu = C::A + ci * C::KB;
                                if (nu >= 0) {
                                    tma_load_3d(fbuf, &a.tmap, tma_bar, 0, pd.x0, pd.prow + nu, C::TMA_BYTES);
                                } else {   // first box of the next pass, if any
                                    PassIter<C> nx = pi;
                                    nx.advance();
                                    if (nx.valid()) {
                                        const PassDesc nd = nx.get();
                                        tma_load_3d(fbuf, &a.tmap, tma_bar, 0, nd.x0, nd.prow, C::TMA_BYTES);
                                    }
                                }
                            }
                            mbar_arrive(&gfull[buf]);
                        }
                    }
                    gs += pass_rows<C>(pd);
                }
            }
        } else {
            // ============================ CONSUMERS ===========================
            // warp 8 + w: pair p = w & 3 (TMEM quarter p); part h = w >> 2 owns output rows
            // h*OR .. h*OR + OR - 1 of every chunk. Both parts run the same code: the window of
            // part h starts h*OR ring rows later (8-row TMEM loads when OR = 8).
            const int p = warp & 3;
            const int h = (warp - C::NA / 32) >> 2;
            const int H0 = h * C::OR;
            const uint32_t tq = tbase + ((uint32_t)(32 * p) << 16);
            const bool active = p < C::NP;
            const long long plane_out = (long long)a.out_rows * a.W;
            const int plane = (p == 0) ? C::D : p - 1;
            constexpr int OR = C::OR;
            constexpr int LR = (OR == 16) ? 16 : 8;                  // ring rows per TMEM load
            constexpr int JB1 = (OR - 1 + 2 * C::R) / LR + 1;        // loads per window
            PassIter<C> pi = pit;
            int q = 0, gs = 0;
            for (; pi.valid(); pi.advance()) {
                const PassDesc pd = pi.get();
                const int np = pd.np, nchunks = pd.nch, ty1 = pd.ty1;
                const int x = pd.x0 + lane;
                const bool xok = x < a.W;
                float *pzp = a.pz + pd.img * a.img_pz + ((long long)pd.slot * (C::D + 1) + plane) * plane_out + x;
                for (int ci = 0; ci < nchunks; ++ci, ++q) {
                    // this item's first visit of the chunk starts its partial sum (the item's first
                    // pass covers chunks cb0.., its second pass the chunks before cb0)
                    const int cabs = pd.cb + ci;
                    const bool first = pd.ip == 0 || (pd.ip == 1 && cabs < pd.cb0);
                    const int cy = pd.ty0 + cabs * C::KB + H0;
                    float *dst = pzp + (long long)(cy - a.out_row0) * a.W;
                    float tot[OR];
#pragma unroll
                    for (int o = 0; o < OR; ++o) {
                        const bool ok = active && xok && (cy + o < ty1);
                        tot[o] = (!first && ok) ? dst[(long long)o * a.W] : 0.f;
                    }
                    mbar_wait(&full[q & 1], (q >> 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const int b0 = (gs + ci * C::KB + H0) % C::HROWS;   // multiple of LR
#pragma unroll 1
                    for (int s = 0; s < np; ++s) {
                        const uint32_t tr = tq + (uint32_t)(s * C::RCOLS);
                        float2 acc[OR], early[OR];
#pragma unroll
                        for (int o = 0; o < OR; ++o) acc[o] = make_float2(0.f, 0.f);
                        float2 v[2][LR];
                        auto slot_of = [&](int bj) {
                            const int slot = b0 + LR * bj;
                            return slot >= C::HROWS ? slot - C::HROWS : slot;
                        };
                        tmem_ld_rows<LR>(tr + 2 * slot_of(0), v[0]);
                        tmem_wait_rows<LR>(v[0]);
                        static_for<JB1>([&](auto B) {
                            constexpr int bj = decltype(B)::value;
                            if constexpr (bj + 1 < JB1) tmem_ld_rows<LR>(tr + 2 * slot_of(bj + 1), v[(bj + 1) & 1]);
                            static_for<LR>([&](auto JJ) {
                                constexpr int j = LR * bj + decltype(JJ)::value;
                                fir_input<C, OR, j>(a, acc, early, v[bj & 1][decltype(JJ)::value]);
                            });
                            if constexpr (bj + 1 < JB1) tmem_wait_rows<LR>(v[(bj + 1) & 1]);
                        });
#ifdef BFVEC_CHECKED
                        if (active && lane == 0) {
                            // every TMEM ring row of this window (loaded above) must still be the
                            // row the window expects, after the loads completed
                            for (int j = 0; j < JB1 * LR; ++j) {
                                const int sl = (b0 + j) % C::HROWS;
                                const int want = gs + ci * C::KB + H0 + j;
                                if (j < C::OR + 2 * C::R) BF_CHECK(ttag[(s * 4 + p) * C::HROWS + sl] == want);
                            }
                            for (int o = 0; o < OR; ++o) {
                                const int row = gs + ci * C::KB + H0 + C::R + o;
                                BF_CHECK(cstag[s * C::RING + row % C::RING] == row);
                            }
                        }
#endif
                        const float2 *csr = csbase + s * CSZ;
                        int slot = (gs + ci * C::KB + H0 + C::R) % C::RING;
#pragma unroll
                        for (int o = 0; o < OR; ++o) {
                            const float2 cs = csr[slot * C::TX + lane];
                            tot[o] = fmaf(cs.x, acc[o].x, fmaf(cs.y, acc[o].y, tot[o]));
                            slot = (slot + 1 == C::RING) ? 0 : slot + 1;
                        }
                    }
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    mbar_arrive(&empty[q & 1]);
                    if (active && xok) {
                        if (a.p2p_world > 0 && pd.last) {
                            // last pass of the group: the finished partial goes to the band owner's
                            // receive slot (peer memory over NVLink), not back to the local tile
#pragma unroll
                            for (int o = 0; o < OR; ++o) {
                                const int row = cy + o;
                                if (row < ty1) {
                                    const int owner = row / a.p2p_rpb;
                                    float *slot = a.peer[owner] +
                                                  ((long long)(a.p2p_rank * a.groups + pd.slot) * (C::D + 1) + plane) *
                                                      a.p2p_rpb * a.W;
                                    slot[(long long)(row - owner * a.p2p_rpb) * a.W + x] = tot[o];
                                }
                            }
                        } else {
#pragma unroll
                            for (int o = 0; o < OR; ++o)
                                if (cy + o < ty1) dst[(long long)o * a.W] = tot[o];
                        }
                    }
                }
                if (a.items && pd.last && active && xok && pi.ue - pi.ub < a.nch_full) {
                    // persistent schedule, end of an item that covered less than a whole pass: its
                    // slot's rows it never visited are zeroed (the normaliser sums every slot the
                    // strip's items wrote, over all rows)
                    const int nf = a.nch_full;
                    const int total = pi.ue - pi.ub, c0 = pi.ub % nf;
                    float *zp = a.pz + ((long long)pd.slot * (C::D + 1) + plane) * plane_out + x;
                    for (int c = 0; c < nf; ++c) {
                        if ((c - c0 + nf) % nf < total) continue;
                        for (int o = 0; o < OR; ++o) {
                            const int row = pd.ty0 + c * C::KB + H0 + o;
                            if (row < ty1) zp[(long long)(row - a.out_row0) * a.W] = 0.f;
                        }
                    }
                }
                gs += pass_rows<C>(pd);
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
cudaError_t launch_tmem2(const FusedArgs &a, dim3 grid, cudaStream_t s) {
    auto k = mcsf_tmem2_kernel<C>;
    static std::atomic<uint64_t> attr{0};
    const cudaError_t e = ensure_smem_attr(k, C::SMEM, attr);
    if (e != cudaSuccess) return e;
    k<<<grid, C::NT, C::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <class C>
void fill_info_tmem2(KernelInfo *info) {
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
    info->sp = C::SP;
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, mcsf_tmem2_kernel<C>) == cudaSuccess) info->regs = fa.numRegs;
    if (cudaFuncSetAttribute(mcsf_tmem2_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM) ==
        cudaSuccess) {
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mcsf_tmem2_kernel<C>, C::NT, C::SMEM) == cudaSuccess)
            info->occupancy = occ;
    }
    cudaGetLastError();
}

}  // namespace
}  // namespace bfvec
