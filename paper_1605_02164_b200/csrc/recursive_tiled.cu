// recursive_tiled.cu -- the O(1)-in-sigma_s engine without intermediate images in HBM
// (option "rec_impl" = 1, the default of engine 1).
//
// Same arithmetic as recursive.cu ("using separability and recursion ... at O(1)
// cost with respect to sigma_s"; Deriche kernel, reading R16; reflected-periodic lines, R1):
// per line x[0..n-1] and pole z_j,
//   u_j[k] = x[k] + z_j u_j[k-1],  v_j[k] = x[k] + z_j v_j[k+1],  y[k] = sum_j Re[A_j (u_j + v_j)] - g0 x[k],
//   u_j[-1] = (S_head + z^n S_tail) / (1 - z^2n),  v_j[n] = u_j[n-1].
// The image is cut into 32 x 32 tiles. By linearity a tile's segment of a line only needs the two
// states entering it, u[x0-1] and v[x0+L], and those follow from per-tile summaries
//   e_t = sum_m z^{L-1-m} x[x0+m]  (causal end state from zero),  b_t = sum_m z^m x[x0+m]
// by a scan along the line:  u[x0_{t+1}-1] = z^{L_t} u[x0_t-1] + e_t,  v[x0_{t-1}+L] = z^{L_t} v[x0_t+L] + b_t,
// with S_tail / S_head the zero-started scans' final values (exact: no head / tail truncation).
// Per batch of samples:
//   pass 0 (tile)  : modulate (Alg. 1), row summaries e, b of the 2(d+1) planes
//   scan rows      : zero-started row states per tile + (u_{-1}, v_n) per row
//   pass 1 (tile)  : exact row blur of the tile into shared memory, column summaries
//   scan columns   : the same along columns
// rec_impl 2 (default) drops pass 1: the column summaries of the row-blurred planes are, by linearity,
// the row blur of the column summaries of the modulated planes -- 8 "virtual lines" per tile row
// (pole, kind, real / imaginary part), formed in pass 0 and appended to the row lines of the row
// scan; the column scan (rect_vscan_kernel) row-blurs their tile segments from their entering states
// and scans the result, so only pass 2 blurs whole tiles.
//   pass 2 (tile)  : exact row blur, exact column blur, Re[conj(H) blur] (Alg. 1) summed
//                    over the group's samples in a shared-memory accumulator, one partial plane
//                    set per group.
// HBM sees f, the summaries (8 B per pixel-sample per axis) and the partial sums only.
// Inside a tile: summaries are dot products with z^m (no dependency chain); an exact segment
// runs its causal and anticausal recursions interleaved (two independent chains); the entering
// states are loaded one stage ahead; each warp owns one (cos, sin) pair of planes, so only the
// modulation needs a CTA barrier.
#include <cuda_runtime.h>

#include "internal.h"
#include "kernel_common.cuh"

namespace bfvec {
namespace {

constexpr int T = kRecT;
constexpr int TP = T + 1;

struct St {              // both poles, (c-part, s-part) of one pair of planes
    float2 ur[2], ui[2];
};

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fma2s(float w, float2 v, float2 acc) {
    return __ffma2_rn(make_float2(w, w), v, acc);
}
__device__ __forceinline__ float2 mul2s(float w, float2 v) { return __fmul2_rn(make_float2(w, w), v); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return f2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return f2(a.x + b.x, a.y + b.y); }

__device__ __forceinline__ void zero(St &s) {
#pragma unroll
    for (int j = 0; j < 2; ++j) s.ur[j] = s.ui[j] = f2(0.f, 0.f);
}
// u <- x + z u for both poles
__device__ __forceinline__ void step(const RecAxis &ax, St &s, float2 x) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const float2 ur = s.ur[j], ui = s.ui[j];
        s.ur[j] = fma2s(ax.zr[j], ur, fma2s(-ax.zi[j], ui, x));
        s.ui[j] = fma2s(ax.zr[j], ui, mul2s(ax.zi[j], ur));
    }
}
// sum_j Re[A_j u_j]
__device__ __forceinline__ float2 re_a(const RecAxis &ax, const St &s) {
    float2 y = mul2s(ax.ar[0], s.ur[0]);
    y = fma2s(-ax.ai[0], s.ui[0], y);
    y = fma2s(ax.ar[1], s.ur[1], y);
    y = fma2s(-ax.ai[1], s.ui[1], y);
    return y;
}

// summary / state arrays: (s, q, j, tile, line) and (s, q, j, line)
__device__ __forceinline__ long long sidx(int s, int q, int j, int t, int line, int NQ, int nt, int nlines) {
    return ((((long long)s * NQ + q) * 2 + j) * nt + t) * nlines + line;
}
__device__ __forceinline__ long long uidx(int s, int q, int j, int line, int NQ, int nlines) {
    return (((long long)s * NQ + q) * 2 + j) * nlines + line;
}

// store the pair's two planes' state (q = 2p: .x parts, q = 2p + 1: .y parts) for both poles
__device__ __forceinline__ void put_state(float2 *A, const St &s, int b, int p, int t, int line, int NQ, int nt,
                                          int nlines) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        A[sidx(b, 2 * p, j, t, line, NQ, nt, nlines)] = f2(s.ur[j].x, s.ui[j].x);
        A[sidx(b, 2 * p + 1, j, t, line, NQ, nt, nlines)] = f2(s.ur[j].y, s.ui[j].y);
    }
}
// The exact states entering tile t of a line from the scanned zero-started ones:
//   L = Lz + z^{x0} u_{-1},  R = Rz + z^{n - x0 - L} v_n.
// load_raw issues the loads a whole sample before their use; the arithmetic that turns them into
// entering states runs only at the use (make_states), so no instruction waits on the loads in
// between (round 2: the cmul / cadd right after the loads were the top long-scoreboard stall sites
// of pass 2)
struct RawSt {
    float2 e[2][2], b[2][2];   // [pole j][plane h]
    float4 uv[2][2];
};
__device__ __forceinline__ void load_raw(const float2 *E, const float2 *B, const float4 *UV, int b, int p, int t,
                                         int line, int NQ, int nt, int nlines, RawSt &r) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int q = 2 * p + h;
            r.e[j][h] = __ldg(E + sidx(b, q, j, t, line, NQ, nt, nlines));
            r.b[j][h] = __ldg(B + sidx(b, q, j, t, line, NQ, nt, nlines));
            r.uv[j][h] = __ldg(UV + uidx(b, q, j, line, NQ, nlines));
        }
}
// pfb[j] = (z_j^{x0}, z_j^{n - x0 - L}) of this tile (shared memory)
__device__ __forceinline__ void make_states(const RawSt &r, const float4 *pfb, St &L, St &R) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const float4 pp = pfb[j];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 uv = r.uv[j][h];
            const float2 l = cadd(r.e[j][h], cmul(f2(pp.x, pp.y), f2(uv.x, uv.y)));
            const float2 rr = cadd(r.b[j][h], cmul(f2(pp.z, pp.w), f2(uv.z, uv.w)));
            if (h == 0) {
                L.ur[j].x = l.x; L.ui[j].x = l.y; R.ur[j].x = rr.x; R.ui[j].x = rr.y;
            } else {
                L.ur[j].y = l.x; L.ui[j].y = l.y; R.ur[j].y = rr.x; R.ui[j].y = rr.y;
            }
        }
    }
}

template <int NP, int MODE>
struct TileSmem {
    static constexpr int D = NP - 1, NQ = 2 * NP;
    static constexpr int OFF_CS = D * T * TP;                 // floats; fs[D][T][TP] first
    static constexpr int OFF_RB = OFF_CS + 2 * T * TP;        // cs: [T][TP] float2
    static constexpr int OFF_ZP = OFF_RB + (MODE >= 1 ? NQ * T * TP : 0);   // zp[2 axes][T] float4
    static constexpr int OFF_PFB = OFF_ZP + 2 * 4 * T;   // pfb[2 axes][2 poles] float4 (make_states)
    // ones: the multiplier of pair 0's planes (cos, sin themselves), so every pair's input is one FMUL2
    // of (cos, sin) by a plane value -- MODE 0 reads it by row and by column ([T][TP]), MODE >= 1 by row only
    static constexpr int OFF_ZQ = OFF_PFB + 16;           // zpq[T] float4 (MODE 0: virtual-line summaries)
    static constexpr int OFF_ONE = OFF_ZQ + 4 * T;
    static constexpr int OFF_ACC = OFF_ONE + (MODE == 0 ? T * TP : T);   // MODE 2: acc[NP][T][T]; MODE 0: vs[NP][2][8][TP]
    static constexpr size_t BYTES =
        sizeof(float) * (size_t)(OFF_ACC + (MODE == 2 ? NP * T * T : MODE == 0 ? NP * 16 * TP : 0));
};

// zero-started summaries of one pair over a segment of n <= T elements,
//   e = sum_m z^{n-1-m} x[m]  (the causal state after the segment),  b = sum_m z^m x[m],
// as dot products with zp[m] = (z_0^m, z_1^m) -- no dependency chain along the segment.
template <bool FULL, class X>
__device__ __forceinline__ void summaries(const float4 *zp, int n, X xat, St &e, St &b) {
    zero(e);
    zero(b);
#pragma unroll 8
    for (int m = 0; m < T; ++m) {
        if (FULL || m < n) {
            const float2 x = xat(m);
            const float4 pb = zp[m], pe = zp[(FULL ? T : n) - 1 - m];
            b.ur[0] = fma2s(pb.x, x, b.ur[0]);
            b.ui[0] = fma2s(pb.y, x, b.ui[0]);
            b.ur[1] = fma2s(pb.z, x, b.ur[1]);
            b.ui[1] = fma2s(pb.w, x, b.ui[1]);
            e.ur[0] = fma2s(pe.x, x, e.ur[0]);
            e.ui[0] = fma2s(pe.y, x, e.ui[0]);
            e.ur[1] = fma2s(pe.z, x, e.ur[1]);
            e.ui[1] = fma2s(pe.w, x, e.ui[1]);
        }
    }
}

// the same for a full segment (n = T) with the pole powers as compile-time-indexed kernel
// parameters: the loop is fully unrolled, so each z^m is a uniform constant operand of the FFMA2s
// instead of two shared-memory loads per element (pass 0 was shared-memory bound, LSU 94 %; round 2:
// pass 0 4.49 -> 3.80 ms, pass 1 13.5 -> 13.2 ms per 16 config-5 samples)
template <class X>
__device__ __forceinline__ void summaries_full(const float4 (&zt)[T], X xat, St &e, St &b) {
    zero(e);
    zero(b);
#pragma unroll
    for (int m = 0; m < T; ++m) {
        const float2 x = xat(m);
        const float4 pb = zt[m], pe = zt[T - 1 - m];
        b.ur[0] = fma2s(pb.x, x, b.ur[0]);
        b.ui[0] = fma2s(pb.y, x, b.ui[0]);
        b.ur[1] = fma2s(pb.z, x, b.ur[1]);
        b.ui[1] = fma2s(pb.w, x, b.ui[1]);
        e.ur[0] = fma2s(pe.x, x, e.ur[0]);
        e.ui[0] = fma2s(pe.y, x, e.ui[0]);
        e.ur[1] = fma2s(pe.z, x, e.ur[1]);
        e.ui[1] = fma2s(pe.w, x, e.ui[1]);
    }
}

// rec_impl 2: index of a virtual-line value (s, q, ty, v, x); v = (k * 2 + kind) * 2 + part for the
// column pole k, kind 0 = e / 1 = b, part 0 = real / 1 = imaginary
__device__ __forceinline__ long long vlidx(int s, int q, int ty, int v, int x, int NQ, int nty, int W) {
    return ((((long long)s * NQ + q) * nty + ty) * 8 + v) * W + x;
}

// summaries of ONE real line over a segment of n <= T elements, both poles in one FFMA2:
// pr/pi = (Re / Im z_0^m, Re / Im z_1^m); e*, b* hold (pole 0, pole 1)
template <bool FULL, class X, class Z>
__device__ __forceinline__ void summaries_line(int n, X xat, Z zat, float2 &er, float2 &ei, float2 &br, float2 &bi) {
    er = ei = br = bi = f2(0.f, 0.f);
#pragma unroll
    for (int m = 0; m < T; ++m) {
        if (FULL || m < n) {
            const float x = xat(m);
            const float4 pb = zat(m), pe = zat((FULL ? T : n) - 1 - m);
            br = fma2s(x, f2(pb.x, pb.y), br);
            bi = fma2s(x, f2(pb.z, pb.w), bi);
            er = fma2s(x, f2(pe.x, pe.y), er);
            ei = fma2s(x, f2(pe.z, pe.w), ei);
        }
    }
}

// exact blur of one pair along a segment from its entering states: r0/r1[m] (the two planes)
// <- sum_j Re[A_j (u_j + v_j)] - g0 x. Full segments run the causal step at m = i and the
// anticausal one at m = T-1-i in the same iteration (two independent chains); the first half of
// the iterations stores, the second half (where the other direction already wrote) adds.
template <bool FULL, class X>
__device__ __forceinline__ void blur_segment(const RecAxis &ax, int n, X xat, const St &l, const St &r, float *r0,
                                             float *r1) {
    St sf = l, sb = r;
    if constexpr (FULL) {
#pragma unroll 4
        for (int i = 0; i < T / 2; ++i) {
            const int mb = T - 1 - i;
            const float2 xf = xat(i), xb = xat(mb);
            step(ax, sf, xf);
            step(ax, sb, xb);
            const float2 yf = fma2s(-ax.g0, xf, re_a(ax, sf));
            const float2 yb = re_a(ax, sb);
            r0[i] = yf.x;
            r1[i] = yf.y;
            r0[mb] = yb.x;
            r1[mb] = yb.y;
        }
#pragma unroll 4
        for (int i = T / 2; i < T; ++i) {
            const int mb = T - 1 - i;
            const float2 xf = xat(i), xb = xat(mb);
            step(ax, sf, xf);
            step(ax, sb, xb);
            const float2 yf = fma2s(-ax.g0, xf, re_a(ax, sf));
            const float2 yb = re_a(ax, sb);
            r0[i] += yf.x;
            r1[i] += yf.y;
            r0[mb] += yb.x;
            r1[mb] += yb.y;
        }
    } else {
        for (int m = 0; m < n; ++m) {
            const float2 x = xat(m);
            step(ax, sf, x);
            const float2 yv = fma2s(-ax.g0, x, re_a(ax, sf));
            r0[m] = yv.x;
            r1[m] = yv.y;
        }
        for (int m = n - 1; m >= 0; --m) {
            step(ax, sb, xat(m));
            const float2 v = re_a(ax, sb);
            r0[m] += v.x;
            r1[m] += v.y;
        }
    }
}

// exact column blur of one pair, folded into acc[m * T] += Re[conj(H) blur] (Alg. 1);
// acc is this thread's column of the group's shared-memory accumulator. Both directions in the
// same iteration (independent chains; the accumulation is a sum, so the order is free).
template <bool FULL>
__device__ __forceinline__ void blur_accumulate(const RecAxis &ax, int n, const float *c0, const float *c1,
                                                const float2 *h, const St &l, const St &r, float *acc) {
    St sf = l, sb = r;
#pragma unroll 4
    for (int i = 0; i < T; ++i) {
        if (FULL || i < n) {
            const int mb = (FULL ? T : n) - 1 - i;
            const float2 xf = f2(c0[i * TP], c1[i * TP]), xb = f2(c0[mb * TP], c1[mb * TP]);
            step(ax, sf, xf);
            step(ax, sb, xb);
            const float2 yf = fma2s(-ax.g0, xf, re_a(ax, sf));
            const float2 yb = re_a(ax, sb);
            const float2 hf = h[i * TP], hb = h[mb * TP];
            acc[i * T] = fmaf(hf.x, yf.x, fmaf(hf.y, yf.y, acc[i * T]));
            acc[mb * T] = fmaf(hb.x, yb.x, fmaf(hb.y, yb.y, acc[mb * T]));
        }
    }
}

// rec_impl 2, pass 0, one warp = pair p: the column summaries of the pair's modulated planes over the
// tile (lane = column) are the tile's segment of the 8 virtual lines per plane,
//   C_{k,e}[x] = sum_m w_k^{Ly-1-m} X[y0+m, x],  C_{k,b}[x] = sum_m w_k^m X[y0+m, x]   (real, imag parts);
// the row blur is linear, so rowblur(C)[x] is the column summary of the row-blurred plane that pass 1
// of rec_impl 1 computed from a full row blur of the tile. The values go to a.vl (read by the
// column scan, rect_vscan_kernel) and, through shared memory vs[h][v][TP], into the row summaries of the virtual
// lines (lane = (h, v), both poles per FFMA2), stored as rows H + 8 ty + v of Eh / Bh.
template <int NP, class XIN>
__device__ __forceinline__ void virtual_lines(const RecTArgs &a, float *vs, const float4 *zp, const float4 *zq, XIN xin, int b, int p,
                                              int tx, int ty, int lane, int Lx, int Ly, bool full) {
    constexpr int NQ = 2 * NP;
    if (lane < Lx) {
        auto xat = [&](int m) -> float2 { return xin(m, lane); };
        St ce, cb;
        if (full) summaries_full(a.zpc, xat, ce, cb);
        else summaries<false>(zp + T, Ly, xat, ce, cb);
        const int x = tx * T + lane;
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int kind = 0; kind < 2; ++kind) {
                const St &sv = kind ? cb : ce;
                const int v = (k * 2 + kind) * 2;
                const float val[2][2] = {{sv.ur[k].x, sv.ui[k].x}, {sv.ur[k].y, sv.ui[k].y}};
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int part = 0; part < 2; ++part) {
                        vs[(h * 8 + v + part) * TP + lane] = val[h][part];
                        a.vl[vlidx(b, 2 * p + h, ty, v + part, x, NQ, a.nty, a.W)] = val[h][part];
                    }
            }
    }
    __syncwarp();
    if (Lx == T) {
        // full segment: all 32 lanes, lane = (half of the segment, line (h, v)); the two halves'
        // partial dot products are summed with one shuffle
        const int hf = lane >> 4, hv = lane & 15, h = hv >> 3, v = hv & 7;
        const float *row = vs + hv * TP + 16 * hf;
        float2 er = f2(0.f, 0.f), ei = er, br = er, bi = er;
#pragma unroll
        for (int mm = 0; mm < 16; ++mm) {
            const int m = 16 * hf + mm;
            const float x = row[mm];
            const float4 pb = zq[m], pe = zq[T - 1 - m];
            br = fma2s(x, f2(pb.x, pb.y), br);
            bi = fma2s(x, f2(pb.z, pb.w), bi);
            er = fma2s(x, f2(pe.x, pe.y), er);
            ei = fma2s(x, f2(pe.z, pe.w), ei);
        }
        float w[8] = {er.x, er.y, ei.x, ei.y, br.x, br.y, bi.x, bi.y};
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] += __shfl_down_sync(0xffffffffu, w[k], 16);
        if (hf == 0) {
            const int q = 2 * p + h, line = a.H + ty * 8 + v;
            a.Eh[sidx(b, q, 0, tx, line, NQ, a.ntx, a.nlh)] = f2(w[0], w[2]);
            a.Eh[sidx(b, q, 1, tx, line, NQ, a.ntx, a.nlh)] = f2(w[1], w[3]);
            a.Bh[sidx(b, q, 0, tx, line, NQ, a.ntx, a.nlh)] = f2(w[4], w[6]);
            a.Bh[sidx(b, q, 1, tx, line, NQ, a.ntx, a.nlh)] = f2(w[5], w[7]);
        }
    } else if (lane < 16) {
        const int h = lane >> 3, v = lane & 7;
        const float *row = vs + (h * 8 + v) * TP;
        float2 er, ei, br, bi;
        auto xat = [&](int m) -> float { return row[m]; };
        summaries_line<false>(Lx, xat, [&](int m) -> float4 {
            const float4 z = zp[m];
            return make_float4(z.x, z.z, z.y, z.w);
        }, er, ei, br, bi);
        const int q = 2 * p + h, line = a.H + ty * 8 + v;
        a.Eh[sidx(b, q, 0, tx, line, NQ, a.ntx, a.nlh)] = f2(er.x, ei.x);
        a.Eh[sidx(b, q, 1, tx, line, NQ, a.ntx, a.nlh)] = f2(er.y, ei.y);
        a.Bh[sidx(b, q, 0, tx, line, NQ, a.ntx, a.nlh)] = f2(br.x, bi.x);
        a.Bh[sidx(b, q, 1, tx, line, NQ, a.ntx, a.nlh)] = f2(br.y, bi.y);
    }
    __syncwarp();   // vs is rewritten for the next sample
}

// minimum CTAs per SM: what shared memory allows (d >= 7 fits one CTA of pass 1 / 2 per SM)
#ifndef BFVEC_REC_P2CTAS
#define BFVEC_REC_P2CTAS 3   // pass 2 is limited to 3 CTAs per SM by its 72 KB of shared memory anyway (A/B: 21.9 -> 21.2 ms)
#endif
#ifndef BFVEC_REC_P0CTAS
#define BFVEC_REC_P0CTAS 4   // A/B: 5 CTAs 8.53 ms, 6 CTAs 8.94 ms (spills) vs 8.09 ms
#endif
template <int NP, int MODE>
constexpr int tile_min_ctas() {
    return NP <= 4 ? (MODE == 2 ? BFVEC_REC_P2CTAS : MODE == 0 ? BFVEC_REC_P0CTAS : 4) : (MODE == 0 || NP <= 7) ? 2 : 1;
}
// A/B: BFVEC_REC_EAGER turns the raw entering-state loads into states right at the load (as before
// round 2's change) instead of at the use
#ifdef BFVEC_REC_EAGER
constexpr bool kEager = true;
#else
constexpr bool kEager = false;
#endif

template <int NP, int MODE>
__global__ void __launch_bounds__(32 * NP, tile_min_ctas<NP, MODE>()) rect_tile_kernel(const __grid_constant__ RecTArgs a) {
    using L = TileSmem<NP, MODE>;
    constexpr int D = L::D, NQ = L::NQ;
    extern __shared__ float sm[];
    float *fs = sm;
    float2 *cs = reinterpret_cast<float2 *>(sm + L::OFF_CS);
    float *rb = sm + L::OFF_RB;

    const int tid = threadIdx.x, lane = tid & 31, p = tid >> 5;
    const int tx = blockIdx.x % a.ntx, ty = blockIdx.x / a.ntx;
    const int x0 = tx * T, y0 = ty * T;
    const int H = a.H, W = a.W;
    const int Lx = min(T, W - x0), Ly = min(T, H - y0);
    if (MODE == 2 && a.tc && Lx == T && Ly == T) return;   // rect_tc2_kernel's tile
    const long long plane = (long long)H * W;
    const int G = (MODE == 2) ? a.g3 : a.g1, g = blockIdx.y;
    const int s0 = (int)((long long)a.ns * g / G), s1 = (int)((long long)a.ns * (g + 1) / G);

    float4 *zp = reinterpret_cast<float4 *>(sm + L::OFF_ZP);   // [0][m]: row axis, [1][m]: column axis
    if (tid < 2 * T) zp[tid] = (tid < T) ? a.th.zp[tid] : a.tv.zp[tid - T];
    float4 *pfb = reinterpret_cast<float4 *>(sm + L::OFF_PFB);   // [0][j]: row axis (tile tx), [1][j]: column (ty)
    if (tid < 4) {
        const int ax = tid >> 1, j = tid & 1;
        const RecTabs &tb = ax ? a.tv : a.th;
        const int t = ax ? ty : tx, nt = ax ? a.nty : a.ntx;
        const float2 pf = tb.pf[j * nt + t], pb = tb.pb[j * nt + t];
        pfb[tid] = make_float4(pf.x, pf.y, pb.x, pb.y);
    }
    for (int e = tid; e < D * T * T; e += 32 * NP) {   // centred f tile (reading R12), zeros outside
        const int c = e / (T * T), i = (e / T) % T, j = e % T;
        fs[(c * T + i) * TP + j] =
            (i < Ly && j < Lx) ? a.f[c * plane + (long long)(y0 + i) * W + x0 + j] - a.mu[c] : 0.f;
    }
    float *acc = sm + L::OFF_ACC + p * T * T + lane;   // MODE 2: this thread's column of pair p
    if (MODE == 2)
        for (int m = 0; m < T; ++m) acc[m * T] = 0.f;

    float4 *zq = reinterpret_cast<float4 *>(sm + L::OFF_ZQ);   // (Re z_0^m, Re z_1^m, Im z_0^m, Im z_1^m)
    if (MODE == 0 && tid < T) zq[tid] = a.zpq[tid];
    float *ones = sm + L::OFF_ONE;
    for (int e = tid; e < (MODE == 0 ? T * TP : T); e += 32 * NP) ones[e] = 1.f;
    // the multiplier plane of pair p (pair 0: ones) and the pair's real input at (row i, column j)
    const float *fpl = (p > 0) ? fs + (p - 1) * T * TP : ones;
    auto xin = [&](int i, int j) -> float2 {
        const float fv = fpl[i * TP + j];
        return __fmul2_rn(cs[i * TP + j], f2(fv, fv));
    };

    // entering states, software-pipelined: the raw loads of sample b + 1's row (column) states are
    // issued right after sample b's row (column) stage and turned into states at their use
    RawSt rraw, craw;
    St rl, rr, cl, cr;
    const bool rb_load = MODE == 2 && a.rbg != nullptr;   // pass 2 reads pass 1's row blur
    __syncthreads();   // pfb
    if (MODE >= 1 && !rb_load && s0 < s1 && lane < Ly) {
        load_raw(a.Eh, a.Bh, a.UVh, s0, p, tx, y0 + lane, NQ, a.ntx, a.nlh, rraw);
        if (kEager) make_states(rraw, pfb, rl, rr);
    }
    if (MODE == 2 && s0 < s1 && lane < Lx) {
        load_raw(a.Ev, a.Bv, a.UVv, s0, p, ty, x0 + lane, NQ, a.nty, W, craw);
        if (kEager) make_states(craw, pfb + 2, cl, cr);
    }
    // the frequencies of the next sample are loaded a sample ahead too
    float tn[D];
    if (s0 < s1) {
#pragma unroll
        for (int c = 0; c < D; ++c) tn[c] = __ldg(a.t + (long long)(a.k0 + s0) * D + c);
    }
    for (int b = s0; b < s1; ++b) {
        float tk[D];
#pragma unroll
        for (int c = 0; c < D; ++c) tk[c] = tn[c];
        if (b + 1 < s1) {
#pragma unroll
            for (int c = 0; c < D; ++c) tn[c] = __ldg(a.t + (long long)(a.k0 + b + 1) * D + c);
        }
        __syncthreads();   // the previous sample's stages are done with cs / rb (and fs is complete)
        for (int e = tid; e < T * T; e += 32 * NP) {
            const int i = e / T, j = e % T;
            float th = 0.f;
#pragma unroll
            for (int c = 0; c < D; ++c) th = fmaf(tk[c], fs[(c * T + i) * TP + j], th);
            float sn, cn;
            __sincosf(th, &sn, &cn);
            cs[i * TP + j] = f2(cn, sn);
        }
        __syncthreads();

        // ---- row stage: lane = row ----
        const bool full = Lx == T && Ly == T;
        if (lane < Ly) {
            const float2 *hrow = cs + lane * TP;
            const float *frow = (p > 0 || MODE == 0) ? fpl + lane * TP : ones;   // MODE >= 1: one ones row
            auto xat = [&](int m) -> float2 {   // the pair's real input at column m of this row
                const float fv = frow[m];
                return __fmul2_rn(hrow[m], f2(fv, fv));
            };
            const int y = y0 + lane;
            if (MODE == 0) {
                St e, bb;
                if (full) summaries_full(a.zpc, xat, e, bb);
                else summaries<false>(zp, Lx, xat, e, bb);
                put_state(a.Eh, e, b, p, tx, y, NQ, a.ntx, a.nlh);
                put_state(a.Bh, bb, b, p, tx, y, NQ, a.ntx, a.nlh);
            } else if (!rb_load) {
                if (!kEager) make_states(rraw, pfb, rl, rr);
                float *r0 = rb + (2 * p * T + lane) * TP, *r1 = rb + ((2 * p + 1) * T + lane) * TP;
                if (full) blur_segment<true>(a.row, T, xat, rl, rr, r0, r1);
                else blur_segment<false>(a.row, Lx, xat, rl, rr, r0, r1);
            }
        }
        if (MODE == 0) {
            if (a.vl != nullptr) virtual_lines<NP>(a, sm + L::OFF_ACC + p * 16 * TP, zp, zq, xin, b, p, tx, ty, lane,
                                                   Lx, Ly, full);
            continue;
        }
        if (rb_load && lane < Lx) {
            // pass 1's exact row blur of this tile (planes 2p, 2p+1): lane = column, coalesced rows
            const float *g0 = a.rbg + (((long long)b * NQ + 2 * p) * H + y0) * W + x0 + lane;
            const float *g1 = g0 + (long long)H * W;
            float *r0 = rb + 2 * p * T * TP + lane, *r1 = rb + (2 * p + 1) * T * TP + lane;
#pragma unroll 8
            for (int m = 0; m < Ly; ++m) {
                r0[m * TP] = __ldg(g0 + (long long)m * W);
                r1[m * TP] = __ldg(g1 + (long long)m * W);
            }
        }
        if (!rb_load && b + 1 < s1 && lane < Ly) {
            load_raw(a.Eh, a.Bh, a.UVh, b + 1, p, tx, y0 + lane, NQ, a.ntx, a.nlh, rraw);
            if (kEager) make_states(rraw, pfb, rl, rr);
        }
        // the column stage of pair p reads only rb planes 2p, 2p+1 (written by this warp) and cs
        // (complete since the barrier after the modulation): a warp barrier suffices
        __syncwarp();

        // ---- column stage: lane = column ----
        if (lane < Lx) {
            const int x = x0 + lane;
            const float *c0 = rb + 2 * p * T * TP + lane, *c1 = rb + (2 * p + 1) * T * TP + lane;
            if (MODE == 1) {
                if (a.rbg) {   // keep the exact row blur for pass 2 (lane = column: coalesced rows)
                    float *g0 = a.rbg + (((long long)b * NQ + 2 * p) * H + y0) * W + x;
                    float *g1 = g0 + (long long)H * W;
#pragma unroll 8
                    for (int m = 0; m < Ly; ++m) {
                        g0[(long long)m * W] = c0[m * TP];
                        g1[(long long)m * W] = c1[m * TP];
                    }
                }
                auto xat = [&](int m) -> float2 { return f2(c0[m * TP], c1[m * TP]); };
                St e, bb;
                if (full) summaries_full(a.zpc, xat, e, bb);
                else summaries<false>(zp + T, Ly, xat, e, bb);
                put_state(a.Ev, e, b, p, ty, x, NQ, a.nty, W);
                put_state(a.Bv, bb, b, p, ty, x, NQ, a.nty, W);
            } else {
                if (!kEager) make_states(craw, pfb + 2, cl, cr);
                if (full) blur_accumulate<true>(a.col, T, c0, c1, cs + lane, cl, cr, acc);
                else blur_accumulate<false>(a.col, Ly, c0, c1, cs + lane, cl, cr, acc);
                if (MODE == 2 && b + 1 < s1) {
                    load_raw(a.Ev, a.Bv, a.UVv, b + 1, p, ty, x0 + lane, NQ, a.nty, W, craw);
                    if (kEager) make_states(craw, pfb + 2, cl, cr);
                }
            }
        }
    }
    if (MODE == 2 && lane < Lx) {
        const int pl = (p == 0) ? D : p - 1;
        float *dst = a.pz + ((long long)g * (D + 1) + pl) * plane + (long long)y0 * W + x0 + lane;
        for (int m = 0; m < Ly; ++m) dst[(long long)m * W] = a.first ? acc[m * T] : dst[(long long)m * W] + acc[m * T];
    }
}

// One chain per (sample, plane, pole, line), two threads per chain: threads [0, 128) of a block run
// the zero-started causal scan over the line's tiles, threads [128, 256) the anticausal one, for
// the same 128 chains (each replaces the summaries in place by the states entering each tile);
// then the line's exact reflected-periodic states (u_{-1}, v_n) from both scans' final values.
// Loads are issued kScanB tiles at a time (independent of the running state), double-buffered: the
// next batch is requested before the current one is scanned and stored (round 2: 8.5 -> 5.3 ms for
// the two scans of 16 config-5 samples, 34 GB at ~6.4 TB/s, i.e. at the HBM bound; 96 registers
// instead of 128 + spills).
constexpr int kScanB = 16;
__global__ void __launch_bounds__(256) rect_scan_kernel(float2 *__restrict__ E, float2 *__restrict__ B,
                                                        float4 *__restrict__ UV, const RecTabs tb,
                                                        const RecAxis ax, int nt, int nlines, long long nchains) {
    __shared__ float2 fin[2][128];
    const int dir = threadIdx.x >> 7;
    const long long id = (long long)blockIdx.x * 128 + (threadIdx.x & 127);
    const bool live = id < nchains;
    const int line = (int)(id % nlines);
    const long long sqj = id / nlines;   // (s * NQ + q) * 2 + j
    const int j = (int)(sqj & 1);
    const long long base = sqj * nt * nlines + line;
    const float2 *zl = tb.zl + j * nt;
    float2 *A = dir ? B : E;
    float2 c = f2(0.f, 0.f);
    if (live) {
        // double-buffered: batch i0 + kScanB is requested before batch i0 is scanned and stored,
        // so the loads overlap the dependent chain and the stores
        float2 v[2][kScanB];
        auto load = [&](int i0, float2 (&vb)[kScanB]) {
#pragma unroll
            for (int u = 0; u < kScanB; ++u) {
                const int t = dir ? nt - 1 - (i0 + u) : i0 + u;
                if (i0 + u < nt) vb[u] = A[base + (long long)t * nlines];
            }
        };
        auto scan = [&](int i0, const float2 (&vb)[kScanB]) {
#pragma unroll
            for (int u = 0; u < kScanB; ++u) {
                const int t = dir ? nt - 1 - (i0 + u) : i0 + u;
                if (i0 + u < nt) {
                    A[base + (long long)t * nlines] = c;
                    c = cadd(cmul(zl[t], c), vb[u]);
                }
            }
        };
        load(0, v[0]);
        for (int i0 = 0; i0 < nt; i0 += 2 * kScanB) {
            if (i0 + kScanB < nt) load(i0 + kScanB, v[1]);
            scan(i0, v[0]);
            if (i0 + kScanB >= nt) break;
            if (i0 + 2 * kScanB < nt) load(i0 + 2 * kScanB, v[0]);
            scan(i0 + kScanB, v[1]);
        }
    }
    fin[dir][threadIdx.x & 127] = c;   // dir 0: S_tail, dir 1: S_head
    __syncthreads();
    if (dir || !live) return;
    const float2 s_tail = c, s_head = fin[1][threadIdx.x];
    const float2 zn = j ? f2(ax.znr[1], ax.zni[1]) : f2(ax.znr[0], ax.zni[0]);   // no dynamic param indexing
    const float2 inv = j ? f2(ax.invr[1], ax.invi[1]) : f2(ax.invr[0], ax.invi[0]);
    const float2 um1 = cmul(cadd(s_head, cmul(zn, s_tail)), inv);
    const float2 vn = cadd(s_tail, cmul(zn, um1));
    UV[sqj * nlines + line] = make_float4(um1.x, um1.y, vn.x, vn.y);
}

// rec_impl 2: the column scan with the virtual lines' row blur folded in. Each warp owns the 32
// columns of one tile column tx for one (sample, plane, column pole k) and one direction (kind e:
// causal scan, kind b: anticausal). Per batch of kVS tile rows: (1) the warp stages the segments of
// the two virtual lines it needs (real and imaginary part of the kind's column summaries) through
// shared memory, coalesced; (2) lane (u, part) row-blurs one segment exactly from the virtual line's
// entering states (row scan), both row poles in one float2 -- by linearity the value is the column
// summary of the row-blurred plane; (3) lane = column, the scan over the batch as in rect_scan_kernel.
// The column summaries never go through HBM (a separate virtual-line kernel writing them for the
// column scan to read and rewrite, round 2's first version, moved 16 B per pixel-sample more:
// 4.4 + 2.7 ms vs 6.6 ms per 16 config-5 samples).
constexpr int kVS = 16;
struct St1 {   // one real line, both poles: (pole 0, pole 1)
    float2 ur, ui;
};

// exact blur of one real line over a segment of n elements from its entering states (l = u[x0-1],
// r = v[x0+n]): y[m] = sum_j Re[A_j (u_j[m] + v_j[m])] - g0 x[m]; full segments interleave the two
// directions as blur_segment does
template <bool FULL>
__device__ __forceinline__ void blur_line(const RecAxis &ax, int n, const float *x, const St1 &l, const St1 &r,
                                          float *y) {
    const float2 zr = f2(ax.zr[0], ax.zr[1]), nzi = f2(-ax.zi[0], -ax.zi[1]), zi = f2(ax.zi[0], ax.zi[1]);
    const float2 ar = f2(ax.ar[0], ax.ar[1]), nai = f2(-ax.ai[0], -ax.ai[1]);
    const float g0 = ax.g0;
    auto step = [&](St1 &st, float xv) {
        const float2 ur = st.ur;
        st.ur = __ffma2_rn(zr, ur, __ffma2_rn(nzi, st.ui, f2(xv, xv)));
        st.ui = __ffma2_rn(zr, st.ui, __fmul2_rn(zi, ur));
    };
    auto out = [&](const St1 &st) {
        const float2 t = __ffma2_rn(ar, st.ur, __fmul2_rn(nai, st.ui));
        return t.x + t.y;
    };
    St1 sf = l, sb = r;
    if constexpr (FULL) {
#pragma unroll 4
        for (int i = 0; i < T / 2; ++i) {
            const int mb = T - 1 - i;
            const float xf = x[i], xb = x[mb];
            step(sf, xf);
            step(sb, xb);
            y[i] = fmaf(-g0, xf, out(sf));
            y[mb] = out(sb);
        }
#pragma unroll 4
        for (int i = T / 2; i < T; ++i) {
            const int mb = T - 1 - i;
            const float xf = x[i], xb = x[mb];
            step(sf, xf);
            step(sb, xb);
            y[i] += fmaf(-g0, xf, out(sf));
            y[mb] += out(sb);
        }
    } else {
        for (int m = 0; m < n; ++m) {
            step(sf, x[m]);
            y[m] = fmaf(-g0, x[m], out(sf));
        }
        for (int m = n - 1; m >= 0; --m) {
            step(sb, x[m]);
            y[m] += out(sb);
        }
    }
}

// the same for a full segment with the two directions packed in one float2 (causal at m = i,
// anticausal at m = T-1-i): St's pair of values is (forward, backward), so step / re_a serve as in
// blur_segment and no horizontal add is needed
__device__ __forceinline__ void blur_line_full(const RecAxis &ax, const float *x, const St1 &l, const St1 &r,
                                               float *y) {
    St st;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        st.ur[j] = f2(j ? l.ur.y : l.ur.x, j ? r.ur.y : r.ur.x);
        st.ui[j] = f2(j ? l.ui.y : l.ui.x, j ? r.ui.y : r.ui.x);
    }
    const float g0 = ax.g0;
#pragma unroll 4
    for (int i = 0; i < T / 2; ++i) {
        const int mb = T - 1 - i;
        const float2 xv = f2(x[i], x[mb]);
        step(ax, st, xv);
        const float2 yv = re_a(ax, st);
        y[i] = fmaf(-g0, xv.x, yv.x);
        y[mb] = yv.y;
    }
#pragma unroll 4
    for (int i = T / 2; i < T; ++i) {
        const int mb = T - 1 - i;
        const float2 xv = f2(x[i], x[mb]);
        step(ax, st, xv);
        const float2 yv = re_a(ax, st);
        y[i] += fmaf(-g0, xv.x, yv.x);
        y[mb] += yv.y;
    }
}

struct VScanSmem {
    static constexpr int WARPS = 8, ROWS = 2 * kVS;
    // per warp: two input buffers (the next batch streams in while the current one is processed), one output
    static constexpr size_t BYTES = sizeof(float) * 3 * WARPS * ROWS * TP + sizeof(float2) * 2 * 128;
};

// loads of one batch that do not depend on the scan: the virtual-line segments (cp.async into vbuf),
// this lane's line's entering-state inputs and its tile's column pole power
struct VBatch {
    float2 e[2], bb[2], z;
    float4 uv[2];
};

__global__ void __launch_bounds__(256, 2) rect_vscan_kernel(const __grid_constant__ RecTArgs a, int NQ,
                                                            long long nsqk) {
    extern __shared__ float smv[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int WB = VScanSmem::ROWS * TP;   // floats per buffer
    float *vbuf = smv + warp * 2 * WB;                                     // inputs [2][u][part][m]
    float *ob = smv + (2 * VScanSmem::WARPS + warp) * WB;                  // row-blurred [u][part][m]
    float2 *fin = reinterpret_cast<float2 *>(smv + 3 * VScanSmem::WARPS * WB);   // [2][128]
    const int dir = threadIdx.x >> 7;
    const int ntx = a.ntx, nty = a.nty, W = a.W;
    const long long id = (long long)blockIdx.x * 128 + (threadIdx.x & 127);
    const long long per = (long long)ntx * 32;
    const long long sqk = id / per;
    const int tx = (int)((id % per) >> 5);
    const int x0 = tx * T, x = x0 + lane;
    const bool wlive = sqk < nsqk;   // warp-uniform
    const bool live = wlive && x < W;
    const int Lx = min(T, W - x0);
    const int k = (int)(sqk & 1);
    const long long sq = sqk >> 1;
    const int q = (int)(sq % NQ), s = (int)(sq / NQ);
    // this lane's blur task in a batch: tile u_me of the batch, virtual line v_me (kind = dir)
    const int u_me = lane & 15, part = lane >> 4, v_me = (k * 2 + dir) * 2 + part;
    float4 pfb[2];   // row-axis tile powers of tx
    if (wlive) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float2 pf = a.th.pf[j * ntx + tx], pb = a.th.pb[j * ntx + tx];
            pfb[j] = make_float4(pf.x, pf.y, pb.x, pb.y);
        }
    }
    float2 *A = dir ? a.Bv : a.Ev;
    const long long base = sqk * nty * (long long)W + x;   // sidx(s, q, k, t, x) = base + t * W
    const float2 *zl = a.tv.zl + k * nty;
    auto tile_of = [&](int i0, int u) { return dir ? nty - 1 - (i0 + u) : i0 + u; };
    // issue the batch starting at tile i0: segments into buffer vb (one coalesced 128 B row per
    // (tile, part), all in flight at once, zero-filled past the image edge), the rest into registers
    auto issue = [&](int i0, float *vb, VBatch &nx) {
        const int nb = min(kVS, nty - i0);
        // segment (u, part) of the batch: src0 + u * ustride + part * W
        const float *src0 = a.vl + vlidx(s, q, tile_of(i0, 0), (k * 2 + dir) * 2, min(x, W - 1), NQ, nty, W);
        const int ustride = (dir ? -8 : 8) * W;   // within one (sample, plane): 32-bit offsets
        const unsigned dst0 = (unsigned)__cvta_generic_to_shared(vb + lane);
        const int bytes = lane < Lx ? 4 : 0;
        const float *sp = src0;
#pragma unroll
        for (int u = 0; u < kVS; ++u) {
            if (u < nb) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst0 + 8u * u * TP), "l"(sp),
                             "r"(bytes)
                             : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst0 + 4u * (2 * u + 1) * TP),
                             "l"(sp + W), "r"(bytes)
                             : "memory");
            }
            sp += ustride;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (u_me < nb) {
            const int t = tile_of(i0, u_me);
            const int line = a.H + t * 8 + v_me;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                nx.e[j] = __ldg(a.Eh + sidx(s, q, j, tx, line, NQ, ntx, a.nlh));
                nx.bb[j] = __ldg(a.Bh + sidx(s, q, j, tx, line, NQ, ntx, a.nlh));
                nx.uv[j] = __ldg(a.UVh + uidx(s, q, j, line, NQ, a.nlh));
            }
            nx.z = zl[t];   // lane u holds tile u's z^{L_t}
        }
    };
    float2 c = f2(0.f, 0.f);
    VBatch cur, nxt;
    if (wlive) issue(0, vbuf, cur);
    for (int i0 = 0, ib = 0; i0 < nty && wlive; i0 += kVS, ib ^= 1) {
        const int nb = min(kVS, nty - i0);
        const float *vb = vbuf + ib * WB;
        if (i0 + kVS < nty) {
            issue(i0 + kVS, vbuf + (ib ^ 1) * WB, nxt);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        // (2) exact row blur of the segment from its entering states: lane (u_me, part)
        if (u_me < nb) {
            St1 l, r;
            float lr[2], li[2], rr_[2], ri[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const float2 lv = cadd(cur.e[j], cmul(f2(pfb[j].x, pfb[j].y), f2(cur.uv[j].x, cur.uv[j].y)));
                const float2 rv = cadd(cur.bb[j], cmul(f2(pfb[j].z, pfb[j].w), f2(cur.uv[j].z, cur.uv[j].w)));
                lr[j] = lv.x; li[j] = lv.y; rr_[j] = rv.x; ri[j] = rv.y;
            }
            l.ur = f2(lr[0], lr[1]); l.ui = f2(li[0], li[1]);
            r.ur = f2(rr_[0], rr_[1]); r.ui = f2(ri[0], ri[1]);
            const int row = u_me * 2 + part;
            if (Lx == T) blur_line_full(a.row, vb + row * TP, l, r, ob + row * TP);
            else blur_line<false>(a.row, Lx, vb + row * TP, l, r, ob + row * TP);
        }
        __syncwarp();
        // (3) the scan over the batch, lane = column: the state entering each tile, then past it
        float2 *dst = A + base + (long long)tile_of(i0, 0) * W;
        const long long tstride = dir ? -(long long)W : (long long)W;
#pragma unroll 4
        for (int u = 0; u < nb; ++u) {
            const float2 val = f2(ob[(2 * u) * TP + lane], ob[(2 * u + 1) * TP + lane]);
            const float2 zt = f2(__shfl_sync(0xffffffffu, cur.z.x, u), __shfl_sync(0xffffffffu, cur.z.y, u));
            if (live) dst[u * tstride] = c;
            c = cadd(cmul(zt, c), val);
        }
        __syncwarp();   // ob and this batch's input buffer are rewritten
        cur = nxt;
    }
    fin[dir * 128 + (threadIdx.x & 127)] = c;   // dir 0: S_tail, dir 1: S_head
    __syncthreads();
    if (dir || !live) return;
    const float2 s_tail = c, s_head = fin[128 + threadIdx.x];
    const RecAxis &ax = a.col;
    const float2 zn = k ? f2(ax.znr[1], ax.zni[1]) : f2(ax.znr[0], ax.zni[0]);
    const float2 inv = k ? f2(ax.invr[1], ax.invi[1]) : f2(ax.invr[0], ax.invi[0]);
    const float2 um1 = cmul(cadd(s_head, cmul(zn, s_tail)), inv);
    const float2 vn = cadd(s_tail, cmul(zn, um1));
    a.UVv[sqk * W + x] = make_float4(um1.x, um1.y, vn.x, vn.y);
}

cudaError_t launch_vscan(const RecTArgs &a, int NQ, cudaStream_t s) {
    static std::atomic<uint64_t> attr{0};
    cudaError_t e = ensure_smem_attr(rect_vscan_kernel, VScanSmem::BYTES, attr);
    if (e != cudaSuccess) return e;
    const long long nsqk = (long long)a.ns * NQ * 2;
    const long long n = nsqk * a.ntx * 32;
    rect_vscan_kernel<<<(unsigned)((n + 127) / 128), 256, VScanSmem::BYTES, s>>>(a, NQ, nsqk);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Tensor-core pass 2 (option rec_tc, d = 3, full tiles). The exact blur of a full segment from its
// entering states is linear in (x[0..31], L_0, L_1, R_0, R_1), so a tile's row blur is one product
//   Y[(q, y)][i] = sum_k A[(q, y)][k] B[i][k],  A = [x row | 8 state reals],  B = [K | state basis]
// (K[i][m] = h(|i - m|), plan.cu rec_tc_matrix), and the column blur the same with A = [Y column |
// column states]: per tile and sample M = 256 rows (8 planes x 32 lines, two M = 128 halves), N = 32,
// K = 40. A lives in tensor memory (written by the line's thread with tcgen05.st), B in shared
// memory; tf32 operands split into hi + lo halves, A_hi B_hi + A_hi B_lo + A_lo B_hi, give fp32
// accuracy. One thread issues the 30 MMAs of a blur and commits them to an mbarrier; the 8 warps
// (warp w: half w / 4, plane 4 (w / 4) + w % 4, lane = line; TMEM lane quarter w % 4) write A, read
// the result, transpose the row blur through shared memory for the column operand, and fold the
// column blur into Re[conj(H) blur] in registers (Alg. 1). Same output as pass 2.
// NP pairs -> NQ = 2 NP planes in NH = ceil(NQ / 4) M halves of 4 planes (the last one padded)
// pitch of pass 2's transpose rows: 36 floats, written as float4 (8 per row; each quarter-warp phase
// hits 8 distinct 4-bank groups) and read down a column (bank 4 m + lane: conflict-free); A/B
// BFVEC_TC_TR33: scalar stores at pitch 33
#ifdef BFVEC_TC_TR33
constexpr int TRP = T + 1;
#else
constexpr int TRP = T + 4;
#endif
// pitch of pass 2's f tile and (cos, sin) planes: 36, the row operand read as float4 (column reads
// stay conflict-free: bank 4 i + lane); A/B BFVEC_TC_ROW33: pitch 33, scalar row reads. Measured with
// the pitch-36 transposes: pass 2 14.51 -> 14.29 -> 14.23 ms per 16 config-5 samples (r2_84, r2_85)
#ifndef BFVEC_TC_ROW33
#define BFVEC_TC_ROWV4
#endif
#ifdef BFVEC_TC_ROWV4
constexpr int CP = T + 4;
#else
constexpr int CP = T + 1;
#endif
template <int NP>
struct TcSmem {
    static constexpr int D = NP - 1, NQ = 2 * NP, NH = (NQ + 3) / 4, WARPS = 4 * NH;
    static constexpr int OFF_FS = 0;                          // fs[D][T][CP]
    static constexpr int OFF_CS = D * T * CP;                 // cs[2 samples][2][T][CP]: cos plane, sin plane
    static constexpr int OFF_B = OFF_CS + 4 * T * CP;         // B: [hi; lo] canonical layout, 16 B aligned
    static constexpr int OFF_TR = OFF_B + kRecTcB;            // transposes [WARPS][T][TRP], 16 B aligned
    static constexpr int OFF_PFB = OFF_TR + WARPS * T * TRP;  // pfb[2 axes][2 poles] float4
    static constexpr int OFF_BAR = OFF_PFB + 16;              // mbarriers [NH], TMEM base
    static constexpr size_t BYTES = sizeof(float) * (OFF_BAR + 2 * NH + 2);
    static constexpr int COLS = NH <= 2 ? 256 : 512;          // tensor memory: 112 columns per half
};
constexpr int kTcCols = 256;   // two M halves (the column scan): D[2] (32 each), A_hi[2] / A_lo[2] (40 each) at 64 + 80 h (+ 40)

struct RawP {   // one plane's entering-state inputs: [pole j]
    float2 e[2], bb[2];
    float4 uv[2];
};
template <int NQ>
__device__ __forceinline__ void load_rawp(const float2 *E, const float2 *B, const float4 *UV, int b, int q, int t,
                                          int line, int nt, int nlines, RawP &r) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        r.e[j] = __ldg(E + sidx(b, q, j, t, line, NQ, nt, nlines));
        r.bb[j] = __ldg(B + sidx(b, q, j, t, line, NQ, nt, nlines));
        r.uv[j] = __ldg(UV + uidx(b, q, j, line, NQ, nlines));
    }
}
// x = hi + lo: hi = x rounded to tf32's 10 mantissa bits (half away from zero, two integer ops; the
// cvt.rna.tf32.f32 instruction is emulated by ~10 instructions on sm_100), lo = the exact fp32
// remainder, whose low 13 bits the tensor core ignores (error <= 2^-21 |x|)
__device__ __forceinline__ void tf32_split(float x, uint32_t &hi, uint32_t &lo) {
    const uint32_t h = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
    hi = h;
    lo = __float_as_uint(x - __uint_as_float(h));
}
__device__ __forceinline__ void tmem_st8(uint32_t t, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32f(uint32_t t, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(t)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// A row of the operand: 32 line values (val(i)) then the 8 entering-state reals, hi and lo halves
template <class V>
__device__ __forceinline__ void tc_write_operand(uint32_t tah, uint32_t tal, V val, const RawP &r,
                                                 const float4 *pfb) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) tf32_split(val(8 * c + j), hi[j], lo[j]);
        tmem_st8(tah + 8 * c, hi);
        tmem_st8(tal + 8 * c, lo);
    }
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const float4 pp = pfb[j];
        const float2 l = cadd(r.e[j], cmul(f2(pp.x, pp.y), f2(r.uv[j].x, r.uv[j].y)));
        const float2 rr = cadd(r.bb[j], cmul(f2(pp.z, pp.w), f2(r.uv[j].z, r.uv[j].w)));
        tf32_split(l.x, hi[2 * j], lo[2 * j]);
        tf32_split(l.y, hi[2 * j + 1], lo[2 * j + 1]);
        tf32_split(rr.x, hi[4 + 2 * j], lo[4 + 2 * j]);
        tf32_split(rr.y, hi[5 + 2 * j], lo[5 + 2 * j]);
    }
    tmem_st8(tah + 32, hi);
    tmem_st8(tal + 32, lo);
}
// the 15 MMAs of one M half of a blur (5 k-steps, 3 tf32 products), one thread; tensor memory of NH
// halves: D[h] at columns 32 h, A_hi[h] / A_lo[h] at 32 NH + 80 h (+ 40)
__device__ __forceinline__ void tc_blur_mmas(uint32_t tb, uint32_t bm, int h, int NH = 2) {
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    auto desc = [](uint32_t start) -> uint64_t {   // K-major, no swizzle: LBO 128 B (K), SBO 1280 B (N)
        return (uint64_t)((start >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(1280 >> 4) << 32) |
               (1ull << 46);
    };
    auto mma = [](uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
            "r"(a), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    };
    const uint32_t td = tb + 32 * h, tah = tb + 32 * NH + 80 * h, tal = tah + 40;
#pragma unroll
    for (int ks = 0; ks < 5; ++ks) {
        const uint64_t bh = desc(bm + ks * 256), bl = desc(bm + 4 * 1280 + ks * 256);
        mma(td, tah + 8 * ks, bh, ks > 0 ? 1u : 0u);
        mma(td, tah + 8 * ks, bl, 1u);
        mma(td, tal + 8 * ks, bh, 1u);
    }
}

// the MMA waits are short (a few hundred cycles): poll without a suspend hint (A/B: BFVEC_TC_SLEEP,
// measured equal)
__device__ __forceinline__ void tc_wait(uint64_t *bar, uint32_t parity) {
#if defined(BFVEC_TC_SLEEP) || defined(BFVEC_CHECKED)
    mbar_wait(bar, parity);   // checked build: with the watchdog
#else
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(saddr(bar)), "r"(parity)
            : "memory");
    } while (!done);
#endif
}

template <int NP>
__global__ void __launch_bounds__(128 * TcSmem<NP>::NH, TcSmem<NP>::NH <= 2 ? 2 : 1)
    rect_tc2_kernel(const __grid_constant__ RecTArgs a) {
    using L = TcSmem<NP>;
    constexpr int D = L::D, NQ = L::NQ, NH = L::NH, NT = 128 * NH;
    extern __shared__ __align__(128) float smt[];
    float *fs = smt + L::OFF_FS;
    float *csb = smt + L::OFF_CS;   // double-buffered: sample b in csb + (b & 1) * 2 T CP
    float *bmat = smt + L::OFF_B;
    float *tr = smt + L::OFF_TR;
    float4 *pfb = reinterpret_cast<float4 *>(smt + L::OFF_PFB);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smt + L::OFF_BAR);
    uint32_t *tbase_s = reinterpret_cast<uint32_t *>(smt + L::OFF_BAR + 2 * NH);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int half = warp >> 2, qw = warp & 3, q = 4 * half + qw, p = q >> 1, part = q & 1;
    const bool real_plane = q < NQ;   // padding planes of the last half: operands only, no output
    const int qq = real_plane ? q : NQ - 1, pp = qq >> 1;   // a valid plane for their (unused) loads
    const int ntxf = a.W / T, ntiles = ntxf * (a.H / T);
    const int H = a.H, W = a.W;
    const long long plane = (long long)H * W;
    const int G = a.g3, g = blockIdx.y;
    const int s0 = (int)((long long)a.ns * g / G), s1 = (int)((long long)a.ns * (g + 1) / G);

    // persistent CTA: the matrix, the barriers and the tensor memory are set up once for all its tiles
    for (int e = tid; e < kRecTcB; e += NT) bmat[e] = __ldg(a.tcb + e);
    if (tid == 0) {
        for (int h = 0; h < NH; ++h) mbar_init(bar + h, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(tbase_s)),
                     "n"(L::COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // B written by threads, read by the MMAs
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = *tbase_s;
    const uint32_t loff = (uint32_t)(qw * 32) << 16;
    const uint32_t td = tb + 32 * half + loff, tah = tb + 32 * NH + 80 * half + loff, tal = tah + 40;
    const uint32_t bm = saddr(bmat);
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int tx = tile % ntxf, ty = tile / ntxf;
    const int x0 = tx * T, y0 = ty * T;
    __syncthreads();   // the previous tile is done with fs, cs, tr and pfb
    for (int e = tid; e < D * T * T; e += NT) {   // centred f tile (reading R12)
        const int c = e / (T * T), i = (e / T) % T, j = e % T;
        fs[(c * T + i) * CP + j] = a.f[c * plane + (long long)(y0 + i) * W + x0 + j] - a.mu[c];
    }
    if (tid < 4) {
        const int ax = tid >> 1, j = tid & 1;
        const RecTabs &tbl = ax ? a.tv : a.th;
        const int t = ax ? ty : tx, nt = ax ? a.nty : a.ntx;
        const float2 pf = tbl.pf[j * nt + t], pb = tbl.pb[j * nt + t];
        pfb[tid] = make_float4(pf.x, pf.y, pb.x, pb.y);
    }
    __syncthreads();

    float acc[T];
#pragma unroll
    for (int i = 0; i < T; ++i) acc[i] = 0.f;
    RawP rraw, craw;
    float tn[D];
    if (s0 < s1) {
        load_rawp<NQ>(a.Eh, a.Bh, a.UVh, s0, qq, tx, y0 + lane, a.ntx, a.nlh, rraw);
        load_rawp<NQ>(a.Ev, a.Bv, a.UVv, s0, qq, ty, x0 + lane, a.nty, W, craw);
#pragma unroll
        for (int c = 0; c < D; ++c) tn[c] = __ldg(a.t + (long long)(a.k0 + s0) * D + c);
    }
    // (cos, sin) of sample b's phases (Alg. 1) into buffer b & 1: the next sample's
    // modulation runs while this sample's column blur is on the tensor cores
    auto modulate = [&](int b, const float (&tk)[D]) {
        float *c = csb + (b & 1) * 2 * T * CP;
        for (int e = tid; e < T * T; e += NT) {
            const int i = e / T, j = e % T;
            float th = 0.f;
#pragma unroll
            for (int cc = 0; cc < D; ++cc) th = fmaf(tk[cc], fs[(cc * T + i) * CP + j], th);
            float sn, cn;
            __sincosf(th, &sn, &cn);
            c[i * CP + j] = cn;
            c[T * CP + i * CP + j] = sn;
        }
    };
    if (s0 < s1) {
        modulate(s0, tn);
        if (s0 + 1 < s1) {
#pragma unroll
            for (int c = 0; c < D; ++c) tn[c] = __ldg(a.t + (long long)(a.k0 + s0 + 1) * D + c);
        }
    }
    __syncthreads();
    for (int b = s0; b < s1; ++b) {
        const float *cs = csb + (b & 1) * 2 * T * CP;
        // row operand of line (q, y = lane): the pair's modulated plane (Alg. 1) + row states;
        // part (cos / sin) and pair 0 (no f factor) are warp-uniform: one instance each, no selects
        {
            const float *hrow = cs + part * T * CP + lane * CP;
            const float *frow = fs + ((pp > 0 ? pp - 1 : 0) * T + lane) * CP;
#ifdef BFVEC_TC_ROWV4
            // rows at pitch 36: float4 loads (each quarter-warp phase: 8 distinct 4-bank groups)
            float xr[T];
            const float4 *h4 = reinterpret_cast<const float4 *>(hrow), *f4 = reinterpret_cast<const float4 *>(frow);
#pragma unroll
            for (int u = 0; u < T / 4; ++u) {
                float4 h = h4[u];
                if (pp > 0) {
                    const float4 fv = f4[u];
                    h = make_float4(h.x * fv.x, h.y * fv.y, h.z * fv.z, h.w * fv.w);
                }
                xr[4 * u] = h.x; xr[4 * u + 1] = h.y; xr[4 * u + 2] = h.z; xr[4 * u + 3] = h.w;
            }
            tc_write_operand(tah, tal, [&](int m) -> float { return xr[m]; }, rraw, pfb);
#else
            if (pp > 0)
                tc_write_operand(tah, tal, [&](int m) -> float { return hrow[m] * frow[m]; }, rraw, pfb);
            else
                tc_write_operand(tah, tal, [&](int m) -> float { return hrow[m]; }, rraw, pfb);
#endif
        }
        if (b + 1 < s1) load_rawp<NQ>(a.Eh, a.Bh, a.UVh, b + 1, qq, tx, y0 + lane, a.ntx, a.nlh, rraw);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        named_sync<128>(1 + half);   // the two M halves run as independent pipelines
        if ((tid & 127) == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            tc_blur_mmas(tb, bm, half, NH);
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             saddr(bar + half))
                         : "memory");
        }
        tc_wait(bar + half, phase);
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // the row blur of line (q, y) -> transpose buffer; column operand of line (q, x = lane)
        {
            float y[T];
            tmem_ld32f(td, y);
            float *trw = tr + (warp * T + lane) * TRP;
#ifdef BFVEC_TC_TR33
#pragma unroll
            for (int i = 0; i < T; ++i) trw[i] = y[i];
#else
#pragma unroll
            for (int i = 0; i < T; i += 4) *reinterpret_cast<float4 *>(trw + i) = make_float4(y[i], y[i + 1], y[i + 2], y[i + 3]);
#endif
        }
        __syncwarp();
        {
            const float *tcol = tr + warp * T * TRP + lane;
            tc_write_operand(tah, tal, [&](int m) -> float { return tcol[m * TRP]; }, craw, pfb + 2);
        }
        if (b + 1 < s1) load_rawp<NQ>(a.Ev, a.Bv, a.UVv, b + 1, qq, ty, x0 + lane, a.nty, W, craw);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        named_sync<128>(1 + half);   // the two M halves run as independent pipelines
        if ((tid & 127) == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            tc_blur_mmas(tb, bm, half, NH);
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             saddr(bar + half))
                         : "memory");
        }
        if (b + 1 < s1) {   // overlaps the column MMAs
            modulate(b + 1, tn);
            if (b + 2 < s1) {
#pragma unroll
                for (int c = 0; c < D; ++c) tn[c] = __ldg(a.t + (long long)(a.k0 + b + 2) * D + c);
            }
        }
        tc_wait(bar + half, phase);
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // the column blur of line (q, x): Re[conj(H) blur] of this plane's part
        {
            float z[T];
            tmem_ld32f(td, z);
            const float *hcol = cs + part * T * CP + lane;
#pragma unroll
            for (int i = 0; i < T; ++i) acc[i] = fmaf(hcol[i * CP], z[i], acc[i]);
        }
        __syncthreads();   // sample b + 1's (cos, sin) complete; tr and buffer b & 1 free for reuse
    }
    // the pair's two planes (warps w, w + 1) summed into the output plane of pair p
    __syncthreads();
    if (part && real_plane) {
        float *o = tr + warp * T * TP + lane;
#pragma unroll
        for (int i = 0; i < T; ++i) o[i * TP] = acc[i];
    }
    __syncthreads();
    if (!part && real_plane) {
        const float *o = tr + (warp + 1) * T * TP + lane;
        const int pl = (p == 0) ? D : p - 1;
        float *dst = a.pz + ((long long)g * (D + 1) + pl) * plane + (long long)y0 * W + x0 + lane;
#pragma unroll
        for (int i = 0; i < T; ++i) {
            const float v = acc[i] + o[i * TP];
            dst[(long long)i * W] = a.first ? v : dst[(long long)i * W] + v;
        }
    }
    }   // tiles
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(L::COLS) : "memory");
}

template <int NP>
cudaError_t launch_tc2(const RecTArgs &a, cudaStream_t s) {
    using L = TcSmem<NP>;
    static std::atomic<uint64_t> attr{0};
    cudaError_t e = ensure_smem_attr(rect_tc2_kernel<NP>, L::BYTES, attr);
    if (e != cudaSuccess) return e;
    static int nsm = 0;
    if (nsm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    // persistent: as many CTAs as fit (tensor memory: two per SM up to two M halves, else one)
    const int ntiles = (a.W / T) * (a.H / T);
    const int ctas = std::min(ntiles, nsm * (L::NH <= 2 ? 2 : 1));
    rect_tc2_kernel<NP><<<dim3(ctas, a.g3), 128 * L::NH, L::BYTES, s>>>(a);
    return cudaGetLastError();
}

// rec_impl 2 + rec_tc: the column scan with the virtual lines' segment blurs on the tensor cores.
// Same work decomposition as rect_vscan_kernel (warp = 32 columns of one tile column, one (sample,
// plane, column pole) and direction; batches of kVS tile rows); the 32 segments a warp blurs per
// batch (lane (u, part)) are rows of the pass-2 product [x | entering states] x [K | state basis]
// (the row axis' B, rec_tc_matrix), the 4 warps of a direction form one M = 128 half: operands by
// tcgen05.st, 15 MMAs issued by one thread, the result read back with tcgen05.ld into the batch's
// (now consumed) input buffer, which the scan then reads. Full tile columns only (W % 32 == 0; the
// plan keeps rect_vscan_kernel otherwise). Every warp takes part in every MMA round (named barrier
// per direction), live or not.
struct VScanTcSmem {
    static constexpr int WARPS = 8, ROWS = 2 * kVS, WB = ROWS * TP;
    static constexpr int OFF_VB = 0;                              // [8 warps][2][ROWS][TP]
    static constexpr int OFF_B = OFF_VB + WARPS * 2 * WB;         // B [hi; lo], 16 B aligned
    static constexpr int OFF_FIN = OFF_B + kRecTcB;               // fin [2][128] float2
    static constexpr int OFF_BAR = OFF_FIN + 2 * 2 * 128;         // mbarriers [2], TMEM base
    static constexpr size_t BYTES = sizeof(float) * (OFF_BAR + 6);
};

__global__ void __launch_bounds__(256, 2) rect_vscan_tc_kernel(const __grid_constant__ RecTArgs a, int NQ,
                                                               long long nsqk) {
    extern __shared__ __align__(128) float smq[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int WB = VScanTcSmem::WB;
    float *vbuf = smq + VScanTcSmem::OFF_VB + warp * 2 * WB;
    const int dir = tid >> 7, qw = warp & 3;
    float *bmat = smq + VScanTcSmem::OFF_B;
    float2 *fin = reinterpret_cast<float2 *>(smq + VScanTcSmem::OFF_FIN);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smq + VScanTcSmem::OFF_BAR);
    uint32_t *tbase_s = reinterpret_cast<uint32_t *>(smq + VScanTcSmem::OFF_BAR + 4);
    const int ntx = a.ntx, nty = a.nty, W = a.W;
    const long long id = (long long)blockIdx.x * 128 + (tid & 127);
    const long long per = (long long)ntx * 32;
    const long long sqk = id / per;
    const int tx = (int)((id % per) >> 5);
    const int x0 = tx * T, x = x0 + lane;
    const bool wlive = sqk < nsqk;   // warp-uniform
    const bool live = wlive && x < W;
    const int Lx = min(T, W - x0);
    const int k = (int)(sqk & 1);
    const long long sq = sqk >> 1;
    const int q = (int)(sq % NQ), s = (int)(sq / NQ);
    const int u_me = lane & 15, part = lane >> 4, v_me = (k * 2 + dir) * 2 + part;

    for (int e = tid; e < kRecTcB; e += 256) bmat[e] = __ldg(a.tcb + e);
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(tbase_s)),
                     "n"(kTcCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = *tbase_s;
    const uint32_t loff = (uint32_t)(qw * 32) << 16;
    const uint32_t td = tb + 32 * dir + loff, tah = tb + 64 + 80 * dir + loff, tal = tah + 40;
    const uint32_t bm = saddr(bmat);

    float4 pfb[2];
    if (wlive) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float2 pf = a.th.pf[j * ntx + tx], pb = a.th.pb[j * ntx + tx];
            pfb[j] = make_float4(pf.x, pf.y, pb.x, pb.y);
        }
    }
    float2 *A = dir ? a.Bv : a.Ev;
    const long long base = sqk * nty * (long long)W + x;
    const float2 *zl = a.tv.zl + k * nty;
    auto tile_of = [&](int i0, int u) { return dir ? nty - 1 - (i0 + u) : i0 + u; };
    auto issue = [&](int i0, float *vb, VBatch &nx) {
        if (!wlive) {
            asm volatile("cp.async.commit_group;" ::: "memory");
            return;
        }
        const int nb = min(kVS, nty - i0);
        const float *src0 = a.vl + vlidx(s, q, tile_of(i0, 0), (k * 2 + dir) * 2, min(x, W - 1), NQ, nty, W);
        const int ustride = (dir ? -8 : 8) * W;
        const unsigned dst0 = (unsigned)__cvta_generic_to_shared(vb + lane);
        const int bytes = lane < Lx ? 4 : 0;
        const float *sp = src0;
#pragma unroll
        for (int u = 0; u < kVS; ++u) {
            if (u < nb) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst0 + 8u * u * TP), "l"(sp),
                             "r"(bytes)
                             : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst0 + 4u * (2 * u + 1) * TP),
                             "l"(sp + W), "r"(bytes)
                             : "memory");
            }
            sp += ustride;
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (u_me < nb) {
            const int t = tile_of(i0, u_me);
            const int line = a.H + t * 8 + v_me;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                nx.e[j] = __ldg(a.Eh + sidx(s, q, j, tx, line, NQ, ntx, a.nlh));
                nx.bb[j] = __ldg(a.Bh + sidx(s, q, j, tx, line, NQ, ntx, a.nlh));
                nx.uv[j] = __ldg(a.UVh + uidx(s, q, j, line, NQ, a.nlh));
            }
            nx.z = zl[t];
        } else {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                nx.e[j] = nx.bb[j] = f2(0.f, 0.f);
                nx.uv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            nx.z = f2(0.f, 0.f);
        }
    };
    float2 c = f2(0.f, 0.f);
    VBatch cur, nxt;
    issue(0, vbuf, cur);
    uint32_t phase = 0;
    for (int i0 = 0, ib = 0; i0 < nty; i0 += kVS, ib ^= 1) {
        const int nb = min(kVS, nty - i0);
        float *vb = vbuf + ib * WB;
        if (i0 + kVS < nty) {
            issue(i0 + kVS, vbuf + (ib ^ 1) * WB, nxt);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        const int row = u_me * 2 + part;
        // the operand: this lane's segment (32 values) and its entering states, tf32 hi / lo
        {
            RawP r;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                r.e[j] = cur.e[j];
                r.bb[j] = cur.bb[j];
                r.uv[j] = cur.uv[j];
            }
            const float *xr = vb + row * TP;
            tc_write_operand(tah, tal, [&](int m) -> float { return xr[m]; }, r, pfb);
        }
        const float *ob = vb;   // consumed: the blurred segments go back into it
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        named_sync<128>(1 + dir);
        if ((tid & 127) == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            tc_blur_mmas(tb, bm, dir);
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             saddr(bar + dir))
                         : "memory");
        }
        tc_wait(bar + dir, phase);
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        {
            float y[T];
            tmem_ld32f(td, y);
            float *yr = vb + row * TP;
#pragma unroll
            for (int i = 0; i < T; ++i) yr[i] = y[i];
        }
        __syncwarp();
        // the scan over the batch, lane = column
        float2 *dst = A + base + (long long)tile_of(i0, 0) * W;
        const long long tstride = dir ? -(long long)W : (long long)W;
#pragma unroll 4
        for (int u = 0; u < nb; ++u) {
            const float2 val = f2(ob[(2 * u) * TP + lane], ob[(2 * u + 1) * TP + lane]);
            const float2 zt = f2(__shfl_sync(0xffffffffu, cur.z.x, u), __shfl_sync(0xffffffffu, cur.z.y, u));
            if (live) dst[u * tstride] = c;
            c = cadd(cmul(zt, c), val);
        }
        __syncwarp();
        cur = nxt;
    }
    fin[dir * 128 + (tid & 127)] = c;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "n"(kTcCols) : "memory");
    if (dir || !live) return;
    const float2 s_tail = c, s_head = fin[128 + tid];
    const RecAxis &ax = a.col;
    const float2 zn = k ? f2(ax.znr[1], ax.zni[1]) : f2(ax.znr[0], ax.zni[0]);
    const float2 inv = k ? f2(ax.invr[1], ax.invi[1]) : f2(ax.invr[0], ax.invi[0]);
    const float2 um1 = cmul(cadd(s_head, cmul(zn, s_tail)), inv);
    const float2 vn = cadd(s_tail, cmul(zn, um1));
    a.UVv[sqk * W + x] = make_float4(um1.x, um1.y, vn.x, vn.y);
}

cudaError_t launch_vscan_tc(const RecTArgs &a, int NQ, cudaStream_t s) {
    static std::atomic<uint64_t> attr{0};
    cudaError_t e = ensure_smem_attr(rect_vscan_tc_kernel, VScanTcSmem::BYTES, attr);
    if (e != cudaSuccess) return e;
    const long long nsqk = (long long)a.ns * NQ * 2;
    const long long n = nsqk * a.ntx * 32;
    rect_vscan_tc_kernel<<<(unsigned)((n + 127) / 128), 256, VScanTcSmem::BYTES, s>>>(a, NQ, nsqk);
    return cudaGetLastError();
}

template <int NP, int MODE>
cudaError_t launch_tile(const RecTArgs &a, int groups, cudaStream_t s) {
    const size_t smem = TileSmem<NP, MODE>::BYTES;
    static std::atomic<uint64_t> attr{0};
    cudaError_t e = ensure_smem_attr(rect_tile_kernel<NP, MODE>, smem, attr);
    if (e != cudaSuccess) return e;
    rect_tile_kernel<NP, MODE><<<dim3(a.ntx * a.nty, groups), 32 * NP, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_scan(float2 *E, float2 *B, float4 *UV, const RecTabs &tb, const RecAxis &ax, int nt, int nlines,
                        long long nq, cudaStream_t s) {
    const long long n = nq * 2 * nlines;
    rect_scan_kernel<<<(unsigned)((n + 127) / 128), 256, 0, s>>>(E, B, UV, tb, ax, nt, nlines, n);
    return cudaGetLastError();
}

// stages (bit mask, DESIGN.md §11 "overlap"): kRecStageP0 = pass 0 (summaries), kRecStageScan = the
// scans (and pass 1 of rec_impl 1), kRecStageP2 = pass 2; all three in order by default
template <int NP>
cudaError_t launch_np(const RecTArgs &a, cudaStream_t s, int stages) {
    const long long nq = (long long)a.ns * 2 * NP;
    cudaError_t e = cudaSuccess;
    if (stages & kRecStageP0) e = launch_tile<NP, 0>(a, a.g1, s);
    if (e == cudaSuccess && (stages & kRecStageScan)) {
        e = launch_scan(a.Eh, a.Bh, a.UVh, a.th, a.row, a.ntx, a.nlh, nq, s);
        if (e == cudaSuccess && a.vl != nullptr) {   // rec_impl 2: virtual-line row blur inside the column scan
            e = a.vtc ? launch_vscan_tc(a, 2 * NP, s) : launch_vscan(a, 2 * NP, s);
        } else {
            if (e == cudaSuccess) e = launch_tile<NP, 1>(a, a.g1, s);
            if (e == cudaSuccess) e = launch_scan(a.Ev, a.Bv, a.UVv, a.tv, a.col, a.nty, a.W, nq, s);
        }
    }
    if (e != cudaSuccess || !(stages & kRecStageP2)) return e;
    if constexpr (NP <= 8) {
        if (a.tc) {   // full tiles on the tensor cores, the rest (if any) on the FP32 path
            if (a.W % T || a.H % T) e = launch_tile<NP, 2>(a, a.g3, s);
            if (e == cudaSuccess && a.W >= T && a.H >= T) e = launch_tc2<NP>(a, s);
            return e;
        }
    }
    return launch_tile<NP, 2>(a, a.g3, s);
}

}  // namespace

cudaError_t launch_recursive_tiled(const RecTArgs &a, cudaStream_t s, int stages) {
    switch (a.d) {
        case 1: return launch_np<2>(a, s, stages);
        case 2: return launch_np<3>(a, s, stages);
        case 3: return launch_np<4>(a, s, stages);
        case 4: return launch_np<5>(a, s, stages);
        case 5: return launch_np<6>(a, s, stages);
        case 6: return launch_np<7>(a, s, stages);
        case 7: return launch_np<8>(a, s, stages);
        case 8: return launch_np<9>(a, s, stages);
    }
    return cudaErrorInvalidValue;
}

}  // namespace bfvec
