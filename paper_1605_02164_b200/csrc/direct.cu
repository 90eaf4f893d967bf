// direct.cu -- the exact bilateral filter, Eq. (2)-(3), on the
// square window [-r, r]^2 with half-sample reflection (reading R1).
// Accuracy reference for the MC path (PSNR, Fig. 5's ground truth), not the MC hot path.
//
// phi(f_j - f_i) = exp(-(f_j - f_i)^T C^-1 (f_j - f_i) / 2) = exp2(-|u_j - u_i|^2)
// with u = sqrt(log2(e)/2) diag(alpha) Q^T f (Eq. (4)); the spatial weight
// w(jx) w(jy) enters the exponent as lw = log2 w(jx) + log2 w(jy), so a pair costs
// d FSUB + d FFMA + one MUFU.EX2 + (d+1) FFMA/FADD = 4d + 1 FP32 ops + 1 MUFU.
//
// Layout: one prep kernel writes U = A f and f itself, reflect-padded
// (r rows / r columns on each side, rows padded to the tile grid), as 2d planes of
// (Hp, Wpp) fp32 -- the hot loop has no index arithmetic beyond a ring-slot offset.
// direct_tiled_kernel: CTA = TXW x TY outputs (TXW = 16 BX, TY = 16; 256 threads, thread =
// BX consecutive outputs of one row). It walks the window's rows jy = -r..r; at step jy the
// CTA needs padded source rows y0 + jy .. y0 + jy + TY - 1, held in a ring of TY + 1 shared-
// memory rows (2d planes each): one new row per step, prefetched with cp.async while the
// step computes. Along the row each thread slides a 2 BX-pixel register window in chunks of
// BX offsets: per chunk ONE vector load per plane serves BX x BX pairs (offset weight
// uniform across the thread's outputs).
#include <cuda_runtime.h>

#include <atomic>

#include "internal.h"
#include "kernel_common.cuh"

namespace bfvec {
namespace {

__device__ __forceinline__ int reflect_idx(long long i, int n) {
    if ((unsigned long long)i < (unsigned long long)n) return (int)i;
    const long long p = 2LL * n;
    i %= p;
    if (i < 0) i += p;
    return (int)(i < n ? i : p - 1 - i);
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

struct RotArgs {
    float A[kMaxD * kMaxD];
    float mu[kMaxD];
};

// UF planes 0..d-1: U = A f, planes d..2d-1: f, at padded (py, px) = reflect(py - r, px - r)
__global__ void direct_prep_kernel(const float *__restrict__ f, int d, int H, int W, int r, int Hp, int Wpp,
                                   const __grid_constant__ RotArgs ra, float *__restrict__ UF) {
    // f is centred by the mid-range mu (reading R12: S[f - mu] + mu = S[f]), halving the
    // magnitude of the weighted sums and of u
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long plane = (long long)Hp * Wpp;
    if (e >= plane) return;
    const int py = (int)(e / Wpp), px = (int)(e - (long long)py * Wpp);
    const int y = reflect_idx((long long)py - r, H), x = reflect_idx((long long)px - r, W);
    const long long npix = (long long)H * W, o = (long long)y * W + x;
    float fv[kMaxD];
    for (int c = 0; c < d; ++c) fv[c] = f[(long long)c * npix + o] - ra.mu[c];
    for (int k = 0; k < d; ++k) {
        float u = 0.f;
        for (int c = 0; c < d; ++c) u = fmaf(ra.A[k * d + c], fv[c], u);
        UF[(long long)k * plane + e] = u;
        UF[(long long)(d + k) * plane + e] = fv[k];
    }
}

constexpr int kDirTYMax = 16;              // output rows per CTA (one per thread row): 4, 8 or 16
constexpr int kDirLw = 2 * kMaxR + 1 + 16; // log2 spatial taps, padded to whole chunks

struct DirectTArgs {
    float lw[kDirLw];     // lw[j + r] = log2 w(|j|) for |j| <= r, -inf beyond (zero weight)
    float mu[kMaxD];      // the centring the output adds back
};

template <int BX>
struct VecT;
template <>
struct VecT<4> {
    using T = float4;
    __device__ static void get(const float *p, float (&v)[4]) {
        const float4 q = *reinterpret_cast<const float4 *>(p);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    }
};
template <>
struct VecT<2> {
    using T = float2;
    __device__ static void get(const float *p, float (&v)[2]) {
        const float2 q = *reinterpret_cast<const float2 *>(p);
        v[0] = q.x; v[1] = q.y;
    }
};

// Shared memory per CTA: ring of NS = TY + 1 rows x 2D planes x SW floats, then the taps.
template <int D, int BX, int TY>
__device__ __forceinline__ void direct_tiled_body(const float *__restrict__ UF, int H, int W, int r, int Hp,
                                                  int Wpp, int SW, int nch, const DirectTArgs &da,
                                                  float *__restrict__ out) {
    constexpr int NP = 2 * D, NS = TY + 1, TXW = 16 * BX, kDirThreads = 16 * TY;
    extern __shared__ __align__(16) float dsm[];
    float *ring = dsm;
    float *s_lw = ring + (size_t)NS * NP * SW;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int x0 = blockIdx.x * TXW, y0 = blockIdx.y * TY;
    const long long plane = (long long)Hp * Wpp;
    const int nvec = SW >> 2;   // 16-byte chunks per plane row

    // padded row y0 + k of every plane -> ring slot `slot`
    auto load_row = [&](int k, int slot) {
        const float *g = UF + (long long)(y0 + k) * Wpp + x0;
        float *s = ring + (size_t)slot * NP * SW;
        for (int i = tid; i < NP * nvec; i += kDirThreads) {
            const int p = i / nvec, v = i - p * nvec;
            cp_async16(s + p * SW + 4 * v, g + p * plane + 4 * v);
        }
        cp_async_commit();
    };
    for (int i = tid; i <= nch * BX; i += kDirThreads) s_lw[i] = i ? da.lw[i - 1] : -INFINITY;
    for (int k = 0; k < TY; ++k) load_row(k, k);

    // this thread's outputs: row y0 + ty, columns x0 + BX tx + b; centre values u_i
    const int y = y0 + ty, xb = x0 + BX * tx;
    float ui[D][BX];
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
        for (int b = 0; b < BX; ++b) ui[c][b] = UF[c * plane + (long long)(y + r) * Wpp + xb + b + r];
    float den[BX], num[D][BX];
#pragma unroll
    for (int b = 0; b < BX; ++b) {
        den[b] = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) num[c][b] = 0.f;
    }
    cp_async_wait_all();
    __syncthreads();

    // Two-level summation: each window row jy accumulates into (rden, rnum), added to the totals
    // once per row -- a single fp32 running sum over (2r+1)^2 terms loses ~(2r+1)^2 eps of the
    // sum (measured 1.3e-3 on config 3), two levels ~2 (2r+1) eps (7e-5, with the centring).
    //
    // Packed pairs (FFMA2): output b (even) at offset index k and output b+1 at k-1 read the SAME
    // source pixel b + k, so the pair's differences, quadratic forms and weighted sums are one
    // FADD2 / FFMA2 each with the source broadcast; only the two ex2 are scalar. k runs over
    // 0..nch*BX-1 >= 2r+1; lw[-1] and lw[k > 2r] are -inf (zero weight), so each output still
    // sees exactly the offsets 0..2r.
    constexpr int BH = BX / 2;
    float2 rden[BH], rnum[D][BH], den2[BH], num2[D][BH], ui2[D][BH];
#pragma unroll
    for (int h = 0; h < BH; ++h) {
        den2[h] = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < D; ++c) {
            num2[c][h] = make_float2(0.f, 0.f);
            ui2[c][h] = make_float2(-ui[c][2 * h], -ui[c][2 * h + 1]);
        }
    }
    // the chunk of offset indices k = BX ch + t (t < BX): pair h reads window pixel 2h + t of
    // (lo | hi) = smem columns BX (tx + ch) .. BX (tx + ch + 2) - 1
    auto chunk = [&](const float (&lo)[NP][BX], const float (&hi)[NP][BX], float lwy, int ch) {
#pragma unroll
        for (int t = 0; t < BX; ++t) {
            // (lw[k] + lwy, lw[k-1] + lwy); s_lw is shifted by one so index k-1 = -1 exists
            const float2 lwt = __fadd2_rn(make_float2(s_lw[BX * ch + t + 1], s_lw[BX * ch + t]),
                                          make_float2(lwy, lwy));
#pragma unroll
            for (int h = 0; h < BH; ++h) {
                const int s = 2 * h + t;
                float2 q = lwt;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const float v = s < BX ? lo[c][s] : hi[c][s - BX];
                    const float2 du = __fadd2_rn(make_float2(v, v), ui2[c][h]);
                    q = __ffma2_rn(make_float2(-du.x, -du.y), du, q);
                }
                const float2 w = make_float2(ex2_approx(q.x), ex2_approx(q.y));
                rden[h] = __fadd2_rn(rden[h], w);
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const float v = s < BX ? lo[D + c][s] : hi[D + c][s - BX];
                    rnum[c][h] = __ffma2_rn(w, make_float2(v, v), rnum[c][h]);
                }
            }
        }
    };

    int slot = ty;               // ring slot of padded row y0 + ty + q
    for (int q = 0; q <= 2 * r; ++q) {
        if (q < 2 * r) load_row(q + TY, (q + TY) % NS);   // the slot step q - 1 released
        const float lwy = s_lw[q + 1];
        const float *srow = ring + (size_t)slot * NP * SW + BX * tx;
#pragma unroll
        for (int h = 0; h < BH; ++h) {
            rden[h] = make_float2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < D; ++c) rnum[c][h] = make_float2(0.f, 0.f);
        }
        float A[NP][BX], B[NP][BX];
#pragma unroll
        for (int p = 0; p < NP; ++p) VecT<BX>::get(srow + p * SW, A[p]);
        int ch = 0;
        for (; ch + 1 < nch; ch += 2) {   // ping-pong: no register copies between chunks
#pragma unroll
            for (int p = 0; p < NP; ++p) VecT<BX>::get(srow + p * SW + BX * (ch + 1), B[p]);
            chunk(A, B, lwy, ch);
#pragma unroll
            for (int p = 0; p < NP; ++p) VecT<BX>::get(srow + p * SW + BX * (ch + 2), A[p]);
            chunk(B, A, lwy, ch + 1);
        }
        if (ch < nch) {
#pragma unroll
            for (int p = 0; p < NP; ++p) VecT<BX>::get(srow + p * SW + BX * (ch + 1), B[p]);
            chunk(A, B, lwy, ch);
        }
#pragma unroll
        for (int h = 0; h < BH; ++h) {
            den2[h] = __fadd2_rn(den2[h], rden[h]);
#pragma unroll
            for (int c = 0; c < D; ++c) num2[c][h] = __fadd2_rn(num2[c][h], rnum[c][h]);
        }
        slot = slot + 1 == NS ? 0 : slot + 1;
        cp_async_wait_all();
        __syncthreads();
    }
#pragma unroll
    for (int h = 0; h < BH; ++h) {
        den[2 * h] = den2[h].x;
        den[2 * h + 1] = den2[h].y;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            num[c][2 * h] = num2[c][h].x;
            num[c][2 * h + 1] = num2[c][h].y;
        }
    }
    if (y >= H) return;
    const long long npix = (long long)H * W;
#pragma unroll
    for (int b = 0; b < BX; ++b) {
        if (xb + b >= W) break;
        const float rd = 1.0f / den[b];
#pragma unroll
        for (int c = 0; c < D; ++c) out[c * npix + (long long)y * W + xb + b] = fmaf(num[c][b], rd, da.mu[c]);
    }
}

// Two entry points over one body: the 256-thread d <= 4 instances are compiled for 3 CTAs per SM
// (80 registers, 72 B of spills outside the inner loop): +2.4 % on config 5 and +2.7 % on config 3
// against the compiler's own choice (102 registers, 2 CTAs per SM; profiles/r02_direct_minblocks.txt);
// the others keep the compiler's choice (an explicit minBlocks = 1 raised d = 3 to 134 registers
// and 1 CTA per SM, and slowed d = 8 by 14 %).
template <int D, int BX, int TY>
__global__ void __launch_bounds__(16 * TY) direct_tiled_kernel(const float *__restrict__ UF, int H, int W, int r,
                                                               int Hp, int Wpp, int SW, int nch,
                                                               const __grid_constant__ DirectTArgs da,
                                                               float *__restrict__ out) {
    direct_tiled_body<D, BX, TY>(UF, H, W, r, Hp, Wpp, SW, nch, da, out);
}
template <int D, int BX, int TY>
__global__ void __launch_bounds__(16 * TY, 3) direct_tiled_kernel_occ3(const float *__restrict__ UF, int H, int W,
                                                                       int r, int Hp, int Wpp, int SW, int nch,
                                                                       const __grid_constant__ DirectTArgs da,
                                                                       float *__restrict__ out) {
    direct_tiled_body<D, BX, TY>(UF, H, W, r, Hp, Wpp, SW, nch, da, out);
}

template <int D>
constexpr int dir_bx() { return D <= 4 ? 4 : 2; }

template <int D, int TY>
cudaError_t launch_direct_dt(const float *UF, int H, int W, int r, int Hp, int Wpp, int SW, int nch,
                             const DirectTArgs &da, float *out, cudaStream_t s) {
    constexpr int BX = dir_bx<D>();
    constexpr int NP = 2 * D, NS = TY + 1;
    const size_t smem = sizeof(float) * ((size_t)NS * NP * SW + kDirLw + 4);
    // the attribute is set once per device, so set it for the largest window (r = kMaxR)
    constexpr int nch_max = (2 * kMaxR + 2 + BX - 1) / BX;
    constexpr int SW_max = (16 * BX + BX * (nch_max + 2) + 3) / 4 * 4;
    constexpr size_t smem_max = sizeof(float) * ((size_t)NS * NP * SW_max + kDirLw + 4);
    static_assert(smem_max <= 227 * 1024, "direct ring exceeds shared memory");
    if (smem > smem_max) return cudaErrorInvalidValue;
    constexpr bool occ3 = TY == 16 && D <= 4;
    auto kern = occ3 ? direct_tiled_kernel_occ3<D, BX, TY> : direct_tiled_kernel<D, BX, TY>;
    static std::atomic<uint64_t> attr_done{0};
    cudaError_t e = ensure_smem_attr(kern, smem_max, attr_done);
    if (e != cudaSuccess) return e;
    dim3 grid((W + 16 * BX - 1) / (16 * BX), (H + TY - 1) / TY);
    kern<<<grid, 16 * TY, smem, s>>>(UF, H, W, r, Hp, Wpp, SW, nch, da, out);
    return cudaGetLastError();
}

template <int D>
cudaError_t launch_direct_d(int ty, const float *UF, int H, int W, int r, int Hp, int Wpp, int SW, int nch,
                            const DirectTArgs &da, float *out, cudaStream_t s) {
    switch (ty) {
        case 4: return launch_direct_dt<D, 4>(UF, H, W, r, Hp, Wpp, SW, nch, da, out, s);
        case 8: return launch_direct_dt<D, 8>(UF, H, W, r, Hp, Wpp, SW, nch, da, out, s);
        case 16: return launch_direct_dt<D, 16>(UF, H, W, r, Hp, Wpp, SW, nch, da, out, s);
    }
    return cudaErrorInvalidValue;
}

// geometry of the padded planes for (d, H, W, r): BX, chunks, smem row width, padded extents
struct DirectGeom {
    int bx, nch, SW, Hp, Wpp;
};
DirectGeom direct_geom(int d, int H, int W, int r) {
    DirectGeom g;
    g.bx = d <= 4 ? 4 : 2;
    const int TXW = 16 * g.bx;
    g.nch = (2 * r + 2 + g.bx - 1) / g.bx;   // offset indices k = 0..2r+1 (packed pairs: b at k, b+1 at k-1)
    g.SW = (TXW + g.bx * (g.nch + 2) + 3) / 4 * 4;   // the last chunk's window + the ping-pong overread
    const int ntx = (W + TXW - 1) / TXW, nty = (H + kDirTYMax - 1) / kDirTYMax;
    g.Hp = nty * kDirTYMax + 2 * r;   // whole 16-row tiles: covers every TY in {4, 8, 16}
    g.Wpp = ((ntx - 1) * TXW + g.SW + 3) / 4 * 4;
    return g;
}

}  // namespace

size_t direct_scratch_bytes(int d, int H, int W, int r) {
    const DirectGeom g = direct_geom(d, H, W, r);
    return sizeof(float) * (size_t)2 * d * g.Hp * g.Wpp;
}

cudaError_t launch_direct(const float *f, int d, int H, int W, int r, const float *w, const float *A,
                          const float *mu, float *UF, float *out, int rows_per_cta, cudaStream_t s) {
    if (r > kMaxR || d < 1 || d > kMaxD) return cudaErrorInvalidValue;
    const DirectGeom g = direct_geom(d, H, W, r);
    RotArgs ra{};
    for (int i = 0; i < d * d; ++i) ra.A[i] = A[i];
    for (int c = 0; c < d; ++c) ra.mu[c] = mu[c];
    const long long plane = (long long)g.Hp * g.Wpp;
    direct_prep_kernel<<<(unsigned)((plane + 255) / 256), 256, 0, s>>>(f, d, H, W, r, g.Hp, g.Wpp, ra, UF);
    DirectTArgs da{};
    for (int c = 0; c < d; ++c) da.mu[c] = mu[c];
    const int ty = rows_per_cta;   // 4, 8 or 16 (plan.cu picks it)
    for (int i = 0; i < kDirLw; ++i) {
        const int j = i - r;
        da.lw[i] = (j <= r && w[j < 0 ? -j : j] > 0.f) ? log2f(w[j < 0 ? -j : j]) : -INFINITY;
    }
    switch (d) {
#define BFV_D(DD) \
    case DD: return launch_direct_d<DD>(ty, UF, H, W, r, g.Hp, g.Wpp, g.SW, g.nch, da, out, s);
        BFV_D(1) BFV_D(2) BFV_D(3) BFV_D(4) BFV_D(5) BFV_D(6) BFV_D(7) BFV_D(8)
#undef BFV_D
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace bfvec
