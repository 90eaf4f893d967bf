// mcsf_fused.cu -- the fused Monte Carlo shiftable-filter kernel for sm_100a.
//
// One CTA owns a strip of TX = 32 output columns x tile_rows output rows and a
// group of samples. For every sample k (Alg. 1) it streams
// the strip top to bottom in chunks of KB output rows:
//
//   modulate  (Alg. 1, Eq. (16))
//       theta = t_k . (f - mu) (d FFMA), (c, s) = sincos(theta) on the SFU,
//       channels (c, s, c f'_q, s f'_q) for the haloed row segment
//       [x0 - R, x0 + TX + R) -> shared memory `mod`;
//   horizontal pass (Alg. 1, "bulk of the computation")
//       (2R+1)-tap FIR along x, taps as constant-bank FFMA operands,
//       -> shared memory row buffer `hb` holding KB + 2R rows;
//   vertical pass + accumulate (Alg. 1, Eq. (18)-(19))
//       (2R+1)-tap FIR along y over `hb`, then
//       Z += c * blur(c) + s * blur(s),  P'_q += c * blur(c f'_q) + s * blur(s f'_q)
//       (= Re[conj(H) blur], reading R4), read-modify-write of the CTA's
//       L2-resident partial tile in global memory.
//
// The complex images H_k, G_k never touch HBM. Separability is exact for the
// square window because omega(j) = w(j_y) w(j_x).
// Boundary: half-sample reflection (reading R1), applied at load time.
#include <cuda_runtime.h>

#include "internal.h"

namespace bfvec {
namespace {

__device__ __forceinline__ int reflect_idx(int i, int n) {
    if ((unsigned)i < (unsigned)n) return i;
    int p = 2 * n;
    i %= p;
    if (i < 0) i += p;
    return i < n ? i : p - 1 - i;
}

constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }
// row stride of the modulated buffer: >= round_up(WIN, 4) and == 4 (mod 32) so that
// the H-pass LDS.128 of 8 lanes (4 column groups x 2 rows) hit 32 distinct banks.
constexpr int mod_stride(int win) {
    int s = round_up(win, 4);
    while (s % 32 != 4) s += 4;
    return s;
}

template <int D_, int R_, int NT_, int KB_, int SH_>
struct Cfg {
    static constexpr int D = D_;
    static constexpr int R = R_;
    static constexpr int NT = NT_;
    static constexpr int KB = KB_;       // output rows per chunk (multiple of 8)
    static constexpr int SH = SH_;       // rows per modulate / H-pass sub-step
    static constexpr int TX = kTX;
    static constexpr int NCH = 2 * (D + 1);
    static constexpr int WIN = TX + 2 * R;
    static constexpr int MSTRIDE = mod_stride(WIN);
    static constexpr int HROWS = KB + 2 * R;
    static constexpr int MOD_FLOATS = NCH * SH * MSTRIDE;
    static constexpr int HB_FLOATS = NCH * HROWS * TX;
    static constexpr int CS_FLOATS = 2 * KB * TX;
    static constexpr size_t SMEM = sizeof(float) * (MOD_FLOATS + HB_FLOATS + CS_FLOATS);
    static_assert(KB % 8 == 0, "KB must be a multiple of 8");
};

template <class C>
__device__ __forceinline__ float phase(const float (&tk)[C::D], const float (&fv)[C::D]) {
    float th = 0.f;
#pragma unroll
    for (int c = 0; c < C::D; ++c) th = fmaf(tk[c], fv[c], th);
    return th;
}

template <class C>
__device__ __forceinline__ void load_pixel(const FusedArgs &a, int yi, int xi, float (&fv)[C::D]) {
    const int yr = min(max(reflect_idx(yi, a.H) - a.slab_row0, 0), a.slab_rows - 1);
    const int xr = reflect_idx(xi, a.W);
    const float *p = a.f + (long long)yr * a.W + xr;
#pragma unroll
    for (int c = 0; c < C::D; ++c) fv[c] = (c < a.d) ? __ldg(p + c * a.plane) - a.mu[c] : 0.f;
}

// modulate rows [img_row0, img_row0 + nrows) of the haloed segment into `mod`
template <class C>
__device__ __forceinline__ void modulate(const FusedArgs &a, float *mod, const float (&tk)[C::D],
                                         int img_row0, int nrows, int x0) {
    for (int it = threadIdx.x; it < C::SH * C::WIN; it += C::NT) {
        const int row = it / C::WIN;
        const int j = it - row * C::WIN;
        if (row >= nrows) continue;
        float fv[C::D];
        load_pixel<C>(a, img_row0 + row, x0 - C::R + j, fv);
        float s, c;
        __sincosf(phase<C>(tk, fv), &s, &c);
        float *m = mod + row * C::MSTRIDE + j;
        constexpr int CH = C::SH * C::MSTRIDE;
        m[0] = c;
        m[CH] = s;
#pragma unroll
        for (int q = 0; q < C::D; ++q) {
            m[(2 + 2 * q) * CH] = c * fv[q];
            m[(3 + 2 * q) * CH] = s * fv[q];
        }
    }
}

// horizontal (2R+1)-tap pass: item = (channel, row, 8-column group)
template <class C>
__device__ __forceinline__ void hpass(const FusedArgs &a, const float *mod, float *hb,
                                      int hb_row0, int nrows) {
    constexpr int ITEMS = C::NCH * C::SH * (C::TX / 8);
    constexpr int NIN = 8 + 2 * C::R;
    constexpr int NV = (NIN + 3) / 4;
    for (int it = threadIdx.x; it < ITEMS; it += C::NT) {
        const int cg = it & 3;
        const int row = (it >> 2) % C::SH;
        const int ch = (it >> 2) / C::SH;
        if (row >= nrows) continue;
        const float *in = mod + (ch * C::SH + row) * C::MSTRIDE + cg * 8;
        float acc[8];
#pragma unroll
        for (int o = 0; o < 8; ++o) acc[o] = 0.f;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const float4 x4 = *reinterpret_cast<const float4 *>(in + 4 * v);
            const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = 4 * v + e;
                if (j < NIN) {
#pragma unroll
                    for (int o = 0; o < 8; ++o) {
                        const int m = j - o - C::R;          // tap offset, compile-time
                        if (m >= -C::R && m <= C::R) acc[o] = fmaf(a.w[m < 0 ? -m : m], xv[e], acc[o]);
                    }
                }
            }
        }
        float *dst = hb + (ch * C::HROWS + hb_row0 + row) * C::TX + cg * 8;
        *reinterpret_cast<float4 *>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        *reinterpret_cast<float4 *>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
}

template <class C>
__global__ void __launch_bounds__(C::NT) mcsf_fused_kernel(const __grid_constant__ FusedArgs a) {
    extern __shared__ __align__(16) float smem[];
    float *mod = smem;
    float *hb = mod + C::MOD_FLOATS;
    float *cs = hb + C::HB_FLOATS;

    const int x0 = blockIdx.x * C::TX;
    const int ty0 = a.out_row0 + blockIdx.y * a.tile_rows;
    const int ty1 = min(ty0 + a.tile_rows, a.out_row0 + a.out_rows);
    const int g = blockIdx.z;
    const int ns = a.k1 - a.k0;
    const int gk0 = a.k0 + (int)((long long)ns * g / a.groups);
    const int gk1 = a.k0 + (int)((long long)ns * (g + 1) / a.groups);
    const long long plane_out = (long long)a.out_rows * a.W;
    float *pzg = a.pz + (long long)g * (C::D + 1) * plane_out;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    constexpr int NWARP = C::NT / 32;
    const int x = x0 + lane;

    for (int k = gk0; k < gk1; ++k) {
        float tk[C::D];
#pragma unroll
        for (int c = 0; c < C::D; ++c) tk[c] = (c < a.d) ? __ldg(a.t + (long long)k * a.d + c) : 0.f;
        const bool first = (k == gk0);

        for (int cy = ty0; cy < ty1; cy += C::KB) {
            int h_img0, hb_dst0, nrows;
            if (cy == ty0) {
                h_img0 = cy - C::R; hb_dst0 = 0; nrows = C::HROWS;
            } else {
                // keep the last 2R horizontally-blurred rows: move rows [KB, KB+2R) -> [0, 2R)
                // in rounds of KB rows (source and destination of a round never overlap)
                for (int r0 = 0; r0 < 2 * C::R; r0 += C::KB) {
                    const int nr = min(C::KB, 2 * C::R - r0);
                    const int n4 = C::NCH * nr * (C::TX / 4);
                    for (int it = threadIdx.x; it < n4; it += C::NT) {
                        const int c4 = it % (C::TX / 4);
                        const int rr = (it / (C::TX / 4)) % nr;
                        const int ch = it / ((C::TX / 4) * nr);
                        float4 *base = reinterpret_cast<float4 *>(hb + ch * C::HROWS * C::TX);
                        base[(r0 + rr) * (C::TX / 4) + c4] = base[(r0 + rr + C::KB) * (C::TX / 4) + c4];
                    }
                    __syncthreads();
                }
                h_img0 = cy + C::R; hb_dst0 = 2 * C::R; nrows = C::KB;
            }
            for (int s0 = 0; s0 < nrows; s0 += C::SH) {
                const int n = min(C::SH, nrows - s0);
                modulate<C>(a, mod, tk, h_img0 + s0, n, x0);
                __syncthreads();
                hpass<C>(a, mod, hb, hb_dst0 + s0, n);
                __syncthreads();
            }
            // (c, s) at the chunk's output pixels (same arithmetic as `modulate`)
            for (int it = threadIdx.x; it < C::KB * C::TX; it += C::NT) {
                const int row = it / C::TX, col = it - row * C::TX;
                float fv[C::D];
                load_pixel<C>(a, cy + row, x0 + col, fv);
                float s, c;
                __sincosf(phase<C>(tk, fv), &s, &c);
                cs[row * C::TX + col] = c;
                cs[(C::KB + row) * C::TX + col] = s;
            }
            __syncthreads();

            // vertical pass + accumulate: warp item = (pair p, 8-row group), lane = column
            constexpr int WITEMS = (C::D + 1) * (C::KB / 8);
            for (int wi = warp; wi < WITEMS; wi += NWARP) {
                const int p = wi % (C::D + 1);          // 0 -> Z, 1 + q -> P'_q
                const int rg = wi / (C::D + 1);
                const int plane = (p == 0) ? C::D : p - 1;
                float *dst = pzg + plane * plane_out + (long long)(cy + rg * 8 - a.out_row0) * a.W + x;
                const bool xok = x < a.W;
                float old[8];
#pragma unroll
                for (int o = 0; o < 8; ++o) {
                    const bool ok = xok && (cy + rg * 8 + o < ty1);
                    old[o] = (!first && ok) ? dst[(long long)o * a.W] : 0.f;
                }
                const float *bc = hb + (2 * p) * C::HROWS * C::TX + rg * 8 * C::TX + lane;
                const float *bs = bc + C::HROWS * C::TX;
                float ac[8], as[8];
#pragma unroll
                for (int o = 0; o < 8; ++o) { ac[o] = 0.f; as[o] = 0.f; }
#pragma unroll
                for (int j = 0; j < 8 + 2 * C::R; ++j) {
                    const float vc = bc[j * C::TX];
                    const float vs = bs[j * C::TX];
#pragma unroll
                    for (int o = 0; o < 8; ++o) {
                        const int m = j - o - C::R;
                        if (m >= -C::R && m <= C::R) {
                            ac[o] = fmaf(a.w[m < 0 ? -m : m], vc, ac[o]);
                            as[o] = fmaf(a.w[m < 0 ? -m : m], vs, as[o]);
                        }
                    }
                }
#pragma unroll
                for (int o = 0; o < 8; ++o) {
                    const int r = rg * 8 + o;
                    if (xok && cy + r < ty1) {
                        const float c = cs[r * C::TX + lane];
                        const float s = cs[(C::KB + r) * C::TX + lane];
                        dst[(long long)o * a.W] = fmaf(c, ac[o], fmaf(s, as[o], old[o]));
                    }
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
// instance table: (D, R) -> Cfg. A plan with radius r uses the smallest
// compiled R >= r (taps beyond r are zero); d uses the smallest D >= d.
// ---------------------------------------------------------------------------
#define BFV_INSTANCES(X)                      \
    X(1, 2, 256, 32, 8) X(1, 6, 256, 32, 8)   \
    X(1, 15, 256, 32, 8) X(1, 32, 256, 32, 8) \
    X(1, 64, 256, 32, 8)                      \
    X(2, 6, 256, 32, 8) X(2, 15, 256, 32, 8)  \
    X(2, 32, 256, 32, 8) X(2, 64, 256, 32, 8) \
    X(3, 2, 256, 32, 8) X(3, 4, 256, 32, 8)   \
    X(3, 6, 256, 32, 8) X(3, 10, 256, 32, 8)  \
    X(3, 15, 256, 32, 8) X(3, 24, 256, 32, 8) \
    X(3, 30, 256, 32, 8) X(3, 48, 256, 32, 8) \
    X(3, 64, 256, 16, 8)                      \
    X(4, 6, 256, 32, 8) X(4, 15, 256, 32, 8)  \
    X(4, 32, 256, 32, 8) X(4, 48, 256, 16, 8) \
    X(8, 6, 288, 32, 4) X(8, 15, 288, 32, 4)  \
    X(8, 24, 288, 32, 4) X(8, 32, 288, 16, 4)

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
