// recursive.cu -- the O(1)-in-sigma_s engine (option "engine" = 1): Algorithm 1 with the
// Gaussian convolutions of step 10 done "using separability and recursion,
// and importantly, at O(1) cost with respect to sigma_s" (Deriche 1993).
//
// Spatial kernel (reading R16): Deriche's 4th-order recursive Gaussian,
//   g(m) = h(|m|) / S,  h(x) = sum_j Re[A_j z_j^x],  z_j = exp((-b_j + i w_j) / sigma_s),
// on the half-sample-reflected, periodically folded image (reading R1), infinite support.
// Per line x[0..n-1] and pole j:
//   u_j[k] = x[k] + z_j u_j[k-1]         (causal,     u_j[-1] = (S_head + z^n S_tail) / (1 - z^2n))
//   v_j[k] = x[k] + z_j v_j[k+1]         (anticausal, v_j[n] = u_j[n-1])
//   y[k]   = sum_j Re[A_j (u_j[k] + v_j[k])] - g0 x[k]
// with S_head = sum_m z^m x[m], S_tail = sum_m z^(n-1-m) x[m] (exact closed form of the
// reflected-periodic initial state; only the first / last Lh terms are above 2^-30).
//
// Staged design (v1): per batch of nb samples,
//   rec_row_kernel : modulation (Alg. 1) + the row pass, one CTA per 32 rows x sample;
//                    forward sweep writes the causal part to y1, backward sweep completes it
//                    in place (y1 = horizontally blurred H and G planes);
//   rec_col_kernel : the column pass on y1 (forward partial in y2), then
//                    Re[conj(H) blur] (Alg. 1) into the partial planes of group b.
// The complex images live in HBM between the two passes (bound by that traffic).
#include <cuda_runtime.h>

#include "internal.h"
#include "kernel_common.cuh"

namespace bfvec {
namespace {

constexpr int kT = 32;   // tile edge: 32 lines x 32 elements per chunk

struct Pole2 {           // both poles, for one real pair (c-part, s-part) of planes
    float2 ur[2], ui[2];
};

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fma2s(float w, float2 v, float2 acc) {
    return __ffma2_rn(make_float2(w, w), v, acc);
}
__device__ __forceinline__ float2 mul2s(float w, float2 v) { return __fmul2_rn(make_float2(w, w), v); }

// u <- x + z u  (complex pole z, real pair input x), both poles
__device__ __forceinline__ void step(const RecAxis &ax, Pole2 &s, float2 x) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const float2 ur = s.ur[j], ui = s.ui[j];
        s.ur[j] = fma2s(ax.zr[j], ur, fma2s(-ax.zi[j], ui, x));
        s.ui[j] = fma2s(ax.zr[j], ui, mul2s(ax.zi[j], ur));
    }
}

// sum_j Re[A_j u_j]
__device__ __forceinline__ float2 re_a(const RecAxis &ax, const Pole2 &s) {
    float2 y = mul2s(ax.ar[0], s.ur[0]);
    y = fma2s(-ax.ai[0], s.ui[0], y);
    y = fma2s(ax.ar[1], s.ur[1], y);
    y = fma2s(-ax.ai[1], s.ui[1], y);
    return y;
}

// running sums S += pw x; pw *= z
struct HeadSum {
    float2 sr[2], si[2];
    float pr[2], pi[2];
    __device__ void init() {
#pragma unroll
        for (int j = 0; j < 2; ++j) { sr[j] = si[j] = f2(0.f, 0.f); pr[j] = 1.f; pi[j] = 0.f; }
    }
    __device__ __forceinline__ void add(const RecAxis &ax, float2 x) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            sr[j] = fma2s(pr[j], x, sr[j]);
            si[j] = fma2s(pi[j], x, si[j]);
            const float nr = ax.zr[j] * pr[j] - ax.zi[j] * pi[j];
            pi[j] = ax.zr[j] * pi[j] + ax.zi[j] * pr[j];
            pr[j] = nr;
        }
    }
};

// u[-1] = (S_head + z^n S_tail) * inv(1 - z^2n), per pole, per real channel of the pair
__device__ __forceinline__ void init_state(const RecAxis &ax, const HeadSum &hd, const HeadSum &tl, Pole2 &s) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        // t = z^n * S_tail
        const float2 tr = fma2s(ax.znr[j], tl.sr[j], mul2s(-ax.zni[j], tl.si[j]));
        const float2 ti = fma2s(ax.znr[j], tl.si[j], mul2s(ax.zni[j], tl.sr[j]));
        const float2 qr = f2(hd.sr[j].x + tr.x, hd.sr[j].y + tr.y);
        const float2 qi = f2(hd.si[j].x + ti.x, hd.si[j].y + ti.y);
        s.ur[j] = fma2s(ax.invr[j], qr, mul2s(-ax.invi[j], qi));
        s.ui[j] = fma2s(ax.invr[j], qi, mul2s(ax.invi[j], qr));
    }
}

// ---------------------------------------------------------------------------------------------
// Row pass: CTA = 32 rows (lane = row) x NP warps (warp = (cos, sin) pair: Z, G_0 .. G_{d-1}) of
// one sample. Chunks of 32 columns are staged through shared memory so every global access is
// coalesced along x; the next chunk's f tile (and, in the backward sweep, its partial tile) is
// prefetched with cp.async while the current chunk's recursions run.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async4(float *dst, const float *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NP>
struct RowSmem {
    static constexpr int D = NP - 1;
    static constexpr int TILE = kT * (kT + 1);           // floats per padded 32 x 32 tile
    static constexpr int OB = 1;                          // partial-tile buffers: one (3 CTAs per SM at d = 3)
    static constexpr int OFF_CS = 2 * D * TILE;          // fs[2][D] tiles first
    static constexpr int OFF_OB = OFF_CS + 2 * TILE;     // cs: TILE float2
    static constexpr size_t BYTES = sizeof(float) * (size_t)(OFF_OB + OB * 2 * NP * TILE);
};

template <int NP>
__global__ void __launch_bounds__(32 * NP) rec_row_kernel(const __grid_constant__ RecArgs a) {
    using L = RowSmem<NP>;
    constexpr int D = L::D, TILE = L::TILE;
    extern __shared__ float sm[];
    auto fs = [&](int buf, int c) { return sm + (buf * D + c) * TILE; };          // [32][33] f - mu
    float2(*cs)[kT + 1] = reinterpret_cast<float2(*)[kT + 1]>(sm + L::OFF_CS);      // [32][33] (c, s)
    auto ob = [&](int buf, int q) { return sm + L::OFF_OB + (buf * 2 * NP + q) * TILE; };

    const int tid = threadIdx.x, lane = tid & 31, p = tid >> 5;
    const int y0 = blockIdx.x * kT;
    const int b = blockIdx.y;
    const int k = a.k0 + b;
    const int H = a.H, W = a.W;
    const long long plane = (long long)H * W;
    float tk[D];
#pragma unroll
    for (int c = 0; c < D; ++c) tk[c] = a.t[(long long)k * D + c];
    float *y1 = a.y1 + (long long)b * (2 * NP) * plane;
    const RecAxis &ax = a.row;
    const int nchunk = (W + kT - 1) / kT;

    // cp.async the raw f tile of chunk cx into fs(buf, .) (zeros outside the image)
    auto issue_f = [&](int cx, int buf) {
        const int x0 = cx * kT;
        for (int e = tid; e < D * kT * kT; e += 32 * NP) {
            const int c = e / (kT * kT), i = (e / kT) % kT, j = e % kT;
            const int x = x0 + j, y = y0 + i;
            const bool ok = x < W && y < H;
            cp_async4(fs(buf, c) + i * (kT + 1) + j, ok ? a.f + c * plane + (long long)y * W + x : a.f, ok);
        }
    };
    auto issue_y1 = [&](int cx, int buf) {
        const int x0 = cx * kT;
        for (int e = tid; e < 2 * NP * kT * kT; e += 32 * NP) {
            const int q = e / (kT * kT), i = (e / kT) % kT, j = e % kT;
            const int x = x0 + j, y = y0 + i;
            const bool ok = x < W && y < H;
            cp_async4(ob(buf, q) + i * (kT + 1) + j, ok ? y1 + q * plane + (long long)y * W + x : y1, ok);
        }
    };
    // centre f (reading R12) and form (c, s) = (cos, sin)(t_k . (f - mu)) of the staged tile
    auto modulate = [&](int buf) {
        for (int e = tid; e < kT * kT; e += 32 * NP) {
            const int i = e / kT, j = e % kT;
            float th = 0.f;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                float *q = fs(buf, c) + i * (kT + 1) + j;
                const float v = *q - a.mu[c];
                *q = v;
                th = fmaf(tk[c], v, th);
            }
            float s, c;
            __sincosf(th, &s, &c);
            cs[i][j] = f2(c, s);
        }
    };
    auto xval = [&](int buf, int i, int j) -> float2 {   // the pair's real input at (row i, column j)
        const float2 h = cs[i][j];
        if (p == 0) return h;
        const float fv = fs(buf, p - 1)[i * (kT + 1) + j];
        return f2(h.x * fv, h.y * fv);
    };
    auto stage_sync = [&](int cx) {   // synchronous staging (initial-state sums only)
        issue_f(cx, 0);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
        modulate(0);
        __syncthreads();
    };

    // ---- reflected-periodic initial state: S_head (first Lh columns), S_tail (last Lh) ----
    HeadSum hd, tl;
    hd.init();
    tl.init();
    const int nh = min(W, ax.lh);
    for (int cx = 0; cx * kT < nh; ++cx) {
        stage_sync(cx);
        for (int j = 0; j < kT && cx * kT + j < nh; ++j) hd.add(ax, xval(0, lane, j));
        __syncthreads();
    }
    const int xt = W - nh;   // first column of the tail range
    for (int cx = nchunk - 1; cx >= 0 && (cx + 1) * kT > xt; --cx) {
        const int x0 = cx * kT;
        stage_sync(cx);
        for (int j = min(kT, W - x0) - 1; j >= 0; --j)
            if (x0 + j >= xt) tl.add(ax, xval(0, lane, j));
        __syncthreads();
    }
    Pole2 st;
    init_state(ax, hd, tl, st);

    // ---- forward sweep: y1 <- sum_j Re[A_j u_j] - g0 x ----
    issue_f(0, 0);
    cp_async_commit();
    for (int cx = 0; cx < nchunk; ++cx) {
        const int buf = cx & 1;
        const int x0 = cx * kT;
        const int nj = min(kT, W - x0);
        if (cx + 1 < nchunk) {
            issue_f(cx + 1, buf ^ 1);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        modulate(buf);
        __syncthreads();
        float *o0 = ob(0, 2 * p) + lane * (kT + 1), *o1 = ob(0, 2 * p + 1) + lane * (kT + 1);
        for (int j = 0; j < nj; ++j) {
            const float2 x = xval(buf, lane, j);
            step(ax, st, x);
            const float2 y = fma2s(-ax.g0, x, re_a(ax, st));
            o0[j] = y.x;
            o1[j] = y.y;
        }
        __syncthreads();
        for (int e = tid; e < 2 * NP * kT * kT; e += 32 * NP) {
            const int q = e / (kT * kT), i = (e / kT) % kT, j = e % kT;
            if (j < nj && y0 + i < H) y1[q * plane + (long long)(y0 + i) * W + x0 + j] = ob(0, q)[i * (kT + 1) + j];
        }
        __syncthreads();
    }
    // ---- backward sweep: v[n] = u[n-1]; y1 += sum_j Re[A_j v_j] ----
    issue_f(nchunk - 1, 0);
    if (L::OB == 2) issue_y1(nchunk - 1, 0);
    cp_async_commit();
    for (int it = 0; it < nchunk; ++it) {
        const int cx = nchunk - 1 - it;
        const int buf = it & 1;
        const int obuf = (L::OB == 2) ? buf : 0;
        const int x0 = cx * kT;
        const int nj = min(kT, W - x0);
        if (it + 1 < nchunk) {
            issue_f(cx - 1, buf ^ 1);
            if (L::OB == 2) issue_y1(cx - 1, buf ^ 1);
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        if (L::OB == 1) {   // no room to prefetch the partial tile: plain coalesced loads
            for (int e = tid; e < 2 * NP * kT * kT; e += 32 * NP) {
                const int q = e / (kT * kT), i = (e / kT) % kT, j = e % kT;
                ob(0, q)[i * (kT + 1) + j] =
                    (j < nj && y0 + i < H) ? y1[q * plane + (long long)(y0 + i) * W + x0 + j] : 0.f;
            }
        }
        __syncthreads();
        modulate(buf);
        __syncthreads();
        float *o0 = ob(obuf, 2 * p) + lane * (kT + 1), *o1 = ob(obuf, 2 * p + 1) + lane * (kT + 1);
        for (int j = nj - 1; j >= 0; --j) {
            step(ax, st, xval(buf, lane, j));
            const float2 y = re_a(ax, st);
            o0[j] += y.x;
            o1[j] += y.y;
        }
        __syncthreads();
        for (int e = tid; e < 2 * NP * kT * kT; e += 32 * NP) {
            const int q = e / (kT * kT), i = (e / kT) % kT, j = e % kT;
            if (j < nj && y0 + i < H) y1[q * plane + (long long)(y0 + i) * W + x0 + j] = ob(obuf, q)[i * (kT + 1) + j];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// Column pass + accumulation: CTA = 32 columns (lane = column) x NP warps (warp = pair) of one
// sample; every access is coalesced along x. The forward partial goes to y2.
// ---------------------------------------------------------------------------------------------
template <int NP>
__global__ void __launch_bounds__(32 * NP) rec_col_kernel(const __grid_constant__ RecArgs a) {
    constexpr int D = NP - 1;
    const int lane = threadIdx.x & 31, p = threadIdx.x >> 5;
    const int x = blockIdx.x * kT + lane;
    const int b = blockIdx.y;
    const int k = a.k0 + b;
    const int H = a.H, W = a.W;
    if (x >= W) return;
    const long long plane = (long long)H * W;
    const float *in0 = a.y1 + ((long long)b * (2 * NP) + 2 * p) * plane + x;
    const float *in1 = in0 + plane;
    float *t0 = a.y2 + ((long long)b * (2 * NP) + 2 * p) * plane + x;
    float *t1 = t0 + plane;
    const RecAxis &ax = a.col;

    HeadSum hd, tl;
    hd.init();
    tl.init();
    const int nh = min(H, ax.lh);
    for (int y = 0; y < nh; ++y) hd.add(ax, f2(in0[(long long)y * W], in1[(long long)y * W]));
    for (int y = H - 1; y >= H - nh; --y) tl.add(ax, f2(in0[(long long)y * W], in1[(long long)y * W]));
    Pole2 st;
    init_state(ax, hd, tl, st);

#pragma unroll 4
    for (int y = 0; y < H; ++y) {
        const long long o = (long long)y * W;
        const float2 xv = f2(in0[o], in1[o]);
        step(ax, st, xv);
        const float2 yv = fma2s(-ax.g0, xv, re_a(ax, st));
        t0[o] = yv.x;
        t1[o] = yv.y;
    }
    float tk[D];
#pragma unroll
    for (int c = 0; c < D; ++c) tk[c] = a.t[(long long)k * D + c];
    const int pl = (p == 0) ? D : p - 1;
    float *pz = a.pz + ((long long)b * (D + 1) + pl) * plane + x;
#pragma unroll 4
    for (int y = H - 1; y >= 0; --y) {
        const long long o = (long long)y * W;
        step(ax, st, f2(in0[o], in1[o]));
        const float2 r = re_a(ax, st);
        const float2 bl = f2(t0[o] + r.x, t1[o] + r.y);
        float th = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) th = fmaf(tk[c], a.f[c * plane + o + x] - a.mu[c], th);
        float s, c;
        __sincosf(th, &s, &c);
        const float v = fmaf(c, bl.x, s * bl.y);   // Re[conj(H) blur], Alg. 1
        pz[o] = a.first ? v : pz[o] + v;
    }
}

template <int NP>
cudaError_t launch_np(const RecArgs &a, cudaStream_t s) {
    const size_t smem = RowSmem<NP>::BYTES;
    static std::atomic<uint64_t> attr{0};
    {
        const cudaError_t e = ensure_smem_attr(rec_row_kernel<NP>, smem, attr);
        if (e != cudaSuccess) return e;
    }
    dim3 grow((a.H + kT - 1) / kT, a.nb), gcol((a.W + kT - 1) / kT, a.nb);
    rec_row_kernel<NP><<<grow, 32 * NP, smem, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    rec_col_kernel<NP><<<gcol, 32 * NP, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_recursive(const RecArgs &a, cudaStream_t s) {
    switch (a.d) {
        case 1: return launch_np<2>(a, s);
        case 2: return launch_np<3>(a, s);
        case 3: return launch_np<4>(a, s);
        case 4: return launch_np<5>(a, s);
        case 5: return launch_np<6>(a, s);
        case 6: return launch_np<7>(a, s);
        case 7: return launch_np<8>(a, s);
        case 8: return launch_np<9>(a, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace bfvec
