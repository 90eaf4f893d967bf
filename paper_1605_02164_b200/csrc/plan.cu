// plan.cu -- host side of libbfvec: the C ABI (include/bfvec.h), Algorithm 1 setup
// (L210-214), scheduling of the fused kernel, and the
// orchestration of the device kernels on the caller's stream.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "internal.h"

using namespace bfvec;

namespace {

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// NVTX range over one C-ABI call (plan, sample, filter, partial, normalise, ...), so an nsys / ncu
// timeline of a multi-GPU run shows each rank's phases by name (`ncu --nvtx --nvtx-include
// "bfvec:filter/"` selects the kernels of one phase). Header-only NVTX3: a no-op unless a tool
// is attached.
// Calls on one plan share its scratch (padded input, partial planes, summaries). A call on a stream
// other than the previous call's first waits (on the device) for the previous call's work, so one
// plan may be driven from several streams without racing on that scratch (found by the checked
// build's timing: an eager call on the legacy stream overlapping the next call on a non-blocking
// stream). Skipped while the stream is being captured by the caller (their graph orders it).
struct StreamOrder {
    bf_vec_plan_t p;
    cudaStream_t s;
    bool active = false;
    StreamOrder(bf_vec_plan_t p_, cudaStream_t s_) : p(p_), s(s_) {
        if (!p || p->device < 0) return;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
            cudaGetLastError();
            return;
        }
        if (!p->order_ev && cudaEventCreateWithFlags(&p->order_ev, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            p->order_ev = nullptr;
            return;
        }
        if (p->order_recorded && p->order_stream != s) cudaStreamWaitEvent(s, p->order_ev, 0);
        active = true;
    }
    ~StreamOrder() {
        if (!active) return;
        if (cudaEventRecord(p->order_ev, s) == cudaSuccess) {
            p->order_stream = s;
            p->order_recorded = true;
        }
        cudaGetLastError();
    }
    StreamOrder(const StreamOrder &) = delete;
    StreamOrder &operator=(const StreamOrder &) = delete;
};

struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx &) = delete;
    Nvtx &operator=(const Nvtx &) = delete;
};

// ---------------------------------------------------------------------------
// Eq. (4): C = Q diag(1/alpha^2) Q^T by cyclic Jacobi rotations
// in fp64, canonical order and signs of reading R8.
// ---------------------------------------------------------------------------
void jacobi_eig(int n, const double *Ain, double *evals, double *V) {
    double A[64];
    std::memcpy(A, Ain, sizeof(double) * n * n);
    for (int i = 0; i < n * n; ++i) V[i] = 0.0;
    for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
    double frob = 0.0;
    for (int i = 0; i < n * n; ++i) frob += A[i] * A[i];
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += A[p * n + q] * A[p * n + q];
        if (off <= 1e-32 * frob) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = A[p * n + q];
                if (std::fabs(apq) < 1e-300) continue;
                const double theta = (A[q * n + q] - A[p * n + p]) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < n; ++k) {
                    const double akp = A[k * n + p], akq = A[k * n + q];
                    A[k * n + p] = c * akp - s * akq;
                    A[k * n + q] = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {
                    const double apk = A[p * n + k], aqk = A[q * n + k];
                    A[p * n + k] = c * apk - s * aqk;
                    A[q * n + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = V[k * n + p], vkq = V[k * n + q];
                    V[k * n + p] = c * vkp - s * vkq;
                    V[k * n + q] = s * vkp + c * vkq;
                }
            }
    }
    for (int i = 0; i < n; ++i) evals[i] = A[i * n + i];
}

bf_status_t diagonalize(int d, const double *C, double *Q, double *alpha) {
    double cmax = 0.0;
    for (int i = 0; i < d * d; ++i) {
        if (!std::isfinite(C[i])) return BF_E_ARG;
        cmax = std::max(cmax, std::fabs(C[i]));
    }
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
            if (std::fabs(C[i * d + j] - C[j * d + i]) > 1e-12 * std::max(1.0, cmax)) return BF_E_NOT_SYMMETRIC;
    bool diag = true;
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
            if (i != j && C[i * d + j] != 0.0) diag = false;
    double lam[8];
    if (diag) {  // reading R8 (i): Q = I, no reordering
        double lmax = 0.0;
        for (int i = 0; i < d; ++i) lmax = std::max(lmax, C[i * d + i]);
        for (int i = 0; i < d; ++i) {
            if (!(C[i * d + i] > 1e-12 * lmax)) return BF_E_NOT_POSDEF;
            alpha[i] = 1.0 / std::sqrt(C[i * d + i]);
        }
        for (int i = 0; i < d * d; ++i) Q[i] = 0.0;
        for (int i = 0; i < d; ++i) Q[i * d + i] = 1.0;
        return BF_OK;
    }
    double V[64];
    jacobi_eig(d, C, lam, V);
    double lmax = 0.0;
    for (int i = 0; i < d; ++i) lmax = std::max(lmax, lam[i]);
    for (int i = 0; i < d; ++i)
        if (!(lam[i] > 1e-12 * lmax)) return BF_E_NOT_POSDEF;
    // reading R8 (ii): C-eigenvalues ascending (alpha descending), stable
    int order[8];
    for (int i = 0; i < d; ++i) order[i] = i;
    std::stable_sort(order, order + d, [&](int a, int b) { return lam[a] < lam[b]; });
    for (int k = 0; k < d; ++k) {
        const int src = order[k];
        double mx = 0.0;
        for (int r = 0; r < d; ++r) mx = std::max(mx, std::fabs(V[r * d + src]));
        double sgn = 1.0;
        for (int r = 0; r < d; ++r)
            if (std::fabs(V[r * d + src]) > 1e-6 * mx) { sgn = V[r * d + src] < 0 ? -1.0 : 1.0; break; }
        for (int r = 0; r < d; ++r) Q[r * d + k] = sgn * V[r * d + src];
        alpha[k] = 1.0 / std::sqrt(lam[src]);
    }
    return BF_OK;
}

bf_status_t cuda_status(cudaError_t e) { return e == cudaSuccess ? BF_OK : BF_E_CUDA; }

#define BF_CUDA(call)                                        \
    do {                                                     \
        cudaError_t _e = (call);                             \
        if (_e != cudaSuccess) return BF_E_CUDA;             \
    } while (0)

// Kernel instance for the plan: the forced variant, else -- box taps whose window is a compiled
// radius -- the running-sum instance (variant 7), else the default order (fused_select).
bool select_kernel(bf_vec_plan_t p) {
    if (p->r > kMaxR) return false;
    if (p->force_variant == 0 && p->spatial == 1) {
        bfvec::KernelInfo ki;
        if (fused_select(p->d, p->r, 7, &ki) && ki.variant == 7) {
            p->kinfo = ki;
            return true;
        }
    }
    return fused_select(p->d, p->r, p->force_variant, &p->kinfo);
}

bf_status_t ensure_device(bf_vec_plan_t p) {
    if (p->device >= 0) return BF_OK;
    int dev = 0;
    BF_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    BF_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10) return BF_E_CUDA;  // sm_100a code only; no fallback
    BF_CUDA(cudaMalloc(&p->dX, sizeof(int32_t) * (size_t)p->M * p->d));
    BF_CUDA(cudaMalloc(&p->dt, sizeof(float) * (size_t)p->M * p->d));
    BF_CUDA(cudaMalloc(&p->dQ, sizeof(double) * 64));
    BF_CUDA(cudaMalloc(&p->dgamma, sizeof(double) * 8));
    BF_CUDA(cudaMalloc(&p->ddiag, 16));
    p->kinfo_ok = select_kernel(p);
    p->device = dev;
    return BF_OK;
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Free device memory for the scratch-budget heuristics, queried once per plan: cudaMemGetInfo
// is a driver round trip that occasionally stalls the host for milliseconds, which showed up as
// outliers in the event-timed short launches.
// The value is the memory available to this plan's scratch: free memory plus what the plan
// already holds, both at the first query -- so later budgets do not drift as the plan allocates.
size_t free_memory(bf_vec_plan_t p) {
    if (p->free_mem == 0) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) free_b = 0;
        cudaGetLastError();
        const size_t avail = free_b ? free_b + p->pz_bytes + p->drec_bytes : 0;
        p->free_mem = avail ? avail : 1;
    }
    return p->free_mem > 1 ? p->free_mem : 0;
}

// An allocation failed: other users of the device (e.g. torch's caching allocator) took memory
// since the cached query. Drop the cache and the failed error so the caller can re-plan its
// scratch against what is free now and retry once.
bool refresh_free_memory(bf_vec_plan_t p) {
    cudaGetLastError();
    p->free_mem = 0;
    return free_memory(p) > 0;
}

// Choose (tile_rows, groups) for one fused launch by a simple cost model:
// per CTA time ~ samples x (H-pass rows + V-pass rows + per-chunk overhead),
// whole launch ~ waves x CTA time + the partial-sum traffic of G groups.
void choose_schedule(const bf_vec_plan_t p, int out_rows, int ns, int *tile_rows, int *groups, int nimg = 1) {
    const KernelInfo &ki = p->kinfo;
    const int KB = ki.kb, R = ki.R, D = ki.D;
    const int nx = (p->W + kTX - 1) / kTX;
    const int occ = std::max(1, ki.occupancy);
    const long long slots = (long long)sm_count() * occ;
    // seconds per "row unit" (one 32-column row of one FIR pass for all channels) per CTA,
    // at ~60 % of the FP32 pipe shared by `occ` CTAs
    const double row_unit = 32.0 * 2.0 * (D + 1) * (2 * R + 1) / (128.0 / occ) / 1.9e9 / 0.6;
    double best = 1e300;
    int bt = KB, bg = 1;
    const int rmax = (out_rows + KB - 1) / KB * KB;
    const size_t free_b = free_memory(p);
    const double pz_budget = std::min(0.25 * (double)free_b, 24.0 * 1073741824.0);
    for (int ty = KB;; ty *= 2) {
        const int t = std::min(ty, rmax);
        const int ny = (out_rows + t - 1) / t;
        const int chunks = (std::min(t, out_rows) + KB - 1) / KB;
        for (int G = 1; G <= std::min(ns, 256); ++G) {
            const long long ctas = (long long)nx * ny * G * nimg;
            if (ctas > 2147483647LL / 2 || (long long)ny * nimg > 65535) continue;
            // partial sums: G x (D+1) planes; keep them within a quarter of the free memory
            // (at most 24 GiB), or 4 groups, whichever is larger
            const double pz_bytes = (double)G * (D + 1) * out_rows * (double)p->W * 4.0;
            if (G > 1 && pz_bytes > std::max(pz_budget, 4.0 * (D + 1) * out_rows * (double)p->W * 4.0)) continue;
            // samples per group, rounded up to whole passes (v5 pairs samples: an odd group
            // ends with a one-sample pass that costs about as much as a pair)
            const int sp = std::max(1, ki.sp);
            const int mg = ((ns + G - 1) / G + sp - 1) / sp * sp;
            // per sample: H rows (chunks*KB + 2R) and V rows (chunks*KB) run concurrently in
            // the two warp groups; the 2R halo rows of the first chunk are not overlapped
            const double cta = mg * (2.0 * chunks * KB + 4.0 * R + 2.0 * chunks) * row_unit + 2e-6;
            const long long waves = (ctas + slots - 1) / slots;
            double tt = waves * cta;
            if (G > 1) tt += (double)G * (D + 1) * out_rows * (double)p->W * 4.0 * 2.0 / 5e12;
            if (tt < best * 0.999) { best = tt; bt = t; bg = G; }
        }
        if (ty >= rmax) break;
    }
    if (p->force_tile_rows > 0) bt = (p->force_tile_rows + KB - 1) / KB * KB;
    if (p->force_groups > 0) bg = std::min(p->force_groups, ns);
    *tile_rows = bt;
    *groups = bg;
}

bf_status_t ensure_pz(bf_vec_plan_t p, size_t bytes) {
    if (p->pz_bytes >= bytes) return BF_OK;
    if (p->dpz) cudaFree(p->dpz);
    p->dpz = nullptr;
    p->pz_bytes = 0;
    BF_CUDA(cudaMalloc(&p->dpz, bytes));
    p->gen += 1;   // a captured filter graph holds the old pointer: re-capture
    p->pz_bytes = bytes;
    return BF_OK;
}

void fill_mu(bf_vec_plan_t p) {
    for (int c = 0; c < 8; ++c) p->mu[c] = (c < p->d) ? (float)(0.5 * p->value_range) : 0.f;
    if (p->lab) { p->mu[0] = 50.f; p->mu[1] = 0.f; p->mu[2] = 0.f; }   // mid L*, neutral a*, b*
}

// Lab mode: the Lab copy of `rows` rows of the caller's sRGB input (plan scratch)
bf_status_t to_lab(bf_vec_plan_t p, const float *f, int rows, const float **out, cudaStream_t s) {
    const size_t bytes = sizeof(float) * 3 * (size_t)rows * p->W;
    if (p->dlab_bytes < bytes) {
        cudaFree(p->dlab);
        p->dlab = nullptr;
        p->dlab_bytes = 0;
        BF_CUDA(cudaMalloc(&p->dlab, bytes));
        p->gen += 1;   // a captured filter graph holds the old pointer: re-capture
        p->dlab_bytes = bytes;
    }
    BF_CUDA(launch_srgb_to_lab(f, p->dlab, (long long)rows * p->W, s));
    *out = p->dlab;
    return BF_OK;
}

// fold every pending fused-launch event interval into the running total
void collect_profile(bf_vec_plan_t p) {
    while (p->ev_count > 0) {
        const int i = (p->ev_head - p->ev_count + bf_vec_plan_s::kEvRing) % bf_vec_plan_s::kEvRing;
        float ms = 0.f;
        if (cudaEventSynchronize(p->ev[i][1]) == cudaSuccess &&
            cudaEventElapsedTime(&ms, p->ev[i][0], p->ev[i][1]) == cudaSuccess) {
            p->fused_ms_total += ms;
            p->fused_calls += 1;
        }
        p->ev_count -= 1;
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bf_status_t encode_tmap(CUtensorMap *map, float *base, int dp, int Wp, int Hp, int win, int sh) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !ptr)
            return BF_E_CUDA;
        fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    const cuuint64_t dims[3] = {(cuuint64_t)dp, (cuuint64_t)Wp, (cuuint64_t)Hp};
    const cuuint64_t strides[2] = {(cuuint64_t)dp * 4, (cuuint64_t)Wp * dp * 4};
    const cuuint32_t box[3] = {(cuuint32_t)dp, (cuuint32_t)win, (cuuint32_t)sh};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? BF_OK : BF_E_CUDA;
}

// one fused launch: output rows [out_row0, out_row0+out_rows), samples [k0, k1)
struct P2POut {
    float *const *peer;   // world receive-slot bases (device pointers), or null for local partials
    int world, rank, slots;
};

// realisation batching for bf_vec_mse_sweep: group g filters samples [k0, k1) of realisation g,
// whose draws are rows [g * stride, (g + 1) * stride) of the table t
struct RealBatch {
    const float *t;
    int groups, stride;
};

// The items of the persistent schedule (see plan_persistent): per CTA its items (strip, u_begin,
// u_end, slot) over the strip's work line u = pass * nf + chunk, and per strip the number of slots
// handed out. Returns the busiest CTA's cost under the chunk-step model. Host-only and pure (the
// CPU tests check its coverage and slot invariants through bfvec_test_persistent_items).
double persistent_items(long long nx, long long nf, long long P, long long nC, long long Gc, double fill,
                        std::vector<std::vector<int4>> &mine, std::vector<int> &nslot) {
    mine.assign(nC, {});
    nslot.assign(nx, 0);   // slots handed out per strip, in item order
    auto unit = [&](long long u, long long &x, long long &g, long long &pb, long long &pe) {
        x = u % nx;
        g = u / nx;
        pb = P * g / Gc;
        pe = P * (g + 1) / Gc;
    };
    const long long units = nx * Gc, rounds = units / nC;
    for (long long r = 0; r < rounds; ++r)
        for (long long c = 0; c < nC; ++c) {
            long long x, g, pb, pe;
            unit(r * nC + c, x, g, pb, pe);
            if (pe > pb) mine[c].push_back(make_int4((int)x, (int)(pb * nf), (int)(pe * nf), nslot[x]++));
        }
    // the tail: units [rounds * nC, units), strip-major, the tail units of one strip merged into
    // one pass range (consecutive groups are consecutive passes), as one work line of chunk steps
    // cut into nC shares
    std::vector<long long> tx, tpb, tpe;   // per tail range: strip, first pass, end pass
    {
        std::vector<long long> lo(nx, -1), hi(nx, -1);
        for (long long u = rounds * nC; u < units; ++u) {
            long long x, g, pb, pe;
            unit(u, x, g, pb, pe);
            if (lo[x] < 0 || pb < lo[x]) lo[x] = pb;
            hi[x] = std::max(hi[x], pe);
        }
        for (long long x = 0; x < nx; ++x)
            if (lo[x] >= 0 && hi[x] > lo[x]) { tx.push_back(x); tpb.push_back(lo[x]); tpe.push_back(hi[x]); }
    }
    std::vector<long long> start(1, 0);
    for (size_t i = 0; i < tx.size(); ++i) start.push_back(start.back() + (tpe[i] - tpb[i]) * nf);
    const long long TW = start.back();
    const double tshare = (double)TW / nC;
    const long long gran = (tshare / nf >= 50.0) ? nf : 1;
    auto cut = [&](long long c) { return c >= nC ? TW : (TW * c / nC + gran / 2) / gran * gran; };
    for (long long c = 0; c < nC && TW > 0; ++c) {
        long long w0 = cut(c);
        const long long w1 = cut(c + 1);
        while (w0 < w1) {
            const long long i = std::upper_bound(start.begin(), start.end(), w0) - start.begin() - 1;
            const long long x = tx[i], pb = tpb[i];
            const long long e = std::min(w1, start[i + 1]);
            const long long a0 = w0 - start[i], a1 = e - start[i];
            mine[c].push_back(make_int4((int)x, (int)(pb * nf + a0), (int)(pb * nf + a1), nslot[x]++));
            w0 = e;
        }
    }
    // busiest CTA under the cost model: chunk steps + one fill per pass an item streams
    double t_pers = 0.0;
    for (long long c = 0; c < nC; ++c) {
        double tc = 0.0;
        for (const int4 &it : mine[c]) {
            const long long passes = (it.z - 1) / nf - it.y / nf + 1;
            tc += (double)(it.z - it.y) + passes * fill;
        }
        t_pers = std::max(t_pers, tc);
    }
    return t_pers;
}

// Persistent schedule for the v6 kernel (FusedArgs::items): one CTA per SM slot running a list of
// items (strip, range of its (pass, chunk) work line, partial slot), instead of whole (strip,
// tile, sample group) CTAs whose count rarely divides into whole waves (config 2: 128 CTAs on 148
// SMs). The classic units (strip x, sample group g: a range of two-sample passes over the full
// height) are dealt out in whole rounds -- CTA c takes units c, c + nC, ... -- so at any time the
// CTAs sweep neighbouring strips at the same rows and share their halo columns of f in L2, as the
// classic waves do; the units left over after the last whole round (config 5: 136 of 1024; config
// 2: all 128) are cut into nC equal shares of their (pass, chunk) work line, on whole passes when a
// share spans >= 50 passes (else mid-pass: a partial pass streams its own A-row halo first). A
// unit's first piece writes slot g, further pieces extra slots >= the group count; an item that
// covers less than a whole pass zeroes the rows it never visited and each strip's last item zeroes
// the slots no CTA uses for it, so the normaliser sums the same slot count everywhere. Chosen when
// the chunk-step cost model (incl. the A/KB-chunk pipeline fill per pass) of the busiest CTA beats
// the classic grid by > 0.5 %. Returns the slot count (groups) or 0 when the classic grid stays.
int plan_persistent(bf_vec_plan_t p, int out_rows, int ns, int tile_rows, int groups, cudaStream_t s) {
    const KernelInfo &ki = p->kinfo;
    if (p->persistent == 0 || (ki.variant != 4 && ki.variant != 7)) return 0;
    // a forced (tile_rows, groups) schedule is honoured unless persistent = 2 forces this one
    if (p->persistent == 1 && (p->force_groups > 0 || p->force_tile_rows > 0)) return 0;
    const long long nx = (p->W + kTX - 1) / kTX;
    const long long nf = (out_rows + ki.kb - 1) / ki.kb;
    const long long P = (ns + ki.sp - 1) / ki.sp;
    const long long nC = (long long)sm_count() * std::max(1, ki.occupancy);
    if (p->persistent != 2 && nx * P * nf < 4 * nC) return 0;   // forced: any size (idle CTAs get no items)
    const long long Gc = std::max(1LL, std::min<long long>(groups, P));
    const long long key[5] = {nx, nf, P, nC, (ki.variant * 2 + (p->persistent == 2 ? 1 : 0)) * 65536 + Gc};
    if (std::equal(key, key + 5, p->pers_key)) return p->pers_groups;
    const double fill = (double)((ki.kb + 2 * ki.R + 15) / 16 * 16) / ki.kb;   // A / KB chunk-times per pass
    // classic grid: whole waves of CTAs, each ceil(samples / SP) passes over its tile
    const long long ny = (out_rows + tile_rows - 1) / tile_rows;
    const long long ctas = nx * ny * groups;
    const long long waves = (ctas + nC - 1) / nC;
    const long long gpass = ((ns + groups - 1) / groups + ki.sp - 1) / ki.sp;
    const double t_classic = (double)waves * gpass * ((tile_rows + ki.kb - 1) / ki.kb + fill);

    std::vector<std::vector<int4>> mine;
    std::vector<int> nslot;
    const double t_pers = persistent_items(nx, nf, P, nC, Gc, fill, mine, nslot);
    // measured: config 2 predicted 0.91, measured 0.90 (kernel time); config 5 (whole rounds +
    // tail) predicted 0.99; config 3 stays classic
    if (p->persistent == 1 && !(t_pers < 0.995 * t_classic)) {
        std::copy(key, key + 5, p->pers_key);
        p->pers_groups = 0;
        return 0;
    }
    std::vector<int4> items;
    std::vector<int> off(nC + 1);
    for (long long c = 0; c < nC; ++c) {
        off[c] = (int)items.size();
        for (const int4 &it : mine[c]) items.push_back(it);
    }
    off[nC] = (int)items.size();
    int G = 1;
    for (long long x = 0; x < nx; ++x) G = std::max(G, nslot[x]);
    if (p->dstrip_cap < (size_t)nx) {
        cudaFree(p->dstrip_slots);
        p->dstrip_slots = nullptr;
        p->dstrip_cap = 0;
        if (cudaMalloc(&p->dstrip_slots, sizeof(int) * nx) != cudaSuccess) { cudaGetLastError(); return 0; }
        p->dstrip_cap = nx;
        p->gen += 1;
    }
    if (p->ditems_cap < items.size()) {
        cudaFree(p->ditems);
        p->ditems = nullptr;
        p->ditems_cap = 0;
        if (cudaMalloc(&p->ditems, sizeof(int4) * items.size()) != cudaSuccess) { cudaGetLastError(); return 0; }
        p->ditems_cap = items.size();
        p->gen += 1;   // a captured filter graph holds the old pointer: re-capture
    }
    if (p->ditem_off_cap < off.size()) {
        cudaFree(p->ditem_off);
        p->ditem_off = nullptr;
        p->ditem_off_cap = 0;
        if (cudaMalloc(&p->ditem_off, sizeof(int) * off.size()) != cudaSuccess) { cudaGetLastError(); return 0; }
        p->ditem_off_cap = off.size();
        p->gen += 1;
    }
    // ordered before the launches that read it (the copy is synchronous; it runs once per schedule)
    if (cudaStreamSynchronize(s) != cudaSuccess ||
        cudaMemcpy(p->ditems, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->ditem_off, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(p->dstrip_slots, nslot.data(), sizeof(int) * nx, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    std::copy(key, key + 5, p->pers_key);
    p->gen += 1;   // the tables were rewritten: a captured filter graph of another shape must re-capture
    p->pers_groups = G;
    p->pers_items = (int)items.size();
    p->pers_ctas = (int)nC;
    return G;
}

bf_status_t run_fused(bf_vec_plan_t p, const float *f, int slab_rows, int slab_row0, int out_row0,
                      int out_rows, int k0, int k1, cudaStream_t s, int *groups_out, const P2POut *p2p = nullptr,
                      const RealBatch *rb = nullptr, int nimg = 1) {
    if (!p->kinfo_ok) return BF_E_UNSUPPORTED;   // r > 64 or no compiled instance: engine 1 only
    int tile_rows = 0, groups = 1;
    choose_schedule(p, out_rows, k1 - k0, &tile_rows, &groups, nimg);
    if (p2p) groups = p2p->slots;   // one receive slot per (rank, group) on every owner
    if (rb) groups = rb->groups;    // one realisation per group
    const KernelInfo &ki = p->kinfo;
    // the persistent schedule: single images without peer stores or realisation batches
    cudaStreamCaptureStatus capst = cudaStreamCaptureStatusNone;
    const bool capturing = cudaStreamIsCapturing(s, &capst) == cudaSuccess && capst != cudaStreamCaptureStatusNone;
    cudaGetLastError();
    int pers = 0;
    if (!p2p && !rb && nimg == 1) {
        const long long key_nf = (out_rows + ki.kb - 1) / ki.kb;
        const long long key_P = (k1 - k0 + ki.sp - 1) / std::max(1, ki.sp);
        const bool cached = p->pers_key[1] == key_nf && p->pers_key[2] == key_P &&
                            p->pers_key[0] == (p->W + kTX - 1) / kTX && p->pers_key[4] / 65536 / 2 == ki.variant;
        // never allocate or copy while the stream is captured: only a cached schedule may be used
        if (!capturing || cached) pers = plan_persistent(p, out_rows, k1 - k0, tile_rows, groups, s);
        if (pers) {
            groups = pers;
            tile_rows = (out_rows + ki.kb - 1) / ki.kb * ki.kb;
        }
    }
    size_t img_pz = (size_t)groups * (ki.D + 1) * out_rows * (size_t)p->W;   // partial floats per image
    bf_status_t st = ensure_pz(p, sizeof(float) * img_pz * nimg);
    if (st == BF_E_CUDA && !p2p && !rb && !pers && refresh_free_memory(p)) {
        // memory taken since the cached query: re-plan the groups against what is free now
        choose_schedule(p, out_rows, k1 - k0, &tile_rows, &groups, nimg);
        img_pz = (size_t)groups * (ki.D + 1) * out_rows * (size_t)p->W;
        st = ensure_pz(p, sizeof(float) * img_pz * nimg);
    }
    if (st != BF_OK) return st;
    // reflect-padded, centred, interleaved copy of the rows this launch reads (pad.cu)
    const int R = ki.R;
    const int Hp = out_rows + 2 * R, Wp = p->W + 2 * R;
    const size_t fbytes = sizeof(float) * (size_t)Hp * Wp * ki.dp * nimg;
    if (p->fpad_bytes < fbytes) {
        cudaFree(p->dfpad);
        p->dfpad = nullptr;
        p->fpad_bytes = 0;
        BF_CUDA(cudaMalloc(&p->dfpad, fbytes));
        p->gen += 1;   // a captured filter graph holds the old pointer: re-capture
        p->fpad_bytes = fbytes;
    }
    fill_mu(p);
    for (int b = 0; b < nimg; ++b)   // image b of a batch: input at b * d * slab_rows * W, padded block b
        BF_CUDA(launch_pad(f + (size_t)b * p->d * slab_rows * p->W, (long long)slab_rows * p->W, p->d, p->H, p->W,
                           slab_row0, slab_rows, out_row0 - R, Hp, Wp, R, ki.dp, p->mu,
                           p->dfpad + (size_t)b * Hp * Wp * ki.dp, s));
    FusedArgs a;
    std::memset(&a, 0, sizeof(a));
    st = encode_tmap(&a.tmap, p->dfpad, ki.dp, Wp, Hp * nimg, ki.win, ki.sh);
    if (st != BF_OK) return st;
    a.d = p->d;
    a.W = p->W;
    a.out_row0 = out_row0;
    a.out_rows = out_rows;
    a.tile_rows = tile_rows;
    a.groups = groups;
    a.k0 = k0;
    a.k1 = k1;
    a.t = rb ? rb->t : p->dt;
    a.gstride = rb ? rb->stride : 0;
    a.pz = p->dpz;
    for (int i = 0; i <= kMaxR; ++i) a.w[i] = (i <= p->r) ? p->taps[i] : 0.f;
    if (p2p) {
        for (int i = 0; i < p2p->world; ++i) a.peer[i] = p2p->peer[i];
        a.p2p_world = p2p->world;
        a.p2p_rank = p2p->rank;
        a.p2p_rpb = p->H / p2p->world;
    }
    const int ny = (out_rows + tile_rows - 1) / tile_rows;
    if (nimg > 1) {
        a.tiles_per_img = ny;
        a.img_prows = Hp;
        a.img_pz = (long long)img_pz;
    }
    dim3 grid((p->W + kTX - 1) / kTX, ny * nimg, groups);
    if (pers) {
        a.items = p->ditems;
        a.item_off = p->ditem_off;
        a.nch_full = (out_rows + ki.kb - 1) / ki.kb;
        grid = dim3(p->pers_ctas, 1, 1);
    }
    p->last_persistent = pers ? 1 : 0;
    p->last_strip_slots = pers ? p->dstrip_slots : nullptr;
    p->last_tile_rows = tile_rows;
    p->last_groups = groups;
    p->last_ctas = (long long)grid.x * grid.y * grid.z;
    int slot = -1;
    if (p->profile) {
        if (p->ev_count == bf_vec_plan_s::kEvRing) collect_profile(p);
        slot = p->ev_head;
        for (int j = 0; j < 2; ++j)
            if (!p->ev[slot][j]) BF_CUDA(cudaEventCreate(&p->ev[slot][j]));
        BF_CUDA(cudaEventRecord(p->ev[slot][0], s));
    }
    BF_CUDA(fused_launch(ki, a, grid, s));
    if (slot >= 0) {
        BF_CUDA(cudaEventRecord(p->ev[slot][1], s));
        p->ev_head = (p->ev_head + 1) % bf_vec_plan_s::kEvRing;
        p->ev_count += 1;
    }
    *groups_out = groups;
    return BF_OK;
}

// Separable spatial taps w(|m|), m in [-r, r], normalised to sum 1 in fp64 (reading R3) and
// rounded once to fp32. Eq. (1) gives the Gaussian; PAPER.md:205 allows "any
// arbitrary spatial filter (such as a box or hat filter)" (reading R15: same window r).
void make_taps(bf_vec_plan_t p) {
    const int r = p->r;
    if (r > kMaxR) {                       // FIR / direct unsupported at this radius
        for (int m = 0; m <= kMaxR; ++m) p->taps[m] = 0.f;
        return;
    }
    double w[kMaxR + 1], sum = 0.0;
    for (int m = 0; m <= r; ++m) {
        if (p->spatial == 1) w[m] = 1.0;                                   // box
        else if (p->spatial == 2) w[m] = (double)(r + 1 - m);              // hat
        else w[m] = std::exp(-(double)m * m / (2.0 * p->sigma_s * p->sigma_s));   // Gaussian
        sum += (m == 0 ? 1.0 : 2.0) * w[m];
    }
    for (int m = 0; m <= kMaxR; ++m) p->taps[m] = (m <= r) ? (float)(w[m] / sum) : 0.f;
}

// ---------------------------------------------------------------------------------------------
// Recursive engine (reading R16): Deriche's 4th-order recursive Gaussian
// (PAPER.md:204). The plan computes, in fp64, the poles z_j = exp((-b_j + i w_j) / sigma_s),
// the residues A_j = (a_j - i a'_j) / S normalised so that the kernel sums to one
// (S = 2 Re sum_j A_j / (1 - z_j) - h(0), the closed-form sum of h(|m|) over all integers m),
// and per axis of length n the reflected-periodic initial-state factors z^n and 1 / (1 - z^2n).
// ---------------------------------------------------------------------------------------------
struct Cplx {
    double r, i;
};
Cplx cmul(Cplx a, Cplx b) { return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
Cplx cdiv(Cplx a, Cplx b) {
    const double den = b.r * b.r + b.i * b.i;
    return {(a.r * b.r + a.i * b.i) / den, (a.i * b.r - a.r * b.i) / den};
}
Cplx cexp_(double re, double im) { return {std::exp(re) * std::cos(im), std::exp(re) * std::sin(im)}; }

void rec_axis(double sigma, int n, RecAxis *ax) {
    // Deriche (1993) smoothing constants: h(x) = (a0 cos(w0 x/s) + a1 sin(w0 x/s)) e^{-b0 x/s}
    //                                           + (c0 cos(w1 x/s) + c1 sin(w1 x/s)) e^{-b1 x/s}
    const double a0 = 1.68, a1 = 3.735, b0 = 1.783, b1 = 1.723, c0 = -0.6803, c1 = -0.2598, w0 = 0.6318,
                 w1 = 1.997;
    const double bj[2] = {b0, b1}, wj[2] = {w0, w1};
    const Cplx Aj[2] = {{a0, -a1}, {c0, -c1}};
    Cplx z[2];
    double S = -(a0 + c0);
    for (int j = 0; j < 2; ++j) {
        z[j] = cexp_(-bj[j] / sigma, wj[j] / sigma);
        S += 2.0 * cdiv(Aj[j], Cplx{1.0 - z[j].r, -z[j].i}).r;
    }
    for (int j = 0; j < 2; ++j) {
        ax->zr[j] = (float)z[j].r;
        ax->zi[j] = (float)z[j].i;
        ax->ar[j] = (float)(Aj[j].r / S);
        ax->ai[j] = (float)(Aj[j].i / S);
        const Cplx zn = cexp_(-bj[j] * n / sigma, wj[j] * n / sigma);
        const Cplx inv = cdiv(Cplx{1.0, 0.0}, Cplx{1.0 - cmul(zn, zn).r, -cmul(zn, zn).i});
        ax->znr[j] = (float)zn.r;
        ax->zni[j] = (float)zn.i;
        ax->invr[j] = (float)inv.r;
        ax->invi[j] = (float)inv.i;
    }
    ax->g0 = (float)((a0 + c0) / S);
    // head / tail terms above 2^-30: |z|^m = e^{-min(b) m / sigma}
    const double lh = std::ceil(30.0 * std::log(2.0) * sigma / std::min(b0, b1));
    ax->lh = (int)std::min<double>(n, lh);
}

bf_status_t ensure_rec_scratch(bf_vec_plan_t p, int nb) {
    const size_t per = sizeof(float) * (size_t)2 * (p->d + 1) * p->H * (size_t)p->W;
    if (p->drec_bytes < 2 * per * nb) {
        cudaFree(p->drec);
        p->drec = nullptr;
        p->drec_bytes = 0;
        BF_CUDA(cudaMalloc(&p->drec, 2 * per * nb));
        p->gen += 1;   // a captured filter graph holds the old pointer: re-capture
        p->drec_bytes = 2 * per * nb;
    }
    return BF_OK;
}

// Tiled engine: per axis of length n in tiles of kRecT, the pole powers z_j^{L_t}, z_j^{x0_t} and
// z_j^{n - x0_t - L_t} (each exp(m (-b_j + i w_j) / sigma_s) in fp64), both axes in p->drtab.
// Tensor-core pass 2 (option rec_tc): the exact blur of a full 32-element segment of a line from its
// entering states (blur_segment) is one matrix product, y[i] = sum_m K[i][m] x[m] + sum_k S[i][k] s[k],
// K[i][m] = h(|i - m|) = sum_j Re[A_j z_j^|i-m|] (the Deriche kernel; the diagonal counts the sample
// once: 2 Re A - g0 = Re A), and the state basis for s = (L_0, L_1, R_0, R_1) as (re, im) pairs,
// S[i][2j] + i S[i][2j+1] = conj-free split of A_j z_j^{i+1} (L_j) and A_j z_j^{32-i} (R_j):
// Re[c L] = Re c L.r - Im c L.i. The 32 x 40 matrix B = [K | S] is split into tf32 halves
// (hi = round-to-nearest tf32, lo = tf32 of the rest) so three tf32 products give fp32 accuracy, and
// laid out as the MMA's K-major no-swizzle B operand: rows n (0..31 hi, 32..63 lo), core matrices of
// 8 rows x 4 columns, (n / 8, k / 4) at ((n / 8) * 10 + k / 4) * 32 floats.
static float tf32_rna(float x) {
    uint32_t b;
    std::memcpy(&b, &x, 4);
    b = (b + 0x1000u) & ~0x1FFFu;
    float r;
    std::memcpy(&r, &b, 4);
    return r;
}
void rec_tc_matrix(double sigma, float *out) {
    const double a0 = 1.68, a1 = 3.735, b0 = 1.783, b1 = 1.723, c0 = -0.6803, c1 = -0.2598, w0 = 0.6318,
                 w1 = 1.997;
    const double bj[2] = {b0, b1}, wj[2] = {w0, w1};
    Cplx Aj[2] = {{a0, -a1}, {c0, -c1}};
    double S = -(a0 + c0);
    Cplx z[2];
    for (int j = 0; j < 2; ++j) {
        z[j] = cexp_(-bj[j] / sigma, wj[j] / sigma);
        S += 2.0 * cdiv(Aj[j], Cplx{1.0 - z[j].r, -z[j].i}).r;
    }
    for (int j = 0; j < 2; ++j) Aj[j] = {Aj[j].r / S, Aj[j].i / S};
    auto azp = [&](int j, int n) {   // A_j z_j^n
        const Cplx zn = cexp_(-bj[j] * n / sigma, wj[j] * n / sigma);
        return cmul(Aj[j], zn);
    };
    double B[kRecT][40];
    for (int i = 0; i < kRecT; ++i) {
        for (int m = 0; m < kRecT; ++m) B[i][m] = azp(0, std::abs(i - m)).r + azp(1, std::abs(i - m)).r;
        for (int j = 0; j < 2; ++j) {
            const Cplx l = azp(j, i + 1), r = azp(j, kRecT - i);
            B[i][32 + 2 * j] = l.r;
            B[i][33 + 2 * j] = -l.i;
            B[i][36 + 2 * j] = r.r;
            B[i][37 + 2 * j] = -r.i;
        }
    }
    for (int n = 0; n < 64; ++n)
        for (int k = 0; k < 40; ++k) {
            const int i = n & 31;
            const float hi = tf32_rna((float)B[i][k]);
            const float v = n < 32 ? hi : tf32_rna((float)(B[i][k] - (double)hi));
            out[((n / 8) * 10 + k / 4) * 32 + (n % 8) * 4 + (k % 4)] = v;
        }
}

bf_status_t ensure_rec_tabs(bf_vec_plan_t p, RecTabs *th, RecTabs *tv) {
    const int ntx = (p->W + kRecT - 1) / kRecT, nty = (p->H + kRecT - 1) / kRecT;
    // + zp: (z_0^m, z_1^m), m < kRecT; + the tensor-core tile-blur matrix (kRecTcB floats)
    const size_t n = (size_t)6 * (ntx + nty) + 2 * kRecT + kRecTcB / 2;
    if (p->drtab_n != n) {
        const double bj[2] = {1.783, 1.723}, wj[2] = {0.6318, 1.997};   // rec_axis's poles
        std::vector<float2> h(n);
        size_t o = 0;
        for (int ax = 0; ax < 2; ++ax) {
            const int len = ax == 0 ? p->W : p->H, nt = ax == 0 ? ntx : nty;
            for (int kind = 0; kind < 3; ++kind)
                for (int j = 0; j < 2; ++j)
                    for (int t = 0; t < nt; ++t) {
                        const int x0 = t * kRecT, L = std::min(kRecT, len - x0);
                        const int m = kind == 0 ? L : kind == 1 ? x0 : len - x0 - L;
                        const Cplx z = cexp_(-bj[j] * m / p->sigma_s, wj[j] * m / p->sigma_s);
                        h[o++] = make_float2((float)z.r, (float)z.i);
                    }
        }
        for (int m = 0; m < kRecT; ++m)
            for (int j = 0; j < 2; ++j) {
                const Cplx z = cexp_(-bj[j] * m / p->sigma_s, wj[j] * m / p->sigma_s);
                h[o++] = make_float2((float)z.r, (float)z.i);
            }
        rec_tc_matrix(p->sigma_s, reinterpret_cast<float *>(h.data() + o));
        cudaFree(p->drtab);
        p->drtab = nullptr;
        p->drtab_n = 0;
        BF_CUDA(cudaMalloc(&p->drtab, sizeof(float2) * n));
        p->gen += 1;   // a captured filter graph holds the old pointer: re-capture
        BF_CUDA(cudaMemcpy(p->drtab, h.data(), sizeof(float2) * n, cudaMemcpyHostToDevice));
        p->drtab_n = n;
    }
    th->zl = p->drtab;
    th->pf = th->zl + 2 * ntx;
    th->pb = th->pf + 2 * ntx;
    tv->zl = th->pb + 2 * ntx;
    tv->pf = tv->zl + 2 * nty;
    tv->pb = tv->pf + 2 * nty;
    th->zp = tv->zp = reinterpret_cast<const float4 *>(tv->pb + 2 * nty);
    return BF_OK;
}

#ifndef BFVEC_REC_BATCH_CAP
#define BFVEC_REC_BATCH_CAP 48
#endif
constexpr int kRecBatchCap = BFVEC_REC_BATCH_CAP;
bf_status_t run_recursive_tiled(bf_vec_plan_t p, const float *f, int k0, int k1, cudaStream_t s, int *groups_out) {
    const int ns = k1 - k0;
    const int NQ = 2 * (p->d + 1);
    const int ntx = (p->W + kRecT - 1) / kRecT, nty = (p->H + kRecT - 1) / kRecT;
    const long long tiles = (long long)ntx * nty;
    const size_t px = (size_t)p->H * p->W;
    // rec_impl 2: the row arrays also hold 8 virtual lines per tile row
    const bool vlines = p->rec_impl == 2;
    const int nlh = p->H + (vlines ? 8 * nty : 0);
    // per sample in flight: row / column summaries (E, B) and line states (+ virtual-line values)
    const size_t sum_h = (size_t)NQ * 2 * ntx * nlh, sum_v = (size_t)NQ * 2 * nty * p->W;
    const size_t uv_h = (size_t)NQ * 2 * nlh, uv_v = (size_t)NQ * 2 * p->W;
    const size_t rb_per = (p->rec_store && !vlines) ? sizeof(float) * (size_t)NQ * px : 0;   // stored row blur
    const size_t vl_per = vlines ? sizeof(float) * (size_t)NQ * nty * 8 * p->W : 0;
    const size_t per = sizeof(float2) * 2 * (sum_h + sum_v) + sizeof(float4) * (uv_h + uv_v) + rb_per + vl_per;
    int nb = 1, g = 1, sets = 1;
    bf_status_t st = BF_OK;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const size_t free_b = free_memory(p);
        // batch: up to 256 samples within 40 % of the free memory, but no more than kRecBatchCap samples
        // or 4 GiB of summaries (whichever allows more). Each batch costs ~2.5 ms beyond its samples'
        // work on config 5 (launch drains, the partial-plane read-modify-write): 16 -> 32 -> 48 samples
        // per batch measured 3.27 -> 3.42 -> 3.46e10 pixel*samples/s
        const double cap = std::max((double)kRecBatchCap, 4.0 * 1024 * 1024 * 1024 / (double)per);
        const double sets_max = p->rec_overlap ? 2.0 : 1.0;   // overlap: two scratch sets in flight
        nb = (int)std::max(1.0, std::min({256.0, 0.4 * (double)free_b / (sets_max * (double)per), cap}));
        if (p->force_batch > 0) nb = p->force_batch;
        nb = std::min(nb, ns);
        sets = (p->rec_overlap && ns > nb) ? 2 : 1;
        // sample groups: enough CTAs for ~8 per SM where the tile count alone does not give them
        const long long want = 8LL * sm_count();
        g = (int)std::min<long long>(nb, std::max<long long>(1, (want + tiles - 1) / tiles));
        st = BF_OK;
        if (p->drec_bytes < per * nb * sets) {
            cudaFree(p->drec);
            p->drec = nullptr;
            p->drec_bytes = 0;
            if (cudaMalloc(&p->drec, per * nb * sets) != cudaSuccess) {
                p->drec = nullptr;
                st = BF_E_CUDA;
            } else {
                p->gen += 1;   // a captured filter graph holds the old pointer: re-capture
                p->drec_bytes = per * nb * sets;
            }
        }
        if (st == BF_OK) st = ensure_pz(p, sizeof(float) * (size_t)g * (p->d + 1) * px);
        // memory taken since the cached query: re-plan the batch against what is free now
        if (st != BF_E_CUDA || attempt == 1 || !refresh_free_memory(p)) break;
    }
    if (st != BF_OK) return st;
    RecTArgs a;
    std::memset(&a, 0, sizeof(a));
    st = ensure_rec_tabs(p, &a.th, &a.tv);
    if (st != BF_OK) return st;
    fill_mu(p);
    a.f = f;
    a.t = p->dt;
    a.pz = p->dpz;
    for (int c = 0; c < kMaxD; ++c) a.mu[c] = p->mu[c];
    a.d = p->d;
    a.H = p->H;
    a.W = p->W;
    a.ntx = ntx;
    a.nty = nty;
    a.g1 = g;
    a.g3 = g;
    // scratch set k (of `sets`): summaries, line states, stored row blur / virtual-line values
    auto set_scratch = [&](RecTArgs &x, int k) {
        float2 *base = reinterpret_cast<float2 *>(reinterpret_cast<char *>(p->drec) + per * nb * k);
        x.Eh = base;
        x.Bh = x.Eh + (size_t)nb * sum_h;
        x.Ev = x.Bh + (size_t)nb * sum_h;
        x.Bv = x.Ev + (size_t)nb * sum_v;
        x.UVh = reinterpret_cast<float4 *>(x.Bv + (size_t)nb * sum_v);
        x.UVv = x.UVh + (size_t)nb * uv_h;
        x.rbg = rb_per ? reinterpret_cast<float *>(x.UVv + (size_t)nb * uv_v) : nullptr;
        x.vl = vlines ? reinterpret_cast<float *>(x.UVv + (size_t)nb * uv_v) : nullptr;
    };
    set_scratch(a, 0);
    a.nlh = nlh;
    a.tcb = reinterpret_cast<const float *>(a.th.zp + kRecT);
    a.tc = (p->rec_tc && p->d <= 7) ? 1 : 0;   // up to four M halves (16 planes) in tensor memory
    a.vtc = (p->rec_vtc && p->rec_tc && p->W % kRecT == 0) ? 1 : 0;
    rec_axis(p->sigma_s, p->W, &a.row);
    rec_axis(p->sigma_s, p->H, &a.col);
    {   // the pole powers z_j^m, m < kRecT (as in ensure_rec_tabs), as kernel parameters
        const double bj[2] = {1.783, 1.723}, wj[2] = {0.6318, 1.997};
        for (int m = 0; m < kRecT; ++m) {
            const Cplx z0 = cexp_(-bj[0] * m / p->sigma_s, wj[0] * m / p->sigma_s);
            const Cplx z1 = cexp_(-bj[1] * m / p->sigma_s, wj[1] * m / p->sigma_s);
            a.zpc[m] = make_float4((float)z0.r, (float)z0.i, (float)z1.r, (float)z1.i);
            a.zpq[m] = make_float4((float)z0.r, (float)z1.r, (float)z0.i, (float)z1.i);
        }
    }
    int slot = -1;
    if (p->profile) {
        if (p->ev_count == bf_vec_plan_s::kEvRing) collect_profile(p);
        slot = p->ev_head;
        for (int j = 0; j < 2; ++j)
            if (!p->ev[slot][j]) BF_CUDA(cudaEventCreate(&p->ev[slot][j]));
        BF_CUDA(cudaEventRecord(p->ev[slot][0], s));
    }
    auto batch = [&](int i) {   // batch i's arguments: samples [k0 + i nb, ...), scratch set i % sets
        RecTArgs x = a;
        x.k0 = k0 + i * nb;
        x.ns = std::min(nb, k1 - x.k0);
        x.first = (i == 0) ? 1 : 0;
        set_scratch(x, i % sets);
        return x;
    };
    const int nbat = (ns + nb - 1) / nb;
    if (sets == 1) {
        for (int i = 0; i < nbat; ++i) BF_CUDA(launch_recursive_tiled(batch(i), s));
    } else {
        // overlap (option rec_overlap): batch i's scans on the auxiliary stream while batch i + 1's
        // pass 0 runs on s; pass 2 of batch i (which accumulates into the shared partial planes) on s
        // after both. Set (i + 1) % 2 is free when pass 0 of batch i + 1 starts: pass 2 of batch i - 1,
        // its last reader, precedes it on s.
        if (!p->rec_aux || p->rec_aux_prio != p->rec_overlap) {
            if (p->rec_aux) {
                cudaStreamSynchronize(p->rec_aux);
                cudaStreamDestroy(p->rec_aux);
                p->rec_aux = nullptr;
            }
            int lo = 0, hi = 0;
            BF_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            BF_CUDA(cudaStreamCreateWithPriority(&p->rec_aux, cudaStreamNonBlocking, p->rec_overlap == 1 ? hi : lo));
            p->rec_aux_prio = p->rec_overlap;
        }
        for (int j = 0; j < 2; ++j)
            if (!p->rec_ev[j]) BF_CUDA(cudaEventCreateWithFlags(&p->rec_ev[j], cudaEventDisableTiming));
        BF_CUDA(launch_recursive_tiled(batch(0), s, kRecStageP0));
        for (int i = 0; i < nbat; ++i) {
            const RecTArgs x = batch(i);
            BF_CUDA(cudaEventRecord(p->rec_ev[0], s));
            BF_CUDA(cudaStreamWaitEvent(p->rec_aux, p->rec_ev[0], 0));
            BF_CUDA(launch_recursive_tiled(x, p->rec_aux, kRecStageScan));
            BF_CUDA(cudaEventRecord(p->rec_ev[1], p->rec_aux));
            if (i + 1 < nbat) BF_CUDA(launch_recursive_tiled(batch(i + 1), s, kRecStageP0));
            BF_CUDA(cudaStreamWaitEvent(s, p->rec_ev[1], 0));
            BF_CUDA(launch_recursive_tiled(x, s, kRecStageP2));
        }
    }
    if (slot >= 0) {
        BF_CUDA(cudaEventRecord(p->ev[slot][1], s));
        p->ev_head = (p->ev_head + 1) % bf_vec_plan_s::kEvRing;
        p->ev_count += 1;
    }
    p->last_batch = nb;
    p->last_groups = g;
    p->last_tile_rows = kRecT;
    p->last_ctas = tiles * g;
    *groups_out = g;
    return BF_OK;
}

// samples [k0, k1) of the recursive engine into p->dpz (groups = samples per batch)
bf_status_t run_recursive(bf_vec_plan_t p, const float *f, int k0, int k1, cudaStream_t s, int *groups_out) {
    if (p->rec_impl >= 1) return run_recursive_tiled(p, f, k0, k1, s, groups_out);
    const int ns = k1 - k0;
    const size_t px = (size_t)p->H * p->W;
    // per sample in flight: y1 + y2 (2 x 2(d+1) planes) + one partial group ((d+1) planes)
    const double per = 4.0 * px * (4.0 * (p->d + 1) + (p->d + 1));
    int nb = 1;
    bf_status_t st = BF_OK;
    for (int attempt = 0; attempt < 2; ++attempt) {
        const size_t free_b = free_memory(p);
        nb = (int)std::max(1.0, std::min<double>(256.0, 0.4 * (double)free_b / per));
        if (p->force_batch > 0) nb = p->force_batch;
        nb = std::min(nb, ns);
        st = ensure_rec_scratch(p, nb);
        if (st == BF_OK) st = ensure_pz(p, sizeof(float) * (size_t)nb * (p->d + 1) * px);
        // memory taken since the cached query: re-plan the batch against what is free now
        if (st != BF_E_CUDA || attempt == 1 || !refresh_free_memory(p)) break;
    }
    if (st != BF_OK) return st;
    RecArgs a;
    std::memset(&a, 0, sizeof(a));
    fill_mu(p);
    a.f = f;
    a.t = p->dt;
    a.y1 = p->drec;
    a.y2 = p->drec + (size_t)nb * 2 * (p->d + 1) * px;
    a.pz = p->dpz;
    for (int c = 0; c < kMaxD; ++c) a.mu[c] = p->mu[c];
    a.d = p->d;
    a.H = p->H;
    a.W = p->W;
    rec_axis(p->sigma_s, p->W, &a.row);
    rec_axis(p->sigma_s, p->H, &a.col);
    int slot = -1;
    if (p->profile) {
        if (p->ev_count == bf_vec_plan_s::kEvRing) collect_profile(p);
        slot = p->ev_head;
        for (int j = 0; j < 2; ++j)
            if (!p->ev[slot][j]) BF_CUDA(cudaEventCreate(&p->ev[slot][j]));
        BF_CUDA(cudaEventRecord(p->ev[slot][0], s));
    }
    for (int kb = k0; kb < k1; kb += nb) {
        a.k0 = kb;
        a.nb = std::min(nb, k1 - kb);
        a.first = (kb == k0) ? 1 : 0;
        BF_CUDA(launch_recursive(a, s));
    }
    if (slot >= 0) {
        BF_CUDA(cudaEventRecord(p->ev[slot][1], s));
        p->ev_head = (p->ev_head + 1) % bf_vec_plan_s::kEvRing;
        p->ev_count += 1;
    }
    p->last_batch = nb;
    p->last_groups = nb;
    p->last_tile_rows = p->H;
    p->last_ctas = (long long)((p->H + 31) / 32 + (p->W + 31) / 32) * nb;
    *groups_out = nb;
    return BF_OK;
}

// the plan's draw set for key `seed` (iid or stratified, option "sampler")
bf_status_t draw(bf_vec_plan_t p, uint64_t seed, cudaStream_t s) {
    if (p->sampler == 1) {
        if (!p->dkeys) BF_CUDA(cudaMalloc(&p->dkeys, sizeof(uint64_t) * (size_t)p->M * p->d));
        BF_CUDA(launch_sampler_stratified(p->M, p->d, p->N, seed, p->dQ, p->dgamma, p->dkeys, p->dX, p->dt, s));
    } else {
        BF_CUDA(launch_sampler(p->M, p->d, p->N, seed, p->dQ, p->dgamma, p->dX, p->dt, s));
    }
    return BF_OK;
}

bool valid_plan(bf_vec_plan_t p) { return p != nullptr; }

}  // namespace

extern "C" {

const char *bf_vec_status_string(bf_status_t st) {
    switch (st) {
        case BF_OK: return "BF_OK";
        case BF_E_ARG: return "BF_E_ARG: invalid argument";
        case BF_E_NOT_SYMMETRIC: return "BF_E_NOT_SYMMETRIC: covariance not symmetric";
        case BF_E_NOT_POSDEF: return "BF_E_NOT_POSDEF: covariance not positive definite";
        case BF_E_UNSUPPORTED: return "BF_E_UNSUPPORTED: configuration outside the compiled kernel set";
        case BF_E_CUDA: return "BF_E_CUDA: CUDA error or no sm_100 device";
        case BF_E_STATE: return "BF_E_STATE: call order violated";
        case BF_W_ALIAS: return "BF_W_ALIAS: raised cosine leaves its main lobe on the data range";
        case BF_W_SMALL_Z: return "BF_W_SMALL_Z: some pixels have Z/M below z_floor";
    }
    return "unknown status";
}

bf_status_t bf_vec_plan(int H, int W, int d, double sigma_s, const double *C, int N, int M,
                        uint64_t seed, bf_vec_plan_t *out) {
    Nvtx nvtx_("bfvec:plan");
    if (!out || !C) return BF_E_ARG;
    *out = nullptr;
    if (H < 1 || W < 1 || d < 1 || d > kMaxD || M < 1) return BF_E_ARG;
    if (!(sigma_s > 0.0) || !std::isfinite(sigma_s)) return BF_E_ARG;
    if (N < 2 || N > 64 || (N & 1)) return BF_E_ARG;
    const int r = (int)std::ceil(3.0 * sigma_s - 1e-12);   // reading R2
    if (r < 1 || r > kMaxRec) return BF_E_ARG;
    bf_vec_plan_t p = new (std::nothrow) bf_vec_plan_s();
    if (!p) return BF_E_ARG;
    p->H = H; p->W = W; p->d = d; p->N = N; p->M = M; p->r = r;
    p->sigma_s = sigma_s;
    p->seed = seed;
    std::memcpy(p->C, C, sizeof(double) * d * d);
    bf_status_t st = diagonalize(d, C, p->Q, p->alpha);
    if (st != BF_OK) { delete p; return st; }
    make_taps(p);
    // alias warning (reading R14): (pi/2) sqrt(N) < alpha_c R ||q_c||_1
    p->alias = false;
    for (int c = 0; c < d; ++c) {
        double l1 = 0.0;
        for (int rr = 0; rr < d; ++rr) l1 += std::fabs(p->Q[rr * d + c]);
        if (0.5 * M_PI * std::sqrt((double)N) < p->alpha[c] * p->value_range * l1) p->alias = true;
    }
    fill_mu(p);
    *out = p;
    return BF_OK;
}

void bf_vec_plan_destroy(bf_vec_plan_t p) {
    if (!p) return;
    if (p->device >= 0) {
        if (p->last) cudaStreamSynchronize(p->last);
        cudaFree(p->dX); cudaFree(p->dt); cudaFree(p->dQ); cudaFree(p->dgamma);
        cudaFree(p->dpz); cudaFree(p->ddiag); cudaFree(p->dU); cudaFree(p->dfpad);
        cudaFree(p->dhost_in); cudaFree(p->dhost_out); cudaFree(p->drec); cudaFree(p->drtab); cudaFree(p->drun); cudaFree(p->dmse);
        cudaFree(p->dkeys); cudaFree(p->dlab); cudaFree(p->dt_batch); cudaFree(p->dX_batch);
        cudaFree(p->ditems); cudaFree(p->ditem_off); cudaFree(p->dstrip_slots);
        if (p->gexec) cudaGraphExecDestroy(p->gexec);
        if (p->copy_out) cudaStreamSynchronize(p->copy_out);
        if (p->order_ev) {
            cudaEventSynchronize(p->order_ev);
            cudaEventDestroy(p->order_ev);
        }
        for (int i = 0; i < 2; ++i) {
            cudaFree(p->dasync_in[i]); cudaFree(p->dasync_out[i]);
            for (cudaEvent_t e : {p->ev_in[i], p->ev_comp[i], p->ev_out[i]})
                if (e) cudaEventDestroy(e);
        }
        if (p->rec_aux) {
            cudaStreamSynchronize(p->rec_aux);
            cudaStreamDestroy(p->rec_aux);
        }
        for (cudaEvent_t e : p->rec_ev)
            if (e) cudaEventDestroy(e);
        if (p->copy_in) cudaStreamDestroy(p->copy_in);
        if (p->copy_out) cudaStreamDestroy(p->copy_out);
        for (auto &pair : p->ev)
            for (auto &e : pair)
                if (e) cudaEventDestroy(e);
    }
    delete p;
}

bf_status_t bf_vec_sample_freqs(bf_vec_plan_t p, void *stream) {
    Nvtx nvtx_("bfvec:sample");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p)) return BF_E_ARG;
    bf_status_t st = ensure_device(p);
    if (st != BF_OK) return st;
    double gamma[8];
    for (int c = 0; c < p->d; ++c) gamma[c] = p->alpha[c] / std::sqrt((double)p->N);
    BF_CUDA(cudaMemcpy(p->dQ, p->Q, sizeof(double) * p->d * p->d, cudaMemcpyHostToDevice));
    BF_CUDA(cudaMemcpy(p->dgamma, gamma, sizeof(double) * p->d, cudaMemcpyHostToDevice));
    st = draw(p, p->seed, S(stream));
    if (st != BF_OK) return st;
    p->sampled = true;
    p->gen += 1;
    p->last = S(stream);
    return BF_OK;
}

bf_status_t bf_vec_get_draws(bf_vec_plan_t p, int32_t *X, float *t, double *Q, double *alpha) {
    if (!valid_plan(p)) return BF_E_ARG;
    if (Q) std::memcpy(Q, p->Q, sizeof(double) * p->d * p->d);
    if (alpha) std::memcpy(alpha, p->alpha, sizeof(double) * p->d);
    if (X || t) {
        if (!p->sampled) return BF_E_STATE;
        BF_CUDA(cudaStreamSynchronize(p->last));
        if (X) BF_CUDA(cudaMemcpy(X, p->dX, sizeof(int32_t) * (size_t)p->M * p->d, cudaMemcpyDeviceToHost));
        if (t) BF_CUDA(cudaMemcpy(t, p->dt, sizeof(float) * (size_t)p->M * p->d, cudaMemcpyDeviceToHost));
    }
    return BF_OK;
}

static bf_status_t filter_band(bf_vec_plan_t p, const float *slab, int slab_rows, int slab_row0,
                               int row0, int row1, float *out, cudaStream_t s) {
    if (!p->sampled) return BF_E_STATE;
    if (p->lab) {   // RGB -> CIE-Lab, filter in Lab, back to RGB
        bf_status_t st = to_lab(p, slab, slab_rows, &slab, s);
        if (st != BF_OK) return st;
    }
    int groups = 1;
    int D = p->kinfo.D;
    bf_status_t st;
    if (p->engine == 1) {
        // the recursion runs along whole columns: full images only (no band sharding)
        if (row0 != 0 || row1 != p->H || slab_row0 != 0 || slab_rows != p->H) return BF_E_UNSUPPORTED;
        st = run_recursive(p, slab, 0, p->M, s, &groups);
        D = p->d;
    } else {
        st = run_fused(p, slab, slab_rows, slab_row0, row0, row1 - row0, 0, p->M, s, &groups);
    }
    if (st != BF_OK) return st;
    BF_CUDA(launch_diag_reset(p->ddiag, s));
    BF_CUDA(launch_normalize_groups(p->dpz, groups, D, p->d, row1 - row0, p->W, p->mu, out,
                                    p->ddiag, 1.0f / p->M, (float)p->z_floor, s,
                                    p->engine == 1 ? nullptr : p->last_strip_slots));
    if (p->lab) BF_CUDA(launch_lab_to_srgb(out, out, (long long)(row1 - row0) * p->W, s));
    // engine 1 per batch: staged 2 kernels (row, column), tiled 5 (3 tile passes, 2 scans), tiled with
    // virtual lines 4 (2 tile passes, 2 scans)
    // engine 0: pad, fused kernel (variant 8: two launches), diagnostics reset, normalise
    // tensor-core pass 2 on an image with partial tiles: + the FP32 pass 2 for those tiles
    const int tc_split = (p->engine == 1 && p->rec_impl >= 1 && p->rec_tc && p->d <= 7 &&
                          (p->W % kRecT || p->H % kRecT) && p->W >= kRecT && p->H >= kRecT) ? 1 : 0;
    p->last_launches = ((p->engine == 1) ? 2 + ((p->rec_impl == 2 ? 4 : p->rec_impl == 1 ? 5 : 2) + tc_split) *
                                                   ((p->M + p->last_batch - 1) / p->last_batch)
                                         : 4 + (p->kinfo.variant == 8 ? 1 : 0)) + (p->lab ? 2 : 0);
    p->last = s;
    return p->alias ? BF_W_ALIAS : BF_OK;
}

// bf_vec_filter through a CUDA graph: the first call with a given (f, out, stream, options) runs
// eagerly (it allocates scratch and picks the schedule), the second captures the same launch
// sequence (pad, fused kernel, diagnostics reset, normalise) into a graph, and later calls replay it
// with one cudaGraphLaunch -- the host cost of a small image drops to one launch.
bf_status_t filter_graph(bf_vec_plan_t p, const float *f, float *out, cudaStream_t s) {
    const bool same = p->gexec && p->g_f == f && p->g_out == out && p->g_stream == s && p->g_gen == p->gen;
    if (same) {
        int slot = -1;
        if (p->profile) {   // time the whole replay (the fused kernel is > 99.7 % of it on configs 2-5)
            if (p->ev_count == bf_vec_plan_s::kEvRing) collect_profile(p);
            slot = p->ev_head;
            for (int j = 0; j < 2; ++j)
                if (!p->ev[slot][j]) BF_CUDA(cudaEventCreate(&p->ev[slot][j]));
            BF_CUDA(cudaEventRecord(p->ev[slot][0], s));
        }
        BF_CUDA(cudaGraphLaunch(p->gexec, s));
        if (slot >= 0) {
            BF_CUDA(cudaEventRecord(p->ev[slot][1], s));
            p->ev_head = (p->ev_head + 1) % bf_vec_plan_s::kEvRing;
            p->ev_count += 1;
        }
        p->last_launches = p->g_launches;
        p->last = s;
        return p->g_status;
    }
    const bool key_seen = p->g_f == f && p->g_out == out && p->g_stream == s && p->g_gen == p->gen;
    if (!key_seen) {   // first call with this key: eager, remember the key
        if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
        p->g_f = f; p->g_out = out; p->g_stream = s;
        const bf_status_t st = filter_band(p, f, p->H, 0, 0, p->H, out, s);
        p->g_gen = p->gen;   // after the call: its scratch allocations bump gen
        return st;
    }
    // second call: capture (profiling events stay outside the graph)
    const bool prof = p->profile;
    p->profile = false;
    BF_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    const bf_status_t st = filter_band(p, f, p->H, 0, 0, p->H, out, s);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(s, &graph);
    p->profile = prof;
    if (st < 0 || ce != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        cudaGetLastError();
        p->use_graph = false;            // fall back to eager launches for this plan
        return st < 0 ? st : filter_band(p, f, p->H, 0, 0, p->H, out, s);
    }
    const cudaError_t ie = cudaGraphInstantiate(&p->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
        p->gexec = nullptr;
        cudaGetLastError();
        p->use_graph = false;
        return filter_band(p, f, p->H, 0, 0, p->H, out, s);
    }
    p->g_launches = p->last_launches;
    p->g_status = st;
    return filter_graph(p, f, out, s);   // replay now
}

bf_status_t bf_vec_filter(bf_vec_plan_t p, const float *f, float *out, void *stream) {
    Nvtx nvtx_("bfvec:filter");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p) || !f || !out || f == out) return BF_E_ARG;
    if (p->device < 0) return BF_E_STATE;
    cudaStream_t s = S(stream);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    // the legacy default stream cannot be captured; a stream the caller is capturing already
    // records our launches into the caller's graph
    if (p->use_graph && p->sampled && s != nullptr && cudaStreamIsCapturing(s, &cs) == cudaSuccess &&
        cs == cudaStreamCaptureStatusNone)
        return filter_graph(p, f, out, s);
    cudaGetLastError();
    return filter_band(p, f, p->H, 0, 0, p->H, out, s);
}

bf_status_t bf_vec_filter_batch(bf_vec_plan_t p, const float *f, float *out, int nimg, void *stream) {
    Nvtx nvtx_("bfvec:filter_batch");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p) || !f || !out || f == out || nimg < 1) return BF_E_ARG;
    if (p->device < 0 || !p->sampled) return BF_E_STATE;
    if (p->engine != 0 || p->lab) return BF_E_UNSUPPORTED;
    if ((long long)((p->H + 15) / 16) * nimg > 65535) return BF_E_UNSUPPORTED;   // grid.y
    cudaStream_t s = S(stream);
    int groups = 1;
    bf_status_t st = run_fused(p, f, p->H, 0, 0, p->H, 0, p->M, s, &groups, nullptr, nullptr, nimg);
    if (st != BF_OK) return st;
    const size_t img_pz = (size_t)groups * (p->kinfo.D + 1) * p->H * (size_t)p->W;
    BF_CUDA(launch_diag_reset(p->ddiag, s));
    for (int b = 0; b < nimg; ++b)
        BF_CUDA(launch_normalize_groups(p->dpz + b * img_pz, groups, p->kinfo.D, p->d, p->H, p->W, p->mu,
                                        out + (size_t)b * p->d * p->H * p->W, p->ddiag, 1.0f / p->M,
                                        (float)p->z_floor, s));
    p->last_launches = 2 * nimg + 2;
    p->last = s;
    return p->alias ? BF_W_ALIAS : BF_OK;
}

bf_status_t bf_vec_filter_host(bf_vec_plan_t p, const float *f_host, float *out_host, void *stream) {
    Nvtx nvtx_("bfvec:filter_host");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p) || !f_host || !out_host) return BF_E_ARG;
    if (p->device < 0) return BF_E_STATE;
    const size_t bytes = sizeof(float) * (size_t)p->d * p->H * p->W;
    if (p->dhost_bytes < bytes) {
        cudaFree(p->dhost_in); cudaFree(p->dhost_out);
        p->dhost_in = p->dhost_out = nullptr;
        p->dhost_bytes = 0;
        BF_CUDA(cudaMalloc(&p->dhost_in, bytes));
        BF_CUDA(cudaMalloc(&p->dhost_out, bytes));
        p->dhost_bytes = bytes;
    }
    cudaStream_t s = S(stream);
    BF_CUDA(cudaMemcpyAsync(p->dhost_in, f_host, bytes, cudaMemcpyHostToDevice, s));
    bf_status_t st = filter_band(p, p->dhost_in, p->H, 0, 0, p->H, p->dhost_out, s);
    if (st < 0) return st;
    BF_CUDA(cudaMemcpyAsync(out_host, p->dhost_out, bytes, cudaMemcpyDeviceToHost, s));
    BF_CUDA(cudaStreamSynchronize(s));
    return st;
}

// Pipelined frames: H2D of frame i+1 and D2H of frame i-1 run on two copy
// streams while frame i computes on the caller's stream. Device slots alternate by call parity;
// events order every reuse: the H2D into slot s waits for the compute that last read it, the compute
// writing output slot s waits for the D2H that last read it.
bf_status_t bf_vec_filter_host_async(bf_vec_plan_t p, const float *f_host, float *out_host, void *stream) {
    Nvtx nvtx_("bfvec:filter_host_async");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    // f_host == out_host would let this frame's D2H race the next frames' H2D reads
    if (!valid_plan(p) || !f_host || !out_host || f_host == out_host) return BF_E_ARG;
    if (p->device < 0 || !p->sampled) return BF_E_STATE;
    const size_t bytes = sizeof(float) * (size_t)p->d * p->H * p->W;
    if (!p->copy_in) {
        BF_CUDA(cudaStreamCreateWithFlags(&p->copy_in, cudaStreamNonBlocking));
        BF_CUDA(cudaStreamCreateWithFlags(&p->copy_out, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            BF_CUDA(cudaEventCreateWithFlags(&p->ev_in[i], cudaEventDisableTiming));
            BF_CUDA(cudaEventCreateWithFlags(&p->ev_comp[i], cudaEventDisableTiming));
            BF_CUDA(cudaEventCreateWithFlags(&p->ev_out[i], cudaEventDisableTiming));
        }
    }
    if (p->dasync_bytes < bytes) {
        BF_CUDA(cudaStreamSynchronize(p->copy_out));   // no frame in flight uses the old slots
        for (int i = 0; i < 2; ++i) {
            cudaFree(p->dasync_in[i]); cudaFree(p->dasync_out[i]);
            p->dasync_in[i] = p->dasync_out[i] = nullptr;
        }
        p->dasync_bytes = 0;
        for (int i = 0; i < 2; ++i) {
            BF_CUDA(cudaMalloc(&p->dasync_in[i], bytes));
            BF_CUDA(cudaMalloc(&p->dasync_out[i], bytes));
        }
        p->dasync_bytes = bytes;
        p->async_calls = 0;
    }
    cudaStream_t s = S(stream);
    const int slot = (int)(p->async_calls & 1);
    const bool reuse = p->async_calls >= 2;
    if (reuse) BF_CUDA(cudaStreamWaitEvent(p->copy_in, p->ev_comp[slot], 0));   // frame i-2 read the slot
    BF_CUDA(cudaMemcpyAsync(p->dasync_in[slot], f_host, bytes, cudaMemcpyHostToDevice, p->copy_in));
    BF_CUDA(cudaEventRecord(p->ev_in[slot], p->copy_in));
    BF_CUDA(cudaStreamWaitEvent(s, p->ev_in[slot], 0));
    if (reuse) BF_CUDA(cudaStreamWaitEvent(s, p->ev_out[slot], 0));   // frame i-2's output was copied out
    bf_status_t st = filter_band(p, p->dasync_in[slot], p->H, 0, 0, p->H, p->dasync_out[slot], s);
    if (st < 0) return st;
    BF_CUDA(cudaEventRecord(p->ev_comp[slot], s));
    BF_CUDA(cudaStreamWaitEvent(p->copy_out, p->ev_comp[slot], 0));
    BF_CUDA(cudaMemcpyAsync(out_host, p->dasync_out[slot], bytes, cudaMemcpyDeviceToHost, p->copy_out));
    BF_CUDA(cudaEventRecord(p->ev_out[slot], p->copy_out));
    p->async_calls += 1;
    p->last = p->copy_out;
    return st;
}

bf_status_t bf_vec_host_sync(bf_vec_plan_t p) {
    if (!valid_plan(p)) return BF_E_ARG;
    if (p->device < 0) return BF_E_STATE;
    if (p->copy_out) BF_CUDA(cudaStreamSynchronize(p->copy_out));
    return BF_OK;
}

bf_status_t bf_vec_filter_partial(bf_vec_plan_t p, const float *f, int k0, int k1, float *PZ,
                                  int rows_per_band, void *stream) {
    Nvtx nvtx_("bfvec:filter_partial");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p) || !f || !PZ) return BF_E_ARG;
    if (k0 < 0 || k1 > p->M || k0 > k1 || rows_per_band < 1 || rows_per_band > p->H) return BF_E_ARG;
    if (p->device < 0 || !p->sampled) return BF_E_STATE;
    cudaStream_t s = S(stream);
    if (k0 == k1) {
        BF_CUDA(cudaMemsetAsync(PZ, 0, sizeof(float) * (size_t)(p->d + 1) * p->H * p->W, s));
        return BF_OK;
    }
    if (p->lab) {
        bf_status_t st = to_lab(p, f, p->H, &f, s);
        if (st != BF_OK) return st;
    }
    int groups = 1;
    bf_status_t st = (p->engine == 1) ? run_recursive(p, f, k0, k1, s, &groups)
                                      : run_fused(p, f, p->H, 0, 0, p->H, k0, k1, s, &groups);
    if (st != BF_OK) return st;
    BF_CUDA(launch_finalize_partial(p->dpz, groups, p->engine == 1 ? p->d : p->kinfo.D, p->d, p->H, p->W, p->mu,
                                    rows_per_band, PZ, s,
                                    p->engine == 1 ? nullptr : p->last_strip_slots));
    p->last_launches = 3;
    p->last = s;
    return BF_OK;
}

bf_status_t bf_vec_filter_partial_p2p(bf_vec_plan_t p, const float *f, int k0, int k1, float *const *peer_slots,
                                      int world, int rank, int slots_per_rank, void *stream) {
    Nvtx nvtx_("bfvec:filter_partial_p2p");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p) || !f || !peer_slots) return BF_E_ARG;
    if (world < 1 || world > 8 || rank < 0 || rank >= world || slots_per_rank < 1) return BF_E_ARG;
    if (k0 < 0 || k1 > p->M || k1 - k0 < slots_per_rank) return BF_E_ARG;   // every group non-empty
    for (int i = 0; i < world; ++i)
        if (!peer_slots[i]) return BF_E_ARG;
    if (p->device < 0 || !p->sampled) return BF_E_STATE;
    if (p->H % world != 0 || p->engine != 0 || p->lab || !p->kinfo_ok || p->kinfo.variant != 4)
        return BF_E_UNSUPPORTED;
    const P2POut o{peer_slots, world, rank, slots_per_rank};
    int groups = 1;
    bf_status_t st = run_fused(p, f, p->H, 0, 0, p->H, k0, k1, S(stream), &groups, &o);
    if (st != BF_OK) return st;
    p->p2p_world = world;            // the receive-slot layout bf_vec_normalize_slots must match
    p->p2p_slots = slots_per_rank;
    p->last_launches = 2;
    p->last = S(stream);
    return BF_OK;
}

bf_status_t bf_vec_normalize_slots(bf_vec_plan_t p, const float *slots, int nslots, int row0, int row1,
                                   float *out_band, void *stream) {
    Nvtx nvtx_("bfvec:normalize_slots");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p) || !slots || !out_band || nslots < 1) return BF_E_ARG;
    if (row0 < 0 || row1 > p->H || row0 >= row1) return BF_E_ARG;
    if (p->device < 0 || !p->kinfo_ok || p->p2p_world < 1) return BF_E_STATE;
    // the slots hold (D+1, H/world, W) planes of ONE owner's band: anything else would read past
    // the receive buffer or misread its layout
    const int band_rows = p->H / p->p2p_world;
    if (row1 - row0 != band_rows || row0 % band_rows != 0 || nslots > p->p2p_world * p->p2p_slots)
        return BF_E_ARG;
    cudaStream_t s = S(stream);
    fill_mu(p);
    BF_CUDA(launch_diag_reset(p->ddiag, s));
    BF_CUDA(launch_normalize_groups(slots, nslots, p->kinfo.D, p->d, row1 - row0, p->W, p->mu, out_band, p->ddiag,
                                    1.0f / p->M, (float)p->z_floor, s));
    p->last_launches = 2;
    p->last = s;
    return BF_OK;
}

bf_status_t bf_vec_normalize(bf_vec_plan_t p, const float *PZ_band, int row0, int row1, float *out_band,
                             void *stream) {
    Nvtx nvtx_("bfvec:normalize");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p) || !PZ_band || !out_band) return BF_E_ARG;
    if (row0 < 0 || row1 > p->H || row0 >= row1) return BF_E_ARG;
    bf_status_t st = ensure_device(p);
    if (st != BF_OK) return st;
    cudaStream_t s = S(stream);
    BF_CUDA(launch_diag_reset(p->ddiag, s));
    BF_CUDA(launch_normalize_raw(PZ_band, p->d, row1 - row0, p->W, out_band, p->ddiag, 1.0f / p->M,
                                 (float)p->z_floor, s));
    p->last_launches = 2;
    p->last = s;
    return BF_OK;
}

bf_status_t bf_vec_filter_rows(bf_vec_plan_t p, const float *slab, int slab_row0, int slab_rows, int row0,
                               int row1, float *out_band, void *stream) {
    Nvtx nvtx_("bfvec:filter_rows");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p) || !slab || !out_band) return BF_E_ARG;
    if (row0 < 0 || row1 > p->H || row0 >= row1) return BF_E_ARG;
    if (slab_row0 < 0 || slab_rows < 1 || slab_row0 + slab_rows > p->H) return BF_E_ARG;
    if (p->device < 0) return BF_E_STATE;
    // every reflected row within r of the band must be in the slab (rows the
    // compiled radius reads beyond r carry zero taps and are clamped in-kernel)
    for (long long y = (long long)row0 - p->r; y < (long long)row1 + p->r; ++y) {
        const long long n = p->H, q = 2 * n;
        long long i = y % q;
        if (i < 0) i += q;
        const long long yr = i < n ? i : q - 1 - i;
        if (yr < slab_row0 || yr >= slab_row0 + slab_rows) return BF_E_ARG;
    }
    return filter_band(p, slab, slab_rows, slab_row0, row0, row1, out_band, S(stream));
}

bf_status_t bf_vec_direct(bf_vec_plan_t p, const float *f, float *out, void *stream) {
    Nvtx nvtx_("bfvec:direct");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p) || !f || !out || f == out) return BF_E_ARG;
    if (p->r > kMaxR) return BF_E_UNSUPPORTED;
    bf_status_t st = ensure_device(p);
    if (st != BF_OK) return st;
    const size_t bytes = direct_scratch_bytes(p->d, p->H, p->W, p->r);
    if (p->dU_bytes < bytes) {
        cudaFree(p->dU);
        p->dU = nullptr;
        p->dU_bytes = 0;
        BF_CUDA(cudaMalloc(&p->dU, bytes));
        p->dU_bytes = bytes;
    }
    // A = sqrt(log2(e)/2) diag(alpha) Q^T  (Eq. (4)): |A (f_j - f_i)|^2 = log2(e) x^T C^-1 x / 2
    float A[64];
    const double sc = std::sqrt(0.5 / std::log(2.0));
    for (int k = 0; k < p->d; ++k)
        for (int c = 0; c < p->d; ++c) A[k * p->d + c] = (float)(sc * p->alpha[k] * p->Q[c * p->d + k]);
    cudaStream_t s = S(stream);
    if (p->lab) {
        st = to_lab(p, f, p->H, &f, s);
        if (st != BF_OK) return st;
    }
    fill_mu(p);
    // rows per CTA: 16 (measured fastest from 512^2 up, profiles/r02_direct_rows_sweep.txt) unless
    // the image has fewer 16-row tiles than SMs; option "direct_rows" forces it
    int ty = p->force_direct_rows;
    if (ty <= 0) {
        const long long ntx = (p->W + 16 * (p->d <= 4 ? 4 : 2) - 1) / (16 * (p->d <= 4 ? 4 : 2));
        ty = 16;
        while (ty > 4 && ntx * ((p->H + ty - 1) / ty) < sm_count()) ty /= 2;
    }
    BF_CUDA(launch_direct(f, p->d, p->H, p->W, p->r, p->taps, A, p->mu, p->dU, out, ty, s));
    if (p->lab) BF_CUDA(launch_lab_to_srgb(out, out, (long long)p->H * p->W, s));
    p->last_launches = 2;
    p->last = s;
    return BF_OK;
}

bf_status_t bf_vec_mse_sweep(bf_vec_plan_t p, const float *f, const float *ref, int n_seeds, const uint64_t *seeds,
                             int n_t, const int *t_list, double *mse, void *stream) {
    Nvtx nvtx_("bfvec:mse_sweep");
    StreamOrder order_(valid_plan(p) ? p : nullptr, S(stream));
    if (!valid_plan(p) || !f || !ref || !seeds || !t_list || !mse || n_seeds < 1 || n_t < 1) return BF_E_ARG;
    for (int j = 0; j < n_t; ++j)
        if (t_list[j] < 1 || t_list[j] > p->M || (j > 0 && t_list[j] <= t_list[j - 1])) return BF_E_ARG;
    if (p->device < 0 || !p->sampled) return BF_E_STATE;
    if (p->lab) return BF_E_UNSUPPORTED;
    cudaStream_t s = S(stream);
    const long long npix = (long long)p->H * p->W;
    const size_t run_bytes = sizeof(float) * (size_t)(p->d + 1) * npix;
    if (p->drun_bytes < run_bytes) {
        cudaFree(p->drun);
        p->drun = nullptr;
        p->drun_bytes = 0;
        BF_CUDA(cudaMalloc(&p->drun, run_bytes));
        p->drun_bytes = run_bytes;
    }
    if (p->dmse_n < n_t) {
        cudaFree(p->dmse);
        p->dmse = nullptr;
        p->dmse_n = 0;
        BF_CUDA(cudaMalloc(&p->dmse, sizeof(double) * n_t));
        p->dmse_n = n_t;
    }
    bf_status_t st = BF_OK;
    if (p->engine == 0) {
        // realisations batched through the fused kernel's group dimension: per checkpoint ONE fused
        // launch filters the new samples of every realisation of the batch, and one kernel folds
        // them into each realisation's running sums and reduces its squared error
        const int D = p->kinfo.D;
        const double per = 4.0 * npix * ((D + 1) + (p->d + 1));
        int RB = (int)std::max(1.0, std::min<double>(256.0, 0.25 * (double)free_memory(p) / per));
        RB = std::min(RB, n_seeds);
        const size_t tn = (size_t)RB * p->M * p->d;
        if (p->dt_batch_n < tn) {
            cudaFree(p->dt_batch); cudaFree(p->dX_batch);
            p->dt_batch = nullptr; p->dX_batch = nullptr; p->dt_batch_n = 0;
            BF_CUDA(cudaMalloc(&p->dt_batch, sizeof(float) * tn));
            BF_CUDA(cudaMalloc(&p->dX_batch, sizeof(int32_t) * tn));
            p->dt_batch_n = tn;
        }
        const size_t rb_bytes = sizeof(float) * (size_t)RB * (p->d + 1) * npix;
        if (p->drun_bytes < rb_bytes) {
            cudaFree(p->drun);
            p->drun = nullptr; p->drun_bytes = 0;
            BF_CUDA(cudaMalloc(&p->drun, rb_bytes));
            p->drun_bytes = rb_bytes;
        }
        if (p->dmse_n < RB * n_t) {
            cudaFree(p->dmse);
            p->dmse = nullptr; p->dmse_n = 0;
            BF_CUDA(cudaMalloc(&p->dmse, sizeof(double) * RB * n_t));
            p->dmse_n = RB * n_t;
        }
        std::vector<double> host((size_t)RB * n_t);
        for (int r0 = 0; r0 < n_seeds && st == BF_OK; r0 += RB) {
            const int nr = std::min(RB, n_seeds - r0);
            for (int r = 0; r < nr; ++r) {
                const size_t off = (size_t)r * p->M * p->d;
                if (p->sampler == 1) {
                    if (!p->dkeys) BF_CUDA(cudaMalloc(&p->dkeys, sizeof(uint64_t) * (size_t)p->M * p->d));
                    BF_CUDA(launch_sampler_stratified(p->M, p->d, p->N, seeds[r0 + r], p->dQ, p->dgamma, p->dkeys,
                                                      p->dX_batch + off, p->dt_batch + off, s));
                } else {
                    BF_CUDA(launch_sampler(p->M, p->d, p->N, seeds[r0 + r], p->dQ, p->dgamma, p->dX_batch + off,
                                           p->dt_batch + off, s));
                }
            }
            BF_CUDA(cudaMemsetAsync(p->dmse, 0, sizeof(double) * nr * n_t, s));
            int k0 = 0;
            for (int j = 0; j < n_t && st == BF_OK; ++j) {
                const RealBatch rbatch{p->dt_batch, nr, p->M};
                int groups = 1;
                st = run_fused(p, f, p->H, 0, 0, p->H, k0, t_list[j], s, &groups, nullptr, &rbatch);
                if (st != BF_OK) break;
                BF_CUDA(launch_mse_accum_batch(p->dpz, nr, D, p->d, npix, p->mu, p->drun, j == 0 ? 1 : 0, ref,
                                               p->dmse + (size_t)j * nr, s));
                k0 = t_list[j];
            }
            if (st != BF_OK) break;
            BF_CUDA(cudaMemcpyAsync(host.data(), p->dmse, sizeof(double) * nr * n_t, cudaMemcpyDeviceToHost, s));
            BF_CUDA(cudaStreamSynchronize(s));
            for (int r = 0; r < nr; ++r)
                for (int j = 0; j < n_t; ++j)
                    mse[(size_t)(r0 + r) * n_t + j] = host[(size_t)j * nr + r] / ((double)p->d * (double)npix);
        }
        p->last = s;
        p->last_launches = 0;
        return st;
    }
    for (int r = 0; r < n_seeds && st == BF_OK; ++r) {
        // realisation r: the same generator keyed by seeds[r] (reading R9)
        st = draw(p, seeds[r], s);
        if (st != BF_OK) break;
        BF_CUDA(cudaMemsetAsync(p->dmse, 0, sizeof(double) * n_t, s));
        int k0 = 0;
        for (int j = 0; j < n_t && st == BF_OK; ++j) {
            int groups = 1;
            st = (p->engine == 1) ? run_recursive(p, f, k0, t_list[j], s, &groups)
                                  : run_fused(p, f, p->H, 0, 0, p->H, k0, t_list[j], s, &groups);
            if (st != BF_OK) break;
            BF_CUDA(launch_mse_accum(p->dpz, groups, p->engine == 1 ? p->d : p->kinfo.D, p->d, npix, p->mu, p->drun,
                                     j == 0 ? 1 : 0, ref, p->dmse + j, s));
            k0 = t_list[j];
        }
        if (st != BF_OK) break;
        BF_CUDA(cudaMemcpyAsync(mse + (size_t)r * n_t, p->dmse, sizeof(double) * n_t, cudaMemcpyDeviceToHost, s));
        BF_CUDA(cudaStreamSynchronize(s));
        for (int j = 0; j < n_t; ++j) mse[(size_t)r * n_t + j] /= (double)p->d * (double)npix;   // Eq. (20)
    }
    // restore the plan's own draws
    const bf_status_t st2 = draw(p, p->seed, s);
    p->last = s;
    p->last_launches = 0;
    if (st == BF_OK) st = st2;
    return st;
}

bf_status_t bf_vec_srgb_to_lab(const float *rgb, float *lab, long long npix, void *stream) {
    if (!rgb || !lab || npix < 0) return BF_E_ARG;
    BF_CUDA(launch_srgb_to_lab(rgb, lab, npix, S(stream)));
    return BF_OK;
}

bf_status_t bf_vec_lab_to_srgb(const float *lab, float *rgb, long long npix, void *stream) {
    if (!rgb || !lab || npix < 0) return BF_E_ARG;
    BF_CUDA(launch_lab_to_srgb(lab, rgb, npix, S(stream)));
    return BF_OK;
}

bf_status_t bf_vec_diag(bf_vec_plan_t p, float *z_min, long long *n_small_z) {
    if (!valid_plan(p)) return BF_E_ARG;
    if (p->device < 0) return BF_E_STATE;
    BF_CUDA(cudaStreamSynchronize(p->last));
    unsigned long long h[2];
    BF_CUDA(cudaMemcpy(h, p->ddiag, 16, cudaMemcpyDeviceToHost));
    const unsigned int key = (unsigned int)(h[0] & 0xFFFFFFFFull);
    unsigned int u = (key & 0x80000000u) ? (key & 0x7FFFFFFFu) : ~key;
    float zm;
    std::memcpy(&zm, &u, 4);
    if (key == 0xFFFFFFFFu) zm = NAN;
    if (z_min) *z_min = zm;
    if (n_small_z) *n_small_z = (long long)h[1];
    return h[1] ? BF_W_SMALL_Z : BF_OK;
}

bf_status_t bf_vec_set_option(bf_vec_plan_t p, const char *name, double v) {
    if (!valid_plan(p) || !name) return BF_E_ARG;
    if (std::strcmp(name, "profile") != 0) p->gen += 1;   // options may change the captured launches
    if (!std::strcmp(name, "graph")) {
        if (v != 0.0 && v != 1.0) return BF_E_ARG;
        p->use_graph = v != 0.0;
        return BF_OK;
    }
    if (!std::strcmp(name, "z_floor")) { p->z_floor = v; return BF_OK; }
    if (!std::strcmp(name, "value_range")) {
        if (!(v > 0) || !std::isfinite(v)) return BF_E_ARG;
        p->value_range = v;
        fill_mu(p);
        p->alias = false;
        for (int c = 0; c < p->d; ++c) {
            double l1 = 0.0;
            for (int rr = 0; rr < p->d; ++rr) l1 += std::fabs(p->Q[rr * p->d + c]);
            if (0.5 * M_PI * std::sqrt((double)p->N) < p->alpha[c] * v * l1) p->alias = true;
        }
        return BF_OK;
    }
    if (!std::strcmp(name, "tile_rows")) { if (v < 0) return BF_E_ARG; p->force_tile_rows = (int)v; return BF_OK; }
    if (!std::strcmp(name, "direct_rows")) {
        if (v != 0.0 && v != 4.0 && v != 8.0 && v != 16.0) return BF_E_ARG;
        p->force_direct_rows = (int)v;
        return BF_OK;
    }
    if (!std::strcmp(name, "groups")) { if (v < 0) return BF_E_ARG; p->force_groups = (int)v; return BF_OK; }
    if (!std::strcmp(name, "variant")) {
        if (v < 0 || v > 8) return BF_E_ARG;
        p->force_variant = (int)v;
        if (p->device >= 0) {   // re-select the kernel instance
            if (!select_kernel(p)) return BF_E_UNSUPPORTED;
            p->kinfo_ok = true;
        }
        return BF_OK;
    }
    if (!std::strcmp(name, "engine")) {
        if (v != 0.0 && v != 1.0) return BF_E_ARG;
        p->engine = (int)v;
        return BF_OK;
    }
    if (!std::strcmp(name, "colorspace")) {
        if ((v != 0.0 && v != 1.0) || (v == 1.0 && p->d != 3)) return BF_E_ARG;
        p->lab = (int)v;
        fill_mu(p);
        return BF_OK;
    }
    if (!std::strcmp(name, "sampler")) {
        if (v != 0.0 && v != 1.0) return BF_E_ARG;
        p->sampler = (int)v;   // takes effect at the next bf_vec_sample_freqs
        return BF_OK;
    }
    if (!std::strcmp(name, "rec_overlap")) {   // A/B: batch k + 1's pass 0 beside batch k's scans
        if (v != 0.0 && v != 1.0 && v != 2.0) return BF_E_ARG;
        p->rec_overlap = (int)v;
        return BF_OK;
    }
    if (!std::strcmp(name, "rec_vtc")) {   // A/B: the column scan's virtual-line blurs on the tensor cores
        if (v != 0.0 && v != 1.0) return BF_E_ARG;
        p->rec_vtc = (int)v;
        return BF_OK;
    }
    if (!std::strcmp(name, "rec_tc")) {
        if (v != 0.0 && v != 1.0) return BF_E_ARG;
        p->rec_tc = (int)v;
        return BF_OK;
    }
    if (!std::strcmp(name, "rec_impl")) {
        if (v != 0.0 && v != 1.0 && v != 2.0) return BF_E_ARG;
        p->rec_impl = (int)v;
        return BF_OK;
    }
    if (!std::strcmp(name, "persistent")) {
        if (v != 0.0 && v != 1.0 && v != 2.0) return BF_E_ARG;
        p->persistent = (int)v;
        return BF_OK;
    }
    if (!std::strcmp(name, "rec_store")) {
        if (v != 0.0 && v != 1.0) return BF_E_ARG;
        p->rec_store = (int)v;
        return BF_OK;
    }
    if (!std::strcmp(name, "rec_batch")) { if (v < 0) return BF_E_ARG; p->force_batch = (int)v; return BF_OK; }
    if (!std::strcmp(name, "spatial_kernel")) {
        if (v != 0.0 && v != 1.0 && v != 2.0) return BF_E_ARG;
        p->spatial = (int)v;
        make_taps(p);
        if (p->device >= 0) p->kinfo_ok = select_kernel(p);   // box: running-sum instance
        return BF_OK;
    }
    if (!std::strcmp(name, "profile")) {
        collect_profile(p);
        p->profile = v != 0.0;
        p->fused_ms_total = 0.0;
        p->fused_calls = 0;
        return BF_OK;
    }
    return BF_E_ARG;
}

bf_status_t bf_vec_plan_info(bf_vec_plan_t p, const char *name, long long *value) {
    if (!valid_plan(p) || !name || !value) return BF_E_ARG;
    const KernelInfo &k = p->kinfo;
    if (!std::strcmp(name, "fused_ns_total") || !std::strcmp(name, "fused_calls")) {
        collect_profile(p);
        *value = !std::strcmp(name, "fused_calls") ? p->fused_calls : (long long)(p->fused_ms_total * 1e6);
        return BF_OK;
    }
    struct { const char *n; long long v; } tab[] = {
        {"radius", p->r}, {"d", p->d}, {"H", p->H}, {"W", p->W}, {"M", p->M}, {"N", p->N},
        {"tile_rows", p->last_tile_rows}, {"groups", p->last_groups}, {"ctas", p->last_ctas},
        {"launches_per_filter", p->last_launches}, {"smem_bytes", (long long)k.smem},
        {"threads", k.threads}, {"kernel_D", k.D}, {"kernel_R", k.R}, {"regs", k.regs},
        {"occupancy", k.occupancy}, {"alias", p->alias ? 1 : 0}, {"variant", k.variant},
        {"spatial_kernel", p->spatial}, {"graph", p->use_graph ? 1 : 0}, {"graph_ready", p->gexec ? 1 : 0}, {"engine", p->engine}, {"rec_batch", p->last_batch}, {"rec_impl", p->rec_impl}, {"rec_tc", p->rec_tc}, {"rec_vtc", p->rec_vtc}, {"rec_overlap", p->rec_overlap}, {"rec_store", p->rec_store}, {"persistent", p->persistent}, {"last_persistent", p->last_persistent}, {"sampler", p->sampler}, {"colorspace", p->lab},
        {"fir_supported", p->r <= kMaxR ? 1 : 0},
    };
    for (auto &e : tab)
        if (!std::strcmp(e.n, name)) { *value = e.v; return BF_OK; }
    return BF_E_ARG;
}

bf_status_t bf_vec_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]) {
    if (!ctr || !key || !out) return BF_E_ARG;
    philox4x64_10_host(ctr, key, out);
    return BF_OK;
}

}  // extern "C"

// Test hook (not part of include/bfvec.h): the persistent schedule's item table for a given shape,
// so the CPU tests can check that every strip's work line is covered exactly once and its slots are
// distinct (tests/host/test_persistent_items.py). items: 4 ints per item; off: nC + 1 ints; nslot:
// nx ints. Returns the item count, or -1 if `cap` items do not fit.
extern "C" int bfvec_test_persistent_items(int nx, int nf, int P, int nC, int Gc, double fill, int *items, int cap,
                                           int *off, int *nslot, double *t_pers) {
    if (nx < 1 || nf < 1 || P < 1 || nC < 1 || Gc < 1 || Gc > P) return -1;
    std::vector<std::vector<int4>> mine;
    std::vector<int> ns;
    const double t = persistent_items(nx, nf, P, nC, Gc, fill, mine, ns);
    int n = 0;
    for (int c = 0; c < nC; ++c) {
        off[c] = n;
        for (const int4 &it : mine[c]) {
            if (n >= cap) return -1;
            items[4 * n + 0] = it.x;
            items[4 * n + 1] = it.y;
            items[4 * n + 2] = it.z;
            items[4 * n + 3] = it.w;
            ++n;
        }
    }
    off[nC] = n;
    for (int x = 0; x < nx; ++x) nslot[x] = ns[x];
    if (t_pers) *t_pers = t;
    return n;
}
