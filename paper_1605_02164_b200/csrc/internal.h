// internal.h -- private declarations of libbfvec (not part of the C ABI).
// Nothing here is shared with oracle/: the two implementations are independent.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bfvec.h"

namespace bfvec {

constexpr int kMaxD = 8;
constexpr int kMaxR = 64;          // largest FIR radius (truncated-window engine)
constexpr int kMaxRec = 1 << 20;   // largest r = ceil(3 sigma_s) the plan accepts (recursive engine)
constexpr int kTX = 32;            // output columns per strip (one warp of lanes)

// Arguments of the fused MCSF kernel (one launch = one output band, one sample range).
// Passed by value as a __grid_constant__ parameter, so the taps w[] become
// constant-bank / uniform-register operands of the FFMA2s and the tensor map is
// addressable by the TMA unit.
struct alignas(64) FusedArgs {
    CUtensorMap tmap;     // 3-D map over the padded copy: dims {DP, Wp, Hp}, box {DP, WIN, SH}
    int d;                // image channels (<= compiled D; channels d..D-1 are zero)
    int W;                // image width
    int out_row0;         // first output row (image coordinates); pad row 0 = out_row0 - R
    int out_rows;         // number of output rows
    int tile_rows;        // rows per CTA tile (multiple of the kernel's KB)
    int groups;           // sample groups (grid.z)
    int k0, k1;           // sample range
    int gstride;          // 0, or realisation batching: group g filters t rows [g*gstride + k0, g*gstride + k1)
    // image batching (bf_vec_filter_batch): blockIdx.y = image * tiles_per_img + tile; image i's padded
    // rows start at i * img_prows in the tensor map and its partial planes at pz + i * img_pz
    int tiles_per_img, img_prows;
    long long img_pz;
    const float *t;       // (M, d) frequency table, fp32
    float *pz;            // (groups, D+1, out_rows, W): planes 0..D-1 = P' (centred), D = Z
    float w[kMaxR + 1];   // normalised taps w[|m|], zero beyond the plan radius
    // peer-slot output (bf_vec_filter_partial_p2p; v6 kernel only): when p2p_world > 0 the LAST
    // pass of every sample group stores its tile rows straight into the receive slots of the rank
    // that owns each row band: peer[owner] + ((p2p_rank * groups + g) * (D+1) + plane) * p2p_rpb * W
    // + (row - owner * p2p_rpb) * W + x, over NVLink while other CTAs are still computing.
    float *peer[8];
    int p2p_world, p2p_rank, p2p_rpb;
    // persistent schedule (v6 kernel only; null = one (strip, tile, group) per CTA): CTA c runs the
    // items [item_off[c], item_off[c+1]); item = {strip, u_begin, u_end, slot}
    // over the strip's work line u = pass * nch_full + chunk (full-height passes of SP samples,
    // chunks of KB rows), so every CTA gets the same number of chunk-steps
    const int4 *items;
    const int *item_off;
    int nch_full;
};

struct PadMu {
    float v[kMaxD];       // centring offsets (exact invariance S[f-mu]+mu = S[f], reading R12)
};

struct KernelInfo {
    int D, R;             // compiled vector dim and radius (taps beyond r are zero)
    int threads;
    int kb;               // output rows per chunk
    int sh;               // rows per TMA box
    int dp;               // floats per padded pixel
    int win;              // haloed columns per box (32 + 2R)
    size_t smem;
    int regs;
    int occupancy;        // CTAs per SM (from the occupancy API)
    int variant;          // 1: shared-memory ring (v3), 2: tensor-memory ring (v4), 3: v4 with two consumer
                          // warps per pair, 4: v4 with two samples per pass (v5)
    int sp = 1;           // samples per pass over a strip
};

// Kernel-set dispatch (mcsf_fused.cu). Returns false if no instance fits.
bool fused_select(int d, int r, int variant, KernelInfo *info);
cudaError_t fused_launch(const KernelInfo &info, const FusedArgs &a, dim3 grid, cudaStream_t s);

// Reflect-padded, centred, interleaved copy of the input for the TMA loads (pad.cu)
cudaError_t launch_pad(const float *f, long long plane, int d, int H, int W, int slab_row0, int slab_rows,
                       int row_begin, int Hp, int Wp, int R, int DP, const float *mu, float *fpad,
                       cudaStream_t s);

// Sampler (sampler.cu)
cudaError_t launch_sampler(int M, int d, int N, uint64_t seed, const double *dQ,
                           const double *dgamma, int32_t *dX, float *dt, cudaStream_t s);
void philox4x64_10_host(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]);
struct CumTable {
    uint64_t v[65];   // cum(n) = sum_{m <= n} C(N, m) for n < N (all-ones beyond)
};
cudaError_t launch_sampler_stratified(int M, int d, int N, uint64_t seed, const double *dQ, const double *dgamma,
                                      uint64_t *dkeys, int32_t *dX, float *dt, cudaStream_t s);

// Epilogues (normalize.cu)
cudaError_t launch_normalize_groups(const float *pz, int groups, int D, int d, int rows, int W,
                                    const float *mu, float *out, float *diag, float inv_m,
                                    float z_floor, cudaStream_t s, const int *strip_slots = nullptr);
// strip_slots (persistent schedule): slots written per 32-column strip; null = `groups` everywhere
cudaError_t launch_finalize_partial(const float *pz, int groups, int D, int d, int rows, int W,
                                    const float *mu, int rows_per_band, float *PZ, cudaStream_t s,
                                    const int *strip_slots = nullptr);
cudaError_t launch_normalize_raw(const float *PZ, int d, int rows, int W, float *out, float *diag,
                                 float inv_m, float z_floor, cudaStream_t s);
cudaError_t launch_diag_reset(float *diag, cudaStream_t s);

// Recursive engine (recursive.cu; option "engine" = 1, reading R16).
// One axis of the separable recursive Gaussian: two complex poles z_j, residues A_j (normalised
// so the kernel sums to 1), g0 = g(0), z_j^n and 1 / (1 - z_j^2n) for the reflected-periodic
// initial state of a line of length n, and the number of head / tail terms summed for it.
struct RecAxis {
    float zr[2], zi[2];
    float ar[2], ai[2];
    float g0;
    float znr[2], zni[2];
    float invr[2], invi[2];
    int lh;
};
struct RecArgs {
    const float *f;       // (d, H, W) input
    const float *t;       // (M, d) frequency table
    float *y1, *y2;       // (nb, 2(d+1), H, W) scratch: row-pass output, column forward partial
    float *pz;            // (nb, d+1, H, W): planes 0..d-1 = P' (centred), d = Z; group b <- sample k0 + b
    float mu[kMaxD];      // centring (reading R12)
    int d, H, W;
    int k0, nb;           // samples [k0, k0 + nb) of this batch
    int first;            // 1: store into pz, 0: accumulate
    RecAxis row, col;
};
cudaError_t launch_recursive(const RecArgs &a, cudaStream_t s);

// Tiled recursive engine (recursive_tiled.cu, option "rec_impl" = 1): 32 x 32
// tiles, exact tile-boundary states of every line from per-tile summaries and a scan, so the
// blurred planes never leave the SM. kRecT = tile edge; per axis of nt tiles the plan keeps the
// pole powers z_j^{L_t}, z_j^{x0_t}, z_j^{n - x0_t - L_t} (fp64-computed, stored fp32 complex).
constexpr int kRecT = 32;
constexpr int kRecTcB = 64 * 40;   // tensor-core pass 2: [hi; lo] x (32 Toeplitz + 8 state-basis) columns
struct RecTabs {
    const float2 *zl;     // [2][nt]
    const float2 *pf;     // [2][nt]
    const float2 *pb;     // [2][nt]
    const float4 *zp;     // [kRecT]: (z_0^m, z_1^m), m = 0 .. kRecT-1
};
struct RecTArgs {
    const float *f;       // (d, H, W) input
    const float *t;       // (M, d) frequency table
    float *pz;            // (g3, d+1, H, W) partial groups
    float mu[kMaxD];
    int d, H, W, ntx, nty;
    int k0, ns;           // samples [k0, k0 + ns) of this batch (batch-local index s = k - k0)
    int g1, g3;           // sample groups of the summary passes / of the accumulation pass
    int first;
    RecAxis row, col;
    float2 *Eh, *Bh;      // (ns, 2(d+1), 2, ntx, H): row tiles' causal end / anticausal start states
    float2 *Ev, *Bv;      // (ns, 2(d+1), 2, nty, W): the same for the column tiles
    float4 *UVh, *UVv;    // (ns, 2(d+1), 2, nlh) / (.., W): line states (u_{-1}, v_n)
    int nlh;              // lines of the row arrays: H (rec_impl 1), H + 8 nty (rec_impl 2: + virtual lines)
    float *vl;            // rec_impl 2: (ns, 2(d+1), nty, 8, W) virtual-line values (column summaries
                          // of the modulated planes, real / imaginary parts), or null (rec_impl 1)
    float *rbg;           // (ns, 2(d+1), H, W) row-blurred planes written by pass 1 and read by pass 2
                          // (option "rec_store" = 1), or null: pass 2 recomputes the row blur
    RecTabs th, tv;
    float4 zpc[kRecT];    // (z_0^m, z_1^m), m < kRecT, in the parameter space: full tiles' summaries take
                          // them as uniform constant operands (no per-element shared-memory loads)
    const float *tcb;     // rec_tc: the tile-blur matrix [K | state basis] (32 x 40, hi / lo tf32 halves) in the
                          // tensor cores' K-major canonical layout, kRecTcB floats (plan.cu, rec_tc_matrix)
    int tc;               // rec_tc: pass 2 of full tiles on the tensor cores (d <= 7), partial tiles on the FP32 path
    int vtc;              // rec_tc, rec_impl 2: the virtual lines' segment blurs on the tensor cores too
    float4 zpq[kRecT];    // the same regrouped (Re z_0^m, Re z_1^m, Im z_0^m, Im z_1^m): both poles of one
                          // real line in one FFMA2 (rec_impl 2's virtual-line summaries)
};
constexpr int kRecStageP0 = 1, kRecStageScan = 2, kRecStageP2 = 4, kRecStageAll = 7;
cudaError_t launch_recursive_tiled(const RecTArgs &a, cudaStream_t s, int stages = kRecStageAll);

// Error-vs-T sweep (sweep.cu): fold partial groups into running (P', Z), S = P'/Z + mu,
// accumulate sum (ref - S)^2 into *out (double).
struct MuArg {
    float v[kMaxD];
};
cudaError_t launch_mse_accum(const float *pz, int groups, int D, int d, long long npix, const float *mu,
                             float *run, int first, const float *ref, double *out, cudaStream_t s);
// realisation-batched: group r of pz is realisation r; run holds nr (d+1)-plane running sums;
// out[r] += sum (ref - S_r)^2
cudaError_t launch_mse_accum_batch(const float *pz, int nr, int D, int d, long long npix, const float *mu,
                                   float *run, int first, const float *ref, double *out, cudaStream_t s);

// sRGB <-> CIE-Lab (color.cu; reading R18), planar (3, npix), in place allowed
cudaError_t launch_srgb_to_lab(const float *in, float *out, long long npix, cudaStream_t s);
cudaError_t launch_lab_to_srgb(const float *in, float *out, long long npix, cudaStream_t s);

// Direct filter (direct.cu)
// scratch UF: direct_scratch_bytes(d, H, W, r) (2d reflect-padded planes: U = A f, then f)
size_t direct_scratch_bytes(int d, int H, int W, int r);
cudaError_t launch_direct(const float *f, int d, int H, int W, int r, const float *w,
                          const float *A /* d x d: diag(alpha) Q^T scaled */,
                          const float *mu /* d: centring (reading R12) */, float *UF,
                          float *out, int rows_per_cta /* 4, 8, 16 */, cudaStream_t s);

}  // namespace bfvec

struct bf_vec_plan_s {
    int H, W, d, N, M, r;
    double sigma_s;
    uint64_t seed;
    double C[64];
    double Q[64];         // row-major, columns are eigenvectors q_k
    double alpha[8];
    float taps[bfvec::kMaxR + 1];
    bool alias;           // static alias warning (BF_W_ALIAS)
    // options
    double z_floor = 0.05;
    double value_range = 255.0;
    int force_tile_rows = 0;
    int force_groups = 0;
    int force_direct_rows = 0; // exact filter: output rows per CTA (0 auto, 4, 8, 16)
    int persistent = 1;        // v6 kernel: 0 (strip, tile, group) grid, 1 auto, 2 force the persistent schedule
    // cached persistent schedule: key, device item table, slots (groups) it needs
    long long pers_key[5] = {-1, -1, -1, -1, -1};
    int4 *ditems = nullptr;
    int *ditem_off = nullptr;
    int *dstrip_slots = nullptr;      // slots written per strip (the normaliser sums only those)
    size_t dstrip_cap = 0;
    const int *last_strip_slots = nullptr;   // of the last fused launch (null: classic grid)
    size_t ditems_cap = 0, ditem_off_cap = 0;
    int pers_groups = 0, pers_items = 0, pers_ctas = 0, last_persistent = 0;
    int rec_store = 0;         // tiled recursive engine: 1 = pass 1 stores the row blur for pass 2 (measured
                               // 2 % slower on config 5: pass 2 is not bound by the recomputed row blur)
    int force_variant = 0;     // 0 auto, 1 v3 (smem ring), 2 v4 (TMEM ring)
    int spatial = 0;           // spatial taps: 0 Gaussian (Eq. (1)), 1 box, 2 hat (reading R15)
    int engine = 0;            // 0 truncated FIR (Eq. (1) window), 1 recursive Deriche (reading R16)
    int force_batch = 0;       // recursive engine: samples per batch (0 = auto)
    float *drec = nullptr;     // recursive engine scratch (y1, y2; tiled: summaries)
    int rec_impl = 2;          // recursive engine: 0 staged (row / column passes via HBM), 1 tiled, 2 tiled + virtual lines
    int rec_tc = 1;            // tiled engine: 1 = pass 2's tile blurs (d <= 7) as block-Toeplitz GEMMs on the tensor cores
    int rec_vtc = 1;           // with rec_tc: the column scan's virtual-line segment blurs on the tensor cores too
    int rec_overlap = 0;       // tiled engine, > 1 batch: batch k + 1's pass 0 (FP32 pipe) runs beside batch k's
                               // scans (HBM) on a second stream, two scratch sets; 1 = that stream at high
                               // priority, 2 = at default priority
    cudaStream_t rec_aux = nullptr;
    int rec_aux_prio = 0;      // the rec_overlap mode rec_aux was created for
    cudaEvent_t rec_ev[2] = {nullptr, nullptr};   // fork (main -> aux), join (aux -> main)
    float2 *drtab = nullptr;   // tiled recursive engine: pole-power tables of both axes
    size_t drtab_n = 0;
    int sampler = 0;           // 0 iid binomial draws (reading R9), 1 stratified (reading R17)
    int lab = 0;               // 1: filter in CIE-Lab (sRGB in/out, reading R18)
    float *dlab = nullptr;     // Lab copy of the input
    size_t dlab_bytes = 0;
    uint64_t *dkeys = nullptr; // stratified sampler: permutation keys (M d)
    float *dt_batch = nullptr; // error sweep: frequency tables of a batch of realisations
    int32_t *dX_batch = nullptr;
    size_t dt_batch_n = 0;
    float *drun = nullptr;     // error sweep: running (P', Z) planes and per-checkpoint sums
    double *dmse = nullptr;
    size_t drun_bytes = 0;
    int dmse_n = 0;
    size_t drec_bytes = 0;
    int last_batch = 0;
    size_t free_mem = 0;       // free device memory at the first launch (0 = not queried yet)
    int p2p_world = 0, p2p_slots = 0;   // layout of the last bf_vec_filter_partial_p2p (normalize_slots checks it)
    // CUDA-graph replay of bf_vec_filter (option "graph"): the launch sequence of a call is
    // captured on the second call with the same (f, out, stream, option generation) and replayed
    bool use_graph = true;
    int gen = 0;               // bumped by every option change (kernel arguments may differ)
    cudaGraphExec_t gexec = nullptr;
    const float *g_f = nullptr;
    float *g_out = nullptr;
    cudaStream_t g_stream = nullptr;
    int g_gen = -1, g_seen = 0, g_launches = 0;
    bf_status_t g_status = BF_OK;
    // device state (lazily created)
    int device = -1;
    bool sampled = false;
    bfvec::KernelInfo kinfo{};
    bool kinfo_ok = false;
    int32_t *dX = nullptr;
    float *dt = nullptr;
    double *dQ = nullptr, *dgamma = nullptr;
    float *dpz = nullptr;
    size_t pz_bytes = 0;
    float *ddiag = nullptr;     // [0] z_min (ordered-int encoded), [1] count
    float *dfpad = nullptr;     // padded input copy (pad.cu), TMA source
    size_t fpad_bytes = 0;
    float *dU = nullptr;        // direct-filter scratch
    size_t dU_bytes = 0;
    float *dhost_in = nullptr, *dhost_out = nullptr;
    size_t dhost_bytes = 0;
    // bf_vec_filter_host_async: two device slots per direction, copy streams and their events
    float *dasync_in[2] = {nullptr, nullptr}, *dasync_out[2] = {nullptr, nullptr};
    size_t dasync_bytes = 0;
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
    long long async_calls = 0;
    float mu[8];
    cudaStream_t last = nullptr;
    // cross-stream ordering of the plan's shared scratch (StreamOrder in plan.cu): the event
    // recorded after the last call and the stream it was recorded on
    cudaEvent_t order_ev = nullptr;
    cudaStream_t order_stream = nullptr;
    bool order_recorded = false;
    // last schedule
    int last_tile_rows = 0, last_groups = 0;
    long long last_ctas = 0;
    int last_launches = 0;
    // optional event timing of the fused kernel (option "profile")
    bool profile = false;
    static constexpr int kEvRing = 256;
    cudaEvent_t ev[kEvRing][2] = {};
    int ev_head = 0, ev_count = 0;   // pending event pairs (not yet folded into the total)
    double fused_ms_total = 0.0;
    long long fused_calls = 0;
};
