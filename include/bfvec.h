/*
 * bfvec.h -- C ABI of libbfvec.so: the Monte Carlo Shiftable Filter (MCSF) of
 * arXiv 1605.02164 ("Fast bilateral filtering of vector-valued images") on
 * NVIDIA B200 (sm_100a).
 *
 * The filter (Algorithm 1): given a vector-valued image
 * f : Omega -> R^d, a spatial Gaussian omega with window
 * [-3 sigma_s, 3 sigma_s]^2 (Eq. (1)) and a range Gaussian
 * phi(x) = exp(-x^T C^-1 x / 2), the range kernel is replaced by a product of
 * raised cosines of order N (Eq. (9)) and sampled with M
 * binomial frequency vectors (Eq. (13)-(14)). The output is
 *     S(i) = P(i) / Z(i),
 *     Z(i) = sum_k Re[ conj(H_k(i)) (omega * H_k)(i) ],
 *     P(i) = sum_k Re[ conj(H_k(i)) (omega * (H_k f))(i) ],
 *     H_k(i) = exp(iota t_k . f(i)),  t_k = Q (Y_k o alpha / sqrt(N)),
 * with Y_k = N - 2 X_k, X_k ~ B(N, 1/2)^d (Eq. (15)-(19), PAPER.md:172-202;
 * readings R4, R6, R7 of DESIGN.md).
 *
 * Conventions shared by every entry point:
 *  - Images are DEVICE pointers to planar float32 (d, rows, W): channel-major,
 *    row-major within a channel, no padding, 4-byte aligned. The caller owns
 *    them. C is a HOST pointer to a d x d row-major double matrix.
 *  - Boundary: half-sample symmetric reflection (reading R1).
 *  - All filter calls are stream-ordered and asynchronous on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream). Launch
 *    failures are reported as BF_E_CUDA by the call that launched.
 *  - A plan owns its device scratch (frequency table, partial sums,
 *    diagnostics). Calls on one plan are ordered on the device even across
 *    streams: a call on a stream other than the previous call's waits for the
 *    previous call's work (an event recorded per call; skipped while the
 *    caller captures the stream into its own graph, which then orders it).
 *    Host-side, one plan must not be called from two threads at once.
 *  - Outputs may start at any 4-byte-aligned address (vector stores are used
 *    only when a row start is 16-byte aligned).
 *  - No exceptions cross the ABI; every function returns a bf_status_t
 *    (< 0 error, 0 ok, > 0 warning). On error no output is written.
 *  - There is no CPU fallback: if no sm_100 device is present the calls that
 *    launch kernels return BF_E_CUDA.
 */
#ifndef BFVEC_H
#define BFVEC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bf_vec_plan_s *bf_vec_plan_t;   /* opaque, owned by the library */

typedef enum {
    BF_OK = 0,
    BF_E_ARG = -1,            /* invalid argument (sizes, pointers, ranges)           */
    BF_E_NOT_SYMMETRIC = -2,  /* C not symmetric within 1e-12 relative   */
    BF_E_NOT_POSDEF = -3,     /* an eigenvalue of C <= 1e-12 * max eigenvalue          */
    BF_E_UNSUPPORTED = -4,    /* configuration outside the compiled kernel set         */
    BF_E_CUDA = -5,           /* CUDA runtime / launch error                           */
    BF_E_STATE = -6,          /* call order violated (e.g. filter before sample_freqs) */
    BF_W_ALIAS = 1,           /* raised cosine leaves its main lobe on the data range  */
    BF_W_SMALL_Z = 2          /* some pixel has Z/M < z_floor (output still written)   */
} bf_status_t;

/*
 * bf_vec_plan -- Algorithm 1 setup, L210-214.
 *   H, W      image height and width, >= 1
 *   d         vector dimension, 1 <= d <= 8
 *   sigma_s   spatial std-dev (pixels) > 0; window radius r = ceil(3 sigma_s). The
 *             truncated-window (FIR) engine and bf_vec_direct need r <= 64 (else they return
 *             BF_E_UNSUPPORTED); the recursive engine (option "engine" = 1) accepts any
 *             r <= 2^20
 *   C         host, d x d row-major symmetric positive-definite covariance (Eq. (1))
 *   N         raised-cosine order, even, 2 <= N <= 64 (Eq. (9))
 *   M         number of Monte Carlo samples (the paper's T), M >= 1
 *   seed      Philox4x64-10 key (reading R9)
 *   out       receives the plan handle
 * Diagonalises C in fp64 (cyclic Jacobi; canonical order and signs of
 * reading R8), builds the normalised fp32 taps (reading R3), picks the
 * kernel instance, and allocates device scratch on the current device.
 * Errors: BF_E_ARG, BF_E_NOT_SYMMETRIC, BF_E_NOT_POSDEF, BF_E_UNSUPPORTED, BF_E_CUDA.
 */
bf_status_t bf_vec_plan(int H, int W, int d, double sigma_s, const double *C, int N, int M,
                        uint64_t seed, bf_vec_plan_t *out);

/* Frees the plan and its device scratch (synchronises the plan's last stream). */
void bf_vec_plan_destroy(bf_vec_plan_t plan);

/*
 * bf_vec_sample_freqs -- Alg. 1 L221 hoisted (Prop. 2):
 * one device kernel draws X_kc = popcount(philox_word(k*d+c) & (2^N-1)),
 * Y = N - 2X, and the fp32 frequency table t_k = Q (Y_k o alpha / sqrt(N))
 * (computed in fp64, rounded once) into plan scratch. Must be called once
 * before any filter call. Asynchronous on `stream`.
 */
bf_status_t bf_vec_sample_freqs(bf_vec_plan_t plan, void *stream);

/*
 * bf_vec_get_draws -- synchronous host copies for checking against the oracle.
 *   X      (M, d) int32 binomial draws, or NULL
 *   t      (M, d) float32 frequency table, or NULL
 *   Q      (d, d) double row-major eigenbasis (columns q_k), or NULL
 *   alpha  (d) double, or NULL
 * Errors: BF_E_STATE if bf_vec_sample_freqs was never called (X, t).
 */
bf_status_t bf_vec_get_draws(bf_vec_plan_t plan, int32_t *X, float *t, double *Q, double *alpha);

/*
 * bf_vec_filter -- the whole hot path for all M samples: S = P / Z
 * (Alg. 1). f, out: device planar (d, H, W) float32; out may not
 * alias f. Returns BF_OK or BF_W_ALIAS (data leaves the raised cosine's main
 * lobe; output still written). BF_W_SMALL_Z is reported by bf_vec_diag.
 * BF_E_UNSUPPORTED when the FIR engine has no kernel for (d, r): r = ceil(3 sigma_s) > 64, or
 * 5 <= d <= 8 with r > 24 (the nine (cos, sin) pairs' rings exceed shared memory / TMEM there);
 * the recursive engine (option "engine" = 1) covers every (d, sigma_s).
 */
bf_status_t bf_vec_filter(bf_vec_plan_t plan, const float *f, float *out, void *stream);

/*
 * bf_vec_filter_batch -- bf_vec_filter for nimg images of the plan's size in ONE fused launch
 * (the images are independent units): the grid covers every image's strips, so small
 * images fill the GPU. Every image uses the plan's draws (as nimg bf_vec_filter calls would).
 *   f, out   device planar (nimg, d, H, W) float32, contiguous; out may not alias f
 * FIR engine only and no colorspace (else BF_E_UNSUPPORTED); BF_W_ALIAS as bf_vec_filter;
 * bf_vec_diag reports the small-Z statistics over all images.
 */
bf_status_t bf_vec_filter_batch(bf_vec_plan_t plan, const float *f, float *out, int nimg, void *stream);

/*
 * bf_vec_filter_host -- bf_vec_filter on HOST buffers: copies f (d,H,W) to the
 * device, filters, copies out back, and synchronises `stream`. Pinned host
 * memory gives full PCIe bandwidth; pageable memory works but is slower.
 */
bf_status_t bf_vec_filter_host(bf_vec_plan_t plan, const float *f_host, float *out_host,
                               void *stream);

/*
 * bf_vec_filter_host_async -- bf_vec_filter_host for a stream of frames: enqueues the H2D copy of
 * f_host (on a plan-owned copy stream), the filter (on `stream`, after the copy) and the D2H copy
 * into out_host (on a second copy stream, after the filter) and returns without waiting, so frame
 * i+1's input copy and frame i-1's output copy overlap frame i's kernels. Results are bitwise those
 * of bf_vec_filter_host. The plan alternates two device slots per direction; reusing a slot waits
 * (on the device) for the frame that used it two calls earlier.
 *   f_host, out_host  host (d, H, W) fp32; pinned (cudaHostAlloc / torch pin_memory) for the copies
 *                     to be asynchronous. The caller must keep f_host unchanged and out_host alive
 *                     until bf_vec_host_sync returns (or alternate host buffers per frame);
 *                     f_host and out_host must not be the same buffer (BF_E_ARG).
 * Errors: BF_E_STATE before bf_vec_sample_freqs; BF_E_CUDA.
 */
bf_status_t bf_vec_filter_host_async(bf_vec_plan_t plan, const float *f_host, float *out_host, void *stream);

/*
 * bf_vec_host_sync -- wait until every bf_vec_filter_host_async frame enqueued on this plan has been
 * copied back to its out_host buffer.
 */
bf_status_t bf_vec_host_sync(bf_vec_plan_t plan);

/*
 * bf_vec_filter_partial -- raw sums over samples k in [k0, k1) only
 * (0 <= k0 <= k1 <= M), for sample sharding (one NCCL sum afterwards).
 *   PZ         device float32, (d+1) planes per row band: for band b covering
 *              rows [b*rows_per_band, min(H, (b+1)*rows_per_band)) the block
 *              (d+1, band_rows, W) is stored contiguously, bands in order.
 *              Planes 0..d-1 hold P_c, plane d holds Z (raw, uncentred, no 1/M).
 *   rows_per_band  1..H (H gives the plain (d+1, H, W) layout)
 */
bf_status_t bf_vec_filter_partial(bf_vec_plan_t plan, const float *f, int k0, int k1, float *PZ,
                                  int rows_per_band, void *stream);

/*
 * bf_vec_filter_partial_p2p -- sample sharding with the exchange fused into the MC kernel: this
 * rank (of `world`, one process per GPU) filters samples [k0, k1) in `slots_per_rank` sample
 * groups, and the LAST pass of every group stores its finished partial tile rows directly into
 * the receive slots of the rank owning each row band (peer memory over NVLink), while other CTAs
 * are still computing -- the reduce-scatter of bf_vec_filter_partial + NCCL without a separate
 * collective. After every rank's call has completed (e.g. a barrier on the stream), each owner
 * sums and normalises its slots with bf_vec_normalize_slots.
 *   peer_slots      host array of `world` device pointers: rank b's receive buffer of
 *                   world * slots_per_rank slots, slot (r * slots_per_rank + g) holding
 *                   (D+1, H/world, W) fp32 planes (D = bf_vec_plan_info "kernel_D"; P' centred,
 *                   Z last), written for band b = rows [b H/world, (b+1) H/world)
 *   slots_per_rank  >= 1 and <= k1 - k0 (every group gets a sample)
 * Requires H % world == 0, the default FIR engine on the v6 kernel (d <= 3, 10 < r <= 48), no
 * colorspace (else BF_E_UNSUPPORTED). The caller maps peers' buffers (CUDA IPC).
 * Reuse: a receive buffer may only be written again once its owner's bf_vec_normalize_slots of
 * the previous call has completed. Frame-by-frame callers alternate two buffers (call n writes
 * set n % 2) with a stream sync + barrier between the stores and the normalise of each call; a
 * rank then cannot reach call n+2 before every owner finished normalising call n
 * (paper_1605_02164_b200/shard.py P2PSlots).
 */
bf_status_t bf_vec_filter_partial_p2p(bf_vec_plan_t plan, const float *f, int k0, int k1,
                                      float *const *peer_slots, int world, int rank,
                                      int slots_per_rank, void *stream);

/*
 * bf_vec_normalize_slots -- Alg. 1 L231 on a receive buffer of bf_vec_filter_partial_p2p:
 * out_c = (sum_s P'_c,s) / (sum_s Z_s) + mu_c for rows [row0, row1) (the owner's band), summing
 * the nslots slots in order (deterministic). slots: device (nslots, D+1, row1-row0, W).
 * The band must be the owner's band of the last bf_vec_filter_partial_p2p on this plan:
 * row1 - row0 == H/world, row0 a multiple of H/world, nslots <= world * slots_per_rank, else
 * BF_E_ARG; BF_E_STATE before any bf_vec_filter_partial_p2p.
 */
bf_status_t bf_vec_normalize_slots(bf_vec_plan_t plan, const float *slots, int nslots, int row0,
                                   int row1, float *out_band, void *stream);

/*
 * bf_vec_normalize -- Alg. 1: out_c = P_c / Z for rows [row0, row1).
 *   PZ_band   device (d+1, row1-row0, W) block as written by filter_partial
 *             (and summed over shards)
 *   out_band  device (d, row1-row0, W)
 * Updates the plan's diagnostics (z_min, small-Z count; see bf_vec_diag).
 */
bf_status_t bf_vec_normalize(bf_vec_plan_t plan, const float *PZ_band, int row0, int row1,
                             float *out_band, void *stream);

/*
 * bf_vec_filter_rows -- band sharding without communication: output rows
 * [row0, row1) of the full H x W image from an input slab holding image rows
 * [slab_row0, slab_row0 + slab_rows). The slab must contain every reflected
 * row within r of the band (else BF_E_ARG).
 *   slab      device (d, slab_rows, W)
 *   out_band  device (d, row1-row0, W)
 */
bf_status_t bf_vec_filter_rows(bf_vec_plan_t plan, const float *slab, int slab_row0,
                               int slab_rows, int row0, int row1, float *out_band, void *stream);

/*
 * bf_vec_direct -- the exact bilateral filter Eq. (2)-(3) on the
 * same window and boundary, O(r^2) per pixel; the accuracy reference for PSNR.
 * f, out: device planar (d, H, W) float32.
 */
bf_status_t bf_vec_direct(bf_vec_plan_t plan, const float *f, float *out, void *stream);

/*
 * bf_vec_mse_sweep -- the error-vs-T experiment of PAPER.md:271-282 (Fig. 5) on the device:
 * for each realisation r (the sampler keyed by seeds[r] instead of the plan seed, reading R9)
 * and each checkpoint T_j of t_list, the MC filter over the first T_j samples is compared with
 * a reference image and
 *     mse[r * n_t + j] = 1/(d |Omega|) sum_c sum_i (ref_c(i) - S_c(i))^2        (Eq. (20))
 * is written (host, double). Samples are shared between checkpoints (T_j extends T_{j-1}).
 *   f, ref     device planar (d, H, W) float32 (ref: usually bf_vec_direct's output)
 *   seeds      host, n_seeds keys;  t_list  host, n_t strictly increasing values in [1, M]
 *   mse        host, n_seeds x n_t doubles
 * Synchronous on `stream`; the plan's own draws are left as they were. Uses the plan's engine,
 * spatial kernel and sampler options. With the FIR engine the realisations are batched through
 * the fused kernel's sample-group dimension (group g = realisation g; as many per batch as 25 %
 * of the free device memory allows, at most 256): per checkpoint one fused launch and one
 * reduction kernel serve the whole batch. Errors: BF_E_ARG, BF_E_STATE (sample_freqs
 * not called), BF_E_UNSUPPORTED, BF_E_CUDA.
 */
bf_status_t bf_vec_mse_sweep(bf_vec_plan_t plan, const float *f, const float *ref, int n_seeds,
                             const uint64_t *seeds, int n_t, const int *t_list, double *mse,
                             void *stream);

/*
 * bf_vec_srgb_to_lab / bf_vec_lab_to_srgb -- the colour transforms around Lab-space filtering
 * ("we first performed a color transformation from the RGB to the CIE-Lab
 * space, performed the filtering in the CIE-Lab space, and then transformed back to the RGB
 * space"). Reading R18: sRGB transfer of IEC 61966-2-1 on values in [0, 255], RGB -> XYZ from
 * the sRGB primaries and the D65 white, CIE 1976 L*a*b* (L* in [0, 100]). No clipping.
 *   rgb, lab   device planar (3, npix) float32; in == out is allowed (per-pixel in place)
 * Asynchronous on `stream`. Errors: BF_E_ARG (NULL pointer, npix < 0), BF_E_CUDA.
 */
bf_status_t bf_vec_srgb_to_lab(const float *rgb, float *lab, long long npix, void *stream);
bf_status_t bf_vec_lab_to_srgb(const float *lab, float *rgb, long long npix, void *stream);

/*
 * bf_vec_diag -- synchronises the plan's last stream and returns diagnostics of
 * the most recent filter/normalize call: z_min = min over pixels of Z/M and
 * n_small_z = #pixels with Z/M < z_floor (default 0.05). Returns BF_W_SMALL_Z
 * when n_small_z > 0.
 */
bf_status_t bf_vec_diag(bf_vec_plan_t plan, float *z_min, long long *n_small_z);

/*
 * bf_vec_set_option -- tuning / policy knobs (all optional):
 *   "z_floor"     threshold of the small-Z diagnostic (default 0.05)
 *   "value_range" nominal data range R used for the alias warning (default 255)
 *   "tile_rows"   force the row-tile height of the fused kernel (0 = auto)
 *   "groups"      force the number of sample groups (0 = auto)
 *   "persistent"  v6 kernel (variants 4, 7): 1 (default) auto -- a persistent schedule (one CTA per
 *                 SM, each an equal share of the (strip, pass, chunk) work line, possibly starting
 *                 and ending mid-pass) when the cost model says it beats the (strip, tile, group)
 *                 grid by > 0.5 % (CTA counts that are not a whole number of waves: config 2 +10 %,
 *                 config 5 +1 %) and
 *                 no "tile_rows" / "groups" is forced; 0 never; 2 always (where the work allows)
 *   "direct_rows" bf_vec_direct: output rows per CTA, 4, 8 or 16 (0 = auto: 16 unless the
 *                 image has fewer 16-row tiles than SMs)
 *   "variant"     fused-kernel variant: 0 auto (d <= 3: 4 where compiled, else 2, else 1;
 *                 5 <= d <= 8: 8),
 *                 1 shared-memory ring (v3), 2 tensor-memory ring (v4, d <= 3), 3 v4 with two
 *                 consumer warps per (cos, sin) pair (d <= 3, r in (30, 48]), 4 v6: tensor-
 *                 memory double ring, two samples per pass, two consumer warps per pair,
 *                 four dedicated modulation warps (d <= 3, r <= 48 where an instance fits), 5
 *                 v5 with one consumer warp per pair, 6 v5c (v6 without the modulation warps)
 *                 (both d = 3, r in (30, 48]), 7 v6 with running-sum FIRs for box taps (d = 3,
 *                 spatial_kernel = 1, r equal to a compiled radius; chosen automatically for box
 *                 taps), 8 tensor-memory ring for 5 <= d <= 8 (two launches per call: pairs
 *                 {Z, P0..P6} two per TMEM quarter, then P7 for four samples at once; r <= 24); a variant
 *                 not compiled for the plan falls back to the default order
 *   "engine"      how Alg. 1 step 10 convolves: 0 (default) the truncated
 *                 separable window [-r, r] of Eq. (1) / "spatial_kernel", O(r) per pixel-sample
 *                 (fused sm_100a kernel); 1 the recursive O(1)-in-sigma_s engine of PAPER.md:204
 *                 (Deriche 1993): spatial kernel g(m) = h(|m|) / sum h of Deriche's 4th-order
 *                 recursive Gaussian over the reflected-periodic image (reading R16,
 *                 §11). Engine 1 filters whole images only (bf_vec_filter, _host, _partial;
 *                 bf_vec_filter_rows returns BF_E_UNSUPPORTED for a proper band) and ignores
 *                 "spatial_kernel", "variant", "tile_rows" and "groups".
 *   "colorspace"  0 (default): filter the values given; 1 (d = 3 only): f is sRGB in [0, 255]
 *                 and bf_vec_filter / _host / _rows / bf_vec_direct convert it to CIE-Lab, filter
 *                 in Lab (C and "value_range" in Lab units; centring mu = (50, 0, 0)) and convert
 *                 the result back (reading R18). bf_vec_filter_partial returns
 *                 Lab-space sums (convert after bf_vec_normalize); bf_vec_mse_sweep returns
 *                 BF_E_UNSUPPORTED.
 *   "sampler"     frequency draws of the next bf_vec_sample_freqs / bf_vec_mse_sweep:
 *                 0 (default) iid X ~ B(N, 1/2) by popcount (reading R9); 1 stratified: per
 *                 dimension a Latin-hypercube stratification of the binomial CDF over the M
 *                 samples (each stratum [j/M, (j+1)/M) used once, random order; DESIGN.md
 *                 reading R17; the paper's "improving the Monte Carlo integration",
 *                 PAPER.md:313). Same estimator Eq. (14); X still B(N, 1/2)-distributed.
 *   "rec_impl"    engine 1: 2 (default) tiled with virtual lines -- 32 x 32 tiles, the exact
 *                 states entering each tile from per-tile summaries and a scan along every
 *                 line; the column summaries of the row-blurred planes come from the row blur
 *                 of 8 "virtual lines" per tile row (the column summaries of the modulated
 *                 planes; linearity), so only pass 2 blurs whole tiles, and the blurred planes
 *                 stay in shared memory; 1 tiled -- as 2 but pass 1 row-blurs
 *                 every tile to form the column summaries; 0 staged -- a row pass and a column
 *                 pass through HBM scratch. Same arithmetic, results equal to fp32 rounding
 *                 (all three gated against the oracle).
 *   "rec_tc"      engine 1, tiled, d <= 7: 1 (default) pass 2 blurs every full 32 x 32 tile on the
 *                 tensor cores -- the exact blur of a segment from its entering states is one
 *                 product [x | states] x [K | state basis] (K = the Deriche kernel's 32 x 32
 *                 Toeplitz block), run as tcgen05.mma kind::tf32 with operands split into tf32
 *                 hi + lo halves (three products, fp32 accuracy), ceil(2(d+1)/4) M = 128 halves
 *                 of four planes; partial tiles and d = 8 use the FP32 recursion. 0: FP32
 *                 recursion everywhere. Results equal to fp32 rounding.
 *   "rec_vtc"     with rec_tc = 1, rec_impl 2 and W a multiple of 32 (any d): 1 (default) the
 *                 column scan's virtual-line segment blurs run as the same tensor-core product.
 *   "rec_overlap" engine 1, tiled, more than one batch: 1 batch k + 1's pass 0 (FP32 pipe) runs on
 *                 the call's stream while batch k's scans (HBM) run on a plan-owned auxiliary
 *                 stream at high priority, forked from and joined back into the call's stream
 *                 (graph-capturable); two scratch sets in flight instead of one. 2: the same with
 *                 the auxiliary stream at default priority. 0: one stream. Output bitwise equal
 *                 in every mode (the same kernels on the same inputs).
 *   "rec_store"   engine 1, rec_impl 1 (ignored by 2): 1 pass 1 stores its exact row blur (2(d+1) fp32 planes per
 *                 sample in flight) and pass 2 reads it instead of recomputing it; 0 (default)
 *                 recompute (measured 2 % faster on config 5)
 *   "rec_batch"   engine 1: samples per batch (0 = auto: at most 256 and 40 % of the free
 *                 device memory, and for the tiled engine at most max(48 samples, 4 GiB of
 *                 summaries); each sample in flight holds, staged, 5 (d+1) fp32 planes of H x W
 *                 scratch, tiled, 16 (d+1) fp32 values per 32 pixels of each axis' lines)
 *   "spatial_kernel" separable spatial taps on the window [-r, r], r = ceil(3 sigma_s):
 *                 0 Gaussian of Eq. (1) (default), 1 box w(m) = 1, 2 hat w(m) = r + 1 - |m|
 *                 ("any arbitrary spatial filter (such as a box or hat filter)";
 *                 DESIGN.md reading R15); taps are normalised to sum 1. Applies to the MC
 *                 filter and to bf_vec_direct.
 *   "graph"       1 (default): bf_vec_filter on a non-default stream captures its launch sequence
 *                 into a CUDA graph on the second call with the same (f, out, stream) and
 *                 options, and replays it afterwards (one cudaGraphLaunch per call); any option
 *                 change or bf_vec_sample_freqs re-captures. 0: always launch eagerly.
 *   "profile"     1: record CUDA events around every fused-kernel launch on the
 *                 launching stream (read back with bf_vec_plan_info
 *                 "fused_ns_total" / "fused_calls"); 0: off. Setting it resets the totals.
 * Errors: BF_E_ARG on an unknown name or invalid value.
 */
bf_status_t bf_vec_set_option(bf_vec_plan_t plan, const char *name, double value);

/*
 * bf_vec_plan_info -- integers describing the plan (for tooling and tests):
 *   "radius", "d", "H", "W", "M", "N", "tile_rows", "groups", "ctas",
 *   "launches_per_filter", "smem_bytes", "threads", "kernel_D", "kernel_R",
 *   "regs", "occupancy", "alias", "variant", "spatial_kernel", "engine", "rec_batch" (last batch
 *   size), "rec_impl", "rec_tc", "rec_vtc", "fir_supported" (r <= 64), "sampler", "colorspace", "graph", "graph_ready", and (option "profile") "fused_ns_total",
 *   "fused_calls" (synchronises on the recorded events). Returns BF_E_ARG for
 *   an unknown name.
 */
bf_status_t bf_vec_plan_info(bf_vec_plan_t plan, const char *name, long long *value);

/*
 * bf_vec_philox4x64_10 -- host-side evaluation of the Philox4x64-10 block function
 * the device sampler uses (Salmon et al., SC'11; reading R9): out = philox(ctr, key).
 * Needs no GPU; lets the generator be checked against published known answers.
 */
bf_status_t bf_vec_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4]);

/* Human-readable name of a status code (static storage). */
const char *bf_vec_status_string(bf_status_t status);

#ifdef __cplusplus
}
#endif

#endif /* BFVEC_H */
