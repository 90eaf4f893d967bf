// mcsf_inst_d3.cu -- fused-kernel instances for D = 3 (one translation unit per D so
// the large fully-expanded FIR bodies compile in parallel).
//   v3 (shared-memory ring, mcsf_fused.cuh): Cfg<D, R, NA, KB, SH> (NA = producer threads)
//   v4 (tensor-memory ring, mcsf_tmem.cuh):  CfgT<D, R, 16>
#include "mcsf_fused.cuh"
#include "mcsf_tmem.cuh"
#include "mcsf_tmem2.cuh"

namespace bfvec {

// The default build compiles only the instances the default selection can pick (build
// weight): v3 for 48 < r <= 64, v4 for r <= 2 and r = 4 (no v6 instance as tight), v6 elsewhere.
// -DBFVEC_COMPARISON_VARIANTS adds the comparison instances (v3 / v4 at every radius, variants 3,
// 5, 6); forcing a variant that is not compiled falls back to the nearest compiled instance of it
// (a padded radius: taps beyond r are zero) or the default order.
#ifdef BFVEC_COMPARISON_VARIANTS
#define BFV_INSTANCES(X) X(3, 2, 128, 16, 16) X(3, 4, 128, 16, 16) X(3, 6, 128, 16, 16) X(3, 10, 128, 16, 16) X(3, 15, 128, 16, 16) X(3, 24, 256, 16, 16) X(3, 30, 256, 16, 16) X(3, 48, 256, 16, 16) X(3, 64, 64, 8, 8)
#define BFV_TMEM_INSTANCES(X) X(3, 2) X(3, 4) X(3, 6) X(3, 10) X(3, 15) X(3, 24) X(3, 30) X(3, 48)
#else
#define BFV_INSTANCES(X) X(3, 64, 64, 8, 8)
#define BFV_TMEM_INSTANCES(X) X(3, 2) X(3, 4)
#endif
#define BFV_TMEM2_INSTANCES(X) X(3, 3) X(3, 6) X(3, 10) X(3, 15) X(3, 24) X(3, 30) X(3, 48)

// variant: 0 auto (v5 where compiled, else v4, else v3), 1 force v3, 2 force v4, 3 v4 with two
// consumer warps per pair (R = 48), 4 force v5 (two samples per pass, two consumer
// warps per pair), 5 v5 with one consumer warp per pair (R = 48)
bool fused_select_d3(int r, int variant, KernelInfo *info) {
    int best = 1 << 30, bestT = 1 << 30;
#define BFV_PICK(D_, R_, NA_, KB_, SH_) \
    if (R_ >= r && R_ < best) best = R_;
    BFV_INSTANCES(BFV_PICK)
#undef BFV_PICK
#define BFV_PICKT(D_, R_) \
    if (R_ >= r && R_ < bestT) bestT = R_;
    BFV_TMEM_INSTANCES(BFV_PICKT)
#undef BFV_PICKT
    const bool use_t = bestT != (1 << 30) && variant != 1 && (variant == 2 || bestT <= best);
    if (variant == 4 || variant == 0) {   // two samples per pass (mcsf_tmem2.cuh), default where compiled
        int best2 = 1 << 30;
#define BFV_PICK2(D_, R_) \
    if (R_ >= r && R_ < best2) best2 = R_;
        BFV_TMEM2_INSTANCES(BFV_PICK2)
#undef BFV_PICK2
        if (best2 != (1 << 30) && (variant == 4 || best2 <= bestT)) {
#define BFV_FILL2(D_, R_) \
    if (R_ == best2) fill_info_tmem2<CfgT2<D_, R_, 2, 4>>(info);
            BFV_TMEM2_INSTANCES(BFV_FILL2)
#undef BFV_FILL2
            info->variant = 4;
            return true;
        }
    }
    if (variant == 7) {   // box taps with the window exactly R: running-sum FIRs (option spatial_kernel = 1)
#define BFV_FILLB(D_, R_) \
    if (R_ == r) { fill_info_tmem2<CfgT2<D_, R_, 2, 4, true>>(info); info->variant = 7; return true; }
        BFV_TMEM2_INSTANCES(BFV_FILLB)
#undef BFV_FILLB
    }
#ifdef BFVEC_COMPARISON_VARIANTS
    if (variant == 6 && bestT == 48) {   // v5c: modulation by the producer warps (comparison instance)
        fill_info_tmem2<CfgT2<3, 48, 2, 0>>(info);
        info->variant = 6;
        return true;
    }
    if (variant == 5 && bestT == 48) {   // v5 with one consumer warp per pair (comparison instance)
        fill_info_tmem2<CfgT2<3, 48, 1>>(info);
        info->variant = 5;
        return true;
    }
    if (variant == 3 && bestT == 48) {   // two consumer warps per pair (comparison instance)
        fill_info_tmem<CfgT<3, 48, 16, 2>>(info);
        info->variant = 3;
        return true;
    }
#endif
    if (use_t) {
#define BFV_FILLT(D_, R_) \
    if (R_ == bestT) fill_info_tmem<CfgT<D_, R_, 16>>(info);
        BFV_TMEM_INSTANCES(BFV_FILLT)
#undef BFV_FILLT
        info->variant = 2;
        return true;
    }
    if (best == (1 << 30)) return false;
#define BFV_FILL(D_, R_, NA_, KB_, SH_) \
    if (R_ == best) fill_info<Cfg<D_, R_, NA_, KB_, SH_>>(info);
    BFV_INSTANCES(BFV_FILL)
#undef BFV_FILL
    info->variant = 1;
    return true;
}

cudaError_t fused_launch_d3(const KernelInfo &info, const FusedArgs &a, dim3 grid, cudaStream_t s) {
#ifdef BFVEC_COMPARISON_VARIANTS
    if (info.variant == 3) return launch_tmem<CfgT<3, 48, 16, 2>>(a, grid, s);
    if (info.variant == 5) return launch_tmem2<CfgT2<3, 48, 1>>(a, grid, s);
    if (info.variant == 6) return launch_tmem2<CfgT2<3, 48, 2, 0>>(a, grid, s);
#endif
    if (info.variant == 7) {
#define BFV_LAUNCHB(D_, R_) \
    if (info.R == R_) return launch_tmem2<CfgT2<D_, R_, 2, 4, true>>(a, grid, s);
        BFV_TMEM2_INSTANCES(BFV_LAUNCHB)
#undef BFV_LAUNCHB
        return cudaErrorInvalidValue;
    }
    if (info.variant == 4) {
#define BFV_LAUNCH2(D_, R_) \
    if (info.R == R_) return launch_tmem2<CfgT2<D_, R_, 2, 4>>(a, grid, s);
        BFV_TMEM2_INSTANCES(BFV_LAUNCH2)
#undef BFV_LAUNCH2
        return cudaErrorInvalidValue;
    }
    if (info.variant == 2) {
#define BFV_LAUNCHT(D_, R_) \
    if (info.R == R_) return launch_tmem<CfgT<D_, R_, 16>>(a, grid, s);
        BFV_TMEM_INSTANCES(BFV_LAUNCHT)
#undef BFV_LAUNCHT
        return cudaErrorInvalidValue;
    }
#define BFV_LAUNCH(D_, R_, NA_, KB_, SH_) \
    if (info.R == R_) return launch_cfg<Cfg<D_, R_, NA_, KB_, SH_>>(a, grid, s);
    BFV_INSTANCES(BFV_LAUNCH)
#undef BFV_LAUNCH
    return cudaErrorInvalidValue;
}

}  // namespace bfvec
