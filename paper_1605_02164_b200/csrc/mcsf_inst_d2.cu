// mcsf_inst_d2.cu -- fused-kernel instances for D = 2 (one translation unit per D so
// the large fully-expanded FIR bodies compile in parallel).
//   v3 (shared-memory ring, mcsf_fused.cuh): Cfg<D, R, NA, KB, SH> (NA = producer threads)
//   v4 (tensor-memory ring, mcsf_tmem.cuh):  CfgT<D, R, 16>
#include "mcsf_fused.cuh"
#include "mcsf_tmem.cuh"
#include "mcsf_tmem2.cuh"

namespace bfvec {

#define BFV_TMEM2_INSTANCES(X) X(2, 6) X(2, 10) X(2, 15) X(2, 24) X(2, 30) X(2, 48)
#ifdef BFVEC_COMPARISON_VARIANTS   // see mcsf_inst_d3.cu
#define BFV_INSTANCES(X) X(2, 6, 96, 16, 16) X(2, 15, 96, 16, 16) X(2, 32, 96, 16, 16) X(2, 64, 96, 16, 8)
#define BFV_TMEM_INSTANCES(X) X(2, 6) X(2, 15) X(2, 24) X(2, 32) X(2, 48)
#else
#define BFV_INSTANCES(X) X(2, 64, 96, 16, 8)
#define BFV_TMEM_INSTANCES(X) X(2, 32)
#endif

// variant: 0 auto (v5 where compiled, else v4, else v3), 1 force v3, 2 force v4, 4 force v5
bool fused_select_d2(int r, int variant, KernelInfo *info) {
    int best = 1 << 30, bestT = 1 << 30;
#define BFV_PICK(D_, R_, NA_, KB_, SH_) \
    if (R_ >= r && R_ < best) best = R_;
    BFV_INSTANCES(BFV_PICK)
#undef BFV_PICK
#define BFV_PICKT(D_, R_) \
    if (R_ >= r && R_ < bestT) bestT = R_;
    BFV_TMEM_INSTANCES(BFV_PICKT)
#undef BFV_PICKT
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
    const bool use_t = bestT != (1 << 30) && variant != 1 && (variant == 2 || bestT <= best);
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

cudaError_t fused_launch_d2(const KernelInfo &info, const FusedArgs &a, dim3 grid, cudaStream_t s) {
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
