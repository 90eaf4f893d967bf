// mcsf_inst_d8.cu -- fused-kernel instances for D = 8 (one translation unit per D so
// the large fully-expanded FIR bodies compile in parallel). Cfg<D, R, NA, KB, SH> (NA = producer threads).
#include "mcsf_fused.cuh"

namespace bfvec {

#define BFV_INSTANCES(X) X(8, 6, 96, 16, 8) X(8, 15, 96, 16, 8) X(8, 24, 96, 8, 8)

bool fused_select_d8(int r, int variant, KernelInfo *info) {
    if (variant == 6 && r > 15 && r <= 24) {   // comparison instance: one H-pass item per producer thread
        fill_info<Cfg<8, 24, 288, 8, 8>>(info);
        info->variant = 6;
        return true;
    }
    int best = 1 << 30;
#define BFV_PICK(D_, R_, NT_, KB_, SH_) \
    if (R_ >= r && R_ < best) best = R_;
    BFV_INSTANCES(BFV_PICK)
#undef BFV_PICK
    if (best == (1 << 30)) return false;
#define BFV_FILL(D_, R_, NT_, KB_, SH_) \
    if (R_ == best) fill_info<Cfg<D_, R_, NT_, KB_, SH_>>(info);
    BFV_INSTANCES(BFV_FILL)
#undef BFV_FILL
    info->variant = 1;
    return true;
}

cudaError_t fused_launch_d8(const KernelInfo &info, const FusedArgs &a, dim3 grid, cudaStream_t s) {
    if (info.variant == 6) return launch_cfg<Cfg<8, 24, 288, 8, 8>>(a, grid, s);
#define BFV_LAUNCH(D_, R_, NT_, KB_, SH_) \
    if (info.R == R_) return launch_cfg<Cfg<D_, R_, NT_, KB_, SH_>>(a, grid, s);
    BFV_INSTANCES(BFV_LAUNCH)
#undef BFV_LAUNCH
    return cudaErrorInvalidValue;
}

}  // namespace bfvec
