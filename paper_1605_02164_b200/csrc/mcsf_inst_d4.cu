// mcsf_inst_d4.cu -- fused-kernel instances for D = 4 (one translation unit per D so
// the large fully-expanded FIR bodies compile in parallel). Cfg<D, R, NA, KB, SH> (NA = producer threads).
#include "mcsf_fused.cuh"

namespace bfvec {

#define BFV_INSTANCES(X) X(4, 6, 160, 16, 8) X(4, 15, 160, 16, 8) X(4, 32, 160, 16, 8) X(4, 48, 160, 16, 8)

bool fused_select_d4(int r, int variant, KernelInfo *info) {
    (void)variant;   // v3 only for D = 4
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

cudaError_t fused_launch_d4(const KernelInfo &info, const FusedArgs &a, dim3 grid, cudaStream_t s) {
#define BFV_LAUNCH(D_, R_, NT_, KB_, SH_) \
    if (info.R == R_) return launch_cfg<Cfg<D_, R_, NT_, KB_, SH_>>(a, grid, s);
    BFV_INSTANCES(BFV_LAUNCH)
#undef BFV_LAUNCH
    return cudaErrorInvalidValue;
}

}  // namespace bfvec
