// mcsf_inst_d1.cu -- fused-kernel instances for D = 1 (one translation unit per D so
// the large fully-expanded FIR bodies compile in parallel). Cfg<D, R, NA, KB, SH> (NA = producer threads).
#include "mcsf_fused.cuh"

namespace bfvec {

#define BFV_INSTANCES(X) X(1, 2, 64, 16, 16) X(1, 6, 64, 16, 16) X(1, 15, 64, 16, 16) X(1, 32, 64, 16, 16) X(1, 64, 64, 16, 16)

bool fused_select_d1(int r, KernelInfo *info) {
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
    return true;
}

cudaError_t fused_launch_d1(const KernelInfo &info, const FusedArgs &a, dim3 grid, cudaStream_t s) {
#define BFV_LAUNCH(D_, R_, NT_, KB_, SH_) \
    if (info.R == R_) return launch_cfg<Cfg<D_, R_, NT_, KB_, SH_>>(a, grid, s);
    BFV_INSTANCES(BFV_LAUNCH)
#undef BFV_LAUNCH
    return cudaErrorInvalidValue;
}

}  // namespace bfvec
