// mcsf_inst_d8.cu -- fused-kernel instances for D = 8 (one translation unit per D so
// the large fully-expanded FIR bodies compile in parallel). Cfg<D, R, NA, KB, SH> (NA = producer threads).
#include "mcsf_fused.cuh"
#include "mcsf_tmem8.cuh"

namespace bfvec {

// NA = 288 producer threads: one H-pass item (pair, row, 8-column group) per thread per
// sub-step (9 pairs x 8 rows x 4 groups); 14 % faster on config 4 than NA = 96
#define BFV_INSTANCES(X) X(8, 6, 288, 16, 8) X(8, 15, 288, 16, 8) X(8, 24, 288, 8, 8)
// tensor-memory ring, three launches per call (mcsf_tmem8.cuh)
#define BFV_TMEM8_INSTANCES(X) X(6) X(15) X(24)

// variant 0: auto (the tensor-memory ring where an instance fits: 1.08x / 1.07x the shared-memory
// ring at r = 6 / 24, equal at r = 15, profiles/r01_v8_vs_v3.txt), 1: v3 (shared-memory ring),
// 8: tensor-memory ring
bool fused_select_d8(int r, int variant, KernelInfo *info) {
    if (variant == 8 || variant == 0) {
        int best8 = 1 << 30;
#define BFV_PICK8(R_) \
    if (R_ >= r && R_ < best8) best8 = R_;
        BFV_TMEM8_INSTANCES(BFV_PICK8)
#undef BFV_PICK8
        if (best8 != (1 << 30)) {
#define BFV_FILL8(R_) \
    if (R_ == best8) fill_info_tmem8<R_>(info);
            BFV_TMEM8_INSTANCES(BFV_FILL8)
#undef BFV_FILL8
            info->variant = 8;
            return true;
        }
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
    if (info.variant == 8) {
#define BFV_LAUNCH8(R_) \
    if (info.R == R_) return launch_tmem8<R_>(a, grid, s);
        BFV_TMEM8_INSTANCES(BFV_LAUNCH8)
#undef BFV_LAUNCH8
        return cudaErrorInvalidValue;
    }
#define BFV_LAUNCH(D_, R_, NT_, KB_, SH_) \
    if (info.R == R_) return launch_cfg<Cfg<D_, R_, NT_, KB_, SH_>>(a, grid, s);
    BFV_INSTANCES(BFV_LAUNCH)
#undef BFV_LAUNCH
    return cudaErrorInvalidValue;
}

}  // namespace bfvec
