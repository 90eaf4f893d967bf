// mcsf_dispatch.cu -- picks the fused-kernel instance for a plan: the smallest
// compiled D >= d (channels d..D-1 are zero) and, within it, the smallest
// compiled R >= r (taps beyond r are zero).
#include "internal.h"

namespace bfvec {

#define BFV_DS(X) X(1) X(2) X(3) X(4) X(8)
#define BFV_DECL(D)                                                 \
    bool fused_select_d##D(int r, int variant, KernelInfo *info);                \
    cudaError_t fused_launch_d##D(const KernelInfo &info, const FusedArgs &a, dim3 grid, cudaStream_t s);
BFV_DS(BFV_DECL)
#undef BFV_DECL

bool fused_select(int d, int r, int variant, KernelInfo *info) {
#define BFV_TRY(D) \
    if (d <= D) return fused_select_d##D(r, variant, info);
    BFV_DS(BFV_TRY)
#undef BFV_TRY
    return false;
}

cudaError_t fused_launch(const KernelInfo &info, const FusedArgs &a, dim3 grid, cudaStream_t s) {
    switch (info.D) {
#define BFV_CASE(D) \
    case D: return fused_launch_d##D(info, a, grid, s);
        BFV_DS(BFV_CASE)
#undef BFV_CASE
    }
    return cudaErrorInvalidValue;
}

}  // namespace bfvec
