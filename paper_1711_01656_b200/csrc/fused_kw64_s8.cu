// Instantiations of the fused build+match sweep for kw = 64, 8 strip(s) per CTA
// (see fused_kernel.cuh).
#include "fused_kernel.cuh"

namespace spct_fused {
void launch_kw64_s8(bool allb, int sk, dim3 grid, cudaStream_t s, const QuantParams& q, const PixelMode& pm,
                       const spct_ih& out, const BuildPlan& bp, const FusedCarries& fc, const FusedParams& f) {
    launch_kw_impl<64, 8>(allb, sk, grid, s, q, pm, out, bp, fc, f);
}
}  // namespace spct_fused
