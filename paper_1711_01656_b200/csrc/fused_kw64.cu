// Instantiations of the fused build+match sweep for kw = 64
// (see fused_kernel.cuh).
#include "fused_kernel.cuh"

namespace spct_fused {
void launch_kw64(bool allb, bool g8, dim3 grid, cudaStream_t s, const QuantParams& q, const PixelMode& pm, const spct_ih& out,
          const BuildPlan& bp, const FusedCarries& fc, const FusedParams& f) {
    launch_kw_impl<64>(allb, g8, grid, s, q, pm, out, bp, fc, f);
}
size_t smem_bytes() { return kSmemBytes; }
}  // namespace spct_fused

namespace spct_impl {
int fused_ctas_per_sm() {
    static int n = 0;
    if (n) return n;
    int v = 0;
    auto k = spct_fused::sweep_match_kernel<true, true, 64, true, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)spct_fused::kSmemBytes);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, 256, spct_fused::kSmemBytes) != cudaSuccess || v <= 0) {
        cudaGetLastError();
        v = 2;
    }
    return n = v;
}
}  // namespace spct_impl
