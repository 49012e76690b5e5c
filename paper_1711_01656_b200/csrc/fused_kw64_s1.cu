// Instantiations of the fused build+match sweep for kw = 64, 1 strip(s) per CTA
// (see fused_kernel.cuh).
#include "fused_kernel.cuh"

namespace spct_fused {
void launch_kw64_s1(bool allb, int sk, dim3 grid, cudaStream_t s, const QuantParams& q, const PixelMode& pm,
                       const spct_ih& out, const BuildPlan& bp, const FusedCarries& fc, const FusedParams& f) {
    launch_kw_impl<64, 1>(allb, sk, grid, s, q, pm, out, bp, fc, f);
}
}  // namespace spct_fused

namespace spct_fused {
size_t smem_bytes() { return kSmemBytes; }
}  // namespace spct_fused

namespace spct_impl {
int fused_ctas_per_sm(int strips) {
    strips = strips >= 8 ? 8 : (strips >= 4 ? 4 : (strips >= 2 ? 2 : 1));
    return per_device_int(200 + strips, [](int key) {
        const int S = key - 200;
        int v = 0;
        cudaError_t e;
#define SPCT_OCC(SV)                                                                          \
    {                                                                                         \
        auto k = spct_fused::sweep_match_kernel<true, 1, 64, true, 1, SV>;                  \
        ensure_smem(k, spct_fused::smem_bytes_s<SV>());                                       \
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, 256, spct_fused::smem_bytes_s<SV>()); \
    }
        if (S == 1) SPCT_OCC(1) else if (S == 2) SPCT_OCC(2) else if (S == 4) SPCT_OCC(4) else SPCT_OCC(8)
#undef SPCT_OCC
        if (e != cudaSuccess || v <= 0) {
            cudaGetLastError();
            v = 2;
        }
        return v;
    });
}
}  // namespace spct_impl
