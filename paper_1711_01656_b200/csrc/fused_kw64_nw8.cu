// Instantiations of the fused build+match sweep for kw = 64,
// 8 warps per CTA (see fused_kernel.cuh).
#include "fused_kernel.cuh"

namespace spct_fused {
void launch_kw64_nw8(bool allb, int sk, dim3 grid, cudaStream_t s, const QuantParams& q, const PixelMode& pm, const spct_ih& out,
          const BuildPlan& bp, const FusedCarries& fc, const FusedParams& f) {
    launch_kw_impl<64, 8>(allb, sk, grid, s, q, pm, out, bp, fc, f);
}
size_t smem_bytes() { return kSmemBytes; }
}  // namespace spct_fused

namespace spct_impl {
int fused_ctas_per_sm(int nw) {
    nw = nw >= 8 ? 8 : (nw >= 4 ? 4 : 2);
    return per_device_int(200 + nw, [](int key) {
        const int nw = key - 200;
        int v = 0;
        cudaError_t e;
        if (nw == 8) {
            auto k = spct_fused::sweep_match_kernel<true, true, 64, true, 1, 8>;
            ensure_smem(k, spct_fused::smem_bytes_nw<8>());
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, 256, spct_fused::smem_bytes_nw<8>());
        } else if (nw == 4) {
            auto k = spct_fused::sweep_match_kernel<true, true, 64, true, 1, 4>;
            ensure_smem(k, spct_fused::smem_bytes_nw<4>());
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, 128, spct_fused::smem_bytes_nw<4>());
        } else {
            auto k = spct_fused::sweep_match_kernel<true, true, 64, true, 1, 2>;
            ensure_smem(k, spct_fused::smem_bytes_nw<2>());
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k, 64, spct_fused::smem_bytes_nw<2>());
        }
        if (e != cudaSuccess || v <= 0) {
            cudaGetLastError();
            v = 16 / nw;
        }
        return v;
    });
}
}  // namespace spct_impl
