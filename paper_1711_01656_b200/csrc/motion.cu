// Joint-IH temporal median background: MedianBackgroundIH
// (reference motion.cpp:35-99, Alg. 4) on the device.
//
// The joint integral histogram J = sum of the window frames' integral histograms lives in
// HBM as one uint32 tensor (exact while frames * H * W < 2^32); a slide is two passes of
// the build sweep in accumulate mode (spct_cu_ih_accumulate: J += IH(new), J -= IH(old),
// read-modify-write of J, ih_build.cu).  background(): one thread per pixel walks the
// CDF over bins of its clipped m x n window (4-corner reads per bin) and reports the
// bin-centre intensity (motion.cpp:28-30).  median_background_sort (motion.cpp:103-118):
// the per-pixel middle order statistic.  Both bit-identical to the reference.
#include "spct_internal.h"

using namespace spct_impl;

namespace spct_motion {

__device__ __forceinline__ uint32_t Jat(const spct_ih& t, int k, int y, int x) {
    return (y > 0 && x > 0) ? t.data[static_cast<int64_t>(k) * t.plane_pitch + static_cast<int64_t>(y - 1) * t.row_pitch +
                                     (x - 1)]
                            : 0u;
}

__global__ void median_bg_kernel(spct_ih J, int nframes, int m, int n, uint8_t* __restrict__ out, int64_t out_pitch) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int W = J.width, Hh = J.height;
    if (i >= static_cast<int64_t>(W) * Hh) return;
    const int x = static_cast<int>(i % W), y = static_cast<int>(i / W);
    const int rx = (m - 1) / 2, ry = (n - 1) / 2;
    const int x0 = max(0, x - rx), x1 = min(W, x + rx + 1), y0 = max(0, y - ry), y1 = min(Hh, y + ry + 1);
    const uint64_t count = static_cast<uint64_t>(x1 - x0) * (y1 - y0) * nframes;
    const uint64_t need = (count + 1) / 2;
    uint64_t cdf = 0;
    int med = J.bins - 1;
    for (int k = 0; k < J.bins; ++k) {
        cdf += static_cast<uint32_t>(Jat(J, k, y1, x1) - Jat(J, k, y0, x1) - Jat(J, k, y1, x0) + Jat(J, k, y0, x0));
        if (cdf >= need) {
            med = k;
            break;
        }
    }
    out[static_cast<int64_t>(y) * out_pitch + x] = static_cast<uint8_t>((2 * med + 1) * 128 / J.bins);
}

constexpr int kMaxSortFrames = 64;

struct FramePtrs {
    const uint8_t* f[kMaxSortFrames];
};

__global__ void median_sort_kernel(FramePtrs fp, int nf, int w, int h, int64_t pitch, uint8_t* __restrict__ out,
                                   int64_t out_pitch) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<int64_t>(w) * h) return;
    const int x = static_cast<int>(i % w), y = static_cast<int>(i / w);
    const int64_t o = static_cast<int64_t>(y) * pitch + x;
    // the (nf/2)-th smallest value: the v with #{< v} <= nf/2 < #{<= v}
    int med = 0;
    for (int a = 0; a < nf; ++a) {
        const int v = fp.f[a][o];
        int lt = 0, le = 0;
        for (int b = 0; b < nf; ++b) {
            const int u = fp.f[b][o];
            lt += u < v;
            le += u <= v;
        }
        if (lt <= nf / 2 && nf / 2 < le) med = v;
    }
    out[static_cast<int64_t>(y) * out_pitch + x] = static_cast<uint8_t>(med);
}

}  // namespace spct_motion

using namespace spct_motion;

extern "C" spct_status spct_cu_median_background(const spct_ih* J, int nframes, int m, int n, uint8_t* out,
                                                 int64_t out_pitch, void* stream) {
    if (auto st = check_ih(J)) return st;
    if (!J->data || !out || out_pitch < J->width) return contract("median_background_ih: bad arguments");
    if (!(nframes >= 1 && nframes % 2 == 1)) return contract("FrameWindow: window length must be odd");  // motion.cpp:14
    if (!(J->bins >= 1 && J->bins <= 256)) return contract("median_background_ih: bins must be in [1,256]");  // :38
    if (!(m >= 1 && n >= 1 && m % 2 == 1 && n % 2 == 1))
        return contract("median_background_ih: kernel sides must be odd and positive");  // :39-40
    if (m > J->width || n > J->height) return contract("median_background_ih: kernel exceeds image");  // :43
    const int64_t px = static_cast<int64_t>(J->width) * J->height;
    median_bg_kernel<<<static_cast<unsigned>(ceil_div(px, 256)), 256, 0, as_stream(stream)>>>(*J, nframes, m, n, out,
                                                                                               out_pitch);
    return launch_status("median_bg_kernel");
}

extern "C" spct_status spct_cu_median_sort(const uint8_t* const* frames, int nf, int width, int height, int64_t pitch,
                                           uint8_t* out, int64_t out_pitch, void* stream) {
    if (!frames || nf < 1) return contract("FrameWindow: empty window");  // motion.cpp:13
    if (nf % 2 != 1) return contract("FrameWindow: window length must be odd");  // :14
    if (nf > kMaxSortFrames) return contract("median_background_sort: at most 64 frames");
    if (!(width > 0 && height > 0)) return contract("FrameWindow: empty frames");  // :16
    if (!out || pitch < width || out_pitch < width) return contract("median_background_sort: bad arguments");
    FramePtrs fp{};
    for (int f = 0; f < nf; ++f) {
        if (!frames[f]) return contract("median_background_sort: null frame");
        fp.f[f] = frames[f];
    }
    const int64_t px = static_cast<int64_t>(width) * height;
    median_sort_kernel<<<static_cast<unsigned>(ceil_div(px, 256)), 256, 0, as_stream(stream)>>>(fp, nf, width, height,
                                                                                                 pitch, out, out_pitch);
    return launch_status("median_sort_kernel");
}
