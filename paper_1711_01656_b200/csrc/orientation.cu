// Gradient-orientation bins: the orientation channel of the tracking batch (BASELINE
// config 5, SURVEY.md §2 row 6 "input prep for config 5").
//
// Restates, in FP64 with the reference's operation order (no FMA contraction):
//   gradient_maps(GrayImage, sigma)  features.cpp:200-203 -> gradient_maps_impl :78-93
//     to_scalar (imagecore.cpp:55-59), gaussian_smooth :30-51 (gaussian_kernel :14-25,
//     separable, replicated borders), diff_x / diff_y :53-69 (central differences / 2),
//     fold_orientation :71-76 (atan(dy/dx) in degrees, 90 on dx == 0, 0 when flat)
//   orientation_bin(deg, bins)       phog.cpp:15-20 (floor((deg + 90) * bins / 180), clamped)
// The taps are computed on the host with the reference's formula.  Three passes over the
// frame (horizontal blur, vertical blur, gradient + bin); two FP64 scratch planes.
#include <cmath>

#include "spct_internal.h"

using namespace spct_impl;

namespace spct_orient {

constexpr int kMaxRadius = 31;

struct Taps {
    int radius;
    double k[2 * kMaxRadius + 1];
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__global__ void hblur_kernel(const uint8_t* __restrict__ gray, int64_t pitch, int w, int h, Taps t,
                             double* __restrict__ out) {
    const int y = blockIdx.y;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < w; x += gridDim.x * blockDim.x) {
        const uint8_t* row = gray + static_cast<int64_t>(y) * pitch;
        double acc = 0.0;
        for (int i = -t.radius; i <= t.radius; ++i)
            acc = __dadd_rn(acc, __dmul_rn(t.k[i + t.radius], static_cast<double>(row[clampi(x + i, 0, w - 1)])));
        out[static_cast<int64_t>(y) * w + x] = acc;
    }
}

__global__ void vblur_kernel(const double* __restrict__ in, int w, int h, Taps t, double* __restrict__ out) {
    const int y = blockIdx.y;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < w; x += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int i = -t.radius; i <= t.radius; ++i)
            acc = __dadd_rn(acc, __dmul_rn(t.k[i + t.radius], in[static_cast<int64_t>(clampi(y + i, 0, h - 1)) * w + x]));
        out[static_cast<int64_t>(y) * w + x] = acc;
    }
}

__global__ void orient_bin_kernel(const double* __restrict__ base, int w, int h, int bins, uint16_t* __restrict__ out,
                                  int64_t out_pitch) {
    const int y = blockIdx.y;
    const double* row = base + static_cast<int64_t>(y) * w;
    const double* up = base + static_cast<int64_t>(clampi(y - 1, 0, h - 1)) * w;
    const double* dn = base + static_cast<int64_t>(clampi(y + 1, 0, h - 1)) * w;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < w; x += gridDim.x * blockDim.x) {
        const double dx = __ddiv_rn(__dsub_rn(row[clampi(x + 1, 0, w - 1)], row[clampi(x - 1, 0, w - 1)]), 2.0);
        const double dy = __ddiv_rn(__dsub_rn(dn[x], up[x]), 2.0);
        double deg;
        if (dx == 0.0 && dy == 0.0) deg = 0.0;
        else if (dx == 0.0) deg = 90.0;
        else deg = __ddiv_rn(__dmul_rn(atan(__ddiv_rn(dy, dx)), 180.0), 3.14159265358979323846);
        const double f = floor(__ddiv_rn(__dmul_rn(__dadd_rn(deg, 90.0), static_cast<double>(bins)), 180.0));
        int b = f < 0.0 ? 0 : (f >= bins ? bins - 1 : static_cast<int>(f));
        out[static_cast<int64_t>(y) * out_pitch + x] = static_cast<uint16_t>(b);
    }
}

// gaussian_kernel (features.cpp:14-25), same operation order; radius 0 (sigma == 0) is the
// identity (acc = 0 + 1 * v), which gaussian_smooth's early return also is.
Taps make_taps(double sigma) {
    Taps t{};
    if (!(sigma > 0.0)) {
        t.radius = 0;
        t.k[0] = 1.0;
        return t;
    }
    t.radius = static_cast<int>(std::ceil(3.0 * sigma));
    double sum = 0.0;
    for (int i = -t.radius; i <= t.radius; ++i) {
        const double v = std::exp(-(static_cast<double>(i) * i) / (2.0 * sigma * sigma));
        t.k[i + t.radius] = v;
        sum += v;
    }
    for (int i = 0; i < 2 * t.radius + 1; ++i) t.k[i] /= sum;
    return t;
}

}  // namespace spct_orient

using namespace spct_orient;

extern "C" spct_status spct_cu_orientation_workspace(int width, int height, size_t* bytes) {
    if (!bytes) return contract("orientation_workspace: null argument");
    if (!(width > 0 && height > 0)) return contract("gradient_maps: empty image");
    *bytes = 2 * static_cast<size_t>(width) * height * sizeof(double) + 256;
    return SPCT_OK;
}

extern "C" spct_status spct_cu_orientation_bins(const uint8_t* gray, int64_t pitch, int width, int height, double sigma,
                                                int bins, uint16_t* out, int64_t out_pitch, void* workspace,
                                                size_t workspace_bytes, void* stream) {
    if (!(sigma >= 0.0)) return contract("gradient_maps: sigma must be nonnegative");  // features.cpp:201
    if (!(width > 0 && height > 0)) return contract("gradient_maps: empty image");
    if (!(bins >= 1 && bins <= 65536)) return contract("orientation_bins: bins must be in [1, 65536]");
    if (!gray || !out || pitch < width || out_pitch < width) return contract("orientation_bins: bad arguments");
    if (std::ceil(3.0 * sigma) > kMaxRadius) return contract("orientation_bins: sigma too large (radius > 31)");
    const size_t plane = static_cast<size_t>(width) * height * sizeof(double);
    if (!workspace || workspace_bytes < 2 * plane) return contract("orientation_bins: workspace too small");
    double* a = static_cast<double*>(workspace);
    double* b = reinterpret_cast<double*>(static_cast<char*>(workspace) + plane);
    const Taps t = make_taps(sigma);
    cudaStream_t s = as_stream(stream);
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>(ceil_div(width, 256), 64)), static_cast<unsigned>(height));
    hblur_kernel<<<grid, 256, 0, s>>>(gray, pitch, width, height, t, a);
    if (auto st = launch_status("hblur_kernel")) return st;
    vblur_kernel<<<grid, 256, 0, s>>>(a, width, height, t, b);
    if (auto st = launch_status("vblur_kernel")) return st;
    orient_bin_kernel<<<grid, 256, 0, s>>>(b, width, height, bins, out, out_pitch);
    return launch_status("orient_bin_kernel");
}
