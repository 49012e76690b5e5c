// Gradient-orientation bins: the orientation channel of the tracking batch (BASELINE
// config 5, SURVEY.md §2 row 6 "input prep for config 5").
//
// Restates, in FP64 with the reference's operation order (no FMA contraction):
//   gradient_maps(GrayImage, sigma)  features.cpp:200-203 -> gradient_maps_impl :78-93
//     to_scalar (imagecore.cpp:55-59), gaussian_smooth :30-51 (gaussian_kernel :14-25,
//     separable, replicated borders), diff_x / diff_y :53-69 (central differences / 2),
//     fold_orientation :71-76 (atan(dy/dx) in degrees, 90 on dx == 0, 0 when flat)
//   orientation_bin(deg, bins)       phog.cpp:15-20 (floor((deg + 90) * bins / 180), clamped)
// The taps are computed on the host with the reference's formula.
//
// One kernel, one 64 x 32 output tile per CTA: the tile's gray pixels (with the blur and
// difference halo, borders replicated by clamping exactly as the reference indexes) are
// staged in shared memory, the horizontal pass, the vertical pass and the differences all
// run out of shared memory, and only the uint16 bins are written (1 B/px in, 2 B/px out;
// the three-pass form moved 8 B/px plane twice more each way).
//
// The bin of q = dy / dx is found without the FP64 atan: a binary search of the float
// ratio over the bin boundaries in q, t_b = tan(pi (b / bins - 1/2)), b = 1 .. bins - 1
// (deg is monotone in q).  Wherever the float ratio lies more than 4e-6 rad (in angle)
// from both neighbouring boundaries, the reference's rounded deg is inside the same bin,
// so the bin is exact; pixels inside the margin, bins > 256, dx == 0 and extreme
// magnitudes run the reference formula itself (bin_formula).
#include <cmath>
#include <cstdlib>

#include "spct_internal.h"

using namespace spct_impl;

namespace spct_orient {

constexpr int kMaxRadius = 31;
constexpr int kTX = 64, kTY = 32, kThreads = 256, kMaxTable = 255;

struct Taps {
    int radius;
    double k[2 * kMaxRadius + 1];
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ int bin_formula(double dx, double dy, int bins) {
    double deg;
    if (dx == 0.0 && dy == 0.0) deg = 0.0;
    else if (dx == 0.0) deg = 90.0;
    else deg = __ddiv_rn(__dmul_rn(atan(__ddiv_rn(dy, dx)), 180.0), 3.14159265358979323846);
    const double f = floor(__ddiv_rn(__dmul_rn(__dadd_rn(deg, 90.0), static_cast<double>(bins)), 180.0));
    return f < 0.0 ? 0 : (f >= bins ? bins - 1 : static_cast<int>(f));
}

// Shared-memory planes.  Every plane is padded with the reference's replicated borders
// (row / column p holds the value at clamp(p)), so the tap loops index without clamps:
//   G [nby + 2r][nbx + 2r]  gray (bytes) at (clamp(y), clamp(x)), y in [yblo - r, ybhi + r],
//                           x in [xlo - r, xhi + r]
//   H [nby + 2r][nbx]       horizontal pass at the padded rows
//   B [nby][nbx]            vertical pass: the blurred image at [yblo, ybhi] x [xlo, xhi]
// Warp w takes rows w, w + 8, ..., lane l columns l, l + 32, l + 64.
constexpr int kBS = kTX + 2;  // H / B row stride (doubles)
constexpr int kWarps = kThreads / 32;

__host__ __device__ constexpr int g_stride(int r) { return (kBS + 2 * r + 15) / 16 * 16; }  // bytes

// Bin search on the float boundaries: the candidate bin of the float ratio, accepted when
// it sits more than kMargin (in angle, radians; tan' = 1 + q^2) from both neighbouring
// boundaries.  Float errors (the two conversions, the division, the rounded table) stay
// below 2e-7 rad, the reference's FP64 deg below 1e-14, so an accepted bin is the
// reference's bin.
constexpr float kMargin = 4e-6f;

// tf: the boundaries padded as tf[0] = -inf, tf[1 .. nth] = t_1 .. t_nth, +inf up to
// tf[top]; top = the smallest power of two > nth.
__device__ __forceinline__ int bin_fast(double ddx, double ddy, int top, const float* __restrict__ tf) {
    // (ddx, ddy are the un-halved differences: the ratio is the same)
    const double ax = fabs(ddx), ay = fabs(ddy);
    if (!(ax >= 1e-30 && ax <= 1e30) || !(ay == 0.0 || (ay >= 1e-30 && ay <= 1e30))) return -1;
    const float q = __fdiv_rn(static_cast<float>(ddy), static_cast<float>(ddx));
    int lo = 0;  // the largest i with tf[i] <= q: the bin
    for (int step = top >> 1; step; step >>= 1) lo += tf[lo + step] <= q ? step : 0;
    const float m = kMargin * (1.0f + q * q);
    return (q - tf[lo] > m && tf[lo + 1] - q > m) ? lo : -1;
}

// R >= 0: the radius as a compile-time constant (unrolled tap chains);
// R < 0: any radius from the taps.
template <int R>
__global__ void __launch_bounds__(kThreads) orientation_tile_kernel(const uint8_t* __restrict__ gray, int64_t pitch,
                                                                    int w, int h, Taps t, int bins,
                                                                    const float* __restrict__ bounds,
                                                                    uint16_t* __restrict__ out, int64_t out_pitch) {
    extern __shared__ double osm[];
    __shared__ double tap[2 * kMaxRadius + 1];
    __shared__ float tf[kMaxTable + 2];
    const int r = R >= 0 ? R : t.radius;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = blockIdx.x * kTX, y0 = blockIdx.y * kTY;
    // B at the actual columns / rows the differences read (clamped into the image)
    const int xlo = max(0, x0 - 1), xhi = min(w - 1, x0 + kTX);
    const int yblo = max(0, y0 - 1), ybhi = min(h - 1, y0 + kTY);
    const int nbx = xhi - xlo + 1, nby = ybhi - yblo + 1;
    const int gs = g_stride(r), nhy = nby + 2 * r, ngx = nbx + 2 * r;
    const int nth = bins <= kMaxTable + 1 ? bins - 1 : -1;
    int top = 1;
    while (top <= nth) top <<= 1;
    double* H = osm;                           // [nhy][kBS]
    double* B = H + (kTY + 2 + 2 * r) * kBS;   // [nby][kBS]
    uint8_t* G = reinterpret_cast<uint8_t*>(B + (kTY + 2) * kBS);  // [nhy][gs]
    for (int i = threadIdx.x; i <= 2 * r; i += kThreads) tap[i] = t.k[i];
    for (int i = threadIdx.x; i <= top && nth >= 0; i += kThreads)
        tf[i] = i == 0 ? -INFINITY : (i <= nth ? __ldg(bounds + i - 1) : INFINITY);
    const bool interior = xlo - r >= 0 && xlo - r + ngx <= w;  // no column clamping
    for (int ry = warp; ry < nhy; ry += kWarps) {
        const uint8_t* src = gray + static_cast<int64_t>(clampi(yblo - r + ry, 0, h - 1)) * pitch + xlo - r;
        uint8_t* gr = G + ry * gs;
        if (interior) {
#pragma unroll 3
            for (int cx = lane; cx < ngx; cx += 32) gr[cx] = __ldg(src + cx);
        } else {
            for (int cx = lane; cx < ngx; cx += 32) gr[cx] = __ldg(src + clampi(xlo - r + cx, 0, w - 1) - (xlo - r));
        }
    }
    __syncthreads();
    // hblur (features.cpp:35-41): acc += k_i * in(clamp(x + i), y), i ascending
    if constexpr (R >= 0) {
        // lane l takes the consecutive columns 3 l .. 3 l + 2: the 3 + 2R gray values it
        // needs are converted to double once (not once per tap); same products and sums
        // in the same order per output
        constexpr int NV = 3 + 2 * R;
        for (int ry = warp; ry < nhy; ry += kWarps) {
            const uint8_t* g = G + ry * gs;
            const int cb = 3 * lane;
            if (cb >= nbx) continue;
            double v[NV];
#pragma unroll
            for (int i = 0; i < NV; ++i) v[i] = static_cast<double>(g[min(cb + i, ngx - 1)]);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                double acc = 0.0;
#pragma unroll
                for (int k = 0; k <= 2 * R; ++k) acc = __dadd_rn(acc, __dmul_rn(tap[k], v[j + k]));
                if (cb + j < nbx) H[ry * kBS + cb + j] = acc;
            }
        }
    } else
    for (int ry = warp; ry < nhy; ry += kWarps) {
        const uint8_t* g = G + ry * gs;
        double acc[3] = {0.0, 0.0, 0.0};
        int c[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) c[j] = min(lane + 32 * j, nbx - 1);
#pragma unroll
        for (int k = 0; k <= 2 * r; ++k) {
            const double tk = tap[k];
#pragma unroll
            for (int j = 0; j < 3; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(tk, static_cast<double>(g[c[j] + k])));
        }
#pragma unroll
        for (int j = 0; j < 3; ++j)
            if (lane + 32 * j < nbx) H[ry * kBS + lane + 32 * j] = acc[j];
    }
    __syncthreads();
    // vblur (:43-49): acc += k_i * tmp(x, clamp(y + i)), i ascending
    if constexpr (R >= 0) {
        // warp w takes the consecutive output rows [r0, r0 + nr): per column the lane loads
        // the nr + 2R rows of H it needs once (not 2R + 1 per output row)
        constexpr int MR = (kTY + 2 + kWarps - 1) / kWarps;  // rows per warp (5 for 34)
        const int r0 = warp * MR, nr = min(MR, nby - r0);
        if (nr > 0)
            for (int j = 0; j < 3; ++j) {
                const int c = lane + 32 * j;
                if (c >= nbx) break;
                double hv[MR + 2 * R];
#pragma unroll
                for (int i = 0; i < MR + 2 * R; ++i) hv[i] = i < nr + 2 * R ? H[(r0 + i) * kBS + c] : 0.0;
#pragma unroll
                for (int q = 0; q < MR; ++q) {
                    if (q >= nr) break;
                    double acc = 0.0;
#pragma unroll
                    for (int k = 0; k <= 2 * R; ++k) acc = __dadd_rn(acc, __dmul_rn(tap[k], hv[q + k]));
                    B[(r0 + q) * kBS + c] = acc;
                }
            }
    } else
    for (int by = warp; by < nby; by += kWarps) {
        double acc[3] = {0.0, 0.0, 0.0};
        int c[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) c[j] = min(lane + 32 * j, nbx - 1);
#pragma unroll
        for (int k = 0; k <= 2 * r; ++k) {
            const double tk = tap[k];
            const double* hr = H + (by + k) * kBS;
#pragma unroll
            for (int j = 0; j < 3; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(tk, hr[c[j]]));
        }
#pragma unroll
        for (int j = 0; j < 3; ++j)
            if (lane + 32 * j < nbx) B[by * kBS + lane + 32 * j] = acc[j];
    }
    __syncthreads();
    // diff_x / diff_y (:53-69), then the bin of atan(dy / dx)
    for (int ty = warp; ty < kTY; ty += kWarps) {
        const int y = y0 + ty;
        if (y >= h) break;
        const double* brow = B + (y - yblo) * kBS - xlo;
        const double* bup = B + (clampi(y - 1, 0, h - 1) - yblo) * kBS - xlo;
        const double* bdn = B + (clampi(y + 1, 0, h - 1) - yblo) * kBS - xlo;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int x = x0 + lane + 32 * j;
            if (x >= w) continue;
            const double ddx = __dsub_rn(brow[clampi(x + 1, 0, w - 1)], brow[clampi(x - 1, 0, w - 1)]);
            const double ddy = __dsub_rn(bdn[x], bup[x]);
            int b = nth >= 0 ? bin_fast(ddx, ddy, top, tf) : -1;
            if (b < 0) b = bin_formula(__dmul_rn(ddx, 0.5), __dmul_rn(ddy, 0.5), bins);  // "/ 2.0" == "* 0.5"
            out[static_cast<int64_t>(y) * out_pitch + x] = static_cast<uint16_t>(b);
        }
    }
}

// Bin boundaries in q = dy / dx: t_b = tan(pi (b / bins - 1/2)), b = 1 .. bins - 1, as
// floats (the margin covers their rounding).
__global__ void bounds_kernel(int bins, float* __restrict__ tb) {
    const int i = threadIdx.x;
    if (i < bins - 1) tb[i] = static_cast<float>(tan(3.14159265358979323846 * (static_cast<double>(i + 1) / bins - 0.5)));
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

size_t tile_smem(int r) {
    return static_cast<size_t>((kTY + 2 + 2 * r) * kBS + (kTY + 2) * kBS) * sizeof(double) +
           static_cast<size_t>(kTY + 2 + 2 * r) * g_stride(r);
}

}  // namespace spct_orient

using namespace spct_orient;

extern "C" spct_status spct_cu_orientation_workspace(int width, int height, size_t* bytes) {
    if (!bytes) return contract("orientation_workspace: null argument");
    if (!(width > 0 && height > 0)) return contract("gradient_maps: empty image");
    *bytes = (kMaxTable + 1) * sizeof(float);  // the bin boundaries
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
    if (!workspace || workspace_bytes < kMaxTable * sizeof(float))
        return contract("orientation_bins: workspace too small");
    const Taps t = make_taps(sigma);
    cudaStream_t s = as_stream(stream);
    float* bounds = static_cast<float*>(workspace);
    if (bins >= 2 && bins <= kMaxTable + 1) {
        bounds_kernel<<<1, 256, 0, s>>>(bins, bounds);
        if (auto st = launch_status("bounds_kernel")) return st;
    }
    ensure_smem(orientation_tile_kernel<3>, tile_smem(kMaxRadius));
    ensure_smem(orientation_tile_kernel<-1>, tile_smem(kMaxRadius));
    const dim3 grid(static_cast<unsigned>(ceil_div(width, kTX)), static_cast<unsigned>(ceil_div(height, kTY)));
    const size_t smem = tile_smem(t.radius);
    static const bool force_generic = std::getenv("SPCT_ORIENT_GENERIC") != nullptr;
    if (t.radius == 3 && !force_generic)  // sigma in (2/3, 1]: the reference's PHOG / tracker sigma 1
        orientation_tile_kernel<3><<<grid, kThreads, smem, s>>>(gray, pitch, width, height, t, bins, bounds, out,
                                                                 out_pitch);
    else
        orientation_tile_kernel<-1><<<grid, kThreads, smem, s>>>(gray, pitch, width, height, t, bins, bounds, out,
                                                                  out_pitch);
    return launch_status("orientation_tile_kernel");
}
