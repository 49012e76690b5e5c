// hist_distance_map over a stored device tensor (spct_cu_hist_match), reading the tensor
// ONCE.  Replaces likelihood.cpp:193-225 for tensors without a known source frame (IHT1
// files, tensors handed in by a caller).
//
// The reference re-reads four corners of every bin plane per window (b * 4 reads per
// window, region_histogram integral.cpp:561-577).  Here:
//
//   1. ih_bins_kernel streams the tensor row by row (each cell read once, 16-byte loads)
//      and recovers every pixel's bin: the pixel's per-bin count is the 2-D difference
//          p_k(y, x) = H_k(y+1, x+1) - H_k(y, x+1) - H_k(y+1, x) + H_k(y, x)
//      (the previous row is kept in registers, the left column comes from the
//      neighbouring lane).  A tensor built from a bin map has exactly one p_k = 1 per
//      pixel; that is checked exactly for every cell (every p_k in {0, 1}, sum 1).  The
//      bins go to a uint16 BinMap (2 B/px), a violation sets a device flag.
//   2. The fused sweep (fused_kernel.cuh, no tensor store) computes the map from that
//      BinMap: window counts from running column counts, integer p = 1 arithmetic for
//      integral templates, the reference's FP64 terms otherwise.
//   3. Only if the flag is set (a weighted / masked / arbitrary tensor), the exact kernel
//      (hist_match.cu, reference operation order, actual window totals) recomputes the
//      map from the tensor; both of its kernels exit on entry otherwise (no host sync).
#include <algorithm>

#include "spct_internal.h"

using namespace spct_dev;
using namespace spct_impl;

namespace spct_tmatch {

constexpr int kWarps = 16;
constexpr int kBinsPerWarp = 8;
constexpr int kGroup = kWarps * kBinsPerWarp;  // bins per CTA (grid.z = bin groups)
constexpr int kBatch = 4;                      // planes loaded per batch (16-byte loads in flight)

// CTA = (128-column strip, band of rows, group of 128 bins); warp w owns bins
// 128 g + 8 w .. +7; lane l owns columns 4l .. 4l+3 of the strip.  Per row and column the
// warp accumulates the moments of its bins' vertical differences dv_k = H_k(y+1, x+1) -
// H_k(y, x+1):  Mk = sum_k k dv_k and N = sum_k dv_k; their horizontal differences are the
// pixel's bin and count (linearity), and every p_k is checked to lie in {0, 1}.  The 16
// warps' partials are summed through shared memory (double-buffered by row parity, one
// barrier per row).  One group: the bin is final and written as uint16; several groups:
// the partials are added into gsum (u32 bin sum, u32 count) and bins_finalize_kernel
// converts them.
__global__ void __launch_bounds__(512, 1) ih_bins_kernel(spct_ih t, int band_rows, uint16_t* __restrict__ bins,
                                                         int64_t bins_pitch, uint32_t* __restrict__ gsum,
                                                         uint32_t* __restrict__ flag) {
    __shared__ uint32_t part[2][2][kWarps][kStrip];  // [parity][idx | cnt][warp][column]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int xs = blockIdx.x * kStrip, x0 = xs + 4 * lane;
    const int y0 = blockIdx.y * band_rows, y1 = min(t.height, y0 + band_rows);
    const int kb = blockIdx.z * kGroup + warp * kBinsPerWarp;  // warp's first bin
    const int nk = max(0, min(kBinsPerWarp, t.bins - kb));
    const bool lane_live = x0 < t.width;                        // row_pitch is a multiple of 128 B
    const uint32_t* base = t.data + static_cast<int64_t>(kb) * t.plane_pitch + x0;
    const uint32_t* lbase = t.data + static_cast<int64_t>(kb) * t.plane_pitch + (xs - 1);

    uint32_t prev[kBinsPerWarp][4];
#pragma unroll
    for (int i = 0; i < kBinsPerWarp; ++i) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (y0 > 0 && i < nk && lane_live)
            v = *reinterpret_cast<const uint4*>(base + static_cast<int64_t>(i) * t.plane_pitch +
                                                static_cast<int64_t>(y0 - 1) * t.row_pitch);
        prev[i][0] = v.x, prev[i][1] = v.y, prev[i][2] = v.z, prev[i][3] = v.w;
    }
    const bool left_live = lane == 0 && xs > 0;  // lane 0 reads the column left of the strip

    for (int y = y0; y < y1; ++y) {
        const int64_t roff = static_cast<int64_t>(y) * t.row_pitch;
        uint32_t msum[4] = {0, 0, 0, 0}, nsum[4] = {0, 0, 0, 0}, bad = 0;
        uint32_t mL = 0, nL = 0;  // the same moments of the column left of the lane (lane 0: x0 - 1)
#pragma unroll
        for (int b0 = 0; b0 < kBinsPerWarp; b0 += kBatch) {
            uint4 cur[kBatch];
            uint32_t curL[kBatch], prvL[kBatch];
#pragma unroll
            for (int i = 0; i < kBatch; ++i) {
                const int k = b0 + i;
                const int64_t off = static_cast<int64_t>(k) * t.plane_pitch + roff;
                cur[i] = (k < nk && lane_live) ? __ldg(reinterpret_cast<const uint4*>(base + off)) : make_uint4(0, 0, 0, 0);
                curL[i] = (k < nk && left_live) ? __ldg(lbase + off) : 0u;
                prvL[i] = (k < nk && left_live && y > 0) ? __ldg(lbase + off - t.row_pitch) : 0u;
            }
#pragma unroll
            for (int i = 0; i < kBatch; ++i) {
                const int k = b0 + i;
                const uint32_t kk = static_cast<uint32_t>(kb + k);
                const uint32_t c4[4] = {cur[i].x, cur[i].y, cur[i].z, cur[i].w};
                uint32_t dv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    dv[j] = c4[j] - prev[k][j];
                    prev[k][j] = c4[j];
                }
                // the left neighbour's dv of this plane: lane l - 1's column 3, lane 0's own load
                const uint32_t dl = curL[i] - prvL[i];
                uint32_t left = __shfl_up_sync(0xffffffffu, dv[3], 1);
                if (lane == 0) left = dl;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t p = dv[j] - (j ? dv[j - 1] : left);  // the pixel's count of bin kk
                    bad |= p & ~1u;
                    msum[j] += kk * dv[j];
                    nsum[j] += dv[j];
                }
                mL += kk * left;
                nL += left;
            }
        }
        // bin = M(x) - M(x - 1), count = N(x) - N(x - 1); a p_k outside {0, 1} flags the tensor
        if (__any_sync(0xffffffffu, bad != 0) && lane == 0) atomicOr(flag, 1u);
        uint32_t* pi = &part[y & 1][0][warp][4 * lane];
        uint32_t* pc = &part[y & 1][1][warp][4 * lane];
        const uint32_t mprev[4] = {mL, msum[0], msum[1], msum[2]}, nprev[4] = {nL, nsum[0], nsum[1], nsum[2]};
        uint4 wi, wc;
        wi.x = msum[0] - mprev[0], wi.y = msum[1] - mprev[1], wi.z = msum[2] - mprev[2], wi.w = msum[3] - mprev[3];
        wc.x = nsum[0] - nprev[0], wc.y = nsum[1] - nprev[1], wc.z = nsum[2] - nprev[2], wc.w = nsum[3] - nprev[3];
        *reinterpret_cast<uint4*>(pi) = wi;
        *reinterpret_cast<uint4*>(pc) = wc;
        __syncthreads();
        if (threadIdx.x < kStrip) {
            const int c = threadIdx.x, x = xs + c;
            uint32_t si = 0, sc = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                si += part[y & 1][0][w][c];
                sc += part[y & 1][1][w][c];
            }
            if (x < t.width) {
                if (gridDim.z == 1) {
                    const bool ok = sc == 1u && si < static_cast<uint32_t>(t.bins);
                    bins[static_cast<int64_t>(y) * bins_pitch + x] = ok ? static_cast<uint16_t>(si) : 0;
                    if (!ok) atomicOr(flag, 1u);
                } else {
                    uint32_t* g = gsum + 2 * (static_cast<int64_t>(y) * t.width + x);
                    atomicAdd(g, si);
                    atomicAdd(g + 1, sc);
                }
            }
        }
        // the next row writes the other parity; this parity is rewritten two rows on,
        // after the next row's barrier
    }
}

// Several bin groups: the summed moments -> bins (and the flag).
__global__ void bins_finalize_kernel(const uint32_t* __restrict__ gsum, int64_t n, int width, int nbins,
                                     uint16_t* __restrict__ bins, int64_t bins_pitch, uint32_t* __restrict__ flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t si = gsum[2 * i], sc = gsum[2 * i + 1];
        const bool ok = sc == 1u && si < static_cast<uint32_t>(nbins);
        bins[(i / width) * bins_pitch + i % width] = ok ? static_cast<uint16_t>(si) : 0;
        bad |= !ok;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

}  // namespace spct_tmatch

namespace spct_impl {

// Recover the bin map of a one-hot tensor (all bins), see above.  `bins` (dev, width x
// height uint16, row pitch bins_pitch), `flag` (dev u32, zeroed here) = 1 if the tensor is
// not the integral histogram of a bin map.  `gsum` scratch of 8 * width * height bytes is
// needed when bins > 128 (else may be null).
spct_status ih_recover_bins(const spct_ih& t, uint16_t* bins, int64_t bins_pitch, uint32_t* flag, uint32_t* gsum,
                            cudaStream_t s) {
    using namespace spct_tmatch;
    const int ngroups = static_cast<int>(ceil_div(t.bins, kGroup));
    cudaMemsetAsync(flag, 0, sizeof(uint32_t), s);
    if (ngroups > 1) {
        if (!gsum) return contract("ih_recover_bins: scratch needed above 128 bins");
        cudaMemsetAsync(gsum, 0, static_cast<size_t>(t.width) * t.height * 8, s);
    }
    // bands: about four waves of the SMs' resident CTA slots
    const int nstrips = static_cast<int>(ceil_div(t.width, kStrip));
    const int64_t want = std::max<int64_t>(1, ceil_div(static_cast<int64_t>(device_sms()) * 4,
                                                       static_cast<int64_t>(nstrips) * ngroups));
    const int band_rows = static_cast<int>(std::max<int64_t>(16, ceil_div(t.height, want)));
    dim3 grid(nstrips, static_cast<unsigned>(ceil_div(t.height, band_rows)), ngroups);
    const int prof = prof_begin("ih_recover_bins", s);
    ih_bins_kernel<<<grid, 32 * kWarps, 0, s>>>(t, band_rows, bins, bins_pitch, gsum, flag);
    prof_end(prof, s);
    if (auto st = launch_status("ih_bins_kernel")) return st;
    if (ngroups > 1) {
        const int64_t n = static_cast<int64_t>(t.width) * t.height;
        const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 148 * 16));
        bins_finalize_kernel<<<blocks, 256, 0, s>>>(gsum, n, t.width, t.bins, bins, bins_pitch, flag);
        if (auto st = launch_status("bins_finalize_kernel")) return st;
    }
    return SPCT_OK;
}

}  // namespace spct_impl
