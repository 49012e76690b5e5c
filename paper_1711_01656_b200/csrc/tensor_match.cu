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
constexpr int kStages = 3;                     // rows of every plane in flight per warp
constexpr int kRowWords = kStrip + 4;          // staged plane row: 4 words left of the strip + the strip
constexpr size_t kStageBytes = size_t(kWarps) * kBinsPerWarp * kRowWords * 4;
constexpr size_t kSmemBytes = kStages * kStageBytes + 2 * kWarps * kStrip * 4 + kStages * kWarps * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// One bulk (TMA) copy global -> shared that completes on `bar` (16-byte aligned, size % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// CTA = (128-column strip, band of rows, group of 128 bins); warp w owns bins 128 g + 8 w ..
// +7; lane l owns columns 4l .. 4l+3 of the strip.  Each warp streams its own planes:
// lane 0 issues, per row and plane, one bulk copy of the plane row's 132 words (the strip
// and the 4 words to its left) into a 3-stage shared ring armed on the warp's mbarrier,
// so three rows of every plane are in flight without holding registers.  Per row and
// column the warp accumulates the moments of its planes' vertical differences dv_k =
// H_k(y+1, x+1) - H_k(y, x+1): M = sum_k (k - 128 g) dv_k and N = sum_k dv_k, whose
// horizontal differences are the pixel's bin and count (linearity), and checks every
// p_k = dv_k(x) - dv_k(x - 1) to lie in {0, 1}.  The 16 warps' partials (u16 bin | u16
// count) are summed through shared memory, double-buffered by row parity: one barrier
// per row.  One group: the bin is final and written as uint16; several groups: the
// partials are added into gsum (u32 bin, u32 count) and bins_finalize_kernel converts.
__global__ void __launch_bounds__(512, 1) ih_bins_kernel(spct_ih t, int band_rows, uint16_t* __restrict__ bins,
                                                         int64_t bins_pitch, uint32_t* __restrict__ gsum,
                                                         uint32_t* __restrict__ flag) {
    extern __shared__ __align__(128) uint32_t sm[];
    uint32_t* ring = sm;                                                       // [stage][warp][plane][132]
    uint32_t* part = ring + kStages * kStageBytes / 4;                         // [parity][warp][column]
    uint64_t* bars = reinterpret_cast<uint64_t*>(part + 2 * kWarps * kStrip);  // [stage][warp]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int xs = blockIdx.x * kStrip, x0 = xs + 4 * lane;
    const int y0 = blockIdx.y * band_rows, y1 = min(t.height, y0 + band_rows);
    const int g0 = blockIdx.z * kGroup;
    const int kb = g0 + warp * kBinsPerWarp;  // warp's first bin
    const int nk = max(0, min(kBinsPerWarp, t.bins - kb));
    const bool lane_live = x0 < t.width;
    // columns past the image edge (row-pitch padding) carry no pixels: not checked
    const int ncols = min(4, max(0, t.width - x0));
    // bytes of a staged plane row: the strip (clipped to the row pitch) plus, right of the
    // first strip, the 16 bytes before it (column xs - 1 is word 3)
    const int strip_words = static_cast<int>(t.row_pitch - xs < kStrip ? t.row_pitch - xs : kStrip);
    const int lead = xs > 0 ? 4 : 0;
    const uint32_t row_bytes = static_cast<uint32_t>(4 * (strip_words + lead));
    const uint32_t* src0 = t.data + static_cast<int64_t>(kb) * t.plane_pitch + xs - lead;

    if (lane == 0)
        for (int st = 0; st < kStages; ++st) mbar_init(&bars[st * kWarps + warp], 1);
    if (xs == 0)  // nothing left of the first strip: those words stay 0 in every stage
        for (int i = threadIdx.x; i < kStages * kWarps * kBinsPerWarp; i += blockDim.x) {
            uint32_t* r = ring + static_cast<int64_t>(i) * kRowWords;
            r[0] = r[1] = r[2] = r[3] = 0;
        }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    auto issue = [&](int y) {  // lane 0: the warp's planes of row y into stage (y - y0) % kStages
        if (lane != 0 || y >= y1 || nk == 0) return;
        const int st = (y - y0) % kStages;
        uint64_t* bar = &bars[st * kWarps + warp];
        uint32_t* dst = ring + (static_cast<int64_t>(st) * kWarps + warp) * kBinsPerWarp * kRowWords + (4 - lead);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, row_bytes * nk);
        for (int k = 0; k < nk; ++k)
            bulk_g2s(dst + k * kRowWords, src0 + static_cast<int64_t>(k) * t.plane_pitch +
                                              static_cast<int64_t>(y) * t.row_pitch, row_bytes, bar);
    };
    for (int i = 0; i < kStages; ++i) issue(y0 + i);

    uint32_t prev[kBinsPerWarp][4], prevL[kBinsPerWarp];
#pragma unroll
    for (int i = 0; i < kBinsPerWarp; ++i) {
        uint4 v = make_uint4(0, 0, 0, 0);
        uint32_t l = 0;
        if (y0 > 0 && i < nk) {
            const int64_t off = static_cast<int64_t>(i) * t.plane_pitch + static_cast<int64_t>(y0 - 1) * t.row_pitch;
            if (lane_live) v = *reinterpret_cast<const uint4*>(src0 + lead + 4 * lane + off);
            if (lane == 0 && lead) l = src0[off + 3];
        }
        prev[i][0] = v.x, prev[i][1] = v.y, prev[i][2] = v.z, prev[i][3] = v.w;
        prevL[i] = l;
    }

    const uint32_t kbase = static_cast<uint32_t>(warp * kBinsPerWarp);  // bin relative to the group
#pragma unroll 2
    for (int y = y0; y < y1; ++y) {
        const int st = (y - y0) % kStages;
        if (nk) mbar_wait(&bars[st * kWarps + warp], static_cast<uint32_t>(((y - y0) / kStages) & 1));
        const uint32_t* rows = ring + (static_cast<int64_t>(st) * kWarps + warp) * kBinsPerWarp * kRowWords;
        // pbits: OR of every checked p_k; all in {0, 1} <=> (pbits & ~1) == 0
        uint32_t msum[4] = {0, 0, 0, 0}, nsum[4] = {0, 0, 0, 0}, pbits = 0, mL = 0, nL = 0;
#pragma unroll
        for (int k = 0; k < kBinsPerWarp; ++k) {
            if (k >= nk) break;
            const uint4 c = *reinterpret_cast<const uint4*>(rows + k * kRowWords + 4 + 4 * lane);
            const uint32_t cl = rows[k * kRowWords + 3];
            const uint32_t c4[4] = {c.x, c.y, c.z, c.w};
            uint32_t dv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                dv[j] = c4[j] - prev[k][j];
                prev[k][j] = c4[j];
            }
            const uint32_t dl = cl - prevL[k];  // lane 0: the column left of the strip
            prevL[k] = cl;
            uint32_t left = __shfl_up_sync(0xffffffffu, dv[3], 1);
            if (lane == 0) left = dl;
            const uint32_t kk = kbase + static_cast<uint32_t>(k);
            uint32_t p[4];  // the pixels' counts of bin kk
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                p[j] = dv[j] - (j ? dv[j - 1] : left);
                if (j >= ncols) p[j] = 0;
                msum[j] += kk * dv[j];
                nsum[j] += dv[j];
            }
            pbits |= (p[0] | p[1]) | (p[2] | p[3]);
            mL += kk * left;
            nL += left;
        }
        __syncwarp();
        issue(y + kStages);  // this stage is consumed: refill it with row y + 3
        if (__any_sync(0xffffffffu, (pbits & ~1u) != 0) && lane == 0) atomicOr(flag, 1u);
        // with every p_k in {0, 1} the warp's bin partial is < 8 * 128 and its count <= 8
        const uint32_t mprev[4] = {mL, msum[0], msum[1], msum[2]}, nprev[4] = {nL, nsum[0], nsum[1], nsum[2]};
        uint4 w;
        w.x = ((msum[0] - mprev[0]) & 0xFFFFu) | ((nsum[0] - nprev[0]) << 16);
        w.y = ((msum[1] - mprev[1]) & 0xFFFFu) | ((nsum[1] - nprev[1]) << 16);
        w.z = ((msum[2] - mprev[2]) & 0xFFFFu) | ((nsum[2] - nprev[2]) << 16);
        w.w = ((msum[3] - mprev[3]) & 0xFFFFu) | ((nsum[3] - nprev[3]) << 16);
        *reinterpret_cast<uint4*>(part + ((y & 1) * kWarps + warp) * kStrip + 4 * lane) = w;
        __syncthreads();
        if (threadIdx.x < kStrip) {
            const int c = threadIdx.x, x = xs + c;
            uint32_t s = 0;
#pragma unroll
            for (int w2 = 0; w2 < kWarps; ++w2) s += part[((y & 1) * kWarps + w2) * kStrip + c];
            const uint32_t si = (s & 0xFFFFu) + static_cast<uint32_t>(g0), sc = s >> 16;
            if (x < t.width) {
                if (gridDim.z == 1) {
                    const bool ok = sc == 1u && si < static_cast<uint32_t>(t.bins);
                    bins[static_cast<int64_t>(y) * bins_pitch + x] = ok ? static_cast<uint16_t>(si) : 0;
                    if (!ok) atomicOr(flag, 1u);
                } else if (sc) {
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
    ensure_smem(ih_bins_kernel, kSmemBytes);
    ih_bins_kernel<<<grid, 32 * kWarps, kSmemBytes, s>>>(t, band_rows, bins, bins_pitch, gsum, flag);
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
