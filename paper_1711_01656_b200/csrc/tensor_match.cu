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

#include <cuda.h>
#include <cudaTypedefs.h>

#include "spct_internal.h"

using namespace spct_dev;
using namespace spct_impl;

namespace spct_tmatch {

constexpr int kWarps = 8;
constexpr int kPlanes = 16;                    // planes per warp
constexpr int kGroup = kWarps * kPlanes;       // bins per CTA (grid.z = bin groups)
constexpr int kStages = 3;                     // rows of every plane in flight per warp
constexpr int kRowWords = kStrip + 4;          // staged plane row: 4 words left of the strip + the strip
constexpr size_t kStageBytes = size_t(kWarps) * kPlanes * kRowWords * 4;
constexpr size_t kSmemBytes = kStages * kStageBytes + 2 * kStrip * 4 + kStages * kWarps * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Wait for a ring stage; a copy that never lands (a bug, not a data condition) traps after
// ~10 s instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (!mbar_try(bar, parity)) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 10000000000ull) __trap();
    }
}
// One TMA box {132 words, 1 row, 16 planes} of the tensor (tensor map `tm`: x = word of the
// row, y = row, z = plane) at (x, y, z) into shared memory, completing on `bar`.  Elements
// outside the tensor (left of column 0, planes past the slab) arrive as zeros.
constexpr uint32_t kBoxBytes = kPlanes * kRowWords * 4;
__device__ __forceinline__ void tma_box(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// CTA = (128-column strip, band of rows, group of 128 bins); warp w owns bins 128 g + 16 w
// .. +15; lane l owns columns 4l .. 4l+3 of the strip.  Each warp streams its own planes:
// per row, one TMA box (the 16 plane rows of the strip plus the 4 words to its left) into
// a 3-stage shared ring armed on the warp's mbarrier, so three rows of every plane are in
// flight without holding registers.  Per plane and column, with h(x) = H_k(y+1, x+1) -
// H_k(y+1, x) the row's horizontal difference (kept from the previous row in registers),
// the pixel's count of bin k is
//     p_k(y, x) = h_y(x) - h_{y-1}(x)                       (two adds per cell)
// and one IMAD folds it into a packed per-pixel sum s += p_k * (k << 8 | 1): with every
// p_k in {0, 1} (OR-accumulated per column and checked once per band) the low byte is
// the pixel's count over the group's bins and the rest the sum of its bins.  The 8 warps'
// sums meet in shared memory (red.shared.add, double-buffered by row parity): one barrier
// per row.  One group: count == 1 gives the bin, written as uint16; several groups: the
// sums go to gsum (u64: bin sum << 32 | count) and bins_finalize_kernel converts.
__global__ void __launch_bounds__(256, 1) ih_bins_kernel(const __grid_constant__ CUtensorMap tm, spct_ih t,
                                                         int band_rows, uint16_t* __restrict__ bins,
                                                         int64_t bins_pitch, unsigned long long* __restrict__ gsum,
                                                         uint32_t* __restrict__ flag) {
    extern __shared__ __align__(128) uint32_t sm[];
    uint32_t* ring = sm;                                              // [stage][warp][plane][132]
    uint32_t* part = ring + kStages * kStageBytes / 4;                // [parity][column]
    uint64_t* bars = reinterpret_cast<uint64_t*>(part + 2 * kStrip);  // [stage][warp]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int xs = blockIdx.x * kStrip, x0 = xs + 4 * lane;
    const int y0 = blockIdx.y * band_rows, y1 = min(t.height, y0 + band_rows);
    const int yfirst = y0 > 0 ? y0 - 1 : y0;  // row y0 - 1 only seeds h
    const int g0 = blockIdx.z * kGroup;
    const int kb = g0 + warp * kPlanes;  // warp's first bin
    const int nk = max(0, min(kPlanes, t.bins - kb));
    // columns past the image edge (row-pitch padding) carry no pixels: not checked
    const int ncols = min(4, max(0, t.width - x0));
    uint32_t* wring = ring + static_cast<int64_t>(warp) * kPlanes * kRowWords;  // stage 0 of the warp

    if (lane == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(&bars[st * kWarps + warp], 1);
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
    }
    for (int i = threadIdx.x; i < 2 * kStrip; i += blockDim.x) part[i] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    auto issue = [&](int y) {  // the warp's planes of row y into stage (y - yfirst) % kStages
        if (y >= y1 || nk == 0) return;
        __syncwarp();
        if (lane == 0) {
            const int st = (y - yfirst) % kStages;
            uint64_t* bar = &bars[st * kWarps + warp];
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar, kBoxBytes);
            tma_box(wring + st * (kWarps * kPlanes * kRowWords), &tm, xs - 4, y, kb, bar);
        }
    };
    for (int i = 0; i < kStages; ++i) issue(yfirst + i);

    uint32_t hp[kPlanes][4];  // h of the previous row (row -1: 0)
#pragma unroll
    for (int k = 0; k < kPlanes; ++k) hp[k][0] = hp[k][1] = hp[k][2] = hp[k][3] = 0;
    uint32_t bits[4] = {0, 0, 0, 0};  // OR of every p_k per column: all in {0, 1} <=> (bits & ~1) == 0
    bool bad = false;

    // one row of the warp's planes: h, p, packed sums (SEED: only refresh h)
    auto row_pass = [&](int y, auto seed_tag, uint32_t (&acc)[4]) {
        constexpr bool SEED = decltype(seed_tag)::value;
        const int st = (y - yfirst) % kStages;
        mbar_wait(&bars[st * kWarps + warp], static_cast<uint32_t>(((y - yfirst) / kStages) & 1));
        const uint32_t* rows = wring + st * (kWarps * kPlanes * kRowWords);
#pragma unroll
        for (int k = 0; k < kPlanes; ++k) {
            if (k < nk) {
                const uint4 c = *reinterpret_cast<const uint4*>(rows + k * kRowWords + 4 + 4 * lane);
                const uint32_t w3 = rows[k * kRowWords + 3];
                const uint32_t up = __shfl_up_sync(0xffffffffu, c.w, 1);
                const uint32_t left = lane ? up : w3;
                const uint32_t h[4] = {c.x - left, c.y - c.x, c.z - c.y, c.w - c.z};
                if (!SEED) {
                    const uint32_t wk = (static_cast<uint32_t>(warp * kPlanes + k) << 8) | 1u;
                    uint32_t p[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        p[j] = h[j] - hp[k][j];
                        acc[j] += p[j] * wk;
                        bits[j] |= p[j];
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) hp[k][j] = h[j];
            }
        }
        issue(y + kStages);  // this stage is consumed: refill it with row y + 3
    };

    if (nk && yfirst < y0) {
        uint32_t dummy[4];
        row_pass(yfirst, std::true_type{}, dummy);
    }
#pragma unroll 1
    for (int y = y0; y < y1; ++y) {
        uint32_t acc[4] = {0, 0, 0, 0};
        if (nk) {
            row_pass(y, std::false_type{}, acc);
            uint32_t* pr = part + (y & 1) * kStrip + 4 * lane;
#pragma unroll
            for (int j = 0; j < 4; ++j) atomicAdd(pr + j, acc[j]);
        }
        __syncthreads();
        if (threadIdx.x < kStrip) {
            const int c = threadIdx.x, x = xs + c;
            uint32_t* pp = part + (y & 1) * kStrip + c;
            const uint32_t s = *pp;
            *pp = 0;  // reused two rows on, after the next row's barrier
            if (x < t.width) {
                const uint32_t cnt = s & 0xFFu, si = (s >> 8) + static_cast<uint32_t>(g0);
                if (gridDim.z == 1) {
                    const bool ok = cnt == 1u && si < static_cast<uint32_t>(t.bins);
                    bins[static_cast<int64_t>(y) * bins_pitch + x] = ok ? static_cast<uint16_t>(si) : 0;
                    bad |= !ok;
                } else if (cnt) {
                    const unsigned long long add =
                        (static_cast<unsigned long long>((s >> 8) + static_cast<uint32_t>(g0) * cnt) << 32) | cnt;
                    atomicAdd(gsum + static_cast<int64_t>(y) * t.width + x, add);
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) bad |= j < ncols && (bits[j] & ~1u) != 0;
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1u);
}

// Several bin groups: the summed moments -> bins (and the flag).
__global__ void bins_finalize_kernel(const unsigned long long* __restrict__ gsum, int64_t n, int width, int nbins,
                                     uint16_t* __restrict__ bins, int64_t bins_pitch, uint32_t* __restrict__ flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long g = gsum[i];
        const uint32_t si = static_cast<uint32_t>(g >> 32), sc = static_cast<uint32_t>(g);
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
namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}
}  // namespace

spct_status ih_recover_bins(const spct_ih& t, uint16_t* bins, int64_t bins_pitch, uint32_t* flag, uint32_t* gsum,
                            cudaStream_t s) {
    using namespace spct_tmatch;
    // the tensor as a 3-D TMA map: x = word of the row (row_pitch), y = row, z = plane
    CUtensorMap tm;
    {
        const auto encode = tensor_map_encoder();
        if (!encode) return SPCT_ERR_CUDA;
        if (reinterpret_cast<uintptr_t>(t.data) % 16 != 0)
            return contract("hist_match: tensor data must be 16-byte aligned");
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(t.row_pitch), static_cast<cuuint64_t>(t.height),
                                    static_cast<cuuint64_t>(t.bins)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(t.row_pitch) * 4,
                                       static_cast<cuuint64_t>(t.plane_pitch) * 4};
        const cuuint32_t box[3] = {static_cast<cuuint32_t>(kRowWords), 1u, static_cast<cuuint32_t>(kPlanes)};
        const cuuint32_t estr[3] = {1u, 1u, 1u};
        if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(t.data), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return contract("hist_match: tensor layout not expressible as a TMA map");
    }
    const int ngroups = static_cast<int>(ceil_div(t.bins, kGroup));
    cudaMemsetAsync(flag, 0, sizeof(uint32_t), s);
    if (ngroups > 1) {
        if (!gsum) return contract("ih_recover_bins: scratch needed above 128 bins");
        cudaMemsetAsync(gsum, 0, static_cast<size_t>(t.width) * t.height * 8, s);
    }
    // bands: about eight waves of one CTA per SM (each band re-reads one seed row)
    const int nstrips = static_cast<int>(ceil_div(t.width, kStrip));
    const int64_t want = std::max<int64_t>(1, ceil_div(static_cast<int64_t>(device_sms()) * 8,
                                                       static_cast<int64_t>(nstrips) * ngroups));
    const int band_rows = static_cast<int>(std::max<int64_t>(32, ceil_div(t.height, want)));
    dim3 grid(nstrips, static_cast<unsigned>(ceil_div(t.height, band_rows)), ngroups);
    const int prof = prof_begin("ih_recover_bins", s);
    ensure_smem(ih_bins_kernel, kSmemBytes);
    ih_bins_kernel<<<grid, 32 * kWarps, kSmemBytes, s>>>(tm, t, band_rows, bins, bins_pitch,
                                                         reinterpret_cast<unsigned long long*>(gsum), flag);
    prof_end(prof, s);
    if (auto st = launch_status("ih_bins_kernel")) return st;
    if (ngroups > 1) {
        const int64_t n = static_cast<int64_t>(t.width) * t.height;
        const int blocks = static_cast<int>(std::min<int64_t>(ceil_div(n, 256), 148 * 16));
        bins_finalize_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const unsigned long long*>(gsum), n, t.width, t.bins, bins, bins_pitch, flag);
        if (auto st = launch_status("bins_finalize_kernel")) return st;
    }
    return SPCT_OK;
}

}  // namespace spct_impl
