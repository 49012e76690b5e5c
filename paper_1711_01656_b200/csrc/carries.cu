// Carry pre-passes of the banded sweep.
//
//   Lt[s][y][kl] = count of slab bin kl in row y, columns [0, 128 s)      (s >= 1)
//   Hb[j-1][kl][x] = H(y0_j, x+1, bin0+kl) = count of kl in rows < y0_j, cols <= x  (j >= 1)
//
// Both are bandwidth-shaped passes over a 1 B/px frame and ~1.5 % of the tensor bytes:
//   carry_rows_kernel   one warp per row, warp-private shared histogram, one strip at a
//                       time (no CTA barriers), pixels prefetched one strip ahead;
//   carry_bands_kernel  one CTA per (band, 128-column strip, 64-bin chunk): per-column
//                       counts of the band into shared memory (one thread per column);
//   carry_hscan_kernel  inclusive scan along x of every (band, bin) row, in place;
//   carry_vscan_kernel  inclusive prefix over bands per (bin, column), in place.
#include "spct_internal.h"

using namespace spct_dev;

namespace spct_carry {

constexpr int kRowWarps = 8;
constexpr int kRowChunk = 512;   // bins per warp histogram pass
constexpr int kBandChunk = 64;

__global__ void __launch_bounds__(256) carry_rows_kernel(QuantParams q, int bin0, int bins, int Lb, int nstrips,
                                                         uint32_t* __restrict__ Lt) {
    __shared__ uint32_t hist_all[kRowWarps][kRowChunk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int y = blockIdx.x * kRowWarps + warp;
    if (y >= q.height) return;
    uint32_t* hist = hist_all[warp];
    const int kc0 = blockIdx.y * kRowChunk;
    const int kcn = min(kRowChunk, Lb - kc0);
    for (int i = lane; i < kcn; i += 32) hist[i] = 0;
    uint64_t raw[4];
    auto load_strip = [&](int s) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int x = s * kStrip + 4 * lane + j;
            raw[j] = x < q.width ? pixel_raw(q, x, y) : 0ull;
        }
    };
    load_strip(0);
    __syncwarp();
    for (int s = 0; s + 1 < nstrips; ++s) {
        uint64_t cur[4] = {raw[0], raw[1], raw[2], raw[3]};
        load_strip(s + 1);  // prefetch; the last strip's pixels are never counted
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (s * kStrip + 4 * lane + j < q.width) {
                const int kl = bin_of_raw(cur[j], q) - bin0 - kc0;
                if (kl >= 0 && kl < kcn && kl + kc0 < bins) atomicAdd(&hist[kl], 1u);
            }
        }
        __syncwarp();
        uint32_t* dst = Lt + (static_cast<int64_t>(s + 1) * q.height + y) * Lb + kc0;
        for (int i = lane; i < kcn; i += 32) dst[i] = hist[i];
        __syncwarp();
    }
}

__global__ void __launch_bounds__(128) carry_bands_kernel(QuantParams q, int bin0, int bins, int Lb, int Wp,
                                                          int band_rows, uint32_t* __restrict__ CC) {
    __shared__ uint32_t cnt[kBandChunk][kStrip];
    const int x = blockIdx.x * kStrip + threadIdx.x;
    const int j = blockIdx.y;
    const int kc0 = blockIdx.z * kBandChunk;
    const int kcn = min(kBandChunk, Lb - kc0);
    for (int i = 0; i < kcn; ++i) cnt[i][threadIdx.x] = 0;
    const int y0 = j * band_rows, y1 = min(q.height, y0 + band_rows);
    if (x < q.width) {
        constexpr int U = 8;
        int y = y0;
        for (; y + U <= y1; y += U) {
            uint64_t r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = pixel_raw(q, x, y + u);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int kl = bin_of_raw(r[u], q) - bin0 - kc0;
                if (kl >= 0 && kl < kcn && kl + kc0 < bins) cnt[kl][threadIdx.x] += 1;
            }
        }
        for (; y < y1; ++y) {
            const int kl = pixel_bin(q, x, y) - bin0 - kc0;
            if (kl >= 0 && kl < kcn && kl + kc0 < bins) cnt[kl][threadIdx.x] += 1;
        }
    }
    for (int i = 0; i < kcn; ++i) CC[(static_cast<int64_t>(j) * Lb + kc0 + i) * Wp + x] = cnt[i][threadIdx.x];
}

// One CTA per (band slot, bin) row of Wp elements: inclusive scan in place.
__global__ void __launch_bounds__(256) carry_hscan_kernel(int Wp, uint32_t* __restrict__ CC) {
    __shared__ uint32_t wsum[8];
    __shared__ uint32_t carry_s;
    uint32_t* row = CC + static_cast<int64_t>(blockIdx.x) * Wp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < Wp; base += 256 * 4) {
        const int x = base + 4 * threadIdx.x;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (x < Wp) v = *reinterpret_cast<const uint4*>(row + x);
        v.y += v.x;
        v.z += v.y;
        v.w += v.z;
        uint32_t inc = v.w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        uint32_t off = carry_s;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        off += inc - v.w;
        if (x < Wp) *reinterpret_cast<uint4*>(row + x) = make_uint4(v.x + off, v.y + off, v.z + off, v.w + off);
        __syncthreads();
        if (threadIdx.x == 255) carry_s = off + v.w;
        __syncthreads();
    }
}

// One thread per (bin, column): running sum over the band slots, in place.
__global__ void carry_vscan_kernel(int nslots, int64_t row_elems, uint32_t* __restrict__ CC) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= row_elems) return;
    uint32_t acc = 0;
    for (int j = 0; j < nslots; ++j) {
        uint32_t* p = CC + j * row_elems + i;
        acc += *p;
        *p = acc;
    }
}

}  // namespace spct_carry

namespace spct_impl {

using namespace spct_carry;

spct_status build_carries(const QuantParams& q, const spct_ih& out, const BuildPlan& p, void* workspace,
                          size_t ws_bytes, cudaStream_t s, uint32_t** Lt, uint32_t** Hb) {
    *Lt = nullptr;
    *Hb = nullptr;
    if (p.lt_bytes + p.hb_bytes > 0 && (!workspace || ws_bytes < p.lt_bytes + p.hb_bytes))
        return contract("ih_build: workspace too small (query spct_cu_ih_build_workspace)");
    char* ws = static_cast<char*>(workspace);
    if (p.lt_bytes) {
        *Lt = reinterpret_cast<uint32_t*>(ws);
        dim3 g(static_cast<unsigned>(ceil_div(q.height, kRowWarps)), static_cast<unsigned>(ceil_div(p.Lb, kRowChunk)));
        carry_rows_kernel<<<g, 256, 0, s>>>(q, out.bin0, out.bins, p.Lb, p.nstrips, *Lt);
        if (auto st = launch_status("carry_rows_kernel")) return st;
    }
    if (p.hb_bytes) {
        *Hb = reinterpret_cast<uint32_t*>(ws + p.lt_bytes);
        const int nslots = p.nbands - 1;
        dim3 g(p.nstrips, nslots, static_cast<unsigned>(ceil_div(p.Lb, kBandChunk)));
        carry_bands_kernel<<<g, 128, 0, s>>>(q, out.bin0, out.bins, p.Lb, p.Wp, p.band_rows, *Hb);
        if (auto st = launch_status("carry_bands_kernel")) return st;
        carry_hscan_kernel<<<nslots * p.Lb, 256, 0, s>>>(p.Wp, *Hb);
        if (auto st = launch_status("carry_hscan_kernel")) return st;
        const int64_t row_elems = static_cast<int64_t>(p.Lb) * p.Wp;
        carry_vscan_kernel<<<static_cast<unsigned>(ceil_div(row_elems, 256)), 256, 0, s>>>(nslots, row_elems, *Hb);
        if (auto st = launch_status("carry_vscan_kernel")) return st;
    }
    return SPCT_OK;
}

}  // namespace spct_impl
