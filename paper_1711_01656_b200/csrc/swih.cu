// Spatially weighted local histograms (SWIH) on the device — SURVEY §8(f) next #1, the
// tracker's per-frame histogram channel (track_loop.cpp:260-283).
//
//   build_weighted_tensor  integral.cpp:553-559   H(y,x,k) = sum_{r<y,c<x, bin=k} w(r,c), uint64
//                                                  (16.16 fixed-point weights); device layout
//                                                  unpadded + pitched like spct_ih, 8-byte cells
//   build_quadrant_set     swih.cpp:115-126        the four ramp fields (swih.cpp:86-104,
//                                                  field_value :45-53) generated in the kernel
//   swlh_query_fixed       swih.cpp:128-164        exact int64 quadrant arithmetic, including the
//                                                  "sum % pair_sum" consistency check
//   brute_force_swlh_fixed swih.cpp:166-178        direct pyramid-weighted window sums
//   swlh-distance map      track_loop.cpp:264-283  per valid centre L = clamp01(1 - d/2),
//                                                  d = sum |q_k - model_k|, replicate_borders
// Integer results are bit-identical to the reference.  Normalisation divides in FP64
// (the reference divides in x87 long double, then rounds to double: <= 1 ulp apart).
#include <algorithm>

#include "spct_internal.h"

using namespace spct_impl;

namespace spct_swih {

struct Ext {
    int sxl, sxr, syt, syb, c;
};

__host__ __device__ inline Ext extents(int kw, int kh) {  // kernel_extents, swih.cpp:19-27
    Ext e;
    e.sxl = kw / 2;
    e.sxr = kw - e.sxl;
    e.syt = kh / 2;
    e.syb = kh - e.syt;
    e.c = e.sxl + e.syt + 1;
    return e;
}

// field_value (swih.cpp:45-53) for dir NW = 0, NE = 1, SW = 2, SE = 3; an integer-valued
// ramp, so quantize_weight (llround(v * 2^16)) is v << 16 exactly.
__host__ __device__ inline int64_t field_int(int dir, int x, int y, int w, int h, int sx, int sy) {
    switch (dir) {
        case 3: return 1 + int64_t(sx) * (w - 1 - x) + int64_t(sy) * (h - 1 - y);
        case 0: return 1 + int64_t(sx) * x + int64_t(sy) * y;
        case 1: return 1 + int64_t(sx) * (w - 1 - x) + int64_t(sy) * y;
        default: return 1 + int64_t(sx) * x + int64_t(sy) * (h - 1 - y);
    }
}

// Pass 1: one CTA per (row, bin): the row prefix of w * [bin == k] (block scan, uint64).
__global__ void __launch_bounds__(256) wih_row_kernel(const uint16_t* __restrict__ bins, int64_t pitch,
                                                      const uint64_t* __restrict__ wts, int dir, int sx, int sy,
                                                      spct_wih t) {
    __shared__ uint64_t wsum[8];
    const int y = blockIdx.x, k = blockIdx.y;
    const int per = (t.width + 255) / 256;
    const int x0 = threadIdx.x * per, x1 = min(t.width, x0 + per);
    const uint16_t* brow = bins + static_cast<int64_t>(y) * pitch;
    auto weight = [&](int x) -> uint64_t {
        if (wts) return wts[static_cast<int64_t>(y) * pitch + x];
        return static_cast<uint64_t>(field_int(dir, x, y, t.width, t.height, sx, sy)) << 16;
    };
    uint64_t local = 0;
    for (int x = x0; x < x1; ++x)
        if (brow[x] == k) local += weight(x);
    // block exclusive scan of the per-thread sums
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t inc = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint64_t run = inc - local;
    for (int w = 0; w < warp; ++w) run += wsum[w];
    uint64_t* row = t.data + static_cast<int64_t>(k) * t.plane_pitch + static_cast<int64_t>(y) * t.row_pitch;
    for (int x = x0; x < x1; ++x) {
        if (brow[x] == k) run += weight(x);
        row[x] = run;
    }
}

// Pass 2: thread per (bin, column): running sum down the rows, in place.
__global__ void wih_col_kernel(spct_wih t) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<int64_t>(t.bins) * t.width) return;
    const int k = static_cast<int>(i / t.width), x = static_cast<int>(i % t.width);
    uint64_t* p = t.data + static_cast<int64_t>(k) * t.plane_pitch + x;
    uint64_t acc = 0;
    for (int y = 0; y < t.height; ++y) {
        acc += p[static_cast<int64_t>(y) * t.row_pitch];
        p[static_cast<int64_t>(y) * t.row_pitch] = acc;
    }
}

// ---- single-pass build (widths <= 4096): a CTA spans the whole row width, so the only
// carry is the weighted column sum above its band.
constexpr int kSweepThreads = 256;

__device__ __forceinline__ uint64_t pixel_weight(const uint64_t* __restrict__ wts, int64_t pitch, int dir, int sx,
                                                 int sy, int x, int y, int w, int h) {
    if (wts) return __ldg(wts + static_cast<int64_t>(y) * pitch + x);
    return static_cast<uint64_t>(field_int(dir, x, y, w, h, sx, sy)) << 16;
}

// T[j][k][x] = sum over the rows of band j of w * [bin == k], bins [kc0, kc0 + kcn); one
// thread per column (its counters in shared memory, no atomics).
__global__ void __launch_bounds__(kSweepThreads) wih_band_kernel(const uint16_t* __restrict__ bins, int64_t pitch,
                                                                 const uint64_t* __restrict__ wts, int dir, int sx,
                                                                 int sy, int w, int h, int nbins, int band_rows,
                                                                 int kc0, int kcn, uint64_t* __restrict__ T) {
    extern __shared__ uint64_t acc[];  // [kcn][256]
    const int x = blockIdx.x * kSweepThreads + threadIdx.x, j = blockIdx.y;
    for (int k = 0; k < kcn; ++k) acc[k * kSweepThreads + threadIdx.x] = 0;
    if (x < w) {
        const int y0 = j * band_rows, y1 = min(h, y0 + band_rows);
        for (int y = y0; y < y1; ++y) {
            const int b = static_cast<int>(__ldg(bins + static_cast<int64_t>(y) * pitch + x)) - kc0;
            if (static_cast<unsigned>(b) < static_cast<unsigned>(kcn))
                acc[b * kSweepThreads + threadIdx.x] += pixel_weight(wts, pitch, dir, sx, sy, x, y, w, h);
        }
        for (int k = 0; k < kcn; ++k) T[(static_cast<int64_t>(j) * nbins + kc0 + k) * w + x] = acc[k * kSweepThreads + threadIdx.x];
    }
}

// In place over bands: T[j] = column sums over rows < y0_{j+1}.
__global__ void wih_band_prefix_kernel(uint64_t* __restrict__ T, int64_t plane, int nb) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= plane) return;
    uint64_t run = 0;
    constexpr int U = 8;  // loads in flight
    for (int j0 = 0; j0 < nb; j0 += U) {
        uint64_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = j0 + u < nb ? T[(j0 + u) * plane + i] : 0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (j0 + u < nb) {
                run += v[u];
                T[(j0 + u) * plane + i] = run;
            }
    }
}

// Exclusive block scan of NBC values per thread; one barrier (sh double-buffered by the
// caller's parity).
template <int NBC>
__device__ __forceinline__ void block_excl_scan_u64(const uint64_t (&v)[NBC], uint64_t (&e)[NBC], uint64_t* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t inc[NBC];
#pragma unroll
    for (int k = 0; k < NBC; ++k) inc[k] = v[k];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
#pragma unroll
        for (int k = 0; k < NBC; ++k) {
            const uint64_t t = __shfl_up_sync(0xffffffffu, inc[k], o);
            if (lane >= o) inc[k] += t;
        }
    if (lane == 31)
#pragma unroll
        for (int k = 0; k < NBC; ++k) sh[warp * NBC + k] = inc[k];
    __syncthreads();
    // lanes 0..7 hold the 8 warp totals: a 3-step scan, then this warp's exclusive base
#pragma unroll
    for (int k = 0; k < NBC; ++k) {
        const uint64_t wt = lane < 8 ? sh[lane * NBC + k] : 0;
        uint64_t ws = wt;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint64_t t = __shfl_up_sync(0xffffffffu, ws, o);
            if (lane >= o) ws += t;
        }
        e[k] = __shfl_sync(0xffffffffu, ws - wt, warp) + inc[k] - v[k];
    }
}

// CTA = (band, NBC bins); thread t owns columns [t PER, t PER + PER) of every row.
template <int PER, int NBC>
__global__ void __launch_bounds__(kSweepThreads) wih_sweep_kernel(const uint16_t* __restrict__ bins, int64_t pitch,
                                                                  const uint64_t* __restrict__ wts, int dir, int sx,
                                                                  int sy, spct_wih t, int band_rows,
                                                                  const uint64_t* __restrict__ C) {
    __shared__ uint64_t sh[2][8 * NBC];
    const int j = blockIdx.x, k0 = blockIdx.y * NBC;
    const int W = t.width, Hh = t.height;
    const int x0 = threadIdx.x * PER;
    const int y0 = j * band_rows, y1 = min(Hh, y0 + band_rows);
    uint64_t V[NBC][PER];
    {   // the band-top row: row prefix of the column sums above the band
        uint64_t tot[NBC], e[NBC];
#pragma unroll
        for (int k = 0; k < NBC; ++k) {
            uint64_t run = 0;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int x = x0 + i;
                if (j > 0 && x < W && k0 + k < t.bins) run += C[(static_cast<int64_t>(j - 1) * t.bins + k0 + k) * W + x];
                V[k][i] = run;
            }
            tot[k] = run;
        }
        block_excl_scan_u64<NBC>(tot, e, sh[(y0 + 1) & 1]);  // the parity of row y0 - 1
#pragma unroll
        for (int k = 0; k < NBC; ++k)
#pragma unroll
            for (int i = 0; i < PER; ++i) V[k][i] += e[k];
    }
    // the row's bins arrive one row ahead (one vector load when the row is aligned)
    const bool vec = PER >= 4 && (pitch % 4) == 0 && (reinterpret_cast<uintptr_t>(bins) & 7) == 0 && x0 + PER <= W;
    auto load_bins = [&](int y, int (&b)[PER]) {
        const uint16_t* r = bins + static_cast<int64_t>(y) * pitch + x0;
        if (vec) {
#pragma unroll
            for (int i = 0; i < PER; i += 4) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(r + i));
                b[i] = v.x & 0xFFFF;
                b[i + 1] = v.x >> 16;
                b[i + 2] = v.y & 0xFFFF;
                b[i + 3] = v.y >> 16;
            }
        } else {
#pragma unroll
            for (int i = 0; i < PER; ++i) b[i] = x0 + i < W ? static_cast<int>(__ldg(r + i)) : -1;
        }
    };
    int bn[PER];
    if (y0 < y1) load_bins(y0, bn);
    for (int y = y0; y < y1; ++y) {
        int b[PER];
        uint64_t wv[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) b[i] = bn[i];
        if (y + 1 < y1) load_bins(y + 1, bn);
#pragma unroll
        for (int i = 0; i < PER; ++i) wv[i] = x0 + i < W ? pixel_weight(wts, pitch, dir, sx, sy, x0 + i, y, W, Hh) : 0;
        uint64_t p[NBC][PER], tot[NBC], e[NBC];
#pragma unroll
        for (int k = 0; k < NBC; ++k) {
            uint64_t run = 0;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                run += b[i] == k0 + k ? wv[i] : 0;
                p[k][i] = run;
            }
            tot[k] = run;
        }
        block_excl_scan_u64<NBC>(tot, e, sh[y & 1]);
#pragma unroll
        for (int k = 0; k < NBC; ++k) {
            if (k0 + k >= t.bins) break;
            uint64_t* row = t.data + static_cast<int64_t>(k0 + k) * t.plane_pitch + static_cast<int64_t>(y) * t.row_pitch;
#pragma unroll
            for (int i = 0; i < PER; ++i) V[k][i] += e[k] + p[k][i];
            if (PER >= 2 && x0 + PER <= W) {  // 16-byte stores (row pitch is a multiple of 16 cells)
#pragma unroll
                for (int i = 0; i < PER; i += 2)
                    *reinterpret_cast<ulonglong2*>(row + x0 + i) = make_ulonglong2(V[k][i], V[k][i + 1]);
            } else {
#pragma unroll
                for (int i = 0; i < PER; ++i)
                    if (x0 + i < W) row[x0 + i] = V[k][i];
            }
        }
    }
}

__global__ void wih_export_kernel(spct_wih t, int k0, int k1, uint64_t* __restrict__ dst) {
    const int64_t W1 = t.width + 1, H1 = t.height + 1;
    const int64_t n = static_cast<int64_t>(k1 - k0) * H1 * W1;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = i / (H1 * W1), rem = i % (H1 * W1);
        const int64_t y = rem / W1, x = rem % W1;
        dst[i] = (y > 0 && x > 0) ? t.data[(k0 + k) * t.plane_pitch + (y - 1) * t.row_pitch + (x - 1)] : 0ull;
    }
}

// region_count (integral.cpp:569-577) on the unpadded layout, uint64 wrap arithmetic.
__device__ __forceinline__ uint64_t H(const spct_wih& t, int k, int y, int x) {
    return (y > 0 && x > 0) ? t.data[static_cast<int64_t>(k) * t.plane_pitch + static_cast<int64_t>(y - 1) * t.row_pitch +
                                     (x - 1)]
                            : 0ull;
}
__device__ __forceinline__ uint64_t region(const spct_wih& t, int k, int x, int y, int w, int h) {
    return H(t, k, y + h, x + w) - H(t, k, y, x + w) - H(t, k, y + h, x) + H(t, k, y, x);
}

__global__ void wih_region_kernel(spct_wih t, const int32_t* __restrict__ rects, int n, uint64_t* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;  // (rect, bin)
    if (i >= static_cast<int64_t>(n) * t.bins) return;
    const int r = static_cast<int>(i / t.bins), k = static_cast<int>(i % t.bins);
    const int32_t* q = rects + 4 * r;
    out[i] = region(t, k, q[0], q[1], q[2], q[3]);
}

struct QuadSet {
    spct_wih t[4];  // NW, NE, SW, SE
    int kw, kh, sx, sy;
    int64_t pair_sum;
};

// swlh_query_fixed (swih.cpp:128-164) for bin k at centre (cx, cy); sets *bad on the
// reference's consistency failure.
__device__ int64_t swlh_bin(const QuadSet& s, int k, int cx, int cy, unsigned* bad) {
    const Ext e = extents(s.kw, s.kh);
    const int W = s.t[0].width, Hh = s.t[0].height;
    // quadrant_geometry (swih.cpp:57-64): rect and centre-adjacent anchor
    const int rx[4] = {cx - e.sxl, cx, cx - e.sxl, cx}, ry[4] = {cy - e.syt, cy - e.syt, cy, cy};
    const int rw[4] = {e.sxl, e.sxr, e.sxl, e.sxr}, rh[4] = {e.syt, e.syt, e.syb, e.syb};
    const int adx[4] = {-1, 0, -1, 0}, ady[4] = {-1, -1, 0, 0};
    int64_t out = 0;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        if (rw[d] == 0 || rh[d] == 0) continue;
        const int opp = 3 - d;  // NW <-> SE, NE <-> SW
        const int64_t field_at_anchor = field_int(d, cx + adx[d], cy + ady[d], W, Hh, s.sx, s.sy);
        const int64_t true_at_anchor = e.c - abs(adx[d]) - abs(ady[d]);
        const int64_t delta = field_at_anchor - true_at_anchor;
        const uint64_t fd = region(s.t[d], k, rx[d], ry[d], rw[d], rh[d]);
        const uint64_t fo = region(s.t[opp], k, rx[d], ry[d], rw[d], rh[d]);
        const int64_t sum = static_cast<int64_t>(fd + fo);
        if (sum % s.pair_sum != 0) atomicOr(bad, 1u);
        const int64_t count_fx = sum / s.pair_sum;
        out += static_cast<int64_t>(fd) - delta * count_fx;
    }
    return out;
}

__global__ void swlh_query_kernel(QuadSet s, const int32_t* __restrict__ centres, int n, int64_t* __restrict__ out,
                                  unsigned* __restrict__ bad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;  // (centre, bin)
    const int bins = s.t[0].bins;
    if (i >= static_cast<int64_t>(n) * bins) return;
    const int q = static_cast<int>(i / bins), k = static_cast<int>(i % bins);
    out[i] = swlh_bin(s, k, centres[2 * q], centres[2 * q + 1], bad);
}

__global__ void swlh_brute_kernel(const uint16_t* __restrict__ bins, int64_t pitch, int nbins, int kw, int kh,
                                  const int32_t* __restrict__ centres, int n, int64_t* __restrict__ out) {
    const int q = blockIdx.x;
    if (q >= n) return;
    const Ext e = extents(kw, kh);
    const int cx = centres[2 * q], cy = centres[2 * q + 1];
    for (int k = threadIdx.x; k < nbins; k += blockDim.x) {
        int64_t acc = 0;
        for (int dy = -e.syt; dy < e.syb; ++dy)
            for (int dx = -e.sxl; dx < e.sxr; ++dx)
                if (bins[static_cast<int64_t>(cy + dy) * pitch + cx + dx] == k)
                    acc += static_cast<int64_t>(e.c - abs(dx) - abs(dy)) * 65536;
        out[static_cast<int64_t>(q) * nbins + k] = acc;
    }
}

// track_loop.cpp:270-279 at every valid centre; `total` is the (constant) kernel mass.
__global__ void swlh_map_kernel(QuadSet s, const double* __restrict__ model, double total, double* __restrict__ map,
                                unsigned* __restrict__ bad) {
    const Ext e = extents(s.kw, s.kh);
    const int W = s.t[0].width, Hh = s.t[0].height, bins = s.t[0].bins;
    const int nu = W - s.kw + 1, nv = Hh - s.kh + 1;
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<int64_t>(nu) * nv) return;
    const int cx = e.sxl + static_cast<int>(i % nu), cy = e.syt + static_cast<int>(i / nu);
    double d = 0.0;
    for (int k = 0; k < bins; ++k) {
        const double q = __ddiv_rn(static_cast<double>(swlh_bin(s, k, cx, cy, bad)), total);
        d = __dadd_rn(d, fabs(__dsub_rn(q, model[k])));
    }
    const double L = __dsub_rn(1.0, __ddiv_rn(d, 2.0));
    map[static_cast<int64_t>(cy) * W + cx] = L < 0.0 ? 0.0 : (L > 1.0 ? 1.0 : L);
}

// replicate_borders (track_loop.cpp:56-64) of the valid region [x0,x1] x [y0,y1].
__global__ void replicate_kernel(double* __restrict__ map, int W, int Hh, int x0, int x1, int y0, int y1) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<int64_t>(W) * Hh) return;
    const int x = static_cast<int>(i % W), y = static_cast<int>(i / W);
    const int sx = x < x0 ? x0 : (x > x1 ? x1 : x), sy = y < y0 ? y0 : (y > y1 ? y1 : y);
    if (sx != x || sy != y) map[i] = map[static_cast<int64_t>(sy) * W + sx];
}

__global__ void fill_kernel(double* __restrict__ map, int64_t n, double v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        map[i] = v;
}

int blocks_for(int64_t n, int b) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + b - 1) / b, 1 << 30))); }

spct_status check_wih(const spct_wih* t) {
    if (!t || !t->data) return contract("weighted tensor: null descriptor or data");
    if (!(t->width > 0 && t->height > 0 && t->bins >= 1)) return contract("weighted tensor: empty dims");
    if (t->row_pitch < t->width || t->plane_pitch < t->row_pitch * t->height)
        return contract("weighted tensor: bad pitches");
    return SPCT_OK;
}

spct_status check_set(const spct_wih* set4, int kw, int kh, QuadSet* s) {
    for (int d = 0; d < 4; ++d) {
        if (auto st = check_wih(set4 + d)) return st;
        if (set4[d].width != set4[0].width || set4[d].height != set4[0].height || set4[d].bins != set4[0].bins)
            return contract("swlh_query: quadrant tensors differ in shape");
        s->t[d] = set4[d];
    }
    if (!(kw >= 1 && kh >= 1)) return contract("kernel extents must be >= 1");  // swih.cpp:20
    s->kw = kw;
    s->kh = kh;
    s->sx = kw >= 3 ? 1 : 0;  // ramp_slopes, swih.cpp:39-42
    s->sy = kh >= 3 ? 1 : 0;
    // S = w_dir + w_opp at every pixel (swih.cpp:119-120); tensor sums are S * count * 2^16
    s->pair_sum = 2 + int64_t(s->sx) * (set4[0].width - 1) + int64_t(s->sy) * (set4[0].height - 1);
    return SPCT_OK;
}

template <int PER, int NBC>
spct_status wih_sweep_launch(const uint16_t* bins, int64_t pitch, const uint64_t* wts, int dir, int sx, int sy,
                             const spct_wih& t, cudaStream_t s) {
    // bands: about two waves of 256-thread CTAs (two resident per SM at ~124 registers),
    // rows >= 16
    const int groups = static_cast<int>(ceil_div(t.bins, NBC));
    int sms = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t want = static_cast<int64_t>(sms) * 2 * 2;
    int nbands = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(t.height / 16, ceil_div(want, groups))));
    const int band_rows = static_cast<int>(ceil_div(t.height, nbands));
    nbands = static_cast<int>(ceil_div(t.height, band_rows));
    uint64_t* C = nullptr;
    if (nbands > 1) {
        const int64_t plane = static_cast<int64_t>(t.bins) * t.width;
        if (auto st = cuda_status(malloc_async(&C, static_cast<size_t>(nbands - 1) * plane * 8, s), "wih alloc"))
            return st;
        const int kc = std::min(t.bins, 64);
        const size_t smem = static_cast<size_t>(kc) * kSweepThreads * 8;
        ensure_smem(wih_band_kernel, 64 * kSweepThreads * 8);
        for (int kc0 = 0; kc0 < t.bins; kc0 += kc) {
            const int kcn = std::min(kc, t.bins - kc0);
            wih_band_kernel<<<dim3(static_cast<unsigned>(ceil_div(t.width, kSweepThreads)), nbands - 1), kSweepThreads,
                              smem, s>>>(bins, pitch, wts, dir, sx, sy, t.width, t.height, t.bins, band_rows, kc0, kcn,
                                         C);
        }
        if (auto st = launch_status("wih_band_kernel")) {
            cudaFreeAsync(C, s);
            return st;
        }
        wih_band_prefix_kernel<<<blocks_for(plane, 256), 256, 0, s>>>(C, plane, nbands - 1);
    }
    wih_sweep_kernel<PER, NBC><<<dim3(nbands, groups), kSweepThreads, 0, s>>>(bins, pitch, wts, dir, sx, sy, t, band_rows,
                                                                           C);
    const spct_status st = launch_status("wih_sweep_kernel");
    if (C) cudaFreeAsync(C, s);
    return st;
}

spct_status wih_sweep(const uint16_t* bins, int64_t pitch, const uint64_t* wts, int dir, int sx, int sy,
                      const spct_wih& t, cudaStream_t s) {
    const int per = static_cast<int>(ceil_div(t.width, kSweepThreads));
    if (per <= 1) return wih_sweep_launch<1, 16>(bins, pitch, wts, dir, sx, sy, t, s);
    if (per <= 2) return wih_sweep_launch<2, 8>(bins, pitch, wts, dir, sx, sy, t, s);
    if (per <= 4) return wih_sweep_launch<4, 4>(bins, pitch, wts, dir, sx, sy, t, s);
    if (per <= 8) return wih_sweep_launch<8, 2>(bins, pitch, wts, dir, sx, sy, t, s);
    return wih_sweep_launch<16, 1>(bins, pitch, wts, dir, sx, sy, t, s);
}

}  // namespace spct_swih

using namespace spct_swih;

extern "C" spct_status spct_cu_wih_layout(int width, int height, int bins, int64_t* row_pitch, int64_t* plane_pitch,
                                          uint64_t* bytes) {
    if (!(width > 0 && height > 0 && bins >= 1)) return contract("weighted tensor: empty dims");
    if (!row_pitch || !plane_pitch || !bytes) return contract("wih_layout: null argument");
    *row_pitch = round_up(width, 16);  // 128-byte rows of uint64
    *plane_pitch = *row_pitch * height;
    *bytes = static_cast<uint64_t>(*plane_pitch) * bins * 8;
    return SPCT_OK;
}

extern "C" spct_status spct_cu_wih_build(const uint16_t* bins, int64_t pitch, const uint64_t* weights, int field_dir,
                                         int kw, int kh, const spct_wih* out, void* stream) {
    if (auto st = check_wih(out)) return st;
    if (!bins || pitch < out->width) return contract("build_weighted_tensor: bad bin map");
    if (!weights && !(field_dir >= 0 && field_dir <= 3 && kw >= 1 && kh >= 1))
        return contract("build_weighted_tensor: need weights or a quadrant field");
    cudaStream_t s = as_stream(stream);
    const int sx = kw >= 3 ? 1 : 0, sy = kh >= 3 ? 1 : 0;
    if (out->width > kSweepThreads * 16) {  // wider than one CTA's row span: row pass + column pass
        wih_row_kernel<<<dim3(out->height, out->bins), 256, 0, s>>>(bins, pitch, weights, field_dir, sx, sy, *out);
        if (auto st = launch_status("wih_row_kernel")) return st;
        const int64_t nc = static_cast<int64_t>(out->bins) * out->width;
        wih_col_kernel<<<blocks_for(nc, 256), 256, 0, s>>>(*out);
        return launch_status("wih_col_kernel");
    }
    return wih_sweep(bins, pitch, weights, field_dir, sx, sy, *out, s);
}

extern "C" spct_status spct_cu_wih_export_u64(const spct_wih* t, int k0, int k1, uint64_t* dst, void* stream) {
    if (auto st = check_wih(t)) return st;
    if (!(0 <= k0 && k0 <= k1 && k1 <= t->bins)) return contract("wih_export: plane range outside the tensor");
    if (k0 == k1) return SPCT_OK;
    if (!dst) return contract("wih_export: null destination");
    const int64_t n = static_cast<int64_t>(k1 - k0) * (t->height + 1) * (t->width + 1);
    wih_export_kernel<<<blocks_for(std::min<int64_t>(n, 148 * 2048), 256), 256, 0, as_stream(stream)>>>(*t, k0, k1, dst);
    return launch_status("wih_export");
}

extern "C" spct_status spct_cu_wih_region_counts(const spct_wih* t, const int32_t* rects, int n, uint64_t* out,
                                                 void* stream) {
    if (auto st = check_wih(t)) return st;
    if (n < 0 || (n > 0 && !(rects && out))) return contract("region_histogram: bad arguments");
    if (n == 0) return SPCT_OK;
    const int64_t m = static_cast<int64_t>(n) * t->bins;
    wih_region_kernel<<<blocks_for(m, 256), 256, 0, as_stream(stream)>>>(*t, rects, n, out);
    return launch_status("wih_region_kernel");
}

extern "C" spct_status spct_cu_swlh_query(const spct_wih* set4, int kw, int kh, const int32_t* centres_host, int n,
                                          int64_t* out, void* stream) {
    QuadSet s{};
    if (auto st = check_set(set4, kw, kh, &s)) return st;
    if (n < 0 || (n > 0 && !(centres_host && out))) return contract("swlh_query: bad arguments");
    const Ext e = extents(kw, kh);
    for (int q = 0; q < n; ++q) {  // check_window (swih.cpp:66-69), on the host copy
        const int cx = centres_host[2 * q], cy = centres_host[2 * q + 1];
        if (!(cx - e.sxl >= 0 && cy - e.syt >= 0 && cx + e.sxr <= s.t[0].width && cy + e.syb <= s.t[0].height))
            return contract("kernel window must lie inside the image");
    }
    if (n == 0) return SPCT_OK;
    cudaStream_t st = as_stream(stream);
    int32_t* dc = nullptr;
    unsigned* bad = nullptr;
    spct_status r = cuda_status(malloc_async(&dc, 8 * static_cast<size_t>(n) + 16, st), "swlh alloc");
    if (!r) {
        bad = reinterpret_cast<unsigned*>(dc + 2 * n);
        cudaMemsetAsync(bad, 0, 4, st);
        r = cuda_status(cudaMemcpyAsync(dc, centres_host, 8 * static_cast<size_t>(n), cudaMemcpyHostToDevice, st), "H2D");
    }
    if (!r) {
        const int64_t m = static_cast<int64_t>(n) * s.t[0].bins;
        swlh_query_kernel<<<blocks_for(m, 256), 256, 0, st>>>(s, dc, n, out, bad);
        r = launch_status("swlh_query_kernel");
    }
    unsigned hb = 0;
    if (!r) r = cuda_status(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, st), "D2H");
    if (!r) r = cuda_status(cudaStreamSynchronize(st), "swlh_query");
    cudaFreeAsync(dc, st);
    if (!r && hb) return contract("swlh_query: inconsistent quadrant tensors");  // swih.cpp:157
    return r;
}

extern "C" spct_status spct_cu_swlh_brute(const uint16_t* bins, int64_t pitch, int width, int height, int nbins, int kw,
                                          int kh, const int32_t* centres_host, int n, int64_t* out, void* stream) {
    if (!(kw >= 1 && kh >= 1)) return contract("kernel extents must be >= 1");
    if (!bins || pitch < width || nbins < 1 || n < 0 || (n > 0 && !(centres_host && out)))
        return contract("brute_force_swlh: bad arguments");
    const Ext e = extents(kw, kh);
    for (int q = 0; q < n; ++q) {
        const int cx = centres_host[2 * q], cy = centres_host[2 * q + 1];
        if (!(cx - e.sxl >= 0 && cy - e.syt >= 0 && cx + e.sxr <= width && cy + e.syb <= height))
            return contract("kernel window must lie inside the image");
    }
    if (n == 0) return SPCT_OK;
    cudaStream_t st = as_stream(stream);
    int32_t* dc = nullptr;
    spct_status r = cuda_status(malloc_async(&dc, 8 * static_cast<size_t>(n), st), "swlh alloc");
    if (!r) r = cuda_status(cudaMemcpyAsync(dc, centres_host, 8 * static_cast<size_t>(n), cudaMemcpyHostToDevice, st), "H2D");
    if (!r) {
        swlh_brute_kernel<<<n, 128, 0, st>>>(bins, pitch, nbins, kw, kh, dc, n, out);
        r = launch_status("swlh_brute_kernel");
    }
    if (!r) r = cuda_status(cudaStreamSynchronize(st), "brute_force_swlh");
    cudaFreeAsync(dc, st);
    return r;
}

extern "C" spct_status spct_cu_swlh_map(const spct_wih* set4, int kw, int kh, const double* model, double* map,
                                        void* stream) {
    QuadSet s{};
    if (auto st = check_set(set4, kw, kh, &s)) return st;
    if (!model || !map) return contract("swlh_map: null model or map");
    const int W = s.t[0].width, Hh = s.t[0].height;
    cudaStream_t st = as_stream(stream);
    const int64_t n = static_cast<int64_t>(W) * Hh;
    if (W < kw || Hh < kh) {  // track_loop.cpp:265-267: a flat 0.5 map
        fill_kernel<<<blocks_for(std::min<int64_t>(n, 148 * 2048), 256), 256, 0, st>>>(map, n, 0.5);
        return launch_status("fill_kernel");
    }
    const Ext e = extents(kw, kh);
    // kernel mass (constant for windows inside the image): 2^16 * sum (c - |dx| - |dy|)
    int64_t mass = 0;
    for (int dy = -e.syt; dy < e.syb; ++dy)
        for (int dx = -e.sxl; dx < e.sxr; ++dx) mass += e.c - std::abs(dx) - std::abs(dy);
    unsigned* bad = nullptr;
    spct_status r = cuda_status(malloc_async(&bad, 4, st), "swlh alloc");
    if (!r) r = cuda_status(cudaMemsetAsync(bad, 0, 4, st), "memset");
    if (!r) {
        const int64_t nc = static_cast<int64_t>(W - kw + 1) * (Hh - kh + 1);
        swlh_map_kernel<<<blocks_for(nc, 128), 128, 0, st>>>(s, model, static_cast<double>(mass << 16), map, bad);
        r = launch_status("swlh_map_kernel");
    }
    if (!r) {
        replicate_kernel<<<blocks_for(n, 256), 256, 0, st>>>(map, W, Hh, e.sxl, W - e.sxr, e.syt, Hh - e.syb);
        r = launch_status("replicate_kernel");
    }
    unsigned hb = 0;
    if (!r) r = cuda_status(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, st), "D2H");
    if (!r) r = cuda_status(cudaStreamSynchronize(st), "swlh_map");
    cudaFreeAsync(bad, st);
    if (!r && hb) return contract("swlh_query: inconsistent quadrant tensors");
    return r;
}
