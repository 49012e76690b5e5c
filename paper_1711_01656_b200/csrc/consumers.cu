// Likelihood-map consumers on the device: the step after the map,
// so a tracker need not copy each map to the host.
//
//   fuse_maps        likelihood.cpp:257-283  weighted sum (weights normalised on the host
//                                            exactly as the reference), map-by-map FP64
//                                            accumulation in the reference order, clamp01
//   find_peaks       likelihood.cpp:285-322  3x3 in-bounds mean (same summation order),
//                                            strict 8-neighbour maxima with the 1e-9 flat
//                                            margin, deterministic row-major compaction, then
//                                            a stable LSD radix sort by height (descending)
//   score_map        likelihood.cpp:332-339  rank of the best peak inside gt (k + 1 if none),
//                                            counted without sorting
//   camshift_refine  tracker.cpp:77-113      one warp per start point; the three window
//                                            sums stay sequential chains (same rounding)
// All results are bit-identical to the reference (no reassociation, no FMA contraction).
#include <cmath>
#include <cstring>
#include <utility>
#include <vector>

#include "spct_internal.h"

using namespace spct_impl;

namespace spct_cons {

constexpr int kMaxFuse = 8;

struct FuseArgs {
    const double* maps[kMaxFuse];
    double wt[kMaxFuse];
    int nmaps, first, last;
};

__device__ __forceinline__ double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

__global__ void fuse_kernel(FuseArgs a, int64_t n, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double acc = a.first ? 0.0 : out[i];
        for (int m = 0; m < a.nmaps; ++m) acc = __dadd_rn(acc, __dmul_rn(a.wt[m], __ldg(a.maps[m] + i)));
        out[i] = a.last ? clamp01(acc) : acc;
    }
}

// ---------------------------------------------------------------- find_peaks

constexpr int kSortTile = 2048;   // keys per radix block (256 threads x 8)

// RN(a / d) for d in {6, 9} (y = RN(1 / d)): q = a y, then one FMA correction with the exact
// remainder (Markstein) — the correctly rounded quotient for |a| in [2^-1000, 2^1000] (checked
// on 6e8 samples against IEEE division); zero, tiny, huge and non-finite `a` divide.
__device__ __forceinline__ double div_small(double a, double d, double y) {
    const double q = __dmul_rn(a, y);
    const double aa = fabs(a);
    if (aa == 0.0) return q;
    if (!(aa >= 0x1p-1000 && aa <= 0x1p1000)) return __ddiv_rn(a, d);
    return fma(fma(-q, d, a), y, q);
}

// Smoothing and peak flags in one pass over the map (find_peaks / score_map front end):
// per CTA a 64 x 32 tile, its raw map with a 2-cell halo and the smoothed map with a
// 1-cell halo staged in shared memory; the smoothed tile is stored, and the peak flags
// leave as one bit per pixel (mask[y][x / 32], bit x % 32, one warp ballot per word).
// Same arithmetic as the reference (likelihood.cpp:288-322): in-image neighbours only,
// row-major order, then / count; the exact negation of `n + 1e-9 >= v`.  Tiles whose halo
// lies inside the map run without bounds checks.
constexpr int kSmX = 64, kSmY = 32;

__global__ void __launch_bounds__(256) smooth_peaks_kernel(const double* __restrict__ map, int w, int h,
                                                           double* __restrict__ s, uint32_t* __restrict__ mask,
                                                           int mw) {
    __shared__ double raw[kSmY + 4][kSmX + 4];
    __shared__ double sm[kSmY + 2][kSmX + 2];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = blockIdx.x * kSmX, y0 = blockIdx.y * kSmY;
    const bool inner = x0 >= 2 && y0 >= 2 && x0 + kSmX + 2 <= w && y0 + kSmY + 2 <= h;
    {   // warp = row, lane = column; every load of the thread in flight before the stores
        constexpr int RR = (kSmY + 4 + 7) / 8, CC = (kSmX + 4 + 31) / 32;
        double v[RR][CC];
#pragma unroll
        for (int k = 0; k < RR; ++k) {
            const int r = warp + 8 * k, gy = y0 - 2 + r;
            const double* row = map + static_cast<int64_t>(gy) * w;
#pragma unroll
            for (int j = 0; j < CC; ++j) {
                const int c = lane + 32 * j, gx = x0 - 2 + c;
                v[k][j] = (r < kSmY + 4 && c < kSmX + 4 && (inner || (gx >= 0 && gy >= 0 && gx < w && gy < h)))
                              ? __ldg(row + gx)
                              : 0.0;
            }
        }
#pragma unroll
        for (int k = 0; k < RR; ++k)
#pragma unroll
            for (int j = 0; j < CC; ++j)
                if (warp + 8 * k < kSmY + 4 && lane + 32 * j < kSmX + 4) raw[warp + 8 * k][lane + 32 * j] = v[k][j];
    }
    __syncthreads();
    constexpr double kInv9 = 1.0 / 9.0, kInv6 = 1.0 / 6.0;
    for (int r = warp; r < kSmY + 2; r += 8)
        for (int c = lane; c < kSmX + 2; c += 32) {
            const int gy = y0 - 1 + r, gx = x0 - 1 + c;
            double v = 0.0;
            if (inner) {
                double acc = raw[r][c];
                acc = __dadd_rn(acc, raw[r][c + 1]);
                acc = __dadd_rn(acc, raw[r][c + 2]);
                acc = __dadd_rn(acc, raw[r + 1][c]);
                acc = __dadd_rn(acc, raw[r + 1][c + 1]);
                acc = __dadd_rn(acc, raw[r + 1][c + 2]);
                acc = __dadd_rn(acc, raw[r + 2][c]);
                acc = __dadd_rn(acc, raw[r + 2][c + 1]);
                acc = __dadd_rn(acc, raw[r + 2][c + 2]);
                v = div_small(acc, 9.0, kInv9);
            } else if (gx >= 0 && gy >= 0 && gx < w && gy < h) {
                double acc = 0.0;
                int cnt = 0;
#pragma unroll
                for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int nx = gx + dx, ny = gy + dy;
                        if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
                        acc = __dadd_rn(acc, raw[r + 1 + dy][c + 1 + dx]);
                        ++cnt;
                    }
                v = cnt == 9 ? div_small(acc, 9.0, kInv9)
                             : (cnt == 6 ? div_small(acc, 6.0, kInv6) : __ddiv_rn(acc, static_cast<double>(cnt)));
            }
            sm[r][c] = v;
        }
    __syncthreads();
    for (int r = warp; r < kSmY; r += 8) {
        const int gy = y0 + r;
#pragma unroll
        for (int hw = 0; hw < kSmX / 32; ++hw) {  // a warp: one 32-column mask word
            const int c = 32 * hw + lane, gx = x0 + c;
            const bool in = inner || (gx < w && gy < h);
            bool peak = false;
            if (in) {
                const double v = sm[r + 1][c + 1];
                s[static_cast<int64_t>(gy) * w + gx] = v;
                if (inner) {
                    const double* u = &sm[r][c];
                    const double* m = &sm[r + 1][c];
                    const double* d = &sm[r + 2][c];
                    peak = !(__dadd_rn(u[0], 1e-9) >= v) & !(__dadd_rn(u[1], 1e-9) >= v) &
                           !(__dadd_rn(u[2], 1e-9) >= v) & !(__dadd_rn(m[0], 1e-9) >= v) &
                           !(__dadd_rn(m[2], 1e-9) >= v) & !(__dadd_rn(d[0], 1e-9) >= v) &
                           !(__dadd_rn(d[1], 1e-9) >= v) & !(__dadd_rn(d[2], 1e-9) >= v);
                } else {
                    peak = true;
#pragma unroll
                    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (dx == 0 && dy == 0) continue;
                            const int nx = gx + dx, ny = gy + dy;
                            if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
                            if (__dadd_rn(sm[r + 1 + dy][c + 1 + dx], 1e-9) >= v) peak = false;
                        }
                }
            }
            const uint32_t b = __ballot_sync(0xffffffffu, peak);
            if (lane == 0 && gy < h && x0 + 32 * hw < w) mask[static_cast<int64_t>(gy) * mw + ((x0 >> 5) + hw)] = b;
        }
    }
}

__device__ __forceinline__ bool mask_bit(const uint32_t* mask, int mw, int x, int y) {
    return (mask[static_cast<int64_t>(y) * mw + (x >> 5)] >> (x & 31)) & 1u;
}

// Exclusive prefix of the mask words' popcounts within runs of 1024 words (woff) and the
// runs' totals (runtot; scanned afterwards by excl_scan_kernel).
__global__ void __launch_bounds__(1024) mask_scan_kernel(const uint32_t* __restrict__ mask, int64_t nwords,
                                                         uint32_t* __restrict__ woff, uint32_t* __restrict__ runtot) {
    __shared__ uint32_t wsum[32];
    const int64_t i = static_cast<int64_t>(blockIdx.x) * 1024 + threadIdx.x;
    const uint32_t x = i < nwords ? static_cast<uint32_t>(__popc(mask[i])) : 0u;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t ws = wsum[lane];
        uint32_t wi = ws;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        wsum[lane] = wi - ws;
        if (lane == 31) runtot[blockIdx.x] = wi;
    }
    __syncthreads();
    if (i < nwords) woff[i] = wsum[warp] + inc - x;
}

// Exclusive scan of n values in place (1024 threads, sequential chunks); CTA b scans the
// b-th run of n values (v + b n) and writes its sum to total[b].
__global__ void __launch_bounds__(1024) excl_scan_kernel(uint32_t* __restrict__ v, int64_t n, uint32_t* total) {
    v += static_cast<int64_t>(blockIdx.x) * n;
    if (total) total += blockIdx.x;
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t b = 0; b < n; b += 1024) {
        const int64_t i = b + threadIdx.x;
        const uint32_t x = i < n ? v[i] : 0u;
        uint32_t inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) wsum[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const uint32_t ws = wsum[lane];
            uint32_t wi = ws;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += t;
            }
            wsum[lane] = wi - ws;  // exclusive warp offsets
        }
        __syncthreads();
        const uint32_t c0 = carry;
        if (i < n) v[i] = c0 + wsum[warp] + inc - x;
        __syncthreads();
        if (threadIdx.x == 1023) carry = c0 + wsum[warp] + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

// Descending order of heights as ascending uint64 keys.
__device__ __forceinline__ uint64_t desc_key(double h) {
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(h));
    const uint64_t asc = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
    return ~asc;
}

// Row-major compaction of the flagged peaks (thread per mask word), with the key range.
__global__ void __launch_bounds__(256) peak_compact_mask_kernel(const double* __restrict__ s, int w, int mw,
                                                                int64_t nwords, const uint32_t* __restrict__ mask,
                                                                const uint32_t* __restrict__ woff,
                                                                const uint32_t* __restrict__ runoff,
                                                                uint64_t* __restrict__ keys, uint32_t* __restrict__ idx,
                                                                unsigned long long* __restrict__ kminmax, int64_t cap) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    unsigned long long kmin = ~0ull, kmax = 0ull;
    if (i < nwords) {
        uint32_t bits = mask[i];
        uint32_t pos = woff[i] + runoff[i >> 10];
        const int64_t y = i / mw, xb = (i % mw) * 32;
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t p = y * w + xb + b;
            const unsigned long long k = desc_key(s[p]);
            if (pos < cap) {  // NaN maps can hold more peaks than the n / 4 + 2 of strict maxima
                keys[pos] = k;
                idx[pos] = static_cast<uint32_t>(p);
            }
            ++pos;
            kmin = k < kmin ? k : kmin;
            kmax = k > kmax ? k : kmax;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmin = a < kmin ? a : kmin;
        kmax = b > kmax ? b : kmax;
    }
    if ((threadIdx.x & 31) == 0 && kmin <= kmax) {
        atomicMin(kminmax, kmin);
        atomicMax(kminmax + 1, kmax);
    }
}

// Radix pass p: digit (key >> 8p) & 255.  counts are digit-major: counts[d * nblk + b].
__global__ void __launch_bounds__(256) radix_hist_kernel(const uint64_t* __restrict__ keys, int64_t n, int shift,
                                                         int nblk, uint32_t* __restrict__ counts) {
    __shared__ uint32_t c[256];
    c[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kSortTile;
    for (int j = threadIdx.x; j < kSortTile; j += 256)
        if (base + j < n) atomicAdd(&c[(keys[base + j] >> shift) & 255u], 1u);
    __syncthreads();
    counts[static_cast<int64_t>(threadIdx.x) * nblk + blockIdx.x] = c[threadIdx.x];
}

// Stable scatter: elements are ranked in index order (round-major, then thread order).
// offs: per digit, the exclusive prefix over blocks (digit-major); dstart: the digits' starts.
__global__ void __launch_bounds__(256) radix_scatter_kernel(const uint64_t* __restrict__ kin,
                                                            const uint32_t* __restrict__ vin, int64_t n, int shift,
                                                            int nblk, const uint32_t* __restrict__ offs,
                                                            const uint32_t* __restrict__ dstart,
                                                            uint64_t* __restrict__ kout, uint32_t* __restrict__ vout) {
    __shared__ uint32_t run[256];       // per digit: elements of this block already placed
    __shared__ uint32_t wcnt[8][256];   // this round's per-warp digit counts, then prefixes
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    run[threadIdx.x] = dstart[threadIdx.x] + offs[static_cast<int64_t>(threadIdx.x) * nblk + blockIdx.x];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kSortTile;
    for (int r = 0; r < kSortTile / 256; ++r) {
        for (int k = 0; k < 8; ++k) wcnt[k][threadIdx.x] = 0;
        __syncthreads();
        const int64_t i = base + r * 256 + threadIdx.x;
        const bool live = i < n;
        const uint64_t key = live ? kin[i] : 0;
        const uint32_t d = live ? static_cast<uint32_t>((key >> shift) & 255u) : 256u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        if (live && rank == 0) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        uint32_t acc = 0;  // thread = digit: exclusive prefix over the warps, round total
        for (int k = 0; k < 8; ++k) {
            const uint32_t c = wcnt[k][threadIdx.x];
            wcnt[k][threadIdx.x] = acc;
            acc += c;
        }
        __syncthreads();
        if (live) {
            const uint32_t pos = run[d] + wcnt[warp][d] + rank;
            kout[pos] = key;
            vout[pos] = vin[i];
        }
        __syncthreads();
        run[threadIdx.x] += acc;
    }
}

__global__ void peak_gather_kernel(const uint32_t* __restrict__ idx, const double* __restrict__ s, int w, int64_t n,
                                   int32_t* __restrict__ xs, int32_t* __restrict__ ys, double* __restrict__ hs) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t p = idx[i];
        xs[i] = static_cast<int32_t>(p % static_cast<uint32_t>(w));
        ys[i] = static_cast<int32_t>(p / static_cast<uint32_t>(w));
        hs[i] = s[p];
    }
}

// First sorted position whose peak lies inside gt (min over a device counter).
// score_map without the sort: the first in-rect peak of the sorted list is the in-rect
// peak with the smallest (descending-height key, index) — stable_sort keeps row-major
// order among equal heights — and its rank is 1 + the number of peaks before it in that
// order (or, with no peak in the rect, the peak count + 1).
__global__ void rect_best_key_kernel(const double* __restrict__ s, const uint32_t* __restrict__ mask, int mw, int w,
                                     int gx, int gy, int gw, int gh, unsigned long long* __restrict__ best_key) {
    const int64_t n = static_cast<int64_t>(gw) * gh;
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = gx + static_cast<int>(j % gw), y = gy + static_cast<int>(j / gw);
        if (mask_bit(mask, mw, x, y))
            atomicMin(best_key, static_cast<unsigned long long>(desc_key(s[static_cast<int64_t>(y) * w + x])));
    }
}

__global__ void rect_best_idx_kernel(const double* __restrict__ s, const uint32_t* __restrict__ mask, int mw, int w,
                                     int gx, int gy, int gw, int gh, const unsigned long long* __restrict__ best_key,
                                     unsigned* __restrict__ best_idx) {
    const int64_t n = static_cast<int64_t>(gw) * gh;
    const unsigned long long bk = *best_key;
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = gx + static_cast<int>(j % gw), y = gy + static_cast<int>(j / gw);
        const int64_t i = static_cast<int64_t>(y) * w + x;
        if (mask_bit(mask, mw, x, y) && desc_key(s[i]) == bk) atomicMin(best_idx, static_cast<unsigned>(i));
    }
}

// found: count the peaks ordered before (best_key, best_idx); else count every peak
// (thread per mask word: only the flagged pixels' heights are read).
__global__ void __launch_bounds__(256) rank_count_kernel(const double* __restrict__ s, int w, int mw, int64_t nwords,
                                                         const uint32_t* __restrict__ mask,
                                                         const unsigned* __restrict__ best_idx,
                                                         const unsigned long long* __restrict__ best_key,
                                                         unsigned long long* __restrict__ count) {
    const unsigned bi = *best_idx;
    const bool found = bi != 0xFFFFFFFFu;
    const unsigned long long bk = *best_key;
    unsigned c = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nwords;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint32_t bits = mask[i];
        if (!found) {
            c += __popc(bits);
            continue;
        }
        const int64_t y = i / mw, xb = (i % mw) * 32;
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t p = y * w + xb + b;
            const unsigned long long k = desc_key(s[p]);
            c += k < bk || (k == bk && static_cast<unsigned>(p) < bi);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, static_cast<unsigned long long>(c));
}

// ---------------------------------------------------------------- camshift_refine

// camshift_refine (tracker.cpp:77-113) for n start points, one warp per start: the warp
// streams the window in 32-pixel chunks through shared memory (the next chunk's loads in
// flight while the current one is summed) and
// lanes 0, 1, 2 run the three sums m00, m10, m01 — each still one sequential chain in the
// reference's row-major order, so every bit matches.
constexpr int kCamWarps = 4;

__global__ void __launch_bounds__(32 * kCamWarps) camshift_warp_kernel(
    const double* __restrict__ map, int w, int h, const double* __restrict__ starts, int n, int win_w, int win_h,
    double delta, int max_iter, double* __restrict__ out, int32_t* __restrict__ iters, int32_t* __restrict__ zero_mass) {
    __shared__ double buf[kCamWarps][2][32];
    __shared__ double mom[kCamWarps][3];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int q = blockIdx.x * kCamWarps + wi;
    if (q >= n) return;
    double cx = starts[2 * q], cy = starts[2 * q + 1];
    int it_done = 0, zm = 0;
    for (int it = 0; it < max_iter; ++it) {
        const int x0 = static_cast<int>(llround(__dsub_rn(cx, (win_w - 1) / 2.0)));
        const int y0 = static_cast<int>(llround(__dsub_rn(cy, (win_h - 1) / 2.0)));
        const int xa = max(x0, 0), ya = max(y0, 0), xb = min(x0 + win_w, w), yb = min(y0 + win_h, h);
        const int rw = max(0, xb - xa), nch = (rw + 31) / 32;
        const int64_t total = static_cast<int64_t>(max(0, yb - ya)) * nch;  // chunks, row-major
        double acc = 0.0;  // lane 0: m00, lane 1: m10, lane 2: m01
        auto load = [&](int64_t c) {
            const int y = ya + static_cast<int>(c / nch), x = xa + static_cast<int>(c % nch) * 32 + lane;
            return x < xb ? __ldg(map + static_cast<int64_t>(y) * w + x) : 0.0;
        };
        double nxt = total > 0 ? load(0) : 0.0;
        for (int64_t c = 0; c < total; ++c) {
            buf[wi][c & 1][lane] = nxt;
            __syncwarp();
            if (c + 1 < total) nxt = load(c + 1);
            if (lane < 3) {
                const int y = ya + static_cast<int>(c / nch), xs = xa + static_cast<int>(c % nch) * 32;
                const int m = min(32, xb - xs);
                const double* b = buf[wi][c & 1];
                if (lane == 0)
                    for (int i = 0; i < m; ++i) acc = __dadd_rn(acc, b[i]);
                else if (lane == 1)
                    for (int i = 0; i < m; ++i) acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(xs + i), b[i]));
                else
                    for (int i = 0; i < m; ++i) acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(y), b[i]));
            }
            __syncwarp();
        }
        if (lane < 3) mom[wi][lane] = acc;
        __syncwarp();
        const double m00 = mom[wi][0], m10 = mom[wi][1], m01 = mom[wi][2];
        __syncwarp();
        if (m00 <= 0.0) {
            zm = 1;
            break;
        }
        const double nx = __ddiv_rn(m10, m00), ny = __ddiv_rn(m01, m00);
        const double d = hypot(__dsub_rn(nx, cx), __dsub_rn(ny, cy));
        cx = nx;
        cy = ny;
        ++it_done;
        if (d < delta) break;
    }
    if (lane == 0) {
        out[2 * q] = cx;
        out[2 * q + 1] = cy;
        iters[q] = it_done;
        zero_mass[q] = zm;
    }
}

// (columns of 256 threads, rows) for the row-wise 2-D kernels, about 16 CTAs per SM
dim3 grid2d(int w, int h) {
    const unsigned gx = static_cast<unsigned>(std::min<int64_t>(ceil_div(w, 256), 16));
    return dim3(gx, static_cast<unsigned>(std::min<int64_t>(h, std::max<int64_t>(1, 148 * 16 / gx))));
}

int grid1(int64_t n) { return static_cast<int>(std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 148 * 16)); }

struct PeakWs {
    double* s;
    uint32_t* mask;    // [h][mw] peak flags, mw = ceil(w / 32)
    uint32_t* woff;    // per mask word: exclusive popcount prefix within its run of 1024 words
    uint32_t* runoff;  // per run: exclusive prefix over the runs
    uint64_t* k[2];
    uint32_t* v[2];
    uint32_t* counts;
    uint32_t* scalars;  // [0] total peaks, [1] score best
    void* extra;        // stream-ordered overflow buffers (freed by the caller after use), or null
};

int64_t mask_words(int w, int h) { return static_cast<int64_t>(h) * ceil_div(w, 32); }

// nblk_peak: runs of 1024 mask words
size_t peak_ws_bytes(int w, int h, int64_t* nblk_peak, int64_t* nblk_sort) {
    const int64_t n = static_cast<int64_t>(w) * h, nw = mask_words(w, h);
    const int64_t cap = n / 4 + 2;  // strict 8-neighbour maxima: at most one per 2 x 2 cell
    *nblk_peak = ceil_div(nw, 1024);
    *nblk_sort = std::max<int64_t>(1, ceil_div(cap, kSortTile));
    auto r = [](int64_t b) { return static_cast<size_t>(round_up(b, 256)); };
    return r(n * 8) + 2 * r(nw * 4) + r(*nblk_peak * 4) + 2 * r(cap * 8) + 2 * r(cap * 4) + r(256 * *nblk_sort * 4) +
           r(16 + 1024 + 16);
}

PeakWs carve(void* ws, int w, int h) {
    int64_t nbp, nbs;
    peak_ws_bytes(w, h, &nbp, &nbs);
    const int64_t n = static_cast<int64_t>(w) * h, cap = n / 4 + 2;
    char* p = static_cast<char*>(ws);
    auto take = [&](int64_t bytes) {
        char* q = p;
        p += round_up(bytes, 256);
        return q;
    };
    PeakWs s;
    s.s = reinterpret_cast<double*>(take(n * 8));
    s.mask = reinterpret_cast<uint32_t*>(take(mask_words(w, h) * 4));
    s.woff = reinterpret_cast<uint32_t*>(take(mask_words(w, h) * 4));
    s.runoff = reinterpret_cast<uint32_t*>(take(nbp * 4));
    s.k[0] = reinterpret_cast<uint64_t*>(take(cap * 8));
    s.k[1] = reinterpret_cast<uint64_t*>(take(cap * 8));
    s.v[0] = reinterpret_cast<uint32_t*>(take(cap * 4));
    s.v[1] = reinterpret_cast<uint32_t*>(take(cap * 4));
    s.counts = reinterpret_cast<uint32_t*>(take(256 * nbs * 4));
    // [0]: peak count, [4 .. 259]: digit starts, [260 .. 263]: key min / max (u64)
    s.scalars = reinterpret_cast<uint32_t*>(take(16 + 1024 + 16));
    s.extra = nullptr;
    return s;
}

// Peaks of `map` sorted (keys/values end in k[0]/v[0]); returns the count (synchronises).
spct_status sorted_peaks(const double* map, int w, int h, void* ws, size_t ws_bytes, cudaStream_t st, PeakWs* out,
                         int64_t* count) {
    int64_t nbp, nbs;
    if (!ws || ws_bytes < peak_ws_bytes(w, h, &nbp, &nbs)) return contract("find_peaks: workspace too small");
    PeakWs P = carve(ws, w, h);
    const int64_t n = static_cast<int64_t>(w) * h, nw = mask_words(w, h);
    const int mw = static_cast<int>(ceil_div(w, 32));
    smooth_peaks_kernel<<<dim3(static_cast<unsigned>(ceil_div(w, kSmX)), static_cast<unsigned>(ceil_div(h, kSmY))), 256,
                          0, st>>>(map, w, h, P.s, P.mask, mw);
    mask_scan_kernel<<<static_cast<unsigned>(nbp), 1024, 0, st>>>(P.mask, nw, P.woff, P.runoff);
    excl_scan_kernel<<<1, 1024, 0, st>>>(P.runoff, nbp, P.scalars);
    unsigned long long* kminmax = reinterpret_cast<unsigned long long*>(P.scalars + 260);
    const unsigned long long init[2] = {~0ull, 0ull};
    cudaMemcpyAsync(kminmax, init, 16, cudaMemcpyHostToDevice, st);
    const int64_t cap = n / 4 + 2;
    const unsigned ncb = static_cast<unsigned>(ceil_div(nw, 256));  // one thread per mask word
    peak_compact_mask_kernel<<<ncb, 256, 0, st>>>(P.s, w, mw, nw, P.mask, P.woff, P.runoff, P.k[0], P.v[0], kminmax,
                                                  cap);
    if (auto e = launch_status("find_peaks compaction")) return e;
    uint32_t hdr[264];
    if (auto e = cuda_status(cudaMemcpyAsync(hdr, P.scalars, sizeof(hdr), cudaMemcpyDeviceToHost, st), "find_peaks count"))
        return e;
    if (auto e = cuda_status(cudaStreamSynchronize(st), "find_peaks")) return e;
    const int64_t m = hdr[0];
    if (m > cap) {
        // more peaks than strict maxima allow (NaN cells pass the reference's test,
        // likelihood.cpp:316): compact again into buffers sized for the real count
        const int64_t nbm = ceil_div(m, kSortTile);
        const size_t kb = round_up(m * 8, 256), vb = round_up(m * 4, 256);
        char* x = nullptr;
        if (auto e = cuda_status(malloc_async(&x, 2 * kb + 2 * vb + 256 * nbm * 4, st), "find_peaks alloc")) return e;
        P.k[0] = reinterpret_cast<uint64_t*>(x);
        P.k[1] = reinterpret_cast<uint64_t*>(x + kb);
        P.v[0] = reinterpret_cast<uint32_t*>(x + 2 * kb);
        P.v[1] = reinterpret_cast<uint32_t*>(x + 2 * kb + vb);
        P.counts = reinterpret_cast<uint32_t*>(x + 2 * kb + 2 * vb);
        P.extra = x;
        cudaMemcpyAsync(kminmax, init, 16, cudaMemcpyHostToDevice, st);
        peak_compact_mask_kernel<<<ncb, 256, 0, st>>>(P.s, w, mw, nw, P.mask, P.woff, P.runoff, P.k[0], P.v[0],
                                                      kminmax, m);
        if (auto e = launch_status("find_peaks compaction")) return e;
        if (auto e = cuda_status(cudaMemcpyAsync(hdr, P.scalars, sizeof(hdr), cudaMemcpyDeviceToHost, st), "find_peaks"))
            return e;
        if (auto e = cuda_status(cudaStreamSynchronize(st), "find_peaks")) return e;
    }
    int cur = 0;
    if (m > 1) {
        const int nb = static_cast<int>(ceil_div(m, kSortTile));
        uint32_t* digit = P.scalars + 4;  // [256] digit totals -> digit starts
        // digits above the highest bit in which two keys differ are the same for every key:
        // those passes would be identity permutations
        unsigned long long kmin, kmax;
        std::memcpy(&kmin, hdr + 260, 8);
        std::memcpy(&kmax, hdr + 262, 8);
        const unsigned long long diff = kmin ^ kmax;
        const int npass = diff ? (63 - __builtin_clzll(diff)) / 8 + 1 : 0;
        for (int pass = 0; pass < npass; ++pass) {
            radix_hist_kernel<<<nb, 256, 0, st>>>(P.k[cur], m, 8 * pass, nb, P.counts);
            // per digit (one CTA each): prefix over the blocks; then the digits' starts
            excl_scan_kernel<<<256, 1024, 0, st>>>(P.counts, nb, digit);
            excl_scan_kernel<<<1, 1024, 0, st>>>(digit, 256, nullptr);
            radix_scatter_kernel<<<nb, 256, 0, st>>>(P.k[cur], P.v[cur], m, 8 * pass, nb, P.counts, digit,
                                                     P.k[cur ^ 1], P.v[cur ^ 1]);
            cur ^= 1;
        }
        if (auto e = launch_status("find_peaks sort")) return e;
    }
    if (cur) {  // an odd number of passes: the sorted data is in buffer 1
        std::swap(P.k[0], P.k[1]);
        std::swap(P.v[0], P.v[1]);
    }
    *out = P;
    *count = m;
    return SPCT_OK;
}

}  // namespace spct_cons

using namespace spct_cons;

extern "C" spct_status spct_cu_fuse_maps(const double* const* maps, int nmaps, const double* weights, int nweights,
                                         int64_t n, double* out, void* stream) {
    if (nmaps < 1 || !maps) return contract("fuse_maps: no maps to fuse");  // likelihood.cpp:258
    if (nweights != 0 && nweights != nmaps) return contract("fuse_maps: weight count mismatch");  // :263
    if (n < 0 || (n > 0 && !out)) return contract("fuse_maps: bad output");
    std::vector<double> wv(nmaps);
    for (int m = 0; m < nmaps; ++m) wv[m] = nweights ? weights[m] : 1.0 / nmaps;  // :262
    double wsum = 0.0;
    for (double x : wv) {
        if (!(x >= 0.0)) return contract("fuse_maps: negative weight");  // :266
        wsum += x;
    }
    if (!(wsum > 0.0)) return contract("fuse_maps: weights sum to zero");  // :269
    if (n == 0) return SPCT_OK;
    cudaStream_t s = as_stream(stream);
    for (int m0 = 0; m0 < nmaps; m0 += kMaxFuse) {
        FuseArgs a{};
        a.nmaps = std::min(kMaxFuse, nmaps - m0);
        for (int j = 0; j < a.nmaps; ++j) {
            if (!maps[m0 + j]) return contract("fuse_maps: null map");
            a.maps[j] = maps[m0 + j];
            a.wt[j] = wv[m0 + j] / wsum;  // :278
        }
        a.first = m0 == 0;
        a.last = m0 + a.nmaps == nmaps;
        fuse_kernel<<<grid1(n), 256, 0, s>>>(a, n, out);
        if (auto st = launch_status("fuse_kernel")) return st;
    }
    return SPCT_OK;
}

extern "C" spct_status spct_cu_find_peaks_workspace(int w, int h, size_t* bytes) {
    if (!bytes) return contract("find_peaks_workspace: null argument");
    if (!(w > 0 && h > 0)) return contract("find_peaks: empty map");  // likelihood.cpp:286
    int64_t a, b;
    *bytes = peak_ws_bytes(w, h, &a, &b);
    return SPCT_OK;
}

extern "C" spct_status spct_cu_find_peaks(const double* map, int w, int h, int32_t* xs, int32_t* ys, double* heights,
                                          int64_t max_out, int64_t* count, void* workspace, size_t workspace_bytes,
                                          void* stream) {
    if (!(w > 0 && h > 0)) return contract("find_peaks: empty map");  // likelihood.cpp:286
    if (!map || !count || max_out < 0 || (max_out > 0 && !(xs && ys && heights)))
        return contract("find_peaks: bad arguments");
    cudaStream_t s = as_stream(stream);
    PeakWs P;
    int64_t m = 0;
    if (auto st = sorted_peaks(map, w, h, workspace, workspace_bytes, s, &P, &m)) return st;
    *count = m;
    const int64_t k = std::min(m, max_out);
    spct_status st = SPCT_OK;
    if (k > 0) {
        peak_gather_kernel<<<grid1(k), 256, 0, s>>>(P.v[0], P.s, w, k, xs, ys, heights);
        st = launch_status("peak_gather_kernel");
    }
    if (P.extra) cudaFreeAsync(P.extra, s);
    return st;
}

extern "C" spct_status spct_cu_score_map(const double* map, int w, int h, int gx, int gy, int gw, int gh, int64_t* rank,
                                         void* workspace, size_t workspace_bytes, void* stream) {
    if (!(gw > 0 && gh > 0 && gx >= 0 && gy >= 0 && gx + gw <= w && gy + gh <= h))  // likelihood.cpp:333-334
        return contract("score_map: ground truth rect must lie inside the map");
    if (!map || !rank) return contract("score_map: bad arguments");
    int64_t nbp, nbs;
    if (!workspace || workspace_bytes < peak_ws_bytes(w, h, &nbp, &nbs)) return contract("find_peaks: workspace too small");
    cudaStream_t s = as_stream(stream);
    PeakWs P = carve(workspace, w, h);
    // scalars: [0..1] best key (u64), [2] best index, [4..5] count (u64)
    unsigned long long* bk = reinterpret_cast<unsigned long long*>(P.scalars);
    unsigned* bi = P.scalars + 2;
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(P.scalars + 4);
    cudaMemsetAsync(P.scalars, 0xFF, 12, s);  // key and index: "none"
    cudaMemsetAsync(cnt, 0, 8, s);
    const int mw = static_cast<int>(ceil_div(w, 32));
    const int64_t nw = mask_words(w, h);
    smooth_peaks_kernel<<<dim3(static_cast<unsigned>(ceil_div(w, kSmX)), static_cast<unsigned>(ceil_div(h, kSmY))), 256,
                          0, s>>>(map, w, h, P.s, P.mask, mw);
    const int64_t nr = static_cast<int64_t>(gw) * gh;
    rect_best_key_kernel<<<grid1(nr), 256, 0, s>>>(P.s, P.mask, mw, w, gx, gy, gw, gh, bk);
    rect_best_idx_kernel<<<grid1(nr), 256, 0, s>>>(P.s, P.mask, mw, w, gx, gy, gw, gh, bk, bi);
    rank_count_kernel<<<grid1(nw), 256, 0, s>>>(P.s, w, mw, nw, P.mask, bi, bk, cnt);
    if (auto st = launch_status("score_map")) return st;
    unsigned long long c = 0;
    if (auto st = cuda_status(cudaMemcpyAsync(&c, cnt, 8, cudaMemcpyDeviceToHost, s), "score")) return st;
    if (auto st = cuda_status(cudaStreamSynchronize(s), "score_map")) return st;
    *rank = static_cast<int64_t>(c) + 1;
    return SPCT_OK;
}

extern "C" spct_status spct_cu_camshift(const double* map, int w, int h, const double* starts, int n, int win_w,
                                        int win_h, double delta, int max_iter, double* out, int32_t* iterations,
                                        int32_t* zero_mass, void* stream) {
    if (!(w > 0 && h > 0)) return contract("camshift_refine: empty map");  // tracker.cpp:79
    if (!(win_w >= 1 && win_h >= 1)) return contract("camshift_refine: empty window");  // :82
    if (!(delta > 0.0)) return contract("camshift_refine: delta must be positive");  // :83
    if (!(max_iter >= 1)) return contract("camshift_refine: need at least one iteration");  // :84
    if (n < 0 || (n > 0 && !(map && starts && out && iterations && zero_mass)))
        return contract("camshift_refine: bad arguments");
    for (int q = 0; q < n; ++q) {  // host copy of the start points: the reference's check (:80-81)
        const double cx = starts[2 * q], cy = starts[2 * q + 1];
        if (!(cx >= 0 && cy >= 0 && cx < w && cy < h)) return contract("camshift_refine: start point outside the map");
    }
    if (n == 0) return SPCT_OK;
    cudaStream_t s = as_stream(stream);
    double *dstart = nullptr, *dout = nullptr;
    int32_t* dint = nullptr;
    spct_status st = cuda_status(malloc_async(&dstart, 2 * n * sizeof(double), s), "camshift alloc");
    if (!st) st = cuda_status(malloc_async(&dout, 2 * n * sizeof(double), s), "camshift alloc");
    if (!st) st = cuda_status(malloc_async(&dint, 2 * n * sizeof(int32_t), s), "camshift alloc");
    if (!st) st = cuda_status(cudaMemcpyAsync(dstart, starts, 2 * n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    if (!st) {
        camshift_warp_kernel<<<static_cast<unsigned>(ceil_div(n, kCamWarps)), 32 * kCamWarps, 0, s>>>(
            map, w, h, dstart, n, win_w, win_h, delta, max_iter, dout, dint, dint + n);
        st = launch_status("camshift_warp_kernel");
    }
    if (!st) st = cuda_status(cudaMemcpyAsync(out, dout, 2 * n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    if (!st) st = cuda_status(cudaMemcpyAsync(iterations, dint, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s), "D2H");
    if (!st) st = cuda_status(cudaMemcpyAsync(zero_mass, dint + n, n * sizeof(int32_t), cudaMemcpyDeviceToHost, s), "D2H");
    if (!st) st = cuda_status(cudaStreamSynchronize(s), "camshift_refine");
    cudaFreeAsync(dstart, s);
    cudaFreeAsync(dout, s);
    cudaFreeAsync(dint, s);
    return st;
}
