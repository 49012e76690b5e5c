// The tracker's swlh-distance map in one sweep over the BinMap, without the quadrant
// tensors (track_loop.cpp:264-283 on top of swih.cpp:115-197).
//
// The reference builds four 16.16 weighted integral histograms and answers every centre
// with quadrant algebra; the answer is the exact pyramid-weighted window histogram
//     F_k(cx, cy) = 2^16 * W_k,  W_k = sum_{window} (c - |dx| - |dy|) [bin = k],
// so it can be computed straight from running sums (all integers, exact):
//     W_k = c N_k - Gx_k - Gy_k,
//   N_k  = sum over the window's columns of v(x), v = the column's count of k over the
//          window rows,
//   Gy_k = sum over the window's columns of m(x), m = sum over the window rows of |r - cy|,
//   Gx_k = sum over the window's columns of |x - cx| v(x)   (from prefix sums of v, x v).
// Per column and bin the sweep keeps a (rows above the centre row), b (rows from it on)
// and m, packed as a | b << 8 | m << 16 (a <= 127, b <= 128, m <= 16256 for kh <= 255).
// Moving the centre row down: m += a - b for every bin (every above-row moves one further,
// every below-row one closer), then three sparse updates for the pixel crossing the
// centre line, the row leaving at the top and the row entering at the bottom.
// The map value is then exactly the quadrant path's: q_k = W_k / mass (= F_k / 2^16 mass),
// d = sum_k |q_k - model_k| in bin order, L = clamp01(1 - d / 2) (FP64, no contraction).
//
// CTA = (strip of 128 centres, band of centre rows); thread t owns extended column
// u0 + t (128 + kw - 1 <= 255 columns: kw <= 128).  Bins go in groups of 32; with more
// bins the partial d of the earlier groups is carried in a global buffer (order kept).
#include <algorithm>
#include <cmath>

#include "spct_internal.h"

using namespace spct_impl;

namespace spct_swlhf {

constexpr int kNC = 128;   // centres per strip
constexpr int kNT = 256;   // threads (>= extended columns)
constexpr int kNBG = 32;   // bins per pass
constexpr int kWarps = kNT / 32;
constexpr int kPS = kNT + 1 + (kNT + 1) / 32 + 1;  // prefix array with one pad word per 32

// Prefix index with a pad word every 32: lane l's eight entries 8l .. 8l + 7 then fall
// into 32 different banks for each i (8-way conflicts without the pad).
__device__ __forceinline__ int pidx(int t) { return t + (t >> 5); }

__global__ void qtab_kernel(double* __restrict__ q, int64_t mass) {
    for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w <= mass;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x)
        q[w] = __ddiv_rn(static_cast<double>(w), static_cast<double>(mass));
}

struct Params {
    const uint16_t* bins;
    int64_t pitch;
    int W, H, k0, nbg;
    int kw, kh, sxl, syt, syb, c;
    const double* qtab;   // qtab[W] = W / mass (correctly rounded), W = 0 .. mass
    const double* model;  // the group's bins
    double* dpart;        // nu * nv partial distances (groups before / after this one), or null
    double* map;          // final group only
    int first, last, band_rows;
};

__device__ __forceinline__ int pix(const Params& p, int x, int y) {
    return static_cast<int>(__ldg(p.bins + static_cast<int64_t>(y) * p.pitch + x)) - p.k0;
}

__global__ void __launch_bounds__(kNT, 2) swlh_fused_kernel(Params p) {
    extern __shared__ uint32_t sm[];
    uint32_t* S = sm;                                            // [kNBG][kNT] column state
    int32_t* Pw = reinterpret_cast<int32_t*>(S + kNBG * kNT);     // [warp][3][kPS] prefixes (padded)
    int32_t* Wb = Pw + kWarps * 3 * kPS;                          // [kNBG][kNC] window sums
    double* Tm = reinterpret_cast<double*>(Wb + kNBG * kNC);      // [kNBG][kNC] |q - model|
    double* mdl = Tm + kNBG * kNC;                                // [kNBG]
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int nu = p.W - p.kw + 1, nv = p.H - p.kh + 1;
    const int u0 = blockIdx.x * kNC;  // first centre of the strip: cx = sxl + u
    const int v0 = blockIdx.y * p.band_rows, v1 = min(nv, v0 + p.band_rows);
    const int ne = kNC + p.kw - 1;     // extended columns: image x = u0 + t
    const int x = u0 + t;
    const bool col_live = t < ne && x < p.W;
    const int nbg = p.nbg;

    for (int i = t; i < kNBG * kNT; i += kNT) S[i] = 0;
    if (t < nbg) mdl[t] = p.model[t];
    __syncthreads();
    // state at the band's first centre row cy0 = syt + v0: window rows [v0, v0 + kh)
    if (col_live) {
        const int cy0 = p.syt + v0;
        for (int r = v0; r < v0 + p.kh; ++r) {
            const int k = pix(p, x, r);
            if (static_cast<unsigned>(k) < static_cast<unsigned>(nbg))
                S[k * kNT + t] += r < cy0 ? (1u + (static_cast<uint32_t>(cy0 - r) << 16))
                                          : ((1u << 8) + (static_cast<uint32_t>(r - cy0) << 16));
        }
    }
    __syncthreads();

    int32_t* P0 = Pw + warp * 3 * kPS;
    int32_t* P1 = P0 + kPS;
    int32_t* PM = P1 + kPS;
    for (int v = v0; v < v1; ++v) {
        const int cy = p.syt + v;
        // 1. window sums of every bin of the row: warp w takes bins w, w + 8, ...; lane l the
        //    extended columns 8l .. 8l + 7
        for (int k = warp; k < nbg; k += kWarps) {
            const uint4 s0 = *reinterpret_cast<const uint4*>(S + k * kNT + 8 * lane);
            const uint4 s1 = *reinterpret_cast<const uint4*>(S + k * kNT + 8 * lane + 4);
            const uint32_t w8[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            int32_t e0[8], e1[8], em[8];
            int32_t r0 = 0, r1 = 0, rm = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int32_t cnt = static_cast<int32_t>((w8[i] & 0xFFu) + ((w8[i] >> 8) & 0xFFu));
                e0[i] = r0;
                e1[i] = r1;
                em[i] = rm;
                r0 += cnt;
                r1 += (8 * lane + i) * cnt;
                rm += static_cast<int32_t>(w8[i] >> 16);
            }
            int32_t i0 = r0, i1 = r1, im = rm;  // inclusive warp scans of the lane totals
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t a0 = __shfl_up_sync(0xffffffffu, i0, o), a1 = __shfl_up_sync(0xffffffffu, i1, o),
                              am = __shfl_up_sync(0xffffffffu, im, o);
                if (lane >= o) {
                    i0 += a0;
                    i1 += a1;
                    im += am;
                }
            }
            const int32_t b0 = i0 - r0, b1 = i1 - r1, bm = im - rm;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int a = pidx(8 * lane + i);
                P0[a] = b0 + e0[i];
                P1[a] = b1 + e1[i];
                PM[a] = bm + em[i];
            }
            if (lane == 31) {
                P0[pidx(kNT)] = i0;
                P1[pidx(kNT)] = i1;
                PM[pidx(kNT)] = im;
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < kNC / 32; ++j) {
                const int u = lane + 32 * j;  // window columns [u, u + kw), centre column u + sxl
                if (u0 + u >= nu) continue;
                const int uc = u + p.sxl, ue = u + p.kw;
                const int iu = pidx(u), ic = pidx(uc), ie = pidx(ue);
                const int32_t n = P0[ie] - P0[iu];
                const int32_t gy = PM[ie] - PM[iu];
                const int32_t gx = uc * (P0[ic] - P0[iu]) - (P1[ic] - P1[iu]) + (P1[ie] - P1[ic]) - uc * (P0[ie] - P0[ic]);
                Wb[k * kNC + u] = p.c * n - gx - gy;
            }
            __syncwarp();
        }
        __syncthreads();  // A: window sums ready, state reads done
        // 2. state -> centre row cy + 1 (own column): every above-row one further, every
        //    below-row one closer, then the three pixels that change sides
        if (col_live && v + 1 < v1) {
            for (int k = 0; k < nbg; ++k) {
                const uint32_t s = S[k * kNT + t];
                S[k * kNT + t] = s + (static_cast<uint32_t>(static_cast<int32_t>(s & 0xFFu) - static_cast<int32_t>((s >> 8) & 0xFFu)) << 16);
            }
            const int kc = pix(p, x, cy), kt = pix(p, x, cy - p.syt), kb = pix(p, x, cy + p.syb);
            if (static_cast<unsigned>(kc) < static_cast<unsigned>(nbg)) S[kc * kNT + t] += 1u - (1u << 8) + (2u << 16);
            if (static_cast<unsigned>(kt) < static_cast<unsigned>(nbg))
                S[kt * kNT + t] -= 1u + (static_cast<uint32_t>(p.syt + 1) << 16);
            if (static_cast<unsigned>(kb) < static_cast<unsigned>(nbg))
                S[kb * kNT + t] += (1u << 8) + (static_cast<uint32_t>(p.syb - 1) << 16);
        }
        // 3. the per-bin terms |W_k / mass - model_k| (track_loop.cpp:275-276)
        for (int i = t; i < nbg * kNC; i += kNT) {
            const int k = i / kNC, u = i % kNC;
            if (u0 + u >= nu) continue;
            const double q = __ldg(p.qtab + Wb[i]);  // == W / mass, the division done once per W
            Tm[i] = fabs(__dsub_rn(q, mdl[k]));
        }
        __syncthreads();  // B: terms ready, state at cy + 1
        // 4. d in bin order, then the map value (or the partial for the next group)
        if (t < kNC && u0 + t < nu) {
            const int64_t o = static_cast<int64_t>(v) * nu + u0 + t;
            double d = p.first ? 0.0 : p.dpart[o];
            for (int k = 0; k < nbg; ++k) d = __dadd_rn(d, Tm[k * kNC + t]);
            if (p.last) {
                const double L = __dsub_rn(1.0, __ddiv_rn(d, 2.0));
                p.map[static_cast<int64_t>(cy) * p.W + p.sxl + u0 + t] = L < 0.0 ? 0.0 : (L > 1.0 ? 1.0 : L);
            } else {
                p.dpart[o] = d;
            }
        }
    }
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

size_t smem_bytes() {
    return static_cast<size_t>(kNBG) * kNT * 4 + static_cast<size_t>(kWarps) * 3 * kPS * 4 +
           static_cast<size_t>(kNBG) * kNC * 4 + static_cast<size_t>(kNBG) * kNC * 8 + kNBG * 8 + 16;
}

}  // namespace spct_swlhf

using namespace spct_swlhf;

extern "C" spct_status spct_cu_swlh_map_direct(const uint16_t* bins, int64_t pitch, int width, int height, int nbins,
                                               int kw, int kh, const double* model, double* map, void* stream) {
    if (!(kw >= 1 && kh >= 1)) return contract("kernel extents must be >= 1");  // swih.cpp:20
    if (!bins || !model || !map || pitch < width || !(width > 0 && height > 0) || nbins < 1)
        return contract("swlh_map: bad arguments");
    if (kw > 128 || kh > 255) return contract("swlh_map_direct: kernel wider than 128 or taller than 255");
    cudaStream_t s = as_stream(stream);
    const int64_t n = static_cast<int64_t>(width) * height;
    if (width < kw || height < kh) {  // track_loop.cpp:265-267: a flat 0.5 map
        fill_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 148 * 8)), 256, 0, s>>>(map, n, 0.5);
        return launch_status("fill_kernel");
    }
    Params p{};
    p.bins = bins;
    p.pitch = pitch;
    p.W = width;
    p.H = height;
    p.kw = kw;
    p.kh = kh;
    p.sxl = kw / 2;
    p.syt = kh / 2;
    p.syb = kh - p.syt;
    p.c = p.sxl + p.syt + 1;
    int64_t mass = 0;  // sum of the pyramid weights (the constant window mass / 2^16)
    for (int dy = -p.syt; dy < p.syb; ++dy)
        for (int dx = -p.sxl; dx < kw - p.sxl; ++dx) mass += p.c - std::abs(dx) - std::abs(dy);
    const int nu = width - kw + 1, nv = height - kh + 1;
    const int strips = static_cast<int>(ceil_div(nu, kNC));
    // bands: about two waves of the resident CTA slots, at least kh rows each (the
    // band-start state costs kh rows of loads)
    const int sms = device_sms();
    const int64_t want = ceil_div(static_cast<int64_t>(sms) * 2 * 2, strips);
    const int nbands = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, nv / std::max(1, kh))));
    p.band_rows = static_cast<int>(ceil_div(nv, nbands));
    const dim3 grid(strips, static_cast<unsigned>(ceil_div(nv, p.band_rows)));
    const size_t smem = smem_bytes();
    ensure_smem(swlh_fused_kernel, smem);
    // W / mass for every possible window sum W (0 .. mass): one division per value instead
    // of one per window and bin
    double* qtab = nullptr;
    if (auto st = cuda_status(malloc_async(&qtab, static_cast<size_t>(mass + 1) * 8, s), "swlh alloc")) return st;
    qtab_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(mass + 1, 256), 148 * 8)), 256, 0, s>>>(qtab, mass);
    if (auto st = launch_status("qtab_kernel")) {
        cudaFreeAsync(qtab, s);
        return st;
    }
    p.qtab = qtab;
    double* dpart = nullptr;
    const int groups = static_cast<int>(ceil_div(nbins, kNBG));
    if (groups > 1)
        if (auto st = cuda_status(malloc_async(&dpart, static_cast<size_t>(nu) * nv * 8, s), "swlh alloc")) {
            cudaFreeAsync(qtab, s);
            return st;
        }
    spct_status st = SPCT_OK;
    for (int g = 0; g < groups && st == SPCT_OK; ++g) {
        p.k0 = g * kNBG;
        p.nbg = std::min(kNBG, nbins - p.k0);
        p.model = model + p.k0;
        p.dpart = dpart;
        p.map = map;
        p.first = g == 0;
        p.last = g == groups - 1;
        swlh_fused_kernel<<<grid, kNT, smem, s>>>(p);
        st = launch_status("swlh_fused_kernel");
    }
    if (dpart) cudaFreeAsync(dpart, s);
    cudaFreeAsync(qtab, s);
    if (st != SPCT_OK) return st;
    replicate_kernel<<<static_cast<unsigned>(std::max<int64_t>(1, ceil_div(n, 256))), 256, 0, s>>>(
        map, width, height, p.sxl, width - (kw - p.sxl), p.syt, height - p.syb);
    return launch_status("replicate_kernel");
}
