// Integral-histogram construction on sm_100a.
//
// Replaces build_integral_histogram / build_tensor and its four CPU schedules
// (reference proj/src/integral.cpp:348-551).  Data flow:
//
//   carries.cu        row carries Lt16[s][y][kl] (count of each slab bin left of strip s),
//                     column counts above each band C16 and corner sums A32, from which
//                     each warp rebuilds the IH row at the top of its band
//   ih_sweep_kernel   per (band, strip, bin slab): one warp per B-bin slab sweeps the
//                     band top to bottom; lane l owns columns 4l..4l+3 of the strip and
//                     keeps H(y, x, k) for those 4 columns x B bins in registers.  A row
//                     update is  H(y,x,k) = H(y-1,x,k) + L(y,k) + #{c <= x in strip : bin = k},
//                     the in-strip count coming from one-hot shifts (four bins per word)
//                     and one warp shuffle scan of 4 bins packed per word.  Each plane-row of the
//                     strip leaves as one coalesced 512-byte run of 16-byte stores.
//
// The pixel -> bin stage (to_grayscale + quantize) is fused into every load.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "spct_internal.h"
#include "sweep_common.cuh"

using namespace spct_dev;

namespace spct_impl {

// ------------------------------------------------------------------ planning

int device_sms() {
    return per_device_int(0, [](int) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device()) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            return 148;  // B200
        }
        return n;
    });
}

BuildPlan plan_build(int width, int height, int bins, int force_B, int ctas_per_sm, int min_band_rows,
                     int strips_per_cta, int max_waves, bool prefer_more_bands) {
    BuildPlan p{};
    p.strips_per_cta = std::max(1, strips_per_cta);
    p.B = force_B ? force_B : (bins <= 4 ? 4 : (bins <= 8 ? 8 : 16));
    const int nslabs = static_cast<int>(ceil_div(bins, p.B));
    p.warps = std::min(8, nslabs);
    p.slab_groups = static_cast<int>(ceil_div(nslabs, p.warps));
    p.Lb = static_cast<int>(round_up(bins, p.B));
    p.nstrips = static_cast<int>(ceil_div(width, kStrip));
    p.Wp = p.nstrips * kStrip;
    int band_rows = 0;
    if (const char* e = std::getenv("SPCT_BAND_ROWS")) band_rows = std::atoi(e);
    if (band_rows <= 0) {
        // Each (strip, band, slab group) tile is one long-lived CTA.  Pick the band count so
        // the tiles fill whole waves of the resident CTA slots (SMs x CTAs per SM): a
        // partial last wave runs at partial occupancy for a full tile time.  Bands are
        // kept >= min_band_rows (carry tables and the matcher's pre-roll scale with
        // 1 / band_rows).
        const int64_t per_band = ceil_div(p.nstrips, p.strips_per_cta) * p.slab_groups;
        const int64_t slots = static_cast<int64_t>(device_sms()) * std::max(1, ctas_per_sm);
        const int64_t nb_max = std::max<int64_t>(1, height / std::max(1, min_band_rows));
        int64_t best_nb = 1;
        double best_eff = -1.0;
        for (int64_t nb = 1; nb <= nb_max; ++nb) {
            const int br = static_cast<int>(ceil_div(height, nb));
            const int64_t tiles = per_band * ceil_div(height, br);
            const int64_t waves = ceil_div(tiles, slots);
            if (waves > max_waves) break;  // finer than max_waves (8) waves buys nothing
            // load balance x a mild preference for >= 2 waves (tail hiding across tiles)
            const double eff = static_cast<double>(tiles) / static_cast<double>(waves * slots) *
                               (waves >= 2 ? 1.0 : 0.97);
            if (eff > best_eff + 1e-9 || (prefer_more_bands && eff > best_eff - 1e-9)) {
                best_eff = eff;
                best_nb = nb;
            }
        }
        band_rows = static_cast<int>(ceil_div(height, best_nb));
    }
    band_rows = std::max(1, std::min(band_rows, height));
    p.band_rows = band_rows;
    p.nbands = static_cast<int>(ceil_div(height, band_rows));
    return p;
}

spct_status make_quant(const spct_source* src, QuantParams* q) {
    if (!src) return contract("build: null source");
    if (!(src->width > 0 && src->height > 0)) return contract("build: empty bin map");
    if (!(src->nbins >= 1 && src->nbins <= 65536)) return contract("quantize: bins must be in [1, 65536]");
    if (src->pitch < src->width) return contract("source pitch smaller than width");
    if (!src->plane[0]) return contract("source plane 0 is null");
    if (src->kind == SPCT_SRC_RGB_U8 && (!src->plane[1] || !src->plane[2]))
        return contract("RGB source needs three planes");
    if (src->kind < SPCT_SRC_BINS_U16 || src->kind > SPCT_SRC_SCALAR_F64) return contract("unknown source kind");
    if (src->kind != SPCT_SRC_BINS_U16 && !(src->hi > src->lo)) return contract("quantize: hi must exceed lo");
    q->kind = src->kind;
    q->nbins = src->nbins;
    q->lo = src->lo;
    q->scale = src->nbins / (src->hi - src->lo);  // imagecore.cpp:33
    q->fast_u8 = (src->kind == SPCT_SRC_GRAY_U8 || src->kind == SPCT_SRC_RGB_U8) && src->lo == 0.0 &&
                 src->hi == 256.0;
    q->p0 = src->plane[0];
    q->p1 = src->plane[1];
    q->p2 = src->plane[2];
    q->pitch = src->pitch;
    q->width = src->width;
    q->height = src->height;
    return SPCT_OK;
}

spct_status check_ih(const spct_ih* t) {
    if (!t) return contract("null tensor descriptor");
    if (!(t->width > 0 && t->height > 0)) return contract("tensor: empty dims");
    if (!(t->nbins_total >= 1 && t->bins >= 1 && t->bin0 >= 0 && t->bin0 + t->bins <= t->nbins_total))
        return contract("tensor: bin slab outside [0, nbins)");
    if (static_cast<uint64_t>(t->width) * static_cast<uint64_t>(t->height) >= (1ull << 32))
        return contract("tensor: height*width must be < 2^32 for uint32 cells");
    if (t->row_pitch < t->width || t->row_pitch % 32 != 0) return contract("tensor: row_pitch must be >= width and a multiple of 32");
    if (t->plane_pitch < t->row_pitch * t->height || t->plane_pitch % 32 != 0)
        return contract("tensor: plane_pitch must be >= height*row_pitch and a multiple of 32");
    return SPCT_OK;
}

spct_status check_carry_dims(int width, int height) {
    if (width >= 65536 || height >= 65536)
        return contract("build: width and height must be below 65536 (16-bit carry tables)");
    return SPCT_OK;
}

}  // namespace spct_impl

using namespace spct_impl;

namespace spct_build {

// ------------------------------------------------------------------ main sweep

// MODE 3 (slide of a joint tensor, motion.cpp:62-69): one group of four planes of
// J += IH(new) - IH(old) in one read-modify-write — V holds the difference of the two
// frames' integral histograms (uint32 wrap arithmetic: J itself stays exact), the two
// frames' rows scanned side by side (two independent shuffle chains).
template <int B>
__device__ __forceinline__ void vpart_group_slide(uint32_t (&V)[4][B], int g, const uint32_t (&tn)[4],
                                                  const uint32_t (&to)[4], uint4 Ln, uint4 Lo, uint32_t* p,
                                                  int64_t plane_pitch, uint32_t store_mask, const uint4* pre) {
    uint32_t Qn[4], Qo[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t mn = shl_clamp(1u, tn[j] - 32u * g), mo = shl_clamp(1u, to[j] - 32u * g);
        Qn[j] = j ? Qn[j - 1] + mn : mn;
        Qo[j] = j ? Qo[j - 1] + mo : mo;
    }
    uint32_t in = Qn[3], io = Qo[3];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        in = scan_add(in, o);
        io = scan_add(io, o);
    }
    const uint32_t en = in - Qn[3], eo = io - Qo[3];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        Qn[j] += en;
        Qo[j] += eo;
    }
    const uint32_t Ld[4] = {Ln.x - Lo.x, Ln.y - Lo.y, Ln.z - Lo.z, Ln.w - Lo.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = 4 * g + i;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            V[j][k] += Ld[i] + __byte_perm(Qn[j], 0, 0x4440 + i) - __byte_perm(Qo[j], 0, 0x4440 + i);
        if (store_mask & (1u << k)) {
            const uint4 o = pre[i];
            *reinterpret_cast<uint4*>(p) = make_uint4(o.x + V[0][k], o.y + V[1][k], o.z + V[2][k], o.w + V[3][k]);
        }
        p += plane_pitch;
    }
}

template <int B, bool GUARD, int MODE>
__global__ void __launch_bounds__(256) ih_sweep_kernel(QuantParams q, PixelMode pm, spct_ih out, int Lb, int Wp,
                                                       int band_rows, int warps_per_cta, FusedCarries fc,
                                                       QuantParams q2 = {}, PixelMode pm2 = {}, FusedCarries fc2 = {}) {
    const int lane = lane_id();
    const int warp = threadIdx.x >> 5;
    const int strip = blockIdx.x;
    const int band = blockIdx.y;
    const int slab = blockIdx.z * warps_per_cta + warp;
    const int kl0 = slab * B;  // first slab-local bin of this warp
    if (kl0 >= out.bins) return;
    const int k_live = min(B, out.bins - kl0);
    if ((k_live < B) != GUARD) return;  // full slabs run the unguarded variant
    const int x0 = strip * kStrip + 4 * lane;  // first of this lane's 4 columns
    const int y0 = band * band_rows, y1 = min(out.height, y0 + band_rows);
    const bool lane_live = x0 < out.row_pitch;
    const int k0 = out.bin0 + kl0;
    const uint32_t kpat0 = pm.byte_mode ? 0x01010101u * static_cast<uint32_t>(k0) : 0u;
    const uint32_t store_mask = lane_live ? (1u << k_live) - 1u : 0u;

    uint32_t V[4][B];
    vpart_init_ca<B>(V, fc.C, fc.A, band, strip, gridDim.y, gridDim.x, Lb, Wp, kl0, x0);
    if (MODE == 3) {  // the difference of the two frames' band-top rows
        uint32_t Vo[4][B];
        vpart_init_ca<B>(Vo, fc2.C, fc2.A, band, strip, gridDim.y, gridDim.x, Lb, Wp, kl0, x0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int k = 0; k < B; ++k) V[j][k] -= Vo[j][k];
    }
    uint32_t* base_ptr = out.data + static_cast<int64_t>(kl0) * out.plane_pitch + x0;
    LtRows<B> lt{(fc.Lt && strip > 0) ? fc.Lt + (static_cast<int64_t>(strip) * out.height + y0) * Lb + kl0 : nullptr,
                 Lb, y1 - y0};
    lt.start();
    LtRows<B> lt2{(MODE == 3 && fc2.Lt && strip > 0) ? fc2.Lt + (static_cast<int64_t>(strip) * out.height + y0) * Lb + kl0
                                                    : nullptr,
                  Lb, y1 - y0};
    if (MODE == 3) lt2.start();
    const uint32_t kpat2 = (MODE == 3 && pm2.byte_mode) ? 0x01010101u * static_cast<uint32_t>(k0) : 0u;

    // accumulate modes read-modify-write the tensor: its cells of row y + 1 are loaded
    // during row y (B x 16 bytes per lane; only the B <= 8 plans use these modes cheaply)
    constexpr int NPRE = MODE != 0 ? B : 1;
    uint4 pre[NPRE], pnx[NPRE];
    auto load_row = [&](int y, uint4 (&d)[NPRE]) {
        const uint32_t* r = base_ptr + static_cast<int64_t>(y) * out.row_pitch;
#pragma unroll
        for (int k = 0; k < NPRE; ++k)
            d[k] = (store_mask & (1u << k)) ? *reinterpret_cast<const uint4*>(r + static_cast<int64_t>(k) * out.plane_pitch)
                                            : make_uint4(0, 0, 0, 0);
    };
    if (MODE != 0 && y0 < y1) load_row(y0, pnx);

    uint32_t nxt = load_bins4_raw(q, pm, x0, y0, k0, B);
    uint32_t nxt2 = MODE == 3 ? load_bins4_raw(q2, pm2, x0, y0, k0, B) : 0u;
    for (int y = y0; y < y1; ++y) {
        const uint32_t cur = decode_bins4(pm, nxt);
        if (y + 1 < y1) nxt = load_bins4_raw(q, pm, x0, y + 1, k0, B);
        uint32_t cur2 = 0;
        if (MODE == 3) {
            cur2 = decode_bins4(pm2, nxt2);
            if (y + 1 < y1) nxt2 = load_bins4_raw(q2, pm2, x0, y + 1, k0, B);
        }
        if (MODE != 0) {
#pragma unroll
            for (int k = 0; k < NPRE; ++k) pre[k] = pnx[k];
            if (y + 1 < y1) load_row(y + 1, pnx);
        }
        uint32_t t4[4];
        onehot_shifts(cur ^ kpat0, t4);
        lt.row(y - y0);
        uint32_t* prow = base_ptr + static_cast<int64_t>(y) * out.row_pitch;
        if constexpr (MODE == 3) {
            uint32_t t4o[4];
            onehot_shifts(cur2 ^ kpat2, t4o);
            lt2.row(y - y0);
#pragma unroll
            for (int g = 0; g < B / 4; ++g)
                vpart_group_slide<B>(V, g, t4, t4o, lt.group(y - y0, g), lt2.group(y - y0, g),
                                     prow + static_cast<int64_t>(4 * g) * out.plane_pitch, out.plane_pitch, store_mask,
                                     pre + 4 * g);
        } else {
#pragma unroll
            for (int g = 0; g < B / 4; ++g)
                vpart_group_q<B, MODE>(V, g, t4, lt.group(y - y0, g), prow + static_cast<int64_t>(4 * g) * out.plane_pitch,
                                       out.plane_pitch, store_mask, MODE != 0 ? pre + 4 * g : nullptr);
        }
    }
}

// ------------------------------------------------------------------ small kernels

__global__ void gray_kernel(const uint8_t* __restrict__ r, const uint8_t* __restrict__ g,
                            const uint8_t* __restrict__ b, int64_t n, uint8_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<uint8_t>(gray_of(r[i], g[i], b[i]));
}

// 16 pixels per thread (every plane and the output 16-byte aligned): 16-byte loads and
// stores, the division by 3 as a multiply-shift (exact for sums <= 766).
__device__ __forceinline__ uint32_t gray4(uint32_t r, uint32_t g, uint32_t b) {
    uint32_t o = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t s = ((r >> (8 * j)) & 0xFFu) + ((g >> (8 * j)) & 0xFFu) + ((b >> (8 * j)) & 0xFFu) + 1u;
        o |= ((s * 0xAAABu) >> 17) << (8 * j);  // s / 3 for s < 2^15
    }
    return o;
}

__global__ void gray16_kernel(const uint4* __restrict__ r, const uint4* __restrict__ g, const uint4* __restrict__ b,
                              int64_t n16, uint4* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n16;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint4 x = __ldg(r + i), y = __ldg(g + i), z = __ldg(b + i);
        out[i] = make_uint4(gray4(x.x, y.x, z.x), gray4(x.y, y.y, z.y), gray4(x.z, y.z, z.z), gray4(x.w, y.w, z.w));
    }
}

// quantize of an 8-bit gray frame with the default range (bin = v * nbins >> 8), 16 pixels
// per thread on 16-byte aligned rows: one 16-byte load, two 16-byte stores.
__global__ void quantize16_kernel(const uint8_t* __restrict__ src, int64_t pitch, int w, int h, uint32_t nbins,
                                  uint16_t* __restrict__ out) {
    const int per_row = w / 16;
    const int64_t n = static_cast<int64_t>(per_row) * h;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int y = static_cast<int>(i / per_row), c = static_cast<int>(i % per_row);
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + static_cast<int64_t>(y) * pitch) + c);
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t a = wv[j];
            o[2 * j] = (((a & 0xFFu) * nbins) >> 8) | ((((a >> 8) & 0xFFu) * nbins) >> 8) << 16;
            o[2 * j + 1] = ((((a >> 16) & 0xFFu) * nbins) >> 8) | (((a >> 24) * nbins) >> 8) << 16;
        }
        uint4* d = reinterpret_cast<uint4*>(out + static_cast<int64_t>(y) * w) + 2 * c;
        d[0] = make_uint4(o[0], o[1], o[2], o[3]);
        d[1] = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

__global__ void quantize_kernel(QuantParams q, uint16_t* __restrict__ out) {
    const int64_t n = static_cast<int64_t>(q.width) * q.height;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int y = static_cast<int>(i / q.width), x = static_cast<int>(i % q.width);
        out[i] = static_cast<uint16_t>(pixel_bin(q, x, y));
    }
}

__global__ void binmax_kernel(const uint16_t* __restrict__ bins, int64_t pitch, int w, int h, int* out) {
    __shared__ int wmax[8];
    int m = 0;
    for (int y = blockIdx.y; y < h; y += gridDim.y) {
        const uint16_t* row = bins + static_cast<int64_t>(y) * pitch;
        for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < w; x += gridDim.x * blockDim.x)
            m = max(m, static_cast<int>(__ldg(row + x)));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {  // one atomic per block
        for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) m = max(m, wmax[i]);
        atomicMax(out, m);
    }
}

__global__ void export_kernel(spct_ih t, int k0, int k1, uint64_t* __restrict__ dst) {
    const int64_t W1 = t.width + 1, H1 = t.height + 1;
    const int64_t n = static_cast<int64_t>(k1 - k0) * H1 * W1;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = i / (H1 * W1), rem = i % (H1 * W1);
        const int64_t y = rem / W1, x = rem % W1;
        uint64_t v = 0;
        if (y > 0 && x > 0) v = t.data[(k0 + k) * t.plane_pitch + (y - 1) * t.row_pitch + (x - 1)];
        dst[i] = v;
    }
}

int grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    return static_cast<int>(std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 32));
}

}  // namespace spct_build

using namespace spct_build;

namespace spct_impl {

int build_ctas_per_sm(int B, int threads) {
    const int bi = B == 4 ? 0 : (B == 8 ? 1 : 2), wi = std::min(8, std::max(1, threads / 32));
    return per_device_int(100 + 16 * bi + wi, [](int key) {
        const int bi = (key - 100) / 16, threads = 32 * ((key - 100) % 16);
        int n = 0;
        cudaError_t e;
        if (bi == 0) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ih_sweep_kernel<4, false, 0>, threads, 0);
        else if (bi == 1) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ih_sweep_kernel<8, false, 0>, threads, 0);
        else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, ih_sweep_kernel<16, false, 0>, threads, 0);
        if (e != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = 2;
        }
        return n;
    });
}

BuildPlan plan_build_sweep(int width, int height, int bins) {
    // Small histograms: fewer bins per warp so a CTA still has ~4 warps (16 bins as one
    // 16-bin warp left a single warp per strip and band, far too little to hide latency).
    const int B = bins >= 64 ? 16 : (bins >= 32 ? 8 : 4);
    const BuildPlan probe = plan_build(width, height, bins, B, 2, 32);
    return plan_build(width, height, bins, B, build_ctas_per_sm(probe.B, 32 * probe.warps), 32);
}

BuildPlan plan_fused_sweep(int width, int height, int bins) {
    // strips per CTA as in spct_fused::fused_strips (fused_kernel.cuh): 8 warps of 16 bins
    // each, S = 128 / (16 * ceil(bins / 16)) strips side by side for narrow histograms.
    // The band floor trades the band-start window state (kh - 1 pre-roll rows, or the
    // carry tables for narrow CTAs) against filling the GPU.
    const int S = bins > 64 ? 1 : (bins > 32 ? 2 : (bins > 16 ? 4 : 8));
    const int ctas = fused_ctas_per_sm(S);
    // (one-strip CTAs: at most 4 waves, the most bands among equally filled plans — C4's
    // 128-bin groups measured 14.97 ms with the exactly-filled 8 waves of 222-row bands,
    // 14.62-14.69 ms with 228-456-row bands; C3's 4 waves of 111 rows stay)
    const BuildPlan p = S == 1 ? plan_build(width, height, bins, 16, ctas, 64, S, 4, true)
                               : plan_build(width, height, bins, 16, ctas, 16, S);
    // small frames of narrow histograms (C2: 1024^2 x 32 bins) that do not fill one wave of
    // CTAs with 16-row bands: down to 8 rows (C2 0.106 -> 0.097 ms)
    const int64_t tiles = ceil_div(p.nstrips, S) * static_cast<int64_t>(p.nbands) * p.slab_groups;
    if (S > 1 && std::getenv("SPCT_BAND_ROWS") == nullptr && tiles < static_cast<int64_t>(device_sms()) * ctas)
        return plan_build(width, height, bins, 16, ctas, 8, S);
    return p;
}

}  // namespace spct_impl

// ------------------------------------------------------------------ C-ABI

extern "C" spct_status spct_cu_to_grayscale(const uint8_t* r, const uint8_t* g, const uint8_t* b, int64_t n,
                                            uint8_t* out, void* stream) {
    if (n < 0) return contract("to_grayscale: negative size");
    if (n == 0) return SPCT_OK;
    if (!r || !g || !b || !out) return contract("to_grayscale: null plane");
    cudaStream_t s = as_stream(stream);
    const bool vec = ((reinterpret_cast<uintptr_t>(r) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(b) |
                       reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    const int64_t n16 = vec ? n / 16 : 0;
    if (n16 > 0)
        gray16_kernel<<<grid_for(n16, 256), 256, 0, s>>>(reinterpret_cast<const uint4*>(r), reinterpret_cast<const uint4*>(g),
                                                         reinterpret_cast<const uint4*>(b), n16, reinterpret_cast<uint4*>(out));
    if (n > 16 * n16)
        gray_kernel<<<grid_for(n - 16 * n16, 256), 256, 0, s>>>(r + 16 * n16, g + 16 * n16, b + 16 * n16, n - 16 * n16,
                                                                out + 16 * n16);
    return launch_status("to_grayscale");
}

extern "C" spct_status spct_cu_quantize(const spct_source* src, uint16_t* out, void* stream) {
    QuantParams q;
    if (!src) return contract("quantize: null source");
    if (!(src->width > 0 && src->height > 0)) return contract("quantize: empty image");
    if (auto st = make_quant(src, &q)) return st;
    if (!out) return contract("quantize: null output");
    const int64_t n = static_cast<int64_t>(q.width) * q.height;
    if (q.kind == SPCT_SRC_GRAY_U8 && q.fast_u8 && q.width % 16 == 0 && q.pitch % 16 == 0 &&
        reinterpret_cast<uintptr_t>(q.p0) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0) {
        quantize16_kernel<<<grid_for(n / 16, 256), 256, 0, as_stream(stream)>>>(
            static_cast<const uint8_t*>(q.p0), q.pitch, q.width, q.height, static_cast<uint32_t>(q.nbins), out);
        return launch_status("quantize");
    }
    quantize_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(q, out);
    return launch_status("quantize");
}

extern "C" spct_status spct_cu_binmap_max(const uint16_t* bins, int64_t pitch, int width, int height, int* out_max,
                                          void* stream) {
    if (!(width > 0 && height > 0)) return contract("build: empty bin map");
    if (!bins || !out_max || pitch < width) return contract("binmap_max: bad arguments");
    int* d = nullptr;
    cudaStream_t s = as_stream(stream);
    if (auto st = cuda_status(malloc_async(&d, sizeof(int), s), "binmap_max alloc")) return st;
    cudaMemsetAsync(d, 0, sizeof(int), s);
    const unsigned gx = static_cast<unsigned>(std::min<int64_t>(ceil_div(width, 256), 8));
    const unsigned gy = static_cast<unsigned>(std::min<int64_t>(height, std::max<int64_t>(1, 148 * 8 / gx)));
    binmax_kernel<<<dim3(gx, gy), 256, 0, s>>>(bins, pitch, width, height, d);
    spct_status st = launch_status("binmap_max");
    int h = 0;
    if (st == SPCT_OK) st = cuda_status(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s), "binmap_max copy");
    cudaFreeAsync(d, s);
    if (st == SPCT_OK) st = cuda_status(cudaStreamSynchronize(s), "binmap_max sync");
    *out_max = h;
    return st;
}

extern "C" spct_status spct_cu_ih_layout(int width, int height, int bins, int64_t* row_pitch, int64_t* plane_pitch,
                                         uint64_t* bytes) {
    if (!(width > 0 && height > 0 && bins >= 1)) return contract("ih_layout: empty tensor");
    const int64_t rp = round_up(width, 32);
    const int64_t pp = rp * height;
    if (row_pitch) *row_pitch = rp;
    if (plane_pitch) *plane_pitch = pp;
    if (bytes) *bytes = static_cast<uint64_t>(pp) * static_cast<uint64_t>(bins) * 4u;
    return SPCT_OK;
}

extern "C" spct_status spct_cu_ih_build_workspace(const spct_source* src, int bin0, int bins, size_t* bytes) {
    (void)bin0;
    if (!src || !bytes) return contract("ih_build_workspace: null argument");
    if (!(src->width > 0 && src->height > 0 && bins >= 1)) return contract("build: empty bin map");
    const BuildPlan p = plan_build_sweep(src->width, src->height, bins);
    const BuildPlan pf = plan_fused_sweep(src->width, src->height, bins);  // fused sweep: 16 bins per warp
    *bytes = std::max(fused_carry_layout(p, src->height).total, fused_carry_layout(pf, src->height, true).total) +
             fused_prep_bytes(bins) + 256 + (src->kind == SPCT_SRC_RGB_U8 ? fused_gray_bytes(src) : 0);
    return SPCT_OK;
}


namespace {

template <int MODE>
void launch_sweep(const BuildPlan& p, dim3 grid, int threads, cudaStream_t s, const QuantParams& q, const PixelMode& pm,
                  const spct_ih& out, const FusedCarries& fc, const QuantParams& q2 = {}, const PixelMode& pm2 = {},
                  const FusedCarries& fc2 = {}) {
    switch (p.B) {
#define SPCT_SWEEP(BB)                                                                                               \
    ih_sweep_kernel<BB, false, MODE><<<grid, threads, 0, s>>>(q, pm, out, p.Lb, p.Wp, p.band_rows, p.warps, fc, q2,  \
                                                              pm2, fc2);                                             \
    if (out.bins % BB) ih_sweep_kernel<BB, true, MODE><<<grid, threads, 0, s>>>(q, pm, out, p.Lb, p.Wp, p.band_rows, \
                                                                                p.warps, fc, q2, pm2, fc2);
        case 4: SPCT_SWEEP(4) break;
        case 8: SPCT_SWEEP(8) break;
        default: SPCT_SWEEP(16) break;
#undef SPCT_SWEEP
    }
}

spct_status build_mode(const spct_source* src, const spct_ih* out, void* workspace, size_t workspace_bytes,
                       void* stream, int mode) {
    QuantParams q;
    if (auto st = make_quant(src, &q)) return st;
    if (auto st = check_ih(out)) return st;
    if (!out->data) return contract("ih_build: null tensor data");
    if (auto st = check_carry_dims(out->width, out->height)) return st;
    if (out->width != src->width || out->height != src->height || out->nbins_total != src->nbins)
        return contract("ih_build: tensor dims do not match the source");
    if (reinterpret_cast<uintptr_t>(out->data) % 16 != 0) return contract("ih_build: tensor data must be 16-byte aligned");
    const BuildPlan p = plan_build_sweep(out->width, out->height, out->bins);
    cudaStream_t s = as_stream(stream);
    FusedCarries fc{};
    if (auto st = build_fused_carries(q, *out, p, workspace, workspace_bytes, s, &fc)) return st;
    dim3 grid(p.nstrips, p.nbands, p.slab_groups);
    const int threads = 32 * p.warps;
    const int prof = prof_begin(mode ? "ih_accumulate" : "ih_sweep", s);
    const PixelMode pm = make_pixel_mode(q, out->bin0);
    if (mode == 0) launch_sweep<0>(p, grid, threads, s, q, pm, *out, fc);
    else if (mode > 0) launch_sweep<1>(p, grid, threads, s, q, pm, *out, fc);
    else launch_sweep<2>(p, grid, threads, s, q, pm, *out, fc);
    prof_end(prof, s);
    return launch_status("ih_sweep_kernel");
}

}  // namespace

extern "C" spct_status spct_cu_ih_build(const spct_source* src, const spct_ih* out, void* workspace,
                                        size_t workspace_bytes, void* stream) {
    return build_mode(src, out, workspace, workspace_bytes, stream, 0);
}

namespace {
// slide plans keep B <= 8 bins per warp (V and the read-ahead tensor row cost 8 B registers)
BuildPlan plan_slide(int width, int height, int bins) {
    return plan_build(width, height, bins, bins >= 32 ? 8 : 4, 2, 32);
}
size_t slide_half_bytes(const BuildPlan& p, int height) {
    return static_cast<size_t>(round_up(static_cast<int64_t>(fused_carry_layout(p, height).total), 256));
}
}  // namespace

extern "C" spct_status spct_cu_ih_slide_workspace(int width, int height, int bins, size_t* bytes) {
    if (!bytes) return contract("ih_slide_workspace: null argument");
    if (!(width > 0 && height > 0 && bins >= 1)) return contract("build: empty bin map");
    *bytes = 2 * slide_half_bytes(plan_slide(width, height, bins), height) + 256;
    return SPCT_OK;
}

extern "C" spct_status spct_cu_ih_slide(const spct_source* src_new, const spct_source* src_old, const spct_ih* acc,
                                        void* workspace, size_t workspace_bytes, void* stream) {
    QuantParams q[2];
    if (!src_new || !src_old) return contract("ih_slide: null source");
    if (auto st = make_quant(src_new, &q[0])) return st;
    if (auto st = make_quant(src_old, &q[1])) return st;
    if (auto st = check_ih(acc)) return st;
    if (!acc->data) return contract("ih_build: null tensor data");
    if (auto st = check_carry_dims(acc->width, acc->height)) return st;
    for (const spct_source* src : {src_new, src_old})
        if (acc->width != src->width || acc->height != src->height || acc->nbins_total != src->nbins)
            return contract("ih_build: tensor dims do not match the source");
    if (reinterpret_cast<uintptr_t>(acc->data) % 16 != 0) return contract("ih_build: tensor data must be 16-byte aligned");
    const BuildPlan p = plan_slide(acc->width, acc->height, acc->bins);
    const size_t half = slide_half_bytes(p, acc->height);
    if (!workspace || workspace_bytes < 2 * half) return contract("ih_slide: workspace too small (spct_cu_ih_slide_workspace)");
    cudaStream_t s = as_stream(stream);
    void* ws[2] = {workspace, static_cast<char*>(workspace) + half};
    FusedCarries fc[2] = {};
    if (auto st = build_fused_carries_multi(2, q, *acc, p, ws, half, s, fc, 0)) return st;
    dim3 grid(p.nstrips, p.nbands, p.slab_groups);
    const int prof = prof_begin("ih_slide", s);
    const PixelMode pm0 = make_pixel_mode(q[0], acc->bin0), pm1 = make_pixel_mode(q[1], acc->bin0);
    launch_sweep<3>(p, grid, 32 * p.warps, s, q[0], pm0, *acc, fc[0], q[1], pm1, fc[1]);
    prof_end(prof, s);
    return launch_status("ih_sweep_kernel");
}

extern "C" spct_status spct_cu_ih_accumulate(const spct_source* src, const spct_ih* acc, int sign, void* workspace,
                                             size_t workspace_bytes, void* stream) {
    if (sign != 1 && sign != -1) return contract("ih_accumulate: sign must be +1 or -1");
    return build_mode(src, acc, workspace, workspace_bytes, stream, sign);
}

extern "C" spct_status spct_cu_ih_export_u64(const spct_ih* t, int k0, int k1, uint64_t* dst, void* stream) {
    if (auto st = check_ih(t)) return st;
    if (!(0 <= k0 && k0 <= k1 && k1 <= t->bins)) return contract("ih_export: plane range outside the tensor");
    if (k0 == k1) return SPCT_OK;
    if (!dst || !t->data) return contract("ih_export: null pointer");
    const int64_t n = static_cast<int64_t>(k1 - k0) * (t->height + 1) * (t->width + 1);
    export_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(*t, k0, k1, dst);
    return launch_status("ih_export");
}
