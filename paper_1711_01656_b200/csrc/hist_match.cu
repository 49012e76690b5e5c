// Sliding-window histogram matching over a device integral histogram, region
// queries, and the likelihood finalisation.
//
// Replaces hist_distance_map + spread_valid (reference proj/src/likelihood.cpp:44-58,
// :193-225) and region_histogram / region_count (integral.cpp:561-577).
#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>

#include "spct_internal.h"

using namespace spct_dev;
using namespace spct_impl;

namespace spct_impl {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

}  // namespace spct_impl

namespace spct_kern {

// Unpadded device cell with the reference's zero padding folded in:
// returns H(y, x) in reference (padded) coordinates.
__device__ __forceinline__ uint32_t H_at(const uint32_t* __restrict__ plane, int64_t row_pitch, int y, int x) {
    return (y > 0 && x > 0) ? __ldg(plane + static_cast<int64_t>(y - 1) * row_pitch + (x - 1)) : 0u;
}

struct MatchParams {
    int kw, kh, nu, nv;
    double p, inv_p, T, invT;
    int T_pow2;   // kw*kh is a power of two: c / T == c * (1/T) exactly
    int metric;
    int p_kind;   // 1: p == 1, 2: p == 2, 0: general pow
    int norm;     // 1: divide by the window's actual total (full tensors, likelihood.cpp:212-214)
};

// Per-bin term of the window statistic.  MINKOWSKI follows likelihood.cpp:218-219
// operation by operation: q = h[k] / total (IEEE divide; exact multiply when T is a
// power of two), |q - t|, pow(., p) (identity for p == 1, x*x for p == 2).
__device__ __forceinline__ double bin_term(double cd, double t, const MatchParams& m, double total, double inv_total) {
    const double q = inv_total != 0.0 ? __dmul_rn(cd, inv_total) : __ddiv_rn(cd, total);
    switch (m.metric) {
        case SPCT_METRIC_MINKOWSKI: {
            const double a = fabs(__dsub_rn(q, t));
            if (m.p_kind == 1) return a;
            if (m.p_kind == 2) return __dmul_rn(a, a);
            return pow(a, m.p);
        }
        case SPCT_METRIC_INTERSECTION:
            return fmin(q, t);
        case SPCT_METRIC_BHATTACHARYYA:
            return sqrt(__dmul_rn(q, t));
        default: {  // chi-square
            const double den = __dadd_rn(q, t);
            if (!(den > 0.0)) return 0.0;
            const double df = __dsub_rn(q, t);
            return __ddiv_rn(__dmul_rn(df, df), den);
        }
    }
}

__device__ __forceinline__ double finalize_value(double s, const MatchParams& m, double dmax) {
    if (s < 0.0) return 0.0;  // massless window (likelihood.cpp:215): no match
    double L;
    switch (m.metric) {
        case SPCT_METRIC_MINKOWSKI: {
            const double d = m.p_kind == 1 ? s : pow(s, m.inv_p);
            L = __dsub_rn(1.0, __ddiv_rn(d, dmax));
            break;
        }
        case SPCT_METRIC_CHISQ:
            L = __dsub_rn(1.0, __ddiv_rn(s, 2.0));
            break;
        default:
            L = s;
    }
    return L < 0.0 ? 0.0 : (L > 1.0 ? 1.0 : L);
}

// Window count of plane k: region_histogram (integral.cpp:561-577) in the reference's
// uint64 arithmetic (wraps like the reference for a tensor that is not monotone), as the
// double the reference divides.
__device__ __forceinline__ double window_count(const spct_ih& t, int k, int ya, int yb, int xa, int xb) {
    const uint32_t* pl = t.data + static_cast<int64_t>(k) * t.plane_pitch;
    const uint64_t c = static_cast<uint64_t>(H_at(pl, t.row_pitch, yb, xb)) - H_at(pl, t.row_pitch, ya, xb) -
                       H_at(pl, t.row_pitch, yb, xa) + H_at(pl, t.row_pitch, ya, xa);
    return static_cast<double>(c);
}

// One thread per valid window (u, v); planes visited in order k = 0 .. bins-1 so the
// per-window sum has the reference's rounding sequence when the tensor holds every bin
// (likelihood.cpp:211-219).  With m.norm the window's histogram is divided by its actual
// total (the reference's `total`); the first pass assumes total == kw * kh (true for every
// tensor built from a bin map) while summing the real total, and a window whose total
// differs is recomputed; a massless window gets the sentinel -1 (finalised to 0).
// `gate` (optional, device): run only if *gate != 0 (the tensor matcher found a tensor that
// is not the integral histogram of a bin map, tensor_match.cu).
__global__ void __launch_bounds__(256) match_partial_kernel(spct_ih t, const double* __restrict__ tmpl, MatchParams m,
                                                            double* __restrict__ partial, int accumulate,
                                                            const uint32_t* __restrict__ gate) {
    if (gate && *gate == 0) return;
    const int64_t n = static_cast<int64_t>(m.nu) * m.nv;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int u = static_cast<int>(i % m.nu), v = static_cast<int>(i / m.nu);
        const double s0 = accumulate ? partial[i] : 0.0;
        const int ya = v, yb = v + m.kh, xa = u, xb = u + m.kw;
        const double invT = m.T_pow2 ? m.invT : 0.0;
        double s = s0, total = 0.0;
        for (int k = 0; k < t.bins; k += 4) {
            double c[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) c[j] = k + j < t.bins ? window_count(t, k + j, ya, yb, xa, xb) : 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (k + j < t.bins) {
                    total = __dadd_rn(total, c[j]);
                    s = __dadd_rn(s, bin_term(c[j], __ldg(tmpl + t.bin0 + k + j), m, m.T, invT));
                }
        }
        if (m.norm && total != m.T) {
            if (!(total > 0.0)) {
                s = -1.0;
            } else {
                s = s0;
                for (int k = 0; k < t.bins; ++k)
                    s = __dadd_rn(s, bin_term(window_count(t, k, ya, yb, xa, xb), __ldg(tmpl + t.bin0 + k), m, total,
                                              0.0));
            }
        }
        partial[i] = s;
    }
}

// spread_valid (likelihood.cpp:44-58) fused with the finalisation (:220-221).
__global__ void finalize_kernel(const double* __restrict__ partial, int W, int H, MatchParams m, double dmax,
                                double* __restrict__ map, const uint32_t* __restrict__ gate) {
    if (gate && *gate == 0) return;
    const int cx0 = (m.kw - 1) / 2, cy0 = (m.kh - 1) / 2;
    const int64_t n = static_cast<int64_t>(W) * H;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % W), y = static_cast<int>(i / W);
        const int vx = min(max(x, cx0), cx0 + m.nu - 1) - cx0;
        const int vy = min(max(y, cy0), cy0 + m.nv - 1) - cy0;
        map[i] = finalize_value(partial[static_cast<int64_t>(vy) * m.nu + vx], m, dmax);
    }
}

__global__ void region_kernel(spct_ih t, const int32_t* __restrict__ rects, int n, uint32_t* __restrict__ out) {
    const int64_t total = static_cast<int64_t>(n) * t.bins;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(i / t.bins), k = static_cast<int>(i % t.bins);
        const int x1 = rects[4 * r], y1 = rects[4 * r + 1];
        const int x2 = x1 + rects[4 * r + 2], y2 = y1 + rects[4 * r + 3];
        const uint32_t* pl = t.data + static_cast<int64_t>(k) * t.plane_pitch;
        out[i] = H_at(pl, t.row_pitch, y2, x2) - H_at(pl, t.row_pitch, y1, x2) - H_at(pl, t.row_pitch, y2, x1) +
                 H_at(pl, t.row_pitch, y1, x1);
    }
}

int grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    return static_cast<int>(std::min<int64_t>(std::max<int64_t>(g, 1), 148 * 16));
}

}  // namespace spct_kern

using namespace spct_kern;

namespace spct_impl {

spct_status make_match(int width, int height, int kw, int kh, double p, int metric, MatchParams* m) {
    if (!(p >= 1.0)) return contract("hist_distance_map: Minkowski order must be >= 1");
    if (!(kw >= 1 && kh >= 1 && kw <= width && kh <= height)) return contract("hist_distance_map: kernel exceeds image");
    if (metric < SPCT_METRIC_MINKOWSKI || metric > SPCT_METRIC_CHISQ) return contract("hist_match: unknown metric");
    m->kw = kw;
    m->kh = kh;
    m->nu = width - kw + 1;
    m->nv = height - kh + 1;
    m->p = p;
    m->inv_p = 1.0 / p;
    m->metric = metric;
    m->p_kind = p == 1.0 ? 1 : (p == 2.0 ? 2 : 0);
    const int64_t T = static_cast<int64_t>(kw) * kh;
    m->T = static_cast<double>(T);
    m->invT = 1.0 / m->T;
    m->T_pow2 = (T & (T - 1)) == 0;
    m->norm = 0;
    return SPCT_OK;
}

}  // namespace spct_impl

extern "C" const char* spct_cu_last_error(void) { return g_err.c_str(); }

extern "C" int spct_cu_version(void) { return 1; }

extern "C" spct_status spct_cu_device_info(int* major, int* minor, int* sms) {
    int dev = 0;
    if (auto st = cuda_status(cudaGetDevice(&dev), "cudaGetDevice")) return st;
    cudaDeviceProp prop;
    if (auto st = cuda_status(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties")) return st;
    if (major) *major = prop.major;
    if (minor) *minor = prop.minor;
    if (sms) *sms = prop.multiProcessorCount;
    return SPCT_OK;
}

extern "C" spct_status spct_cu_estimate_memory(int w, int h, int bins, int elem, uint64_t* padded, uint64_t* raw,
                                               int* degenerate) {
    // integral.cpp:592-599
    if (w < 0 || h < 0 || bins < 0 || elem < 0) return contract("estimate_memory: negative input");
    if (degenerate) *degenerate = (w == 0 || h == 0 || bins == 0 || elem == 0);
    if (padded) *padded = static_cast<uint64_t>(bins) * (h + 1) * (w + 1) * elem;
    if (raw) *raw = static_cast<uint64_t>(bins) * h * w * elem;
    return SPCT_OK;
}

extern "C" spct_status spct_cu_schedule_stats(int w, int h, int tile, int scan_len, long long* iterations,
                                              long long* tiles, double* eff) {
    // integral.cpp:579-590
    if (!(w > 0 && h > 0 && tile > 0)) return contract("schedule_stats: positive dims required");
    if (!(scan_len >= 2)) return contract("schedule_stats: scan_len must be >= 2");
    const long long tx = (w + tile - 1) / tile, ty = (h + tile - 1) / tile;
    if (iterations) *iterations = tx + ty - 1;
    if (tiles) *tiles = tx * ty;
    const double n = scan_len;
    if (eff) *eff = 3.0 * (n - 1.0) / (n * std::log2(n));
    return SPCT_OK;
}

extern "C" spct_status spct_cu_hist_check(int nbins, int width, int height, const double* tmpl, int ntmpl, int kw,
                                          int kh, double p) {
    // likelihood.cpp:196-206, same predicates and messages
    if (!(p >= 1.0)) return contract("hist_distance_map: Minkowski order must be >= 1");
    if (!(kw >= 1 && kh >= 1 && kw <= width && kh <= height)) return contract("hist_distance_map: kernel exceeds image");
    if (ntmpl != nbins) return contract("hist_distance_map: template bin count mismatch");
    if (!tmpl && ntmpl > 0) return contract("hist_distance_map: null template");
    double tsum = 0.0;
    for (int k = 0; k < ntmpl; ++k) {
        if (!(tmpl[k] >= 0.0)) return contract("hist_distance_map: negative template entry");
        tsum += tmpl[k];
    }
    if (!(std::abs(tsum - 1.0) <= 1e-6)) return contract("hist_distance_map: template must be normalized");
    return SPCT_OK;
}

extern "C" spct_status spct_cu_region_counts(const spct_ih* t, const int32_t* rects, int n, uint32_t* out,
                                             void* stream) {
    if (auto st = check_ih(t)) return st;
    if (n < 0) return contract("region_counts: negative count");
    if (n == 0) return SPCT_OK;
    if (!rects || !out || !t->data) return contract("region_counts: null pointer");
    region_kernel<<<grid_for(static_cast<int64_t>(n) * t->bins, 256), 256, 0, as_stream(stream)>>>(*t, rects, n, out);
    return launch_status("region_counts");
}

namespace {
spct_status hist_partial_impl(const spct_ih* t, const double* tmpl, int kw, int kh, double p, int metric,
                              double* partial, int accumulate, int norm, void* stream, const uint32_t* gate = nullptr) {
    if (auto st = check_ih(t)) return st;
    MatchParams m;
    if (auto st = make_match(t->width, t->height, kw, kh, p, metric, &m)) return st;
    m.norm = norm;
    if (!tmpl || !partial || !t->data) return contract("hist_partial: null pointer");
    const int64_t n = static_cast<int64_t>(m.nu) * m.nv;
    const int prof = prof_begin("match_partial", as_stream(stream));
    match_partial_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(*t, tmpl, m, partial, accumulate, gate);
    prof_end(prof, as_stream(stream));
    return launch_status("match_partial_kernel");
}
}  // namespace

extern "C" spct_status spct_cu_hist_partial(const spct_ih* t, const double* tmpl, int kw, int kh, double p, int metric,
                                            double* partial, int accumulate, void* stream) {
    return hist_partial_impl(t, tmpl, kw, kh, p, metric, partial, accumulate, 0, stream);
}

namespace {
spct_status finalize_impl(const double* partial, int width, int height, int kw, int kh, double p, int metric,
                          double* map, void* stream, const uint32_t* gate) {
    MatchParams m;
    if (!(width > 0 && height > 0)) return contract("hist_finalize: empty map");
    if (auto st = make_match(width, height, kw, kh, p, metric, &m)) return st;
    if (!partial || !map) return contract("hist_finalize: null pointer");
    const double dmax = std::pow(2.0, 1.0 / p);  // likelihood.cpp:208
    const int64_t n = static_cast<int64_t>(width) * height;
    finalize_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(partial, width, height, m, dmax, map, gate);
    return launch_status("finalize_kernel");
}
}  // namespace

extern "C" spct_status spct_cu_hist_finalize(const double* partial, int width, int height, int kw, int kh, double p,
                                             int metric, double* map, void* stream) {
    return finalize_impl(partial, width, height, kw, kh, p, metric, map, stream, nullptr);
}

namespace {
spct_status hist_match_impl(const spct_ih* t, const double* tmpl, int kw, int kh, double p, int metric, double* map,
                            void* stream, bool exact) {
    if (auto st = check_ih(t)) return st;
    if (t->bin0 != 0 || t->bins != t->nbins_total)
        return contract("hist_match: the tensor must hold every bin (use hist_partial for slabs)");
    MatchParams m;
    if (auto st = make_match(t->width, t->height, kw, kh, p, metric, &m)) return st;
    if (!map || !t->data) return contract("hist_match: null pointer");
    cudaStream_t s = as_stream(stream);
    const int64_t n = static_cast<int64_t>(m.nu) * m.nv;
    double* part = nullptr;
    if (auto st = cuda_status(malloc_async(&part, n * sizeof(double), s), "hist_match alloc")) return st;
    spct_status st = SPCT_OK;
    uint32_t* gate = nullptr;
    void* scratch = nullptr;
    if (!exact && spct_cu_fused_window_ok(kw, kh) && t->nbins_total <= 65536 &&
        check_carry_dims(t->width, t->height) == SPCT_OK) {
        // read the tensor once: recover the bin map (tensor_match.cu), then the fused
        // no-store sweep; the exact kernels below run only if the tensor is not one-hot
        const size_t nb = round_up(static_cast<int64_t>(t->width) * t->height * 2, 256);
        const size_t gs = t->bins > 128 ? static_cast<size_t>(t->width) * t->height * 8 : 0;
        size_t ws = 0;
        spct_source src{};
        src.kind = SPCT_SRC_BINS_U16;
        src.pitch = t->width;
        src.width = t->width;
        src.height = t->height;
        src.nbins = t->nbins_total;
        st = spct_cu_ih_build_workspace(&src, 0, t->bins, &ws);
        if (st == SPCT_OK)
            st = cuda_status(malloc_async(&scratch, nb + 256 + gs + ws, s), "hist_match alloc");
        if (st == SPCT_OK) {
            char* sp = static_cast<char*>(scratch);
            uint16_t* bins = reinterpret_cast<uint16_t*>(sp);
            gate = reinterpret_cast<uint32_t*>(sp + nb);
            uint32_t* gsum = gs ? reinterpret_cast<uint32_t*>(sp + nb + 256) : nullptr;
            src.plane[0] = bins;
            st = ih_recover_bins(*t, bins, t->width, gate, gsum, s);
            spct_ih nodata = *t;
            nodata.data = nullptr;
            if (st == SPCT_OK)
                st = spct_cu_ih_build_match_map(&src, &nodata, tmpl, kw, kh, p, metric, map, sp + nb + 256 + gs, ws,
                                                stream);
        }
    }
    // the reference's operation order over the tensor itself, each window normalised by its
    // actual total (gated by the one-hot check above when that ran)
    if (st == SPCT_OK) st = hist_partial_impl(t, tmpl, kw, kh, p, metric, part, 0, 1, stream, gate);
    if (st == SPCT_OK) st = finalize_impl(part, t->width, t->height, kw, kh, p, metric, map, stream, gate);
    cudaFreeAsync(part, s);
    if (scratch) cudaFreeAsync(scratch, s);
    return st;
}
}  // namespace

extern "C" spct_status spct_cu_hist_match(const spct_ih* t, const double* tmpl, int kw, int kh, double p, int metric,
                                          double* map, void* stream) {
    return hist_match_impl(t, tmpl, kw, kh, p, metric, map, stream, std::getenv("SPCT_EXACT_MAPS") != nullptr);
}

extern "C" spct_status spct_cu_hist_match_exact(const spct_ih* t, const double* tmpl, int kw, int kh, double p,
                                                int metric, double* map, void* stream) {
    return hist_match_impl(t, tmpl, kw, kh, p, metric, map, stream, true);
}
