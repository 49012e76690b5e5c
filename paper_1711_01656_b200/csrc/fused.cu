// Fused integral histogram + sliding-window matcher: host side (C-ABI, template prep,
// dispatch).  The kernel is in fused_kernel.cuh.
#include <mutex>

#include "fused_kernel.cuh"

using namespace spct_dev;
using namespace spct_impl;

namespace spct_fused {

// Side streams of a batched call (per device, created once): the sweeps of a batch's
// sources are independent, so sources 1.. run on their own streams, forked from and joined
// back into the caller's stream by events (captured as parallel branches inside a CUDA
// graph).  Each sweep is about one wave of CTAs; side by side, one source's pre-roll and
// tail overlap another's steady state.  The mutex keeps a fork / join sequence's event
// records and waits together when several host threads share the pool.
struct SidePool {
    std::mutex mu;
    cudaStream_t side[kMaxCarryCh] = {};
    cudaEvent_t fork = nullptr, join[kMaxCarryCh] = {};
    bool ok = false;
};

static SidePool* side_pool() {
    static SidePool pools[64];
    static std::mutex init_mu;
    const int dev = current_device();
    if (dev < 0 || dev >= 64) return nullptr;
    SidePool& P = pools[dev];
    std::lock_guard<std::mutex> lk(init_mu);
    if (!P.ok) {
        bool good = cudaEventCreateWithFlags(&P.fork, cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; good && i < kMaxCarryCh; ++i)
            good = cudaStreamCreateWithFlags(&P.side[i], cudaStreamNonBlocking) == cudaSuccess &&
                   cudaEventCreateWithFlags(&P.join[i], cudaEventDisableTiming) == cudaSuccess;
        if (!good) {
            cudaGetLastError();
            return nullptr;
        }
        P.ok = true;
    }
    return &P;
}

// Template prep: s_k = T t_k.  Kind 1 (the exact integer path) iff every s_k of the slab
// is an integer up to FP noise (then the integer formula is exact to ~1e-15) and the metric
// allows it; otherwise kind 2 (integer path on floor(s_k) plus the fractional parts) when
// the host allows it (`frac_ok`: p = 1 / intersection, kw kh <= 4096), else kind 0 (FP64).
// Other metrics: kind `other_kind` (3: integer / FP32 terms, 0: FP64).
// Layout (fused_prep_layout): [0] kind, [1 + k] floor(s_k) replicated in both u16 halves;
// per 128-bin group sum floor(s_k) (int64) and sum r_k (double); r_k per bin (double);
// the MODE 3 constants per bin (float4) and per 16-bin slab (double2), FusedParams::c3.
// One CTA per source of a batch (PrepBatch, blockIdx.x).
struct PrepBatch {
    const double* tmpl[kMaxCarryCh];
    uint32_t* prep[kMaxCarryCh];
    long long* S_group[kMaxCarryCh];
    double* Sr_group[kMaxCarryCh];
    double* rfrac[kMaxCarryCh];
    float4* c3[kMaxCarryCh];
    double2* c3slab[kMaxCarryCh];
};

__global__ void prep_kernel(const __grid_constant__ PrepBatch pb, int bin0, int bins, double T, int fast_metric,
                            int frac_ok, int other_kind, int ngroups) {
    const double* __restrict__ tmpl = pb.tmpl[blockIdx.x];
    uint32_t* __restrict__ prep = pb.prep[blockIdx.x];
    long long* __restrict__ S_group = pb.S_group[blockIdx.x];
    double* __restrict__ Sr_group = pb.Sr_group[blockIdx.x];
    double* __restrict__ rfrac = pb.rfrac[blockIdx.x];
    float4* __restrict__ c3 = pb.c3[blockIdx.x];
    double2* __restrict__ c3slab = pb.c3slab[blockIdx.x];
    __shared__ int all_integral;
    if (threadIdx.x == 0) all_integral = 1;
    __syncthreads();
    for (int k = threadIdx.x; k < bins; k += blockDim.x) {
        const double s = T * tmpl[bin0 + k];
        const double n = rint(s);
        const bool integral = fabs(s - n) <= 8.0 * 2.220446049250313e-16 * fmax(1.0, fabs(s)) && n >= 0.0 && n <= T;
        if (!integral) all_integral = 0;
        // s_k >= 0 (template contract); floor clamped to [0, T] (c_k <= T, so min(c, s) = c above)
        const double fl = integral ? n : fmin(fmax(floor(s), 0.0), T);
        const uint32_t ni = static_cast<uint32_t>(fl);
        prep[1 + k] = ni | (ni << 16);
        rfrac[k] = integral ? 0.0 : fmax(s - fl, 0.0);
        {   // MODE 3 constants (floor and fraction of s_k without the integrality snap)
            const double f3 = fmin(fmax(floor(s), 0.0), T), r3 = s - f3, R = rint(32.0 * r3);
            const int K = static_cast<int>(64.0 * f3 + 2.0 * R);
            c3[k] = make_float4(__int_as_float(K), static_cast<float>(r3 - R / 32.0),
                                static_cast<float>(sqrt(tmpl[bin0 + k] / T)), static_cast<float>(s));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) prep[0] = fast_metric ? (all_integral ? 1u : (frac_ok ? 2u : 0u)) : static_cast<uint32_t>(other_kind);
    for (int sl = threadIdx.x; sl < (bins + 15) / 16; sl += blockDim.x) {
        double a = 0.0, b = 0.0;
        for (int k = 16 * sl; k < min(bins, 16 * sl + 16); ++k) {
            const double sk = T * tmpl[bin0 + k];
            a += sk * sk;
            b += sk;
        }
        c3slab[sl] = make_double2(a, b);
    }
    for (int g = threadIdx.x; g < ngroups; g += blockDim.x) {
        long long acc = 0;
        double racc = 0.0;
        for (int k = g * kGroupBins; k < min(bins, (g + 1) * kGroupBins); ++k) {
            acc += prep[1 + k] & 0xFFFFu;
            racc += rfrac[k];
        }
        S_group[g] = acc;
        Sr_group[g] = racc;
    }
}

struct PrepLayout {
    size_t S, Sr, r, c3, c3slab, total;
};
inline PrepLayout fused_prep_layout(int bins) {
    const size_t ng = (static_cast<size_t>(bins) + kGroupBins - 1) / kGroupBins;
    PrepLayout l;
    l.S = round_up((static_cast<int64_t>(bins) + 1) * 4, 256);
    l.Sr = l.S + round_up(static_cast<int64_t>(ng) * 8, 256);
    l.r = l.Sr + round_up(static_cast<int64_t>(ng) * 8, 256);
    l.c3 = l.r + round_up(static_cast<int64_t>(bins) * 8, 256);
    l.c3slab = l.c3 + round_up(static_cast<int64_t>(bins) * 16, 256);
    l.total = l.c3slab + round_up(static_cast<int64_t>((bins + 15) / 16) * 16, 256);
    return l;
}

}  // namespace spct_fused

using namespace spct_fused;

namespace spct_impl {
size_t fused_prep_bytes(int bins) { return fused_prep_layout(bins).total; }
}  // namespace spct_impl

namespace spct_fused {

// Shared body of spct_cu_ih_build_match (partial != null), spct_cu_ih_build_match_map (map
// != null) and the batched spct_cu_ih_build_match_map_multi: n same-shape sources (one
// tensor, template, output and workspace each) share one launch of each carry kernel and of
// the template prep; the sweeps run per source.
spct_status build_match(int n, const spct_source* srcs, const spct_ih* outs, const double* const* tmpls, int kw,
                        int kh, double p, int metric, double* const* partials, double* const* maps,
                        void* const* workspaces, size_t workspace_bytes, void* stream) {
    if (n < 1 || n > kMaxCarryCh) return contract("ih_build_match_map_multi: 1 .. 8 sources");
    QuantParams qs[kMaxCarryCh];
    for (int c = 0; c < n; ++c) {
        const spct_source* src = &srcs[c];
        const spct_ih* out = &outs[c];
        if (auto st = make_quant(src, &qs[c])) return st;
        if (auto st = check_ih(out)) return st;
        if (out->width != src->width || out->height != src->height || out->nbins_total != src->nbins)
            return contract("ih_build_match: tensor dims do not match the source");
        if (auto st = check_carry_dims(out->width, out->height)) return st;
        if (out->data && reinterpret_cast<uintptr_t>(out->data) % 16 != 0)
            return contract("ih_build_match: tensor data must be 16-byte aligned");
        if (!(p >= 1.0)) return contract("hist_distance_map: Minkowski order must be >= 1");
        if (!(kw >= 1 && kh >= 1 && kw <= src->width && kh <= src->height))
            return contract("hist_distance_map: kernel exceeds image");
        if (metric < SPCT_METRIC_MINKOWSKI || metric > SPCT_METRIC_CHISQ) return contract("hist_match: unknown metric");
        if (!tmpls[c] || !((partials && partials[c]) || (maps && maps[c])))
            return contract("ih_build_match: null template or output");
        if (maps && (out->bin0 != 0 || out->bins != out->nbins_total))
            return contract("ih_build_match_map: the slab must hold every bin (use the partial form for slabs)");
        if (c > 0 && (out->width != outs[0].width || out->height != outs[0].height || out->bins != outs[0].bins ||
                      out->bin0 != outs[0].bin0 || out->nbins_total != outs[0].nbins_total ||
                      (out->data != nullptr) != (outs[0].data != nullptr)))
            return contract("ih_build_match_map_multi: the sources must share one shape (and all store or none)");
    }
    const spct_ih* out = &outs[0];
    cudaStream_t s = as_stream(stream);
    const int64_t T = static_cast<int64_t>(kw) * kh;
    const bool fusable = spct_cu_fused_window_ok(kw, kh) != 0;
    const int ngroups = static_cast<int>(ceil_div(out->bins, kGroupBins));
    if (n > 1 && (!fusable || (maps && ngroups > 1))) {  // one source at a time
        for (int c = 0; c < n; ++c) {
            double* pc = partials ? partials[c] : nullptr;
            double* mc = maps ? maps[c] : nullptr;
            if (auto st = build_match(1, &srcs[c], &outs[c], &tmpls[c], kw, kh, p, metric, partials ? &pc : nullptr,
                                      maps ? &mc : nullptr, &workspaces[c], workspace_bytes, stream))
                return st;
        }
        return SPCT_OK;
    }
    double* const map0 = maps ? maps[0] : nullptr;
    double* group_part = nullptr;  // > 128 bins with a finished map: the earlier groups' partial sums (n == 1)
    if (fusable && map0 && ngroups > 1) {
        const size_t nw = static_cast<size_t>(out->width - kw + 1) * (out->height - kh + 1);
        if (auto st = cuda_status(malloc_async(&group_part, nw * sizeof(double), s), "ih_build_match_map alloc"))
            return st;
    }
    struct FreeAsync {
        double* p;
        cudaStream_t s;
        ~FreeAsync() { if (p) cudaFreeAsync(p, s); }
    } free_part{group_part, s};
    if (!fusable) {
        // two passes: window too large for the 16-bit running-histogram cells (n == 1 here)
        if (!out->data) return contract("ih_build_match: this shape needs tensor storage (two-pass schedule)");
        if (auto st = spct_cu_ih_build(&srcs[0], out, workspaces[0], workspace_bytes, stream)) return st;
        if (map0) return spct_cu_hist_match(out, tmpls[0], kw, kh, p, metric, map0, stream);
        return spct_cu_hist_partial(out, tmpls[0], kw, kh, p, metric, partials[0], 0, stream);
    }
    const BuildPlan bp = plan_fused_sweep(out->width, out->height, out->bins);
    // Band tops start their running column counts from the carry tables when that takes
    // fewer load rounds than re-reading the kh - 1 rows above (narrow histograms, several
    // strips per CTA); with a full 128-bin group the row pre-roll costs the same and needs
    // no extra table (the kernel reads the tables only for groups under 128 bins).
    const int S = fused_strips(out->bins), ext = kStrip * (S + 1), nt = 256;
    const int64_t table_rounds = ceil_div(static_cast<int64_t>(std::min(out->bins, kGroupBins)) * (ext / 2), 8 * nt);
    const int64_t preroll_rounds = ceil_div(ceil_div(ext, nt) * (kh - 1), 8);
    const int win_kh = (kh > 1 && out->bins < kGroupBins && table_rounds < preroll_rounds) ? kh : 0;
    const size_t carry_bytes = out->data ? fused_carry_layout(bp, out->height, win_kh > 1).total : 0;
    const size_t need = carry_bytes + fused_prep_bytes(out->bins);
    for (int c = 0; c < n; ++c) {
        const size_t gray = srcs[c].kind == SPCT_SRC_RGB_U8 ? fused_gray_bytes(&srcs[c]) : 0;
        if (!workspaces[c] || workspace_bytes < need + gray) return contract("ih_build_match: workspace too small");
        if (gray) {
            // planar RGB: to_grayscale (imagecore.cpp:17-24) once into the workspace, then the
            // 8-bit source path (prefetched staging, 4-pixel carry loads) — the same bins as
            // the per-pixel conversion in the load stage, for 4 extra bytes per pixel
            uint8_t* g = static_cast<uint8_t*>(workspaces[c]) + need;
            const int64_t np = srcs[c].pitch * static_cast<int64_t>(srcs[c].height);
            if (auto st = spct_cu_to_grayscale(static_cast<const uint8_t*>(srcs[c].plane[0]),
                                               static_cast<const uint8_t*>(srcs[c].plane[1]),
                                               static_cast<const uint8_t*>(srcs[c].plane[2]), np, g, stream))
                return st;
            spct_source gs = srcs[c];
            gs.kind = SPCT_SRC_GRAY_U8;
            gs.plane[0] = g;
            gs.plane[1] = gs.plane[2] = nullptr;
            if (auto st = make_quant(&gs, &qs[c])) return st;
        }
    }
    FusedCarries fcs[kMaxCarryCh] = {};
    if (out->data)
        if (auto st = build_fused_carries_multi(n, qs, *out, bp, workspaces, workspace_bytes, s, fcs, win_kh)) return st;
    // integer paths: packed 16-bit window counts (kw * kh <= 24576, fused_kernel.cuh); the
    // fractional flags need every count <= 4096
    const int fast_metric = ((metric == SPCT_METRIC_MINKOWSKI && p == 1.0) || metric == SPCT_METRIC_INTERSECTION) &&
                            T <= 24576;
    const int frac_ok = fast_metric && T <= 4096;
    // p = 2 (int32 sums need kw kh <= 4096), Bhattacharyya and chi-square: integer / FP32 terms
    const int f32_ok = (metric == SPCT_METRIC_MINKOWSKI && p == 2.0 && T <= 4096) ||
                       metric == SPCT_METRIC_BHATTACHARYYA || metric == SPCT_METRIC_CHISQ;
    // Bhattacharyya / chi-square in the quarter layout (MODE 4 / 5, packed 16-bit window counts)
    const int quarter = T <= 24576 ? (metric == SPCT_METRIC_BHATTACHARYYA ? 4 : (metric == SPCT_METRIC_CHISQ ? 5 : 0)) : 0;
    // p = 2 (kw kh <= 4096): MODE 3's exact integer + FP32 split in the quarter layout (MODE 6)
    const int p2q = metric == SPCT_METRIC_MINKOWSKI && p == 2.0 && T <= 4096 && !std::getenv("SPCT_P2_MODE3") ? 6 : 0;
    const int path = fast_metric ? 1 : (quarter ? quarter : (p2q ? p2q : (f32_ok ? 3 : 0)));
    const PrepLayout pl = fused_prep_layout(out->bins);
    PrepBatch pbt{};
    for (int c = 0; c < n; ++c) {
        char* ws = static_cast<char*>(workspaces[c]) + carry_bytes;
        pbt.tmpl[c] = tmpls[c];
        pbt.prep[c] = reinterpret_cast<uint32_t*>(ws);
        pbt.S_group[c] = reinterpret_cast<long long*>(ws + pl.S);
        pbt.Sr_group[c] = reinterpret_cast<double*>(ws + pl.Sr);
        pbt.rfrac[c] = reinterpret_cast<double*>(ws + pl.r);
        pbt.c3[c] = reinterpret_cast<float4*>(ws + pl.c3);
        pbt.c3slab[c] = reinterpret_cast<double2*>(ws + pl.c3slab);
    }
    prep_kernel<<<n, 256, 0, s>>>(pbt, out->bin0, out->bins, static_cast<double>(T), fast_metric, frac_ok,
                                  path == 1 ? 0 : path, ngroups);
    if (auto st = launch_status("prep_kernel")) return st;

    // sources 1.. on side streams (sweeps only: carries and prep above are batched launches)
    SidePool* pool = n > 1 && !std::getenv("SPCT_NO_SIDE_STREAMS") ? side_pool() : nullptr;
    std::unique_lock<std::mutex> side_lk;
    // a side stream forked and not yet joined (an error return in between) is joined on
    // the way out, so the caller's stream (or graph capture) never leaves one dangling
    struct JoinOnExit {
        SidePool* pool = nullptr;
        cudaStream_t s = nullptr;
        int open = -1;
        ~JoinOnExit() {
            if (open > 0 && cudaEventRecord(pool->join[open], pool->side[open]) == cudaSuccess)
                cudaStreamWaitEvent(s, pool->join[open], 0);
        }
    } joiner{pool, s};
    if (pool) {
        side_lk = std::unique_lock<std::mutex>(pool->mu);
        if (auto st = cuda_status(cudaEventRecord(pool->fork, s), "ih_build_match fork")) return st;
    }
    for (int c = 0; c < n; ++c) {
        cudaStream_t sc = s;
        if (pool && c > 0) {
            sc = pool->side[c];
            if (auto st = cuda_status(cudaStreamWaitEvent(sc, pool->fork, 0), "ih_build_match fork")) return st;
            joiner.open = c;
        }
        FusedParams f{};
        f.kw = kw;
        f.kh = kh;
        f.nu = out->width - kw + 1;
        f.nv = out->height - kh + 1;
        f.metric = metric;
        f.p = p;
        f.inv_p = 1.0 / p;
        f.dmax = std::pow(2.0, 1.0 / p);  // likelihood.cpp:208
        {   // d / dmax == d * (1 / dmax) bit for bit when dmax is a power of two (p = 1: dmax = 2)
            int e = 0;
            f.inv_dmax = std::frexp(f.dmax, &e) == 0.5 ? 1.0 / f.dmax : 0.0;
        }
        f.p_kind = p == 1.0 ? 1 : (p == 2.0 ? 2 : 0);
        f.fp_kind = metric == SPCT_METRIC_MINKOWSKI ? (f.p_kind == 1 ? 0 : (f.p_kind == 2 ? 1 : 2))
                                                    : (metric == SPCT_METRIC_INTERSECTION ? 3
                                                       : (metric == SPCT_METRIC_BHATTACHARYYA ? 4 : 5));
        f.T = static_cast<double>(T);
        f.invT = 1.0 / f.T;
        f.T_pow2 = (T & (T - 1)) == 0;
        f.tmpl = tmpls[c];
        f.prep = pbt.prep[c];
        f.S_group = pbt.S_group[c];
        f.Sr_group = pbt.Sr_group[c];
        f.rfrac = pbt.rfrac[c];
        f.frac = frac_ok;
        f.path = path;
        f.c3 = pbt.c3[c];
        f.c3slab = pbt.c3slab[c];
        double* const mapc = maps ? maps[c] : nullptr;
        f.partial = group_part ? group_part : (partials ? partials[c] : nullptr);
        f.map = group_part ? nullptr : mapc;
        f.W = out->width;
        f.H = out->height;
        const QuantParams& q = qs[c];
        const FusedCarries& fc = fcs[c];
        const spct_ih& oc = outs[c];
        const PixelMode pm = make_pixel_mode(q, oc.bin0);
        for (int g = 0; g < ngroups; ++g) {
            f.group0 = g * kGroupBins;
            f.accumulate = g > 0;
            // several groups into a finished map: groups accumulate into group_part, the last
            // one adds its sums to it and writes the finished map (no finalise pass)
            if (group_part && g == ngroups - 1) f.map = mapc;
            dim3 grid(static_cast<unsigned>(ceil_div(bp.nstrips, S)), bp.nbands, 1);
            const int prof = prof_begin(oc.data ? "ih_sweep_match" : "sweep_match_nostore", sc);
            // the group is the whole histogram: window totals over its bins are kw * kh
            const bool allb = oc.bin0 == 0 && oc.bins == oc.nbins_total && ngroups == 1;
            const bool al4 = ((reinterpret_cast<uintptr_t>(q.p0) | static_cast<uintptr_t>(q.pitch)) & 3) == 0;
            const int sk = (q.kind == SPCT_SRC_GRAY_U8 && q.fast_u8) ? (S >= 4 && al4 && !std::getenv("SPCT_NO_WIDE") ? 3 : 1)
                                                                     : (q.kind == SPCT_SRC_BINS_U16 ? 2 : 0);
#define SPCT_LAUNCH(KW)                                                                                     \
    if (S == 1) launch_##KW##_s1(allb, sk, grid, sc, q, pm, oc, bp, fc, f);                                      \
    else if (S == 2) launch_##KW##_s2(allb, sk, grid, sc, q, pm, oc, bp, fc, f);                                 \
    else if (S == 4) launch_##KW##_s4(allb, sk, grid, sc, q, pm, oc, bp, fc, f);                                 \
    else launch_##KW##_s8(allb, sk, grid, sc, q, pm, oc, bp, fc, f);
            if (kw == 64) {
                SPCT_LAUNCH(kw64)
            } else if (kw == 128) {
                SPCT_LAUNCH(kw128)
            } else {
                SPCT_LAUNCH(kw_any)
            }
#undef SPCT_LAUNCH
            prof_end(prof, sc);
            note_launch();
            if (auto st = launch_status("sweep_match_kernel")) return st;
        }
        if (sc != s) {
            if (auto st = cuda_status(cudaEventRecord(pool->join[c], sc), "ih_build_match join")) return st;
            if (auto st = cuda_status(cudaStreamWaitEvent(s, pool->join[c], 0), "ih_build_match join")) return st;
            joiner.open = -1;
        }
    }
    return SPCT_OK;
}

}  // namespace spct_fused

extern "C" int spct_cu_fused_window_ok(int kw, int kh) {
    // 16-bit running-histogram cells (fused_kernel.cuh)
    return kw >= 1 && kh >= 1 && kw <= 128 && kh <= 255 && static_cast<int64_t>(kw) * kh <= 65535;
}

extern "C" spct_status spct_cu_ih_build_match(const spct_source* src, const spct_ih* out, const double* tmpl, int kw,
                                              int kh, double p, int metric, double* partial, void* workspace,
                                              size_t workspace_bytes, void* stream) {
    if (!partial) return contract("ih_build_match: null partial");
    if (!src || !out) return contract("ih_build_match: null argument");
    return spct_fused::build_match(1, src, out, &tmpl, kw, kh, p, metric, &partial, nullptr, &workspace,
                                   workspace_bytes, stream);
}

extern "C" spct_status spct_cu_ih_build_match_map(const spct_source* src, const spct_ih* out, const double* tmpl, int kw,
                                                  int kh, double p, int metric, double* map, void* workspace,
                                                  size_t workspace_bytes, void* stream) {
    if (!map) return contract("ih_build_match_map: null map");
    if (!src || !out) return contract("ih_build_match_map: null argument");
    return spct_fused::build_match(1, src, out, &tmpl, kw, kh, p, metric, nullptr, &map, &workspace, workspace_bytes,
                                   stream);
}

extern "C" spct_status spct_cu_ih_build_match_map_multi(int n, const spct_source* srcs, const spct_ih* outs,
                                                        const double* const* tmpls, int kw, int kh, double p, int metric,
                                                        double* const* maps, void* const* workspaces,
                                                        size_t workspace_bytes, void* stream) {
    if (!srcs || !outs || !tmpls || !maps || !workspaces) return contract("ih_build_match_map_multi: null argument");
    return spct_fused::build_match(n, srcs, outs, tmpls, kw, kh, p, metric, nullptr, maps, workspaces, workspace_bytes,
                                   stream);
}
