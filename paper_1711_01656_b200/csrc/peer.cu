// Bin-slab reduce over peer memory.
//
// With N ranks, rank r's fused sweep (spct_cu_ih_build_match) writes its slab's partial
// window statistic straight into slot r of a slot buffer that lives on the root GPU
// (an IPC mapping of the root's allocation, NVLink stores from the kernel's epilogue),
// so the transfer overlaps the sweep tile by tile instead of following it as a separate
// collective.  A one-thread signal kernel then publishes the rank's epoch in a flag on
// the root (fence.sc.sys + st.release.sys); the root waits for every flag
// (ld.acquire.sys, bounded by a timeout that raises an error flag instead of hanging),
// sums the N slots in rank order while it finalises the map (spread_valid + the
// likelihood of hist_distance_map, likelihood.cpp:44-58,220-221), and acknowledges the
// epoch in each rank's own flag so slots can be reused (double-buffered by epoch parity).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "spct_internal.h"

using namespace spct_impl;

namespace spct_peer {

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void signal_kernel(uint64_t* flag, uint64_t value) {
    // everything this stream wrote before (the sweep's partials, possibly to peer memory)
    // is ordered before the flag store at system scope
    asm volatile("fence.sc.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

__global__ void wait_kernel(const uint64_t* flags, int n, int64_t stride, uint64_t value, uint64_t timeout_ns,
                            uint32_t* err) {
    const int i = threadIdx.x;
    if (i < n) {
        const uint64_t* f = flags + static_cast<int64_t>(i) * stride;
        const uint64_t t0 = globaltimer();
        while (ld_acquire_sys(f) < value) {
            if (globaltimer() - t0 > timeout_ns) {
                atomicExch(err, 1u);
                break;
            }
            __nanosleep(256);
        }
    }
    __syncthreads();
    asm volatile("fence.acq_rel.sys;" ::: "memory");
}

struct FinParams {
    int W, H, nu, nv, cx0, cy0, metric, p_kind;
    double inv_p, dmax;
};

__device__ __forceinline__ double finalize_L(double s, const FinParams& f) {
    double L;
    if (f.metric == SPCT_METRIC_MINKOWSKI) {
        const double d = f.p_kind == 1 ? s : pow(s, f.inv_p);
        L = __dsub_rn(1.0, __ddiv_rn(d, f.dmax));
    } else if (f.metric == SPCT_METRIC_CHISQ) {
        L = __dsub_rn(1.0, __ddiv_rn(s, 2.0));
    } else {
        L = s;
    }
    return L < 0.0 ? 0.0 : (L > 1.0 ? 1.0 : L);
}

// One thread per output pixel: the slots' partials at the pixel's (clamped) window, summed
// in rank order, then the finalisation.  Border pixels re-read their nearest valid window
// (spread_valid), interior ones read each slot once.
__global__ void __launch_bounds__(256) finalize_slots_kernel(const double* __restrict__ slots, int nslots,
                                                             int64_t slot_stride, FinParams f,
                                                             double* __restrict__ map) {
    const int64_t n = static_cast<int64_t>(f.W) * f.H;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % f.W), y = static_cast<int>(i / f.W);
        const int vx = min(max(x, f.cx0), f.cx0 + f.nu - 1) - f.cx0;
        const int vy = min(max(y, f.cy0), f.cy0 + f.nv - 1) - f.cy0;
        const double* p = slots + static_cast<int64_t>(vy) * f.nu + vx;
        double s = __ldcs(p);
        for (int r = 1; r < nslots; ++r) s = __dadd_rn(s, __ldcs(p + r * slot_stride));
        map[i] = finalize_L(s, f);
    }
}

// ---- band-owned reduce: every rank keeps its partial map in its own HBM; rank r owns the
// valid rows [v0, v1) and pulls them from all N partials (NVLink loads from the peers'
// IPC mappings), sums in rank order, finalises and writes the final map rows (borders
// included, spread_valid) into the map on the root.  The reduction work and the NVLink
// traffic are spread over all ranks instead of converging on the root.
constexpr int kMaxPeers = 16;

struct PeerPtrs {
    const double* p[kMaxPeers];
};

struct FlagPtrs {
    uint64_t* p[kMaxPeers];
};

__global__ void signal_many_kernel(FlagPtrs f, int n, uint64_t value) {
    asm volatile("fence.sc.sys;" ::: "memory");
    const int i = threadIdx.x;
    if (i < n) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f.p[i]), "l"(value) : "memory");
}

__global__ void __launch_bounds__(256) finalize_band_kernel(PeerPtrs src, int nsrc, FinParams f, int v0, int v1,
                                                            double* __restrict__ map) {
    // output rows whose clamped valid row lies in [v0, v1): the band, plus the replicated
    // top (first band) and bottom (last band) borders
    const int y0 = v0 == 0 ? 0 : v0 + f.cy0, y1 = v1 == f.nv ? f.H : v1 + f.cy0;
    const int64_t n = static_cast<int64_t>(y1 - y0) * f.W;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % f.W), y = y0 + static_cast<int>(i / f.W);
        const int vx = min(max(x, f.cx0), f.cx0 + f.nu - 1) - f.cx0;
        const int vy = min(max(y, f.cy0), f.cy0 + f.nv - 1) - f.cy0;
        const int64_t o = static_cast<int64_t>(vy) * f.nu + vx;
        double s = src.p[0][o];
        for (int r = 1; r < nsrc; ++r) s = __dadd_rn(s, src.p[r][o]);
        map[static_cast<int64_t>(y) * f.W + x] = finalize_L(s, f);
    }
}

spct_status make_fin(int width, int height, int kw, int kh, double p, int metric, FinParams* f) {
    if (!(width > 0 && height > 0)) return contract("hist_finalize: empty map");
    if (!(p >= 1.0)) return contract("hist_distance_map: Minkowski order must be >= 1");
    if (!(kw >= 1 && kh >= 1 && kw <= width && kh <= height)) return contract("hist_distance_map: kernel exceeds image");
    if (metric < SPCT_METRIC_MINKOWSKI || metric > SPCT_METRIC_CHISQ) return contract("hist_match: unknown metric");
    *f = FinParams{};
    f->W = width;
    f->H = height;
    f->nu = width - kw + 1;
    f->nv = height - kh + 1;
    f->cx0 = (kw - 1) / 2;
    f->cy0 = (kh - 1) / 2;
    f->metric = metric;
    f->p_kind = p == 1.0 ? 1 : 0;
    f->inv_p = 1.0 / p;
    f->dmax = std::pow(2.0, 1.0 / p);  // likelihood.cpp:208
    return SPCT_OK;
}

}  // namespace spct_peer

using namespace spct_peer;

extern "C" spct_status spct_cu_flag_signal_many(uint64_t* const* flags, int n, uint64_t value, void* stream) {
    if (!flags || n < 1 || n > kMaxPeers) return contract("flag_signal_many: bad arguments");
    FlagPtrs f{};
    for (int i = 0; i < n; ++i) {
        if (!flags[i]) return contract("flag_signal_many: null flag");
        f.p[i] = flags[i];
    }
    signal_many_kernel<<<1, 32, 0, as_stream(stream)>>>(f, n, value);
    return launch_status("signal_many_kernel");
}

extern "C" spct_status spct_cu_hist_finalize_band(const double* const* partials, int nsrc, int width, int height,
                                                  int kw, int kh, double p, int metric, int v0, int v1, double* map,
                                                  void* stream) {
    FinParams f;
    if (auto st = make_fin(width, height, kw, kh, p, metric, &f)) return st;
    if (!partials || !map || nsrc < 1 || nsrc > kMaxPeers || !(0 <= v0 && v0 <= v1 && v1 <= f.nv))
        return contract("hist_finalize_band: bad arguments");
    if (v0 == v1) return SPCT_OK;
    PeerPtrs src{};
    for (int i = 0; i < nsrc; ++i) {
        if (!partials[i]) return contract("hist_finalize_band: null partial");
        src.p[i] = partials[i];
    }
    const int y0 = v0 == 0 ? 0 : v0 + f.cy0, y1 = v1 == f.nv ? f.H : v1 + f.cy0;
    const int64_t n = static_cast<int64_t>(y1 - y0) * width;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
    finalize_band_kernel<<<static_cast<unsigned>(blocks), 256, 0, as_stream(stream)>>>(src, nsrc, f, v0, v1, map);
    return launch_status("finalize_band_kernel");
}

static_assert(sizeof(cudaIpcMemHandle_t) == SPCT_IPC_HANDLE_BYTES, "IPC handle size");

extern "C" spct_status spct_cu_peer_alloc(size_t bytes, void** ptr, void* handle) {
    if (!ptr || !handle || bytes == 0) return contract("peer_alloc: bad arguments");
    *ptr = nullptr;
    if (auto st = cuda_status(cudaMalloc(ptr, bytes), "peer_alloc")) return st;
    if (auto st = cuda_status(cudaMemset(*ptr, 0, bytes), "peer_alloc memset")) {
        cudaFree(*ptr);
        *ptr = nullptr;
        return st;
    }
    cudaIpcMemHandle_t h;
    if (auto st = cuda_status(cudaIpcGetMemHandle(&h, *ptr), "cudaIpcGetMemHandle")) {
        cudaFree(*ptr);
        *ptr = nullptr;
        return st;
    }
    memcpy(handle, &h, sizeof(h));
    return SPCT_OK;
}

extern "C" spct_status spct_cu_peer_free(void* ptr) { return cuda_status(cudaFree(ptr), "peer_free"); }

extern "C" spct_status spct_cu_peer_open(const void* handle, void** ptr) {
    if (!handle || !ptr) return contract("peer_open: bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    return cuda_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

extern "C" spct_status spct_cu_peer_close(void* ptr) {
    return cuda_status(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
}

extern "C" spct_status spct_cu_flag_signal(uint64_t* flag, uint64_t value, void* stream) {
    if (!flag) return contract("flag_signal: null flag");
    signal_kernel<<<1, 1, 0, as_stream(stream)>>>(flag, value);
    return launch_status("signal_kernel");
}

extern "C" spct_status spct_cu_flag_wait(const uint64_t* flags, int n, int64_t stride, uint64_t value,
                                         uint64_t timeout_ns, uint32_t* err, void* stream) {
    if (!flags || !err || n < 1 || n > 1024 || stride < 1) return contract("flag_wait: bad arguments");
    wait_kernel<<<1, ((n + 31) / 32) * 32, 0, as_stream(stream)>>>(flags, n, stride, value, timeout_ns, err);
    return launch_status("wait_kernel");
}

extern "C" spct_status spct_cu_hist_finalize_slots(const double* slots, int nslots, int64_t slot_stride, int width,
                                                   int height, int kw, int kh, double p, int metric, double* map,
                                                   void* stream) {
    if (!(width > 0 && height > 0)) return contract("hist_finalize: empty map");
    if (!(p >= 1.0)) return contract("hist_distance_map: Minkowski order must be >= 1");
    if (!(kw >= 1 && kh >= 1 && kw <= width && kh <= height)) return contract("hist_distance_map: kernel exceeds image");
    if (metric < SPCT_METRIC_MINKOWSKI || metric > SPCT_METRIC_CHISQ) return contract("hist_match: unknown metric");
    FinParams f{};
    f.W = width;
    f.H = height;
    f.nu = width - kw + 1;
    f.nv = height - kh + 1;
    if (!slots || !map || nslots < 1 || slot_stride < static_cast<int64_t>(f.nu) * f.nv)
        return contract("hist_finalize_slots: bad arguments");
    f.cx0 = (kw - 1) / 2;
    f.cy0 = (kh - 1) / 2;
    f.metric = metric;
    f.p_kind = p == 1.0 ? 1 : 0;
    f.inv_p = 1.0 / p;
    f.dmax = std::pow(2.0, 1.0 / p);  // likelihood.cpp:208
    const int64_t n = static_cast<int64_t>(width) * height;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 8);
    finalize_slots_kernel<<<static_cast<unsigned>(blocks), 256, 0, as_stream(stream)>>>(slots, nslots, slot_stride, f,
                                                                                        map);
    return launch_status("finalize_slots_kernel");
}
