// Host-side helpers shared by the C-ABI translation units.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>

#include <cuda_runtime.h>

#include "spct_cuda.h"
#include "spct_device.cuh"

namespace spct_impl {

void set_error(const std::string& msg);

inline spct_status contract(const char* msg) {
    set_error(msg);
    return SPCT_ERR_CONTRACT;
}

inline spct_status cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return SPCT_OK;
    set_error(std::string(where) + ": " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SPCT_ERR_OOM : SPCT_ERR_CUDA;
}

// Instrumentation (profile.cu): count launches; bracket main kernels with events.
void note_launch(int n = 1);
int prof_begin(const char* name, cudaStream_t s);
void prof_end(int id, cudaStream_t s);

inline spct_status launch_status(const char* where) {
    note_launch();
    return cuda_status(cudaGetLastError(), where);
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Per-device launch state (profile.cu).  A process may drive several GPUs from one or more
// host threads, so nothing launch-related is cached process-wide: the dynamic shared-memory
// limit of a kernel is raised once per (device, kernel) and cached occupancy / SM counts
// are keyed by the current device; both are guarded by a mutex.
int current_device();
void ensure_smem(const void* func, size_t bytes);
template <class F>
void ensure_smem(F* func, size_t bytes) {
    ensure_smem(reinterpret_cast<const void*>(func), bytes);
}
// Cached per-device integer: compute() runs once per (device, key).
int per_device_int(int key, int (*compute)(int key));

// Stream-ordered scratch allocation (profile.cu): cudaMallocAsync from the device's default
// pool, which is set once per device to keep freed memory (no release threshold), so
// repeated calls reuse it instead of going back to the driver.
cudaError_t malloc_async(void** p, size_t bytes, cudaStream_t s);
template <class T>
cudaError_t malloc_async(T** p, size_t bytes, cudaStream_t s) {
    return malloc_async(reinterpret_cast<void**>(p), bytes, s);
}

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
inline int64_t ceil_div(int64_t v, int64_t m) { return (v + m - 1) / m; }

// Validate a source and derive the kernel-side quantisation parameters.
spct_status make_quant(const spct_source* src, spct_dev::QuantParams* q);

// Validate a device tensor descriptor.
spct_status check_ih(const spct_ih* t);
// The sweeps' carry tables hold row / column counts as u16 (carries.cu): both image
// dimensions must stay below 2^16 on the build and fused paths.
spct_status check_carry_dims(int width, int height);

// Bins per warp and band height used by the build for a given slab size / image.
struct BuildPlan {
    int B;          // bins per warp (4, 8 or 16)
    int warps;      // warps per CTA (slabs per CTA)
    int Lb;         // slab bins padded to a multiple of B (carry-table row length)
    int nstrips;    // ceil(width / 128)
    int Wp;         // nstrips * 128
    int band_rows;  // rows per band
    int nbands;
    int slab_groups;  // CTAs along the bin axis
    int strips_per_cta;  // fused sweep: strips side by side in one CTA (grid.x = ceil(nstrips / strips_per_cta))
};
BuildPlan plan_build(int width, int height, int bins, int force_B = 0, int ctas_per_sm = 2, int min_band_rows = 32,
                     int strips_per_cta = 1, int max_waves = 8, bool prefer_more_bands = false);

// Resident CTAs per SM of the build sweep (B bins per warp, `threads` per CTA) and of the
// fused sweep; used to size bands in whole waves.  Fall back to 2 without a device.
int build_ctas_per_sm(int B, int threads);
int fused_ctas_per_sm(int strips = 1);
int device_sms();
// The two plans every caller (workspace query included) must agree on.
BuildPlan plan_build_sweep(int width, int height, int bins);
BuildPlan plan_fused_sweep(int width, int height, int bins);

// Recover the bin map of a one-hot device tensor (tensor_match.cu).
spct_status ih_recover_bins(const spct_ih& t, uint16_t* bins, int64_t bins_pitch, uint32_t* flag, uint32_t* gsum,
                            cudaStream_t s);

// Workspace of the fused path's template prep (fused.cu).
size_t fused_prep_bytes(int bins);
// ... and of the gray frame an RGB source is converted to first (pitch x height bytes).
inline size_t fused_gray_bytes(const spct_source* src) {
    return static_cast<size_t>(round_up(src->pitch * static_cast<int64_t>(src->height), 256));
}


// Carry tables of the fused build+match sweep (carries.cu): row carries (u16), column
// counts above each band boundary (u16) and the band x strip corner sums (u32).
struct FusedCarries {
    const uint16_t* Lt;  // [nstrips][H][Lb]        (strip 0 unused)
    const uint16_t* C;   // [nbands - 1][Lb][Wp]
    const uint32_t* A;   // [Lb][nbands - 1][nstrips]
    // matcher window start (kh > 1): S[i][kl][x] = count of kl in column x over rows
    // [y0_i + o, y1_i), o = (-(kh - 1)) mod band_rows; with C it gives the sweep's running
    // column counts at every band top without re-reading the kh - 1 rows above it
    const uint16_t* S;   // [nbands - 1][Lb][Wp] or null
};
struct FusedCarryLayout {
    size_t lt_off, lt_bytes, r_off, r_bytes, c_off, c_bytes, a_off, a_bytes, s_off, s_bytes, total;
};
FusedCarryLayout fused_carry_layout(const BuildPlan& p, int height, bool window = false);
spct_status build_fused_carries(const spct_dev::QuantParams& q, const spct_ih& out, const BuildPlan& p,
                                void* workspace, size_t ws_bytes, cudaStream_t s, FusedCarries* fc, int kh = 0);
// The same for n <= kMaxCarryCh same-shape sources (one workspace each) in one launch per kernel.
constexpr int kMaxCarryCh = 8;
spct_status build_fused_carries_multi(int n, const spct_dev::QuantParams* qs, const spct_ih& out, const BuildPlan& p,
                                      void* const* workspaces, size_t ws_bytes, cudaStream_t s, FusedCarries* fcs,
                                      int kh);

}  // namespace spct_impl
