/*
 * spct_cuda.h — C-ABI of the B200 (sm_100a) integral-histogram / likelihood-map path.
 *
 * This is the drop-in boundary under the reference's C++ API (namespace spct,
 * /root/reference/proj/include/spct/{imagecore,integral,likelihood}.hpp).  The C++
 * host layer (include/spct/*.hpp, paper_1711_01656_b200/csrc/host/) keeps the
 * reference signatures and calls down through these entry points; Python tests and
 * bench.py bind them with ctypes.  No C++ or torch types cross this interface:
 * plain pointers, sizes and a cudaStream_t passed as void*.
 *
 * Conventions
 *   - Every entry point returns an spct_status.  Contract checks run first and use
 *     the reference's predicates, so a call that would throw spct::contract_error in
 *     the reference returns SPCT_ERR_CONTRACT here and launches nothing.
 *   - Device pointers are marked (dev).  Calls are stream-ordered and asynchronous
 *     unless stated; nothing allocates behind the caller's back except where a
 *     workspace is explicitly queried (spct_cu_*_workspace).
 *   - spct_cu_last_error() returns a thread-local message for the last failure.
 *
 * Device tensor layout (struct spct_ih): the reference stores, per bin, a zero-padded
 * (h+1)x(w+1) uint64 plane (integral.hpp:78-93).  The device stores the same values
 * as uint32 WITHOUT the all-zero padding row/column:
 *      data[k*plane_pitch + y*row_pitch + x] == H(bin0+k, y+1, x+1)   (reference indexing)
 * for 0<=k<bins, 0<=y<height, 0<=x<width, with row_pitch a multiple of 32 elements
 * (128-byte rows -> full-line, 16-byte-vector stores).  uint32 is exact because
 * every cell is <= height*width < 2^32 (checked).  spct_cu_ih_export re-creates the
 * reference layout (padding included, widened to uint64) for host mirrors.
 */
#ifndef SPCT_CUDA_H
#define SPCT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPCT_OK = 0,
    SPCT_ERR_CONTRACT = 2, /* spct::contract_error (reference error.hpp:11-14) */
    SPCT_ERR_IO = 3,       /* spct::io_error (error.hpp:17-20) */
    SPCT_ERR_CUDA = 4,     /* CUDA runtime / launch failure */
    SPCT_ERR_OOM = 5       /* device allocation failed */
} spct_status;

/* ScanScheduleKind (reference integral.hpp:21-26).  All kinds produce the same
 * bits; on the device they select nothing — accepted for drop-in. */
enum { SPCT_SCHED_SEQUENTIAL = 0, SPCT_SCHED_STS = 1, SPCT_SCHED_CW_TIS = 2, SPCT_SCHED_WF_TIS = 3 };

/* Window-match metrics.  MINKOWSKI is the reference's hist_distance_map
 * (likelihood.cpp:193-225).  The other three are extensions named by the thesis
 * but absent from the reference: definitions in DESIGN.md. */
enum { SPCT_METRIC_MINKOWSKI = 0, SPCT_METRIC_INTERSECTION = 1, SPCT_METRIC_BHATTACHARYYA = 2,
       SPCT_METRIC_CHISQ = 3 };

/* Pixel source of a build: what the fused load stage reads and how it bins it. */
enum { SPCT_SRC_BINS_U16 = 0, /* a BinMap (imagecore.hpp:65-76), values < nbins           */
       SPCT_SRC_GRAY_U8 = 1,  /* GrayImage -> quantize(img, nbins, lo, hi)  imagecore.cpp:45 */
       SPCT_SRC_RGB_U8 = 2,   /* planar ColorImage -> to_grayscale -> quantize   :17-24      */
       SPCT_SRC_SCALAR_F64 = 3 /* ScalarMap -> quantize(map, nbins, lo, hi)       :50-53      */ };

typedef struct {
    int kind;             /* SPCT_SRC_* */
    const void* plane[3]; /* (dev) plane[0] = bins/gray/R/values; plane[1..2] = G, B for RGB */
    int64_t pitch;        /* elements between rows of each plane (>= width) */
    int width, height;
    int nbins;            /* total bin count b of the histogram */
    double lo, hi;        /* quantisation range (defaults 0, 256) */
} spct_source;

typedef struct {
    uint32_t* data;      /* (dev) see layout above */
    int bins;            /* planes stored (a bin slab when sharded) */
    int bin0;            /* global index of plane 0 (slab start) */
    int nbins_total;     /* b of the full histogram */
    int height, width;   /* source image dims */
    int64_t row_pitch;   /* elements, multiple of 32, >= width */
    int64_t plane_pitch; /* elements, >= height*row_pitch */
} spct_ih;

/* ----------------------------------------------------------------- library */

const char* spct_cu_last_error(void);
/* Returns the library ABI version (1) and reports the CUDA device it will use. */
int spct_cu_version(void);
spct_status spct_cu_device_info(int* sm_major, int* sm_minor, int* num_sms);

/* ----------------------------------------------------------------- imagecore */

/* to_grayscale (imagecore.cpp:17-24): out = lround((r+g+b)/3). (dev) planes, n pixels. */
spct_status spct_cu_to_grayscale(const uint8_t* r, const uint8_t* g, const uint8_t* b, int64_t n,
                                 uint8_t* out, void* stream);

/* quantize (imagecore.cpp:28-53) of a GRAY_U8 / RGB_U8 / SCALAR_F64 source into a
 * dense BinMap (dev, width*height uint16).  Contract: width,height > 0,
 * 1 <= nbins <= 65536, hi > lo (imagecore.cpp:30-31,46,51). */
spct_status spct_cu_quantize(const spct_source* src, uint16_t* out_bins, void* stream);

/* Gradient-orientation BinMap (the orientation channel of the tracking batch): the
 * reference's gradient_maps(GrayImage, sigma) orientation (features.cpp:200-203, :78-93:
 * Gaussian smoothing, central differences, atan fold to degrees) binned by
 * phog.cpp:15-20 orientation_bin.  gray (dev) with row pitch `pitch`; out (dev) uint16
 * with row pitch out_pitch.  Contract: sigma >= 0 (features.cpp:201), width,height > 0,
 * 1 <= bins <= 65536, ceil(3 sigma) <= 31.  Workspace: spct_cu_orientation_workspace (the
 * bin-boundary table, 2 KiB). */
spct_status spct_cu_orientation_workspace(int width, int height, size_t* bytes);
spct_status spct_cu_orientation_bins(const uint8_t* gray, int64_t pitch, int width, int height, double sigma,
                                     int bins, uint16_t* out, int64_t out_pitch, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* Validation pass of build_tensor (integral.cpp:337-343): max BinMap value (dev -> host,
 * synchronises the stream). */
spct_status spct_cu_binmap_max(const uint16_t* bins, int64_t pitch, int width, int height,
                               int* out_max, void* stream);

/* ----------------------------------------------------------------- integral histogram */

/* estimate_memory (integral.cpp:592-599), same arithmetic.  elem_bytes as in the reference. */
spct_status spct_cu_estimate_memory(int w, int h, int bins, int elem_bytes, uint64_t* padded,
                                    uint64_t* raw, int* degenerate);

/* schedule_stats (integral.cpp:579-590). */
spct_status spct_cu_schedule_stats(int w, int h, int tile, int scan_len, long long* iterations,
                                   long long* tiles, double* efficiency);

/* Pitches the library wants for a (width, height, bins) tensor; fills row_pitch,
 * plane_pitch and returns the device bytes needed for data. */
spct_status spct_cu_ih_layout(int width, int height, int bins, int64_t* row_pitch,
                              int64_t* plane_pitch, uint64_t* bytes);

/* Scratch the build needs (row-carry and band-carry tables); 0 is possible. */
spct_status spct_cu_ih_build_workspace(const spct_source* src, int bin0, int bins,
                                       size_t* bytes);

/* build_integral_histogram (integral.cpp:548-551) of bins [out->bin0, out->bin0+out->bins)
 * into the caller-allocated device tensor `out`.  The contract checks of build_tensor
 * (integral.cpp:510-514) are the caller's: the host layer runs them with the
 * reference predicates (including the 2 GiB budget with elem_bytes = 8).  Here the
 * device-side checks are: dims > 0, nbins >= 1, slab inside [0, nbins), h*w < 2^32,
 * pitches aligned.  BinMap sources must already be validated (spct_cu_binmap_max). */
spct_status spct_cu_ih_build(const spct_source* src, const spct_ih* out, void* workspace,
                             size_t workspace_bytes, void* stream);

/* Re-create the reference layout for planes [k0, k1) of the tensor: a (k1-k0) x
 * (height+1) x (width+1) uint64 block with zero padding row/column (dev dst). */
spct_status spct_cu_ih_export_u64(const spct_ih* t, int k0, int k1, uint64_t* dst, void* stream);

/* ----------------------------------------------------------------- map consumers
 * (likelihood.cpp:257-330, tracker.cpp:77-113), bit-identical to the reference.
 * fuse_maps: `maps` is a host array of nmaps device pointers to n doubles each; weights a
 *   host array (nweights == 0: equal weights).  Contract: likelihood.cpp:258-269.
 * find_peaks: peaks of the (w x h) device map sorted by height (descending, ties in
 *   row-major order); the first min(count, max_out) go to xs / ys / heights (device);
 *   rank = index + 1.  Synchronises `stream` (count).
 * score_map: rank of the best peak inside gt (count + 1 if none).  Synchronises.
 * camshift: one refinement per start point (host arrays: starts, out = 2n doubles,
 *   iterations, zero_mass); synchronises. */
spct_status spct_cu_fuse_maps(const double* const* maps, int nmaps, const double* weights, int nweights, int64_t n,
                              double* out, void* stream);
spct_status spct_cu_find_peaks_workspace(int w, int h, size_t* bytes);
spct_status spct_cu_find_peaks(const double* map, int w, int h, int32_t* xs, int32_t* ys, double* heights,
                               int64_t max_out, int64_t* count, void* workspace, size_t workspace_bytes, void* stream);
spct_status spct_cu_score_map(const double* map, int w, int h, int gx, int gy, int gw, int gh, int64_t* rank,
                              void* workspace, size_t workspace_bytes, void* stream);
spct_status spct_cu_camshift(const double* map, int w, int h, const double* starts, int n, int win_w, int win_h,
                             double delta, int max_iter, double* out, int32_t* iterations, int32_t* zero_mass,
                             void* stream);

/* ----------------------------------------------------------------- SWIH (swih.hpp)
 * Weighted integral histogram: uint64 cells (16.16 fixed-point weight sums), unpadded
 * and pitched like spct_ih: data[k*plane_pitch + y*row_pitch + x] == H(k, y+1, x+1). */
typedef struct {
    uint64_t* data;
    int bins;
    int height;
    int width;
    int64_t row_pitch;
    int64_t plane_pitch;
} spct_wih;

spct_status spct_cu_wih_layout(int width, int height, int bins, int64_t* row_pitch, int64_t* plane_pitch,
                               uint64_t* bytes);
/* build_weighted_tensor (integral.cpp:553-559): bins (dev uint16, row pitch `pitch`, values
 * >= out->bins count nowhere) with per-pixel weights (dev uint64, same pitch), or, with
 * weights == NULL, the quadrant ramp field `field_dir` (0 NW, 1 NE, 2 SW, 3 SE; swih.cpp:45-53)
 * of a kw x kh kernel (build_quadrant_set swih.cpp:115-126). */
spct_status spct_cu_wih_build(const uint16_t* bins, int64_t pitch, const uint64_t* weights, int field_dir, int kw,
                              int kh, const spct_wih* out, void* stream);
spct_status spct_cu_wih_export_u64(const spct_wih* t, int k0, int k1, uint64_t* dst, void* stream);
/* region_histogram (integral.cpp:561-577) of a weighted tensor: rects (dev) n x {x, y, w, h}
 * (checked by the caller), out (dev) n x bins uint64. */
spct_status spct_cu_wih_region_counts(const spct_wih* t, const int32_t* rects, int n, uint64_t* out, void* stream);
/* swlh_query_fixed (swih.cpp:128-164) at n centres (host array of (cx, cy)) over the four
 * quadrant tensors set4[NW, NE, SW, SE]; out (dev) n x bins int64, 16.16.  Synchronises. */
spct_status spct_cu_swlh_query(const spct_wih* set4, int kw, int kh, const int32_t* centres, int n, int64_t* out,
                               void* stream);
/* brute_force_swlh_fixed (swih.cpp:166-178) at n centres (host array); out (dev). */
spct_status spct_cu_swlh_brute(const uint16_t* bins, int64_t pitch, int width, int height, int nbins, int kw, int kh,
                               const int32_t* centres, int n, int64_t* out, void* stream);
/* The tracker's swlh-distance map (track_loop.cpp:264-283): model (dev, bins doubles),
 * map (dev, width x height doubles).  Synchronises. */
spct_status spct_cu_swlh_map(const spct_wih* set4, int kw, int kh, const double* model, double* map, void* stream);
/* The same map in one sweep over the BinMap (dev uint16, nbins bins), without the quadrant
 * tensors: exact pyramid-weighted window sums from running column states (swlh_fused.cu),
 * bit-identical to spct_cu_swlh_map.  kw <= 128, kh <= 255. */
spct_status spct_cu_swlh_map_direct(const uint16_t* bins, int64_t pitch, int width, int height, int nbins, int kw,
                                    int kh, const double* model, double* map, void* stream);

/* ----------------------------------------------------------------- joint-IH median (motion.hpp)
 * spct_cu_ih_accumulate: the build of spct_cu_ih_build, added (sign +1) to or subtracted
 * (sign -1) from the tensor already in `acc` (uint32 wrap arithmetic; a joint histogram of
 * frames stays exact while frames * H * W < 2^32) — MedianBackgroundIH::add_frame
 * (motion.cpp:51-60).  spct_cu_median_background: background() (motion.cpp:71-99) of a
 * joint tensor over `nframes` frames, out (dev uint8).  spct_cu_median_sort:
 * median_background_sort (motion.cpp:103-118), frames a host array of nf device planes. */
spct_status spct_cu_ih_accumulate(const spct_source* src, const spct_ih* acc, int sign, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* One slide of a joint integral histogram (reference motion.cpp:62-69, MedianBackgroundIH::
 * slide): acc += IH(src_new) - IH(src_old) in ONE read-modify-write pass of acc (the two
 * frames' carry tables in one launch each, their rows scanned side by side), instead of two
 * spct_cu_ih_accumulate passes.  acc holds every bin of both sources.  Workspace:
 * spct_cu_ih_slide_workspace. */
spct_status spct_cu_ih_slide_workspace(int width, int height, int bins, size_t* bytes);
spct_status spct_cu_ih_slide(const spct_source* src_new, const spct_source* src_old, const spct_ih* acc,
                             void* workspace, size_t workspace_bytes, void* stream);
spct_status spct_cu_median_background(const spct_ih* joint, int nframes, int m, int n, uint8_t* out, int64_t out_pitch,
                                      void* stream);
spct_status spct_cu_median_sort(const uint8_t* const* frames, int nf, int width, int height, int64_t pitch,
                                uint8_t* out, int64_t out_pitch, void* stream);

/* IHT1 wire format (integral.hpp:132-135; dump_tensor / load_tensor integral.cpp:619-659):
 * "IHT1", LE u32 bins/height/width/elem_bytes, then the padded planes as LE elements.
 * spct_cu_ih_dump streams the device tensor (all of its planes) to `path`; elem_bytes 8 is
 * the reference format, 4 an extension.  spct_cu_ih_load_header reads and validates the
 * header (SPCT_ERR_IO with the reference's messages: cannot open / bad magic / truncated
 * header / unsupported element size / bad dimensions); spct_cu_ih_load fills a device
 * tensor of matching dims (truncated payload, nonzero padding or a value above 2^32-1 are
 * SPCT_ERR_IO).  Both synchronise `stream` (host file IO). */
spct_status spct_cu_ih_dump(const spct_ih* t, const char* path, int elem_bytes, void* stream);
spct_status spct_cu_ih_load_header(const char* path, int* bins, int* height, int* width, int* elem_bytes);
spct_status spct_cu_ih_load(const char* path, const spct_ih* t, void* stream);

/* region_histogram / region_count (integral.cpp:561-577), batched: rects (dev) are
 * n x {x, y, w, h} int32; out (dev) is n x t->bins uint32 (counts of planes
 * [0, t->bins)).  Rects are validated on the host by the caller (Rect::inside). */
spct_status spct_cu_region_counts(const spct_ih* t, const int32_t* rects, int n, uint32_t* out,
                                  void* stream);

/* ----------------------------------------------------------------- likelihood maps */

/* Contract checks of hist_distance_map (likelihood.cpp:196-206) on a HOST template. */
spct_status spct_cu_hist_check(int nbins, int width, int height, const double* tmpl_host,
                               int ntmpl, int kw, int kh, double p);

/* hist_distance_map (likelihood.cpp:193-225) over a device tensor that holds ALL bins
 * (t->bin0 == 0, t->bins == t->nbins_total): map (dev) is height x width float64,
 * borders replicated as spread_valid (:44-58).  tmpl (dev) has nbins doubles.
 * MINKOWSKI follows the reference's operation order (k = 0..b-1, divide, pow); each
 * window is divided by its actual total (:212-214; kw*kh for any tensor built from a
 * bin map) and a massless window scores 0 (:215), so arbitrary (e.g. IHT1-loaded)
 * tensors give the reference's map. */
spct_status spct_cu_hist_match(const spct_ih* t, const double* tmpl, int kw, int kh, double p,
                               int metric, double* map, void* stream);
/* The same map computed the reference's way from the tensor: one thread per window, the
 * b planes visited in order k = 0..b-1 with the reference's divide and pow (bit-identical
 * to likelihood.cpp:211-221 for p = 1; 4 b scattered reads per window).  spct_cu_hist_match
 * instead reads the tensor once (tensor_match.cu: per-pixel bins recovered and checked,
 * then the fused sweep; bit-identical for p = 1 with an integral template and a
 * power-of-two kw*kh, within 1e-5 otherwise) and falls back to this arithmetic for tensors
 * that are not the integral histogram of a bin map.  SPCT_EXACT_MAPS=1 makes
 * spct_cu_hist_match take this path too. */
spct_status spct_cu_hist_match_exact(const spct_ih* t, const double* tmpl, int kw, int kh, double p,
                                     int metric, double* map, void* stream);

/* Bin-slab partial of the window statistic over the valid grid (nv x nu, nu = width-kw+1,
 * nv = height-kh+1): partial[v*nu+u] (+)= sum_{k in slab} term_k.  With accumulate = 0
 * the buffer is overwritten.  Summing slab partials (e.g. an NCCL reduce across GPUs)
 * then spct_cu_hist_finalize gives the full map. */
spct_status spct_cu_hist_partial(const spct_ih* t, const double* tmpl, int kw, int kh, double p,
                                 int metric, double* partial, int accumulate, void* stream);

/* partial sums (dev, nv x nu) -> likelihood map (dev, height x width) with the
 * reference's finalisation (likelihood.cpp:220-224) and spread_valid border replication. */
spct_status spct_cu_hist_finalize(const double* partial, int width, int height, int kw, int kh,
                                  double p, int metric, double* map, void* stream);

/* 1 if the fused sweeps below can produce a kw x kh window statistic without a stored
 * tensor (16-bit running-histogram cells: kw <= 128, kh <= 255, kw*kh <= 65535), else 0.
 * Callers recomputing a map from a tensor's source frame take that path only then. */
int spct_cu_fused_window_ok(int kw, int kh);

/* Fused build + match: one pass that writes the integral histogram of the slab
 * [out->bin0, out->bin0+out->bins) AND the slab's partial window statistic (as
 * spct_cu_hist_partial), without re-reading the tensor from HBM.  `out->data` may be
 * NULL to compute the partial map only.  tmpl (dev) holds the FULL template
 * (nbins_total doubles).  Workspace from spct_cu_ih_build_workspace. */
spct_status spct_cu_ih_build_match(const spct_source* src, const spct_ih* out, const double* tmpl,
                                   int kw, int kh, double p, int metric, double* partial,
                                   void* workspace, size_t workspace_bytes, void* stream);

/* Fused build + match producing the finished likelihood map (dev, height x width,
 * spread_valid borders) in the same pass: build_integral_histogram followed by
 * hist_distance_map (tools/spct_main.cpp:332-333) for a tensor that holds every bin
 * (out->bin0 == 0, out->bins == out->nbins_total).  `out->data` may be NULL. */
spct_status spct_cu_ih_build_match_map(const spct_source* src, const spct_ih* out, const double* tmpl,
                                       int kw, int kh, double p, int metric, double* map,
                                       void* workspace, size_t workspace_bytes, void* stream);

/* spct_cu_ih_build_match_map for n (1..8) sources of one shape — the feature channels of a
 * tracking batch (reference: track_loop.cpp's per-channel likelihood fan-out, each channel
 * build_integral_histogram + hist_distance_map): the carry tables and template preps of all
 * channels are computed in one launch per kernel, then one sweep per channel.  outs[c]
 * share width / height / bins and either all store their tensor or none; tmpls[c] and
 * maps[c] are per-channel device pointers; each channel has its own workspace of
 * workspace_bytes (spct_cu_ih_build_workspace of one channel). */
spct_status spct_cu_ih_build_match_map_multi(int n, const spct_source* srcs, const spct_ih* outs,
                                             const double* const* tmpls, int kw, int kh, double p, int metric,
                                             double* const* maps, void* const* workspaces,
                                             size_t workspace_bytes, void* stream);

/* ----------------------------------------------------------------- bin-slab reduce over peer memory
 * (peer.cu).  The multi-GPU form of hist_distance_map (likelihood.cpp:193-225)
 * with the bins sharded across ranks: rank r passes a slot of the root's slot buffer
 * (opened with spct_cu_peer_open) as the `partial` of spct_cu_ih_build_match, so its
 * sweep writes the partial map over NVLink; then publishes with spct_cu_flag_signal.
 * The root waits (spct_cu_flag_wait) and runs spct_cu_hist_finalize_slots, which sums
 * the slots in rank order and finalises (spread_valid + clamp, likelihood.cpp:44-58,
 * 220-221).  Buffers shared this way come from spct_cu_peer_alloc (zeroed cudaMalloc +
 * its IPC handle, SPCT_IPC_HANDLE_BYTES bytes).  Flags are uint64 epochs; a wait that
 * exceeds timeout_ns sets *err (device) to 1 and returns instead of hanging. */
#define SPCT_IPC_HANDLE_BYTES 64
spct_status spct_cu_peer_alloc(size_t bytes, void** ptr, void* handle);
spct_status spct_cu_peer_free(void* ptr);
spct_status spct_cu_peer_open(const void* handle, void** ptr);
spct_status spct_cu_peer_close(void* ptr);
spct_status spct_cu_flag_signal(uint64_t* flag, uint64_t value, void* stream);
spct_status spct_cu_flag_wait(const uint64_t* flags, int n, int64_t stride, uint64_t value, uint64_t timeout_ns,
                              uint32_t* err, void* stream);
spct_status spct_cu_hist_finalize_slots(const double* slots, int nslots, int64_t slot_stride, int width, int height,
                                        int kw, int kh, double p, int metric, double* map, void* stream);
/* Band-owned variant: the caller owns valid rows [v0, v1); `partials` is a
 * host array of nsrc (<= 16) device pointers to the ranks' full (H-kh+1) x (W-kw+1)
 * partial maps (peer mappings), summed in array order; writes the final map rows of the
 * band (with the replicated top / bottom borders for the first / last band) into `map`
 * (W x H, may be a peer mapping).  spct_cu_flag_signal_many publishes one epoch to n
 * (<= 16) flags with one release. */
spct_status spct_cu_hist_finalize_band(const double* const* partials, int nsrc, int width, int height, int kw, int kh,
                                       double p, int metric, int v0, int v1, double* map, void* stream);
spct_status spct_cu_flag_signal_many(uint64_t* const* flags, int n, uint64_t value, void* stream);

/* ----------------------------------------------------------------- instrumentation */

/* Every kernel launch of this library increments a process-wide counter.  With
 * profiling enabled, the main kernels (ih_sweep, ih_sweep_match, match_partial) are
 * bracketed by CUDA events recorded on their launch stream; spct_cu_profile_read
 * synchronises those events and returns the summed device time per kernel name. */
uint64_t spct_cu_launch_count(void);
void spct_cu_profile_enable(int on);
void spct_cu_profile_reset(void);
spct_status spct_cu_profile_read(const char* kernel, double* total_ms, int* launches);

#ifdef __cplusplus
}
#endif
#endif /* SPCT_CUDA_H */
