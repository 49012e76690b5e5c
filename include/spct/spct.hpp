// spct:: drop-in API backed by the B200 C-ABI (include/spct_cuda.h).
//
// A caller of the reference library (/root/reference/proj/include/spct/*.hpp) re-links
// against libspct_b200.so and keeps its source: the names, signatures, argument
// meaning and error behaviour below are the reference's for the hot path
//   to_grayscale / quantize            (imagecore.hpp:95-100)
//   build_integral_histogram           (integral.hpp:98-100)
//   region_histogram / region_count    (integral.hpp:111-114)
//   schedule_stats / estimate_memory   (integral.hpp:116-130)
//   dump_tensor / load_tensor          (integral.hpp:132-135, the IHT1 wire format)
//   hist_distance_map                  (likelihood.hpp:59-61)
//   fuse_maps / find_peaks / score_map (likelihood.hpp:63-88), camshift_refine (tracker.hpp:62-64)
// What changes underneath: the tensor lives in HBM as uint32 (exact, h*w < 2^32) and
// `IntegralHistogramTensor::data` is a host mirror in the reference layout (padded,
// uint64) that is materialised from the device only when a caller touches it.
// imagecore.hpp / integral.hpp / likelihood.hpp / error.hpp in this directory just
// include this file so existing #include lines keep working.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace spct {

// ---------------------------------------------------------------- errors (error.hpp)
struct contract_error : std::invalid_argument {  // CLI exit code 2
    using std::invalid_argument::invalid_argument;
};
struct io_error : std::runtime_error {  // CLI exit code 3
    using std::runtime_error::runtime_error;
};
// CUDA / device failures surface as this (not in the reference: it has no device).
struct device_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
inline void require(bool ok, const std::string& what) {
    if (!ok) throw contract_error(what);
}

// ---------------------------------------------------------------- rasters (imagecore.hpp)
struct Rect {
    int x = 0, y = 0, w = 0, h = 0;
    int right() const { return x + w; }
    int bottom() const { return y + h; }
    long long area() const { return 1LL * w * h; }
    double cx() const { return x + (w - 1) / 2.0; }
    double cy() const { return y + (h - 1) / 2.0; }
    bool contains(double px, double py) const { return px >= x && px < x + w && py >= y && py < y + h; }
    bool inside(int img_w, int img_h) const {
        return x >= 0 && y >= 0 && w >= 0 && h >= 0 && right() <= img_w && bottom() <= img_h;
    }
    bool operator==(const Rect&) const = default;
};
Rect intersect(const Rect& a, const Rect& b);

template <class T>
struct Raster {  // row-major single plane
    int width = 0, height = 0;
    std::vector<T> data;
    Raster() = default;
    Raster(int w, int h, T fill = T{}) : width(w), height(h), data(std::size_t(w) * h, fill) {}
    T& at(int x, int y) { return data[std::size_t(y) * width + x]; }
    T at(int x, int y) const { return data[std::size_t(y) * width + x]; }
};

struct GrayImage : Raster<std::uint8_t> {
    using Raster::Raster;
    bool operator==(const GrayImage& o) const { return width == o.width && height == o.height && data == o.data; }
};

struct ColorImage {  // planar R, G, B
    int width = 0, height = 0;
    std::vector<std::uint8_t> r, g, b;
    ColorImage() = default;
    ColorImage(int w, int h)
        : width(w), height(h), r(std::size_t(w) * h), g(std::size_t(w) * h), b(std::size_t(w) * h) {}
    std::size_t idx(int x, int y) const { return std::size_t(y) * width + x; }
};

struct BinMap : Raster<std::uint16_t> {  // per-pixel bin in [0, bins)
    int bins = 0;
    BinMap() = default;
    BinMap(int w, int h, int b) : Raster(w, h, 0), bins(b) {}
};

struct ScalarMap : Raster<double> {
    std::string kind;
    ScalarMap() = default;
    ScalarMap(int w, int h, double fill = 0.0, std::string k = {}) : Raster(w, h, fill), kind(std::move(k)) {}
};

GrayImage to_grayscale(const ColorImage& img);
BinMap quantize(const GrayImage& img, int bins, double lo = 0.0, double hi = 256.0);
BinMap quantize(const ScalarMap& map, int bins, double lo, double hi);

// ---------------------------------------------------------------- tensor (integral.hpp)
enum class ScanScheduleKind { Sequential, ScanTransposeScan, CrossWeaveTiled, WavefrontTiled };
const char* to_string(ScanScheduleKind k);
ScanScheduleKind schedule_from_string(const std::string& s);

// Accepted for drop-in compatibility.  Every kind yields the same bits; the
// device sweep ignores kind/tile/threads after validating them like the reference.
struct ScanSchedule {
    ScanScheduleKind kind = ScanScheduleKind::Sequential;
    int tile = 32;
    int threads = 1;
};

namespace detail {
struct DeviceTensor;  // owns the HBM allocation (RAII, move-only through shared_ptr)

// Reference-layout host view: b x (h+1) x (w+1) uint64, filled from HBM on first use.
class HostMirror {
public:
    using value_type = std::uint64_t;
    using const_iterator = const std::uint64_t*;
    std::size_t size() const;
    bool empty() const { return size() == 0; }
    const std::uint64_t* data() const;
    std::uint64_t* data();
    const std::uint64_t* begin() const { return data(); }
    const std::uint64_t* end() const { return data() + size(); }
    std::uint64_t operator[](std::size_t i) const { return data()[i]; }
    std::uint64_t& operator[](std::size_t i) { return data()[i]; }
    bool operator==(const HostMirror& o) const;
    bool operator==(const std::vector<std::uint64_t>& o) const;
    void clear();
    bool mirrored() const { return valid_; }  // the host copy is filled (non-reference addition)
    void adopt(std::vector<std::uint64_t>&& host);  // library-internal: install a filled host copy

    std::shared_ptr<DeviceTensor> dev;  // null for a default-constructed tensor
private:
    mutable std::vector<std::uint64_t> host_;
    mutable bool valid_ = false;
    void fill() const;
};
}  // namespace detail

struct IntegralHistogramTensor {
    int bins = 0;
    int height = 0, width = 0;
    detail::HostMirror data;  // plane-major, row-major, padded; lazily mirrored from HBM

    std::size_t plane_stride() const { return std::size_t(height + 1) * (width + 1); }
    std::size_t row_stride() const { return std::size_t(width + 1); }
    std::uint64_t at(int k, int y, int x) const { return data[k * plane_stride() + std::size_t(y) * row_stride() + x]; }
    const std::uint64_t* plane(int k) const { return data.data() + k * plane_stride(); }
    std::uint64_t* plane(int k) { return data.data() + k * plane_stride(); }

    // Device view for kernels that consume the tensor in place (non-reference addition).
    const void* device_descriptor() const;  // -> const spct_ih*
};

inline constexpr std::uint64_t kDefaultMemoryBudget = 2ull << 30;

IntegralHistogramTensor build_integral_histogram(const BinMap& bins, const ScanSchedule& schedule = {},
                                                 std::uint64_t memory_budget = kDefaultMemoryBudget);
// integral.hpp:102-104: each pixel contributes its (16.16 fixed-point) weight instead of 1.
IntegralHistogramTensor build_weighted_tensor(const BinMap& bins, const std::vector<std::uint64_t>& weights,
                                              const ScanSchedule& schedule = {},
                                              std::uint64_t memory_budget = kDefaultMemoryBudget);
std::vector<std::uint64_t> region_histogram(const IntegralHistogramTensor& t, const Rect& r);
std::uint64_t region_count(const IntegralHistogramTensor& t, int bin, const Rect& r);

struct ScheduleStats {
    long long wavefront_iterations;
    long long tile_count;
    double scan_efficiency;
};
ScheduleStats schedule_stats(int w, int h, int tile, int scan_len);

struct MemoryEstimate {
    std::uint64_t padded_bytes;
    std::uint64_t raw_bytes;
    bool degenerate;
};
MemoryEstimate estimate_memory(int w, int h, int bins, int elem_bytes);

// Binary dump (integral.hpp:132-135): magic "IHT1", little-endian u32 bins/h/w/elem_bytes,
// then the planes in storage order as little-endian u64.  Streamed from / to HBM.
void dump_tensor(const IntegralHistogramTensor& t, const std::string& path);
IntegralHistogramTensor load_tensor(const std::string& path);

// ---------------------------------------------------------------- likelihood (likelihood.hpp)
struct LikelihoodMap {
    int width = 0, height = 0;
    std::vector<double> values;  // row-major, in [0, 1]
    std::string tag;
    double& at(int x, int y) { return values[std::size_t(y) * width + x]; }
    double at(int x, int y) const { return values[std::size_t(y) * width + x]; }
};

LikelihoodMap hist_distance_map(const IntegralHistogramTensor& t, const std::vector<double>& template_hist, int kw,
                                int kh, double p = 1.0);

// Map consumers (likelihood.hpp:63-88), computed on the device, bit-identical.
LikelihoodMap fuse_maps(const std::vector<LikelihoodMap>& maps, std::vector<double> weights = {});

struct Peak {
    int x = 0, y = 0;
    double height = 0.0;
    int rank = 0;  // 1 = highest
};
std::vector<Peak> find_peaks(const LikelihoodMap& map);
int score_map(const LikelihoodMap& map, const Rect& gt);

// camshift_refine (tracker.hpp:54-64; the reference declares it next to its Eigen tracker).
struct CamshiftResult {
    double cx = 0, cy = 0;
    int iterations = 0;
    bool zero_mass = false;  // window mass was zero; center left at init
};
CamshiftResult camshift_refine(const LikelihoodMap& map, double cx, double cy, int win_w, int win_h,
                               double delta = 0.5, int max_iter = 20);

// ---------------------------------------------------------------- extensions (not in the reference)
enum class HistMetric { Minkowski = 0, Intersection = 1, Bhattacharyya = 2, ChiSquare = 3 };

// hist_distance_map over a tensor built by this library recomputes the window counts
// from the tensor's source frame in the fused sweep (within the 1e-5 map tolerance).
// With exact maps on (set_exact_maps(true) or SPCT_EXACT_MAPS=1) it reads the tensor
// with the reference's operation order instead: bit-identical for p = 1.
void set_exact_maps(bool on);
bool exact_maps();

// hist_distance_map with a selectable bin-to-bin statistic (thesis PAPER.md:703).
LikelihoodMap hist_match_map(const IntegralHistogramTensor& t, const std::vector<double>& template_hist, int kw,
                             int kh, HistMetric metric, double p = 1.0);

// The same into a caller-owned map whose storage is reused when the size matches: a
// per-frame loop then skips allocating (and page-faulting) W x H doubles every call,
// which at 4096^2 costs more than the whole device computation.
void hist_match_map_into(const IntegralHistogramTensor& t, const std::vector<double>& template_hist, int kw, int kh,
                         HistMetric metric, double p, LikelihoodMap& out);

// quantize -> build -> match in one fused device pass over a gray frame; the tensor is
// returned as well (device resident).  Equivalent to
//   t = build_integral_histogram(quantize(img, bins)); map = hist_distance_map(t, tmpl, kw, kh, p)
LikelihoodMap likelihood_from_frame(const GrayImage& img, int bins, const std::vector<double>& template_hist, int kw,
                                    int kh, double p, IntegralHistogramTensor* tensor_out = nullptr,
                                    std::uint64_t memory_budget = kDefaultMemoryBudget);

}  // namespace spct
