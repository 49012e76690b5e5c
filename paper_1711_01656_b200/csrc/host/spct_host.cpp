// spct:: drop-in host layer (include/spct/spct.hpp) on top of the C-ABI.
//
// Each function re-runs the reference's contract checks with the same predicates
// and messages before touching the device, so reference expectations such as
// CHECK_THROWS_AS(..., contract_error) (test_integral.cpp:190-206) still hold.
// Device failures throw spct::device_error.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include <cuda_runtime.h>

#include "spct/spct.hpp"
#include "spct_cuda.h"

namespace spct {

namespace {
bool g_exact_maps = [] {
    const char* e = std::getenv("SPCT_EXACT_MAPS");
    return e && *e && *e != '0';
}();
}  // namespace

void set_exact_maps(bool on) { g_exact_maps = on; }
bool exact_maps() { return g_exact_maps; }

namespace {

void check(spct_status st) {
    if (st == SPCT_OK) return;
    const std::string msg = spct_cu_last_error();
    if (st == SPCT_ERR_CONTRACT) throw contract_error(msg);
    if (st == SPCT_ERR_IO) throw io_error(msg);
    throw device_error(msg);
}

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw device_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer.
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t bytes) {
        if (bytes) cuda(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

template <class T>
void upload(DevBuf& d, const std::vector<T>& v) {
    cuda(cudaMemcpy(d.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
}

}  // namespace

namespace detail {

struct DeviceTensor {
    spct_ih desc{};
    std::unique_ptr<DevBuf> mem;
    // The frame the tensor was built from (device copy): hist_distance_map recomputes
    // window counts from it (1 B/px) instead of re-reading b*H*W*4 tensor bytes.
    spct_source src{};
    std::unique_ptr<DevBuf> src_mem;
};

std::size_t HostMirror::size() const {
    if (!dev) return host_.size();
    return std::size_t(dev->desc.bins) * std::size_t(dev->desc.height + 1) * std::size_t(dev->desc.width + 1);
}

void HostMirror::fill() const {
    if (valid_ || !dev) return;
    const spct_ih& d = dev->desc;
    const std::size_t plane = std::size_t(d.height + 1) * (d.width + 1);
    host_.resize(plane * d.bins);
    // Export a few planes at a time through a bounded device staging buffer.
    const std::size_t per = std::max<std::size_t>(1, (std::size_t(256) << 20) / (plane * 8));
    DevBuf stage(std::min<std::size_t>(per, d.bins) * plane * 8);
    for (int k0 = 0; k0 < d.bins; k0 += int(per)) {
        const int k1 = std::min<int>(d.bins, k0 + int(per));
        check(spct_cu_ih_export_u64(&d, k0, k1, stage.as<std::uint64_t>(), nullptr));
        cuda(cudaMemcpy(host_.data() + std::size_t(k0) * plane, stage.p, std::size_t(k1 - k0) * plane * 8,
                        cudaMemcpyDeviceToHost),
             "D2H");
    }
    valid_ = true;
}

const std::uint64_t* HostMirror::data() const {
    fill();
    return host_.data();
}

std::uint64_t* HostMirror::data() {
    fill();
    return host_.data();
}

bool HostMirror::operator==(const HostMirror& o) const {
    if (size() != o.size()) return false;
    return std::equal(begin(), end(), o.begin());
}

bool HostMirror::operator==(const std::vector<std::uint64_t>& o) const {
    if (size() != o.size()) return false;
    return std::equal(begin(), end(), o.begin());
}

void HostMirror::clear() {
    dev.reset();
    host_.clear();
    valid_ = false;
}

}  // namespace detail

Rect intersect(const Rect& a, const Rect& b) {
    const int x1 = std::max(a.x, b.x), y1 = std::max(a.y, b.y);
    const int x2 = std::min(a.right(), b.right()), y2 = std::min(a.bottom(), b.bottom());
    if (x2 <= x1 || y2 <= y1) return Rect{x1, y1, 0, 0};
    return Rect{x1, y1, x2 - x1, y2 - y1};
}

GrayImage to_grayscale(const ColorImage& img) {
    GrayImage out(img.width, img.height);
    const std::size_t n = out.data.size();
    if (n == 0) return out;
    DevBuf d(4 * n);
    auto* p = d.as<std::uint8_t>();
    cuda(cudaMemcpy(p, img.r.data(), n, cudaMemcpyHostToDevice), "H2D");
    cuda(cudaMemcpy(p + n, img.g.data(), n, cudaMemcpyHostToDevice), "H2D");
    cuda(cudaMemcpy(p + 2 * n, img.b.data(), n, cudaMemcpyHostToDevice), "H2D");
    check(spct_cu_to_grayscale(p, p + n, p + 2 * n, std::int64_t(n), p + 3 * n, nullptr));
    cuda(cudaMemcpy(out.data.data(), p + 3 * n, n, cudaMemcpyDeviceToHost), "D2H");
    return out;
}

namespace {
template <class T>
BinMap quantize_any(const Raster<T>& img, int kind, int bins, double lo, double hi, const char* empty_msg) {
    require(img.width > 0 && img.height > 0, empty_msg);                      // imagecore.cpp:46 / :51
    require(bins >= 1 && bins <= 65536, "quantize: bins must be in [1, 65536]");  // :30
    require(hi > lo, "quantize: hi must exceed lo");                            // :31
    const std::size_t n = img.data.size();
    DevBuf src(n * sizeof(T)), dst(n * 2);
    upload(src, img.data);
    spct_source s{};
    s.kind = kind;
    s.plane[0] = src.p;
    s.pitch = img.width;
    s.width = img.width;
    s.height = img.height;
    s.nbins = bins;
    s.lo = lo;
    s.hi = hi;
    check(spct_cu_quantize(&s, dst.as<std::uint16_t>(), nullptr));
    BinMap out(img.width, img.height, bins);
    cuda(cudaMemcpy(out.data.data(), dst.p, n * 2, cudaMemcpyDeviceToHost), "D2H");
    return out;
}
}  // namespace

BinMap quantize(const GrayImage& img, int bins, double lo, double hi) {
    return quantize_any(img, SPCT_SRC_GRAY_U8, bins, lo, hi, "quantize: empty image");
}

BinMap quantize(const ScalarMap& map, int bins, double lo, double hi) {
    return quantize_any(map, SPCT_SRC_SCALAR_F64, bins, lo, hi, "quantize: empty map");
}

const char* to_string(ScanScheduleKind k) {
    static const char* names[] = {"sequential", "sts", "cw-tis", "wf-tis"};
    const int i = static_cast<int>(k);
    return (i >= 0 && i < 4) ? names[i] : "?";
}

ScanScheduleKind schedule_from_string(const std::string& s) {  // integral.cpp:63-69
    if (s == "sequential" || s == "seq") return ScanScheduleKind::Sequential;
    if (s == "sts" || s == "scan-transpose-scan") return ScanScheduleKind::ScanTransposeScan;
    if (s == "cw-tis" || s == "crossweave") return ScanScheduleKind::CrossWeaveTiled;
    if (s == "wf-tis" || s == "wavefront") return ScanScheduleKind::WavefrontTiled;
    throw contract_error("unknown schedule '" + s + "'");
}

const void* IntegralHistogramTensor::device_descriptor() const { return data.dev ? &data.dev->desc : nullptr; }

namespace {

// build_tensor's checks (integral.cpp:510-514, 330-343) on the host copy.
void validate_build(const BinMap& bm, const ScanSchedule& schedule, std::uint64_t budget) {
    require(bm.width > 0 && bm.height > 0, "build: empty bin map");
    require(bm.bins >= 1, "build: bins must be >= 1");
    std::uint16_t mx = 0;
    for (std::uint16_t v : bm.data) mx = std::max(mx, v);
    require(mx < bm.bins, "build: bin index out of range");
    require(schedule.tile >= 2 && schedule.tile <= 4096, "build: tile must be in [2, 4096]");
    require(schedule.threads >= 1 && schedule.threads <= 64, "build: threads must be in [1, 64]");
    const MemoryEstimate est = estimate_memory(bm.width, bm.height, bm.bins, 8);
    if (est.padded_bytes > budget)
        throw contract_error("tensor of " + std::to_string(est.padded_bytes) + " bytes exceeds the memory budget of " +
                             std::to_string(budget));
}

IntegralHistogramTensor build_from_source(const spct_source& src, std::unique_ptr<DevBuf> src_mem) {
    auto dt = std::make_shared<detail::DeviceTensor>();
    dt->src = src;
    dt->src_mem = std::move(src_mem);
    spct_ih& d = dt->desc;
    std::uint64_t bytes = 0;
    check(spct_cu_ih_layout(src.width, src.height, src.nbins, &d.row_pitch, &d.plane_pitch, &bytes));
    dt->mem = std::make_unique<DevBuf>(bytes);
    d.data = dt->mem->as<std::uint32_t>();
    d.bins = src.nbins;
    d.bin0 = 0;
    d.nbins_total = src.nbins;
    d.height = src.height;
    d.width = src.width;
    std::size_t ws = 0;
    check(spct_cu_ih_build_workspace(&src, 0, src.nbins, &ws));
    DevBuf work(ws);
    check(spct_cu_ih_build(&src, &d, work.p, ws, nullptr));
    cuda(cudaDeviceSynchronize(), "build");
    IntegralHistogramTensor t;
    t.bins = src.nbins;
    t.height = src.height;
    t.width = src.width;
    t.data.dev = std::move(dt);
    return t;
}

}  // namespace

IntegralHistogramTensor build_integral_histogram(const BinMap& bins, const ScanSchedule& schedule,
                                                 std::uint64_t memory_budget) {
    validate_build(bins, schedule, memory_budget);
    auto src = std::make_unique<DevBuf>(bins.data.size() * 2);
    upload(*src, bins.data);
    spct_source s{};
    s.kind = SPCT_SRC_BINS_U16;
    s.plane[0] = src->p;
    s.pitch = bins.width;
    s.width = bins.width;
    s.height = bins.height;
    s.nbins = bins.bins;
    return build_from_source(s, std::move(src));
}

namespace {
const spct_ih& desc_of(const IntegralHistogramTensor& t) {
    require(t.data.dev != nullptr, "tensor has no device storage");
    return t.data.dev->desc;
}
}  // namespace

std::vector<std::uint64_t> region_histogram(const IntegralHistogramTensor& t, const Rect& r) {
    require(r.w >= 0 && r.h >= 0, "region_histogram: negative extent");       // integral.cpp:562
    require(r.inside(t.width, t.height), "region_histogram: rect outside image");  // :563
    const spct_ih& d = desc_of(t);
    DevBuf rect(16), out(std::size_t(t.bins) * 4);
    const std::int32_t rr[4] = {r.x, r.y, r.w, r.h};
    cuda(cudaMemcpy(rect.p, rr, 16, cudaMemcpyHostToDevice), "H2D");
    check(spct_cu_region_counts(&d, rect.as<std::int32_t>(), 1, out.as<std::uint32_t>(), nullptr));
    std::vector<std::uint32_t> h32(t.bins);
    cuda(cudaMemcpy(h32.data(), out.p, h32.size() * 4, cudaMemcpyDeviceToHost), "D2H");
    return std::vector<std::uint64_t>(h32.begin(), h32.end());
}

std::uint64_t region_count(const IntegralHistogramTensor& t, int bin, const Rect& r) {
    require(bin >= 0 && bin < t.bins, "region_count: bin out of range");     // integral.cpp:570
    require(r.inside(t.width, t.height), "region_count: rect outside image");  // :571
    return region_histogram(t, r)[bin];
}

// IHT1 wire format (integral.cpp:619-659): streamed from / to HBM by the C-ABI.
void dump_tensor(const IntegralHistogramTensor& t, const std::string& path) {
    check(spct_cu_ih_dump(&desc_of(t), path.c_str(), 8, nullptr));
}

IntegralHistogramTensor load_tensor(const std::string& path) {
    int bins = 0, h = 0, w = 0, elem = 0;
    check(spct_cu_ih_load_header(path.c_str(), &bins, &h, &w, &elem));
    auto dt = std::make_shared<detail::DeviceTensor>();
    spct_ih& d = dt->desc;
    std::uint64_t bytes = 0;
    check(spct_cu_ih_layout(w, h, bins, &d.row_pitch, &d.plane_pitch, &bytes));
    dt->mem = std::make_unique<DevBuf>(bytes);
    d.data = dt->mem->as<std::uint32_t>();
    d.bins = bins;
    d.bin0 = 0;
    d.nbins_total = bins;
    d.height = h;
    d.width = w;
    check(spct_cu_ih_load(path.c_str(), &d, nullptr));
    IntegralHistogramTensor t;
    t.bins = bins;
    t.height = h;
    t.width = w;
    t.data.dev = std::move(dt);
    return t;
}

ScheduleStats schedule_stats(int w, int h, int tile, int scan_len) {
    ScheduleStats s{};
    check(spct_cu_schedule_stats(w, h, tile, scan_len, &s.wavefront_iterations, &s.tile_count, &s.scan_efficiency));
    return s;
}

MemoryEstimate estimate_memory(int w, int h, int bins, int elem_bytes) {
    MemoryEstimate e{};
    int deg = 0;
    check(spct_cu_estimate_memory(w, h, bins, elem_bytes, &e.padded_bytes, &e.raw_bytes, &deg));
    e.degenerate = deg != 0;
    return e;
}

LikelihoodMap hist_match_map(const IntegralHistogramTensor& t, const std::vector<double>& th, int kw, int kh,
                             HistMetric metric, double p) {
    check(spct_cu_hist_check(t.bins, t.width, t.height, th.data(), int(th.size()), kw, kh, p));
    const spct_ih& d = desc_of(t);
    DevBuf tm(th.size() * 8), map(std::size_t(t.width) * t.height * 8);
    upload(tm, th);
    const detail::DeviceTensor& dt = *t.data.dev;
    if (dt.src_mem && !exact_maps()) {
        // recompute the window counts from the source in the fused sweep (no tensor re-read)
        spct_ih nodata = d;
        nodata.data = nullptr;
        std::size_t ws = 0;
        check(spct_cu_ih_build_workspace(&dt.src, 0, d.bins, &ws));
        DevBuf work(ws);
        check(spct_cu_ih_build_match_map(&dt.src, &nodata, tm.as<double>(), kw, kh, p, int(metric), map.as<double>(),
                                         work.p, ws, nullptr));
    } else {
        check(spct_cu_hist_match(&d, tm.as<double>(), kw, kh, p, int(metric), map.as<double>(), nullptr));
    }
    LikelihoodMap out;
    out.width = t.width;
    out.height = t.height;
    out.tag = metric == HistMetric::Minkowski ? "hist-distance" : "hist-match";
    out.values.resize(std::size_t(t.width) * t.height);
    cuda(cudaMemcpy(out.values.data(), map.p, out.values.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    return out;
}

LikelihoodMap hist_distance_map(const IntegralHistogramTensor& t, const std::vector<double>& th, int kw, int kh,
                                double p) {
    return hist_match_map(t, th, kw, kh, HistMetric::Minkowski, p);
}

namespace {
std::unique_ptr<DevBuf> upload_map(const LikelihoodMap& m) {
    require(m.values.size() == std::size_t(m.width) * std::size_t(m.height), "map: values do not match width * height");
    auto d = std::make_unique<DevBuf>(m.values.size() * 8);
    upload(*d, m.values);
    return d;
}
}  // namespace

LikelihoodMap fuse_maps(const std::vector<LikelihoodMap>& maps, std::vector<double> weights) {
    require(!maps.empty(), "fuse_maps: no maps to fuse");  // likelihood.cpp:258
    const int w = maps[0].width, h = maps[0].height;
    for (const auto& m : maps) require(m.width == w && m.height == h, "fuse_maps: map dimensions differ");
    std::vector<std::unique_ptr<DevBuf>> dev;
    std::vector<const double*> ptrs;
    for (const auto& m : maps) {
        dev.push_back(upload_map(m));
        ptrs.push_back(dev.back()->as<double>());
    }
    const std::size_t n = std::size_t(w) * h;
    DevBuf out(n * 8);
    check(spct_cu_fuse_maps(ptrs.data(), int(ptrs.size()), weights.data(), int(weights.size()), std::int64_t(n),
                            out.as<double>(), nullptr));
    LikelihoodMap f;
    f.width = w;
    f.height = h;
    f.tag = "fused";
    f.values.resize(n);
    cuda(cudaMemcpy(f.values.data(), out.p, n * 8, cudaMemcpyDeviceToHost), "D2H");
    return f;
}

std::vector<Peak> find_peaks(const LikelihoodMap& map) {
    require(map.width > 0 && map.height > 0, "find_peaks: empty map");  // likelihood.cpp:286
    auto d = upload_map(map);
    std::size_t ws = 0;
    check(spct_cu_find_peaks_workspace(map.width, map.height, &ws));
    DevBuf work(ws);
    const std::int64_t cap = std::int64_t(map.width) * map.height / 4 + 2;
    DevBuf xs(cap * 4), ys(cap * 4), hs(cap * 8);
    std::int64_t count = 0;
    check(spct_cu_find_peaks(d->as<double>(), map.width, map.height, xs.as<std::int32_t>(), ys.as<std::int32_t>(),
                             hs.as<double>(), cap, &count, work.p, ws, nullptr));
    std::vector<std::int32_t> hx(count), hy(count);
    std::vector<double> hh(count);
    if (count) {
        cuda(cudaMemcpy(hx.data(), xs.p, count * 4, cudaMemcpyDeviceToHost), "D2H");
        cuda(cudaMemcpy(hy.data(), ys.p, count * 4, cudaMemcpyDeviceToHost), "D2H");
        cuda(cudaMemcpy(hh.data(), hs.p, count * 8, cudaMemcpyDeviceToHost), "D2H");
    }
    std::vector<Peak> peaks(count);
    for (std::int64_t i = 0; i < count; ++i) peaks[i] = Peak{hx[i], hy[i], hh[i], int(i) + 1};
    return peaks;
}

int score_map(const LikelihoodMap& map, const Rect& gt) {
    require(gt.w > 0 && gt.h > 0 && gt.inside(map.width, map.height),
            "score_map: ground truth rect must lie inside the map");  // likelihood.cpp:325-326
    auto d = upload_map(map);
    std::size_t ws = 0;
    check(spct_cu_find_peaks_workspace(map.width, map.height, &ws));
    DevBuf work(ws);
    std::int64_t rank = 0;
    check(spct_cu_score_map(d->as<double>(), map.width, map.height, gt.x, gt.y, gt.w, gt.h, &rank, work.p, ws, nullptr));
    return int(rank);
}

CamshiftResult camshift_refine(const LikelihoodMap& map, double cx, double cy, int win_w, int win_h, double delta,
                               int max_iter) {
    require(map.width > 0 && map.height > 0, "camshift_refine: empty map");  // tracker.cpp:79
    auto d = upload_map(map);
    const double start[2] = {cx, cy};
    double out[2] = {cx, cy};
    std::int32_t it = 0, zm = 0;
    check(spct_cu_camshift(d->as<double>(), map.width, map.height, start, 1, win_w, win_h, delta, max_iter, out, &it,
                           &zm, nullptr));
    return CamshiftResult{out[0], out[1], int(it), zm != 0};
}

LikelihoodMap likelihood_from_frame(const GrayImage& img, int bins, const std::vector<double>& th, int kw, int kh,
                                    double p, IntegralHistogramTensor* tensor_out, std::uint64_t memory_budget) {
    require(img.width > 0 && img.height > 0, "quantize: empty image");
    require(bins >= 1 && bins <= 65536, "quantize: bins must be in [1, 65536]");
    const MemoryEstimate est = estimate_memory(img.width, img.height, bins, 8);
    if (est.padded_bytes > memory_budget)
        throw contract_error("tensor of " + std::to_string(est.padded_bytes) + " bytes exceeds the memory budget of " +
                             std::to_string(memory_budget));
    check(spct_cu_hist_check(bins, img.width, img.height, th.data(), int(th.size()), kw, kh, p));
    auto src = std::make_unique<DevBuf>(img.data.size());
    DevBuf tm(th.size() * 8);
    upload(*src, img.data);
    upload(tm, th);
    spct_source s{};
    s.kind = SPCT_SRC_GRAY_U8;
    s.plane[0] = src->p;
    s.pitch = img.width;
    s.width = img.width;
    s.height = img.height;
    s.nbins = bins;
    s.lo = 0.0;
    s.hi = 256.0;
    auto dt = std::make_shared<detail::DeviceTensor>();
    spct_ih& d = dt->desc;
    std::uint64_t bytes = 0;
    check(spct_cu_ih_layout(img.width, img.height, bins, &d.row_pitch, &d.plane_pitch, &bytes));
    dt->mem = std::make_unique<DevBuf>(bytes);
    d.data = dt->mem->as<std::uint32_t>();
    d.bins = bins;
    d.nbins_total = bins;
    d.height = img.height;
    d.width = img.width;
    std::size_t ws = 0;
    check(spct_cu_ih_build_workspace(&s, 0, bins, &ws));
    DevBuf work(ws);
    DevBuf map(std::size_t(img.width) * img.height * 8);
    check(spct_cu_ih_build_match_map(&s, &d, tm.as<double>(), kw, kh, p, SPCT_METRIC_MINKOWSKI, map.as<double>(),
                                     work.p, ws, nullptr));
    LikelihoodMap out;
    out.width = img.width;
    out.height = img.height;
    out.tag = "hist-distance";
    out.values.resize(std::size_t(img.width) * img.height);
    cuda(cudaMemcpy(out.values.data(), map.p, out.values.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    if (tensor_out) {
        tensor_out->bins = bins;
        tensor_out->height = img.height;
        tensor_out->width = img.width;
        tensor_out->data.clear();
        dt->src = s;
        dt->src_mem = std::move(src);
        tensor_out->data.dev = std::move(dt);
    }
    return out;
}

}  // namespace spct
