// spct:: drop-in host layer (include/spct/spct.hpp) on top of the C-ABI.
//
// Each function re-runs the reference's contract checks with the same predicates
// and messages before touching the device, so reference expectations such as
// CHECK_THROWS_AS(..., contract_error) (test_integral.cpp:190-206) still hold.
// Device failures throw spct::device_error.
#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include <sys/mman.h>

#include <cuda_runtime.h>

#include "spct/motion.hpp"
#include "spct/spct.hpp"
#include "spct/swih.hpp"
#include "spct_cuda.h"

namespace spct_impl {
cudaError_t malloc_async(void** p, size_t bytes, cudaStream_t s);  // profile.cu
}

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

// RAII device buffer, stream-ordered on the legacy default stream that every call of this
// layer uses, from the library's retaining pool: a caller building one tensor per frame
// reuses the previous frame's memory instead of a cudaMalloc / cudaFree of gigabytes.
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t bytes) {
        if (bytes) cuda(spct_impl::malloc_async(&p, bytes, nullptr), "cudaMallocAsync");
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, nullptr);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Host <-> device copies of large pageable buffers (the reference API's std::vectors)
// through two pinned 8 MiB chunks: the DMA of one chunk overlaps the host memcpy of the
// other, instead of the driver's serial pageable staging.
constexpr std::size_t kChunk = std::size_t(8) << 20;

struct PinnedStage {
    std::mutex mu;
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    bool ready() {
        if (buf[0]) return true;
        for (int i = 0; i < 2; ++i) {
            if (cudaMallocHost(&buf[i], kChunk) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
        }
        return true;
    }
};

// memcpy between pinned staging and pageable memory on a few host threads (one thread
// moves ~10 GB/s; the PCIe link moves ~50).
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool* p = new CopyPool();  // never destroyed: workers outlive static teardown
        return *p;
    }
    // Fault in the pages of fresh (untouched) memory on every worker: the kernel's
    // first-touch cost (~1.4 us per 4 KiB page) dominates a large new result vector.
    void touch_par(void* dst, std::size_t n) { memcpy_par(dst, nullptr, n); }
    void memcpy_par(void* dst, const void* src, std::size_t n) {
        if (n < (std::size_t(1) << 20) || workers_.empty()) {
            copy_or_touch(dst, src, n);
            return;
        }
        const std::size_t parts = workers_.size() + 1, step = (n / parts + 63) / 64 * 64;
        {
            std::lock_guard<std::mutex> lock(mu_);
            for (std::size_t i = 1; i < parts; ++i) {
                const std::size_t off = std::min(n, i * step), len = std::min(n, off + step) - off;
                jobs_.push_back({static_cast<char*>(dst) + off, src ? static_cast<const char*>(src) + off : nullptr, len});
            }
            pending_ += parts - 1;
        }
        cv_.notify_all();
        copy_or_touch(dst, src, std::min(n, step));
        std::unique_lock<std::mutex> lock(mu_);
        done_cv_.wait(lock, [&] { return pending_ == 0; });
    }

private:
    struct Job {
        char* dst;
        const char* src;
        std::size_t len;
    };
    static void copy_or_touch(void* dst, const void* src, std::size_t n) {
        if (src) {
            std::memcpy(dst, src, n);
            return;
        }
        volatile char* d = static_cast<volatile char*>(dst);
        for (std::size_t o = 0; o < n; o += 4096) d[o] = 0;
    }
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        const unsigned n = hw >= 16 ? 7 : (hw >= 8 ? 3 : (hw >= 4 ? 1 : 0));
        for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { run(); }).detach();
    }
    void run() {
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> lock(mu_);
                cv_.wait(lock, [&] { return !jobs_.empty(); });
                j = jobs_.back();
                jobs_.pop_back();
            }
            copy_or_touch(j.dst, j.src, j.len);
            std::lock_guard<std::mutex> lock(mu_);
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<Job> jobs_;
    std::size_t pending_ = 0;
    std::vector<std::thread> workers_;
};

PinnedStage& stage() {
    static PinnedStage* s = new PinnedStage();  // never destroyed: outlives static tensors
    return *s;
}

void copy_d2h(void* dst, const void* src, std::size_t bytes) {
    PinnedStage& st = stage();
    std::unique_lock<std::mutex> lock(st.mu);
    if (bytes < 2 * kChunk || !st.ready()) {
        cuda(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "D2H");
        return;
    }
    const std::size_t n = (bytes + kChunk - 1) / kChunk;
    for (std::size_t i = 0; i <= n; ++i) {
        if (i < n) {
            const std::size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
            cuda(cudaMemcpyAsync(st.buf[i & 1], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost,
                                 nullptr),
                 "D2H");
            cuda(cudaEventRecord(st.ev[i & 1], nullptr), "event");
        }
        if (i > 0) {  // chunk i - 1 landed: move it while chunk i is in flight
            const std::size_t off = (i - 1) * kChunk, len = std::min(kChunk, bytes - off);
            cuda(cudaEventSynchronize(st.ev[(i - 1) & 1]), "D2H");
            CopyPool::get().memcpy_par(static_cast<char*>(dst) + off, st.buf[(i - 1) & 1], len);
        }
    }
}

// Ask for transparent huge pages on the 2 MiB-aligned interior of a fresh buffer (a 134 MB
// map is 64 faults instead of 32768 where THP is enabled; a no-op where it is not).
void advise_huge(void* p, std::size_t bytes) {
    constexpr std::uintptr_t kHuge = std::uintptr_t(2) << 20;
    const std::uintptr_t a = (reinterpret_cast<std::uintptr_t>(p) + kHuge - 1) & ~(kHuge - 1);
    const std::uintptr_t b = (reinterpret_cast<std::uintptr_t>(p) + bytes) & ~(kHuge - 1);
    if (b > a) madvise(reinterpret_cast<void*>(a), b - a, MADV_HUGEPAGE);
}

// Size a result vector of the reference API (LikelihoodMap::values) to n doubles.  A new
// large vector's pages are faulted in on the copy pool's threads before std::vector
// zero-fills them, instead of one page fault at a time inside that fill.
void resize_prefaulted(std::vector<double>& v, std::size_t n) {
    if (v.size() == n) return;
    if (v.capacity() < n && n * sizeof(double) >= (std::size_t(16) << 20)) {
        std::vector<double> fresh;
        fresh.reserve(n);
        advise_huge(fresh.data(), n * sizeof(double));
        CopyPool::get().touch_par(fresh.data(), n * sizeof(double));
        fresh.resize(n);
        v.swap(fresh);
        return;
    }
    v.resize(n);
}

// values := the n doubles at device `src` (reference API result vectors, by value): the
// vector is faulted in on the copy pool (huge pages where THP allows) before std::vector's
// value-initialising resize, then filled through the pinned stage.  (A whole-result pinned
// stage whose DMA overlapped the resize measured the same, 17 ms at 4096^2: the host-side
// zero-fill of the new vector is the floor of a by-value result.)
void fill_from_device(std::vector<double>& v, const void* src, std::size_t n) {
    resize_prefaulted(v, n);  // no-op when the caller's map already has this size
    copy_d2h(v.data(), src, n * sizeof(double));
}

void copy_h2d(void* dst, const void* src, std::size_t bytes) {
    PinnedStage& st = stage();
    std::unique_lock<std::mutex> lock(st.mu);
    if (bytes < 2 * kChunk || !st.ready()) {
        cuda(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "H2D");
        return;
    }
    const std::size_t n = (bytes + kChunk - 1) / kChunk;
    for (std::size_t i = 0; i < n; ++i) {
        const std::size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        if (i >= 2) cuda(cudaEventSynchronize(st.ev[i & 1]), "H2D");  // chunk i - 2 has left this buffer
        CopyPool::get().memcpy_par(st.buf[i & 1], static_cast<const char*>(src) + off, len);
        cuda(cudaMemcpyAsync(static_cast<char*>(dst) + off, st.buf[i & 1], len, cudaMemcpyHostToDevice, nullptr), "H2D");
        cuda(cudaEventRecord(st.ev[i & 1], nullptr), "event");
    }
    cuda(cudaEventSynchronize(st.ev[(n - 1) & 1]), "H2D");
}

template <class T>
void upload(DevBuf& d, const std::vector<T>& v) {
    copy_h2d(d.p, v.data(), v.size() * sizeof(T));
}

}  // namespace

namespace detail {

struct DeviceTensor {
    spct_ih desc{};
    std::unique_ptr<DevBuf> mem;
    // Weighted tensors (build_weighted_tensor, SWIH): uint64 cells in `wdesc` instead.
    bool weighted = false;
    spct_wih wdesc{};
    // The frame the tensor was built from (device copy): hist_distance_map recomputes
    // window counts from it (1 B/px) instead of re-reading b*H*W*4 tensor bytes.
    spct_source src{};
    std::unique_ptr<DevBuf> src_mem;
    // region queries: a reusable device buffer, and a count that switches small tensors to
    // answering from the host mirror (the reference's own arithmetic) after a few queries
    std::unique_ptr<DevBuf> qbuf;
    int queries = 0;
};

std::size_t HostMirror::size() const {
    if (!dev) return host_.size();
    if (dev->weighted)
        return std::size_t(dev->wdesc.bins) * std::size_t(dev->wdesc.height + 1) * std::size_t(dev->wdesc.width + 1);
    return std::size_t(dev->desc.bins) * std::size_t(dev->desc.height + 1) * std::size_t(dev->desc.width + 1);
}

void HostMirror::fill() const {
    if (valid_ || !dev) return;
    if (dev->weighted) {
        const spct_wih& w = dev->wdesc;
        const std::size_t plane = std::size_t(w.height + 1) * (w.width + 1);
        host_.resize(plane * w.bins);
        const std::size_t per = std::max<std::size_t>(1, (std::size_t(256) << 20) / (plane * 8));
        DevBuf stage(std::min<std::size_t>(per, w.bins) * plane * 8);
        for (int k0 = 0; k0 < w.bins; k0 += int(per)) {
            const int k1 = std::min<int>(w.bins, k0 + int(per));
            check(spct_cu_wih_export_u64(&w, k0, k1, stage.as<std::uint64_t>(), nullptr));
            copy_d2h(host_.data() + std::size_t(k0) * plane, stage.p, std::size_t(k1 - k0) * plane * 8);
        }
        valid_ = true;
        return;
    }
    const spct_ih& d = dev->desc;
    const std::size_t plane = std::size_t(d.height + 1) * (d.width + 1);
    host_.resize(plane * d.bins);
    // Export a few planes at a time through a bounded device staging buffer.
    const std::size_t per = std::max<std::size_t>(1, (std::size_t(256) << 20) / (plane * 8));
    DevBuf stage(std::min<std::size_t>(per, d.bins) * plane * 8);
    for (int k0 = 0; k0 < d.bins; k0 += int(per)) {
        const int k1 = std::min<int>(d.bins, k0 + int(per));
        check(spct_cu_ih_export_u64(&d, k0, k1, stage.as<std::uint64_t>(), nullptr));
        copy_d2h(host_.data() + std::size_t(k0) * plane, stage.p, std::size_t(k1 - k0) * plane * 8);
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

void HostMirror::adopt(std::vector<std::uint64_t>&& host) {
    host_ = std::move(host);
    valid_ = true;
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
    copy_h2d(p, img.r.data(), n);
    copy_h2d(p + n, img.g.data(), n);
    copy_h2d(p + 2 * n, img.b.data(), n);
    check(spct_cu_to_grayscale(p, p + n, p + 2 * n, std::int64_t(n), p + 3 * n, nullptr));
    copy_d2h(out.data.data(), p + 3 * n, n);
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
    copy_d2h(out.data.data(), dst.p, n * 2);
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

// build_tensor's checks (integral.cpp:510-514, 330-343) in the reference's order:
// validate_binmap (empty, bins, then the bin range — on the uploaded copy, one device
// max instead of a host pass over the pixels), then tile, threads and the budget.
// Returns the uploaded BinMap.
std::unique_ptr<DevBuf> validated_upload(const BinMap& bm, const ScanSchedule& schedule, std::uint64_t budget) {
    require(bm.width > 0 && bm.height > 0, "build: empty bin map");
    require(bm.bins >= 1, "build: bins must be >= 1");
    require(bm.data.size() == std::size_t(bm.width) * bm.height, "build: bin map size mismatch");
    auto d = std::make_unique<DevBuf>(bm.data.size() * 2);
    upload(*d, bm.data);
    int mx = 0;
    check(spct_cu_binmap_max(d->as<std::uint16_t>(), bm.width, bm.width, bm.height, &mx, nullptr));
    require(mx < bm.bins, "build: bin index out of range");
    require(schedule.tile >= 2 && schedule.tile <= 4096, "build: tile must be in [2, 4096]");
    require(schedule.threads >= 1 && schedule.threads <= 64, "build: threads must be in [1, 64]");
    const MemoryEstimate est = estimate_memory(bm.width, bm.height, bm.bins, 8);
    if (est.padded_bytes > budget)
        throw contract_error("tensor of " + std::to_string(est.padded_bytes) + " bytes exceeds the memory budget of " +
                             std::to_string(budget));
    return d;
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
    auto src = validated_upload(bins, schedule, memory_budget);
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
    require(!t.data.dev->weighted, "operation needs a count tensor (this one is weighted)");
    return t.data.dev->desc;
}
}  // namespace

namespace {
// Mirrors of at most this many cells (256 MiB of uint64) are filled once the device round
// trips (~20 us each) would have cost about as much as the fill (~64 KiB of mirror per
// query); later queries read the host copy like the reference does.
constexpr std::size_t kMirrorCells = std::size_t(32) << 20;
int queries_before_mirror(std::size_t cells) { return static_cast<int>(std::max<std::size_t>(16, cells * 8 >> 16)); }

std::vector<std::uint64_t> region_from_mirror(const IntegralHistogramTensor& t, const Rect& r) {
    std::vector<std::uint64_t> out(t.bins);
    const std::uint64_t* d = t.data.data();
    const std::size_t ps = t.plane_stride(), rs = t.row_stride();
    const std::size_t y1 = r.y, y2 = std::size_t(r.y) + r.h, x1 = r.x, x2 = std::size_t(r.x) + r.w;
    for (int k = 0; k < t.bins; ++k) {  // integral.cpp:569-577, uint64 wrap arithmetic
        const std::uint64_t* pl = d + std::size_t(k) * ps;
        out[k] = pl[y2 * rs + x2] - pl[y1 * rs + x2] - pl[y2 * rs + x1] + pl[y1 * rs + x1];
    }
    return out;
}
}  // namespace

std::vector<std::uint64_t> region_histogram(const IntegralHistogramTensor& t, const Rect& r) {
    require(r.w >= 0 && r.h >= 0, "region_histogram: negative extent");       // integral.cpp:562
    require(r.inside(t.width, t.height), "region_histogram: rect outside image");  // :563
    detail::DeviceTensor* dt = t.data.dev.get();
    if (!dt || t.data.mirrored()) return region_from_mirror(t, r);
    if (t.data.size() <= kMirrorCells && ++dt->queries > queries_before_mirror(t.data.size()))
        return region_from_mirror(t, r);
    const std::size_t cell = dt->weighted ? 8 : 4;
    if (!dt->qbuf) dt->qbuf = std::make_unique<DevBuf>(16 + std::size_t(t.bins) * 8);
    auto* rect = dt->qbuf->as<std::int32_t>();
    void* out = dt->qbuf->as<char>() + 16;
    const std::int32_t rr[4] = {r.x, r.y, r.w, r.h};
    cuda(cudaMemcpy(rect, rr, 16, cudaMemcpyHostToDevice), "H2D");
    if (dt->weighted)
        check(spct_cu_wih_region_counts(&dt->wdesc, rect, 1, static_cast<std::uint64_t*>(out), nullptr));
    else
        check(spct_cu_region_counts(&desc_of(t), rect, 1, static_cast<std::uint32_t*>(out), nullptr));
    std::vector<std::uint64_t> h(t.bins);
    if (cell == 8) {
        cuda(cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    } else {
        std::vector<std::uint32_t> h32(t.bins);
        cuda(cudaMemcpy(h32.data(), out, h32.size() * 4, cudaMemcpyDeviceToHost), "D2H");
        std::copy(h32.begin(), h32.end(), h.begin());
    }
    return h;
}

std::uint64_t region_count(const IntegralHistogramTensor& t, int bin, const Rect& r) {
    require(bin >= 0 && bin < t.bins, "region_count: bin out of range");     // integral.cpp:570
    require(r.inside(t.width, t.height), "region_count: rect outside image");  // :571
    return region_histogram(t, r)[bin];
}

// IHT1 wire format (integral.cpp:619-659): streamed from / to HBM by the C-ABI.
void dump_tensor(const IntegralHistogramTensor& t, const std::string& path) {
    if (t.data.dev && t.data.dev->weighted) {  // uint64 cells: the file is the host mirror itself
        std::FILE* f = std::fopen(path.c_str(), "wb");
        if (!f) throw io_error("cannot write tensor: " + path);  // integral.cpp:621
        unsigned char hdr[20] = {'I', 'H', 'T', '1'};
        const std::uint32_t v[4] = {std::uint32_t(t.bins), std::uint32_t(t.height), std::uint32_t(t.width), 8u};
        for (int i = 0; i < 4; ++i)
            for (int b = 0; b < 4; ++b) hdr[4 + 4 * i + b] = static_cast<unsigned char>(v[i] >> (8 * b));
        bool ok = std::fwrite(hdr, 1, 20, f) == 20;
        ok = ok && std::fwrite(t.data.data(), 8, t.data.size(), f) == t.data.size();
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) throw io_error("write failed: " + path);  // :631
        return;
    }
    check(spct_cu_ih_dump(&desc_of(t), path.c_str(), 8, nullptr));
}

namespace {
// A file whose cells do not fit the uint32 device tensor (a dumped weighted tensor: 16.16
// sums) loads, like the reference's load_tensor, as uint64 cells: the padded payload is
// the host mirror itself, and a weighted device tensor is filled from it plane by plane.
IntegralHistogramTensor load_tensor_u64(const std::string& path, int bins, int h, int w) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw io_error("cannot open tensor: " + path);  // integral.cpp:636
    const std::size_t cells = std::size_t(bins) * (h + 1) * (w + 1);
    std::vector<std::uint64_t> host(cells);
    const bool ok = std::fseek(f, 20, SEEK_SET) == 0 && std::fread(host.data(), 8, cells, f) == cells;
    std::fclose(f);
    if (!ok) throw io_error("truncated tensor payload: " + path);  // :655
    auto dt = std::make_shared<detail::DeviceTensor>();
    dt->weighted = true;
    spct_wih& d = dt->wdesc;
    std::uint64_t bytes = 0;
    check(spct_cu_wih_layout(w, h, bins, &d.row_pitch, &d.plane_pitch, &bytes));
    dt->mem = std::make_unique<DevBuf>(bytes);
    d.data = dt->mem->as<std::uint64_t>();
    d.bins = bins;
    d.height = h;
    d.width = w;
    const std::size_t ps = std::size_t(h + 1) * (w + 1);
    for (int k = 0; k < bins; ++k)  // cells (y, x) >= (1, 1) of plane k, unpadded and pitched
        cuda(cudaMemcpy2D(d.data + std::size_t(k) * d.plane_pitch, d.row_pitch * 8, host.data() + k * ps + (w + 1) + 1,
                          (w + 1) * 8, std::size_t(w) * 8, h, cudaMemcpyHostToDevice),
             "H2D");
    IntegralHistogramTensor t;
    t.bins = bins;
    t.height = h;
    t.width = w;
    t.data.dev = std::move(dt);
    t.data.adopt(std::move(host));
    return t;
}
}  // namespace

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
    const spct_status st = spct_cu_ih_load(path.c_str(), &d, nullptr);
    if (st == SPCT_ERR_IO && elem == 8 &&
        std::string(spct_cu_last_error()).rfind("tensor value exceeds the uint32 device cell", 0) == 0)
        return load_tensor_u64(path, bins, h, w);
    check(st);
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

void hist_match_map_into(const IntegralHistogramTensor& t, const std::vector<double>& th, int kw, int kh,
                         HistMetric metric, double p, LikelihoodMap& out) {
    check(spct_cu_hist_check(t.bins, t.width, t.height, th.data(), int(th.size()), kw, kh, p));
    const spct_ih& d = desc_of(t);
    DevBuf tm(th.size() * 8), map(std::size_t(t.width) * t.height * 8);
    upload(tm, th);
    const detail::DeviceTensor& dt = *t.data.dev;
    if (dt.src_mem && !exact_maps() && spct_cu_fused_window_ok(kw, kh)) {
        // recompute the window counts from the source in the fused sweep (no tensor re-read)
        spct_ih nodata = d;
        nodata.data = nullptr;
        std::size_t ws = 0;
        check(spct_cu_ih_build_workspace(&dt.src, 0, d.bins, &ws));
        DevBuf work(ws);
        check(spct_cu_ih_build_match_map(&dt.src, &nodata, tm.as<double>(), kw, kh, p, int(metric), map.as<double>(),
                                         work.p, ws, nullptr));
    } else {
        // a stored tensor: read once (bins recovered on the device), or the reference's
        // operation order in exact mode
        check((exact_maps() ? spct_cu_hist_match_exact : spct_cu_hist_match)(&d, tm.as<double>(), kw, kh, p,
                                                                           int(metric), map.as<double>(), nullptr));
    }
    out.width = t.width;
    out.height = t.height;
    out.tag = metric == HistMetric::Minkowski ? "hist-distance" : "hist-match";
    fill_from_device(out.values, map.p, std::size_t(t.width) * t.height);  // reuses the caller's map storage
}

LikelihoodMap hist_match_map(const IntegralHistogramTensor& t, const std::vector<double>& th, int kw, int kh,
                             HistMetric metric, double p) {
    LikelihoodMap out;
    hist_match_map_into(t, th, kw, kh, metric, p, out);
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
    fill_from_device(f.values, out.p, n);
    return f;
}

std::vector<Peak> find_peaks(const LikelihoodMap& map) {
    require(map.width > 0 && map.height > 0, "find_peaks: empty map");  // likelihood.cpp:286
    auto d = upload_map(map);
    std::size_t ws = 0;
    check(spct_cu_find_peaks_workspace(map.width, map.height, &ws));
    DevBuf work(ws);
    std::int64_t cap = std::int64_t(map.width) * map.height / 4 + 2;  // strict maxima
    std::int64_t count = 0;
    std::unique_ptr<DevBuf> xs, ys, hs;
    for (;;) {  // NaN cells are peaks too (likelihood.cpp:316): then size for the real count
        xs = std::make_unique<DevBuf>(cap * 4);
        ys = std::make_unique<DevBuf>(cap * 4);
        hs = std::make_unique<DevBuf>(cap * 8);
        check(spct_cu_find_peaks(d->as<double>(), map.width, map.height, xs->as<std::int32_t>(),
                                 ys->as<std::int32_t>(), hs->as<double>(), cap, &count, work.p, ws, nullptr));
        if (count <= cap) break;
        cap = count;
    }
    std::vector<std::int32_t> hx(count), hy(count);
    std::vector<double> hh(count);
    if (count) {
        cuda(cudaMemcpy(hx.data(), xs->p, count * 4, cudaMemcpyDeviceToHost), "D2H");
        cuda(cudaMemcpy(hy.data(), ys->p, count * 4, cudaMemcpyDeviceToHost), "D2H");
        cuda(cudaMemcpy(hh.data(), hs->p, count * 8, cudaMemcpyDeviceToHost), "D2H");
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
    fill_from_device(out.values, map.p, std::size_t(img.width) * img.height);
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

// ---------------------------------------------------------------- weighted tensors (integral.hpp:102-104)
namespace {

// A device weighted tensor over a device bin map: explicit weights (dev uint64, 16.16) or
// the quadrant ramp field `dir` of a kw x kh kernel (spct_cu_wih_build).
IntegralHistogramTensor make_weighted(const std::uint16_t* dbins, int w, int h, int bins, const std::uint64_t* dweights,
                                      int dir, int kw, int kh) {
    auto dt = std::make_shared<detail::DeviceTensor>();
    dt->weighted = true;
    spct_wih& d = dt->wdesc;
    std::uint64_t bytes = 0;
    check(spct_cu_wih_layout(w, h, bins, &d.row_pitch, &d.plane_pitch, &bytes));
    dt->mem = std::make_unique<DevBuf>(bytes);
    d.data = dt->mem->as<std::uint64_t>();
    d.bins = bins;
    d.height = h;
    d.width = w;
    check(spct_cu_wih_build(dbins, w, dweights, dir, kw, kh, &d, nullptr));
    cuda(cudaDeviceSynchronize(), "build_weighted_tensor");
    IntegralHistogramTensor t;
    t.bins = bins;
    t.height = h;
    t.width = w;
    t.data.dev = std::move(dt);
    return t;
}

const spct_wih& wdesc_of(const IntegralHistogramTensor& t) {
    require(t.data.dev != nullptr && t.data.dev->weighted, "swlh_query: quadrant tensors must be weighted tensors");
    return t.data.dev->wdesc;
}

}  // namespace

IntegralHistogramTensor build_weighted_tensor(const BinMap& bins, const std::vector<std::uint64_t>& weights,
                                              const ScanSchedule& schedule, std::uint64_t memory_budget) {
    require(weights.size() == bins.data.size(), "build_weighted_tensor: weight size mismatch");  // integral.cpp:557
    auto db = validated_upload(bins, schedule, memory_budget);
    DevBuf dw(weights.size() * 8);
    upload(dw, weights);
    return make_weighted(db->as<std::uint16_t>(), bins.width, bins.height, bins.bins, dw.as<std::uint64_t>(), -1, 1, 1);
}

// ---------------------------------------------------------------- SWIH (swih.hpp)
const char* to_string(Quadrant q) {
    static const char* names[] = {"NW", "NE", "SW", "SE"};
    const int i = static_cast<int>(q);
    return (i >= 0 && i < 4) ? names[i] : "?";
}

KernelExtents kernel_extents(const KernelSpec& spec) {  // swih.cpp:19-27
    require(spec.kw >= 1 && spec.kh >= 1, "kernel extents must be >= 1");
    const int sxl = spec.kw / 2, syt = spec.kh / 2;
    return KernelExtents{sxl, spec.kw - sxl, syt, spec.kh - syt, sxl + syt + 1};
}

std::uint64_t quantize_weight(double w) {  // swih.cpp:29-32
    require(std::isfinite(w) && w >= 0.0, "weights must be finite and nonnegative");
    return static_cast<std::uint64_t>(std::llround(w * kWeightScale));
}

namespace {
// Slope 1 on an axis the kernel spans with >= 3 cells, else 0 (swih.cpp:40-43).
int ramp_slope(int k) { return k >= 3 ? 1 : 0; }
}  // namespace

std::array<WeightField, 4> quadrant_weight_fields(int img_w, int img_h, const KernelSpec& spec) {
    require(img_w > 0 && img_h > 0, "quadrant_weight_fields: empty image");  // swih.cpp:86
    kernel_extents(spec);
    const int sx = ramp_slope(spec.kw), sy = ramp_slope(spec.kh);
    std::array<WeightField, 4> out;
    for (int d = 0; d < 4; ++d) {
        WeightField& f = out[d];
        f.width = img_w;
        f.height = img_h;
        f.dir = static_cast<Quadrant>(d);
        f.w.resize(std::size_t(img_w) * img_h);
        // the field falls by one per step away from its anchor corner (swih.cpp:45-53):
        // NW / SW count x from the left, NE / SE from the right; NW / NE y from the top
        const bool from_left = f.dir == Quadrant::NW || f.dir == Quadrant::SW;
        const bool from_top = f.dir == Quadrant::NW || f.dir == Quadrant::NE;
        for (int y = 0; y < img_h; ++y)
            for (int x = 0; x < img_w; ++x) {
                const int ax = from_left ? x : img_w - 1 - x, ay = from_top ? y : img_h - 1 - y;
                f.w[std::size_t(y) * img_w + x] = 1.0 + sx * ax + sy * ay;
            }
    }
    return out;
}

IntegralHistogramTensor build_weighted_ih(const BinMap& bins, const WeightField& field, const ScanSchedule& schedule) {
    require(field.width == bins.width && field.height == bins.height,
            "build_weighted_ih: field/bin map size mismatch");  // swih.cpp:104-105
    std::vector<std::uint64_t> wq(field.w.size());
    std::transform(field.w.begin(), field.w.end(), wq.begin(), quantize_weight);
    return build_weighted_tensor(bins, wq, schedule);
}

// The four ramp tensors are built on the device straight from the bin map (the field is
// generated in the build kernel), one upload of the map for all four.
WeightedQuadrantSet build_quadrant_set(const BinMap& bins, const KernelSpec& spec, const ScanSchedule& schedule) {
    require(bins.width > 0 && bins.height > 0, "quadrant_weight_fields: empty image");
    kernel_extents(spec);
    auto db = validated_upload(bins, schedule, kDefaultMemoryBudget);
    WeightedQuadrantSet set;
    set.kernel = spec;
    set.sx = ramp_slope(spec.kw);
    set.sy = ramp_slope(spec.kh);
    set.pair_sum = 2 + std::int64_t(set.sx) * (bins.width - 1) + std::int64_t(set.sy) * (bins.height - 1);
    for (int d = 0; d < 4; ++d)
        set.tensors[d] =
            make_weighted(db->as<std::uint16_t>(), bins.width, bins.height, bins.bins, nullptr, d, spec.kw, spec.kh);
    return set;
}

std::vector<std::int64_t> swlh_query_fixed(const WeightedQuadrantSet& set, int cx, int cy, const KernelSpec& spec) {
    require(spec == set.kernel, "swlh_query: kernel spec differs from the built set");  // swih.cpp:130
    kernel_extents(spec);
    const spct_wih descs[4] = {wdesc_of(set.tensors[0]), wdesc_of(set.tensors[1]), wdesc_of(set.tensors[2]),
                               wdesc_of(set.tensors[3])};
    const std::int32_t c[2] = {cx, cy};
    const int bins = set.tensors[0].bins;
    DevBuf out(std::size_t(bins) * 8);
    check(spct_cu_swlh_query(descs, spec.kw, spec.kh, c, 1, out.as<std::int64_t>(), nullptr));
    std::vector<std::int64_t> h(bins);
    cuda(cudaMemcpy(h.data(), out.p, h.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    return h;
}

namespace {
// Unit-mass normalisation with the reference's extended-precision total (swih.cpp:182-192).
std::vector<double> unit_mass(const std::vector<std::int64_t>& fx) {
    long double total = 0;
    for (std::int64_t v : fx) total += v;
    std::vector<double> out(fx.size(), 0.0);
    if (total > 0)
        for (std::size_t k = 0; k < fx.size(); ++k) out[k] = static_cast<double>(fx[k] / total);
    return out;
}
}  // namespace

std::vector<double> swlh_query(const WeightedQuadrantSet& set, int cx, int cy, const KernelSpec& spec) {
    return unit_mass(swlh_query_fixed(set, cx, cy, spec));
}

std::vector<std::int64_t> brute_force_swlh_fixed(const BinMap& bins, int cx, int cy, const KernelSpec& spec) {
    kernel_extents(spec);
    require(bins.data.empty() || *std::max_element(bins.data.begin(), bins.data.end()) < bins.bins,
            "build: bin index out of range");
    DevBuf db(bins.data.size() * 2), out(std::size_t(std::max(bins.bins, 1)) * 8);
    upload(db, bins.data);
    const std::int32_t c[2] = {cx, cy};
    check(spct_cu_swlh_brute(db.as<std::uint16_t>(), bins.width, bins.width, bins.height, bins.bins, spec.kw, spec.kh, c,
                             1, out.as<std::int64_t>(), nullptr));
    std::vector<std::int64_t> h(bins.bins);
    cuda(cudaMemcpy(h.data(), out.p, h.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    return h;
}

std::vector<double> brute_force_swlh(const BinMap& bins, int cx, int cy, const KernelSpec& spec) {
    return unit_mass(brute_force_swlh_fixed(bins, cx, cy, spec));
}

// Nested-rectangle ("wedding cake") approximation over a plain tensor (swih.cpp:200-262):
// ring l between rect l and rect l+1 gets the exact mean pyramid weight over the ring,
// rounded half up in 16.16.  All rect histograms come from one device query.
std::vector<double> wedding_cake_swlh(const IntegralHistogramTensor& plain, int cx, int cy, const KernelSpec& spec,
                                      int layers) {
    require(layers >= 1, "wedding_cake_swlh: layers must be >= 1");
    const KernelExtents e = kernel_extents(spec);
    require(cx - e.sxl >= 0 && cy - e.syt >= 0 && cx + e.sxr <= plain.width && cy + e.syb <= plain.height,
            "kernel window must lie inside the image");
    struct Ext {
        std::int64_t xl, xr, yt, yb;
        std::int64_t area() const { return (xl + xr) * (yt + yb); }
        // sum over dx in [-xl, xr), dy in [-yt, yb) of (c - |dx| - |dy|)
        std::int64_t mass(std::int64_t c) const {
            const std::int64_t nx = xl + xr, ny = yt + yb;
            const std::int64_t ax = xl * (xl + 1) / 2 + (xr - 1) * xr / 2, ay = yt * (yt + 1) / 2 + (yb - 1) * yb / 2;
            return c * nx * ny - ax * ny - ay * nx;
        }
    };
    std::vector<Ext> ext(layers + 1, Ext{0, 0, 0, 0});  // ext[layers]: the empty rect
    std::vector<std::int32_t> rects;
    for (int l = 0; l < layers; ++l) {
        const double f = static_cast<double>(layers - l) / layers;
        ext[l] = Ext{std::lround(e.sxl * f), std::max<long>(1, std::lround(e.sxr * f)), std::lround(e.syt * f),
                     std::max<long>(1, std::lround(e.syb * f))};
        rects.insert(rects.end(), {std::int32_t(cx - ext[l].xl), std::int32_t(cy - ext[l].yt),
                                   std::int32_t(ext[l].xl + ext[l].xr), std::int32_t(ext[l].yt + ext[l].yb)});
    }
    const spct_ih& d = desc_of(plain);
    const int bins = plain.bins;
    DevBuf drect(rects.size() * 4), dout(std::size_t(layers) * bins * 4);
    upload(drect, rects);
    check(spct_cu_region_counts(&d, drect.as<std::int32_t>(), layers, dout.as<std::uint32_t>(), nullptr));
    std::vector<std::uint32_t> hist(std::size_t(layers) * bins);
    cuda(cudaMemcpy(hist.data(), dout.p, hist.size() * 4, cudaMemcpyDeviceToHost), "D2H");
    std::vector<std::int64_t> acc(bins, 0);
    for (int l = 0; l < layers; ++l) {
        const std::int64_t d_area = ext[l].area() - ext[l + 1].area();
        if (d_area <= 0) continue;
        const std::int64_t d_mass = ext[l].mass(e.c) - ext[l + 1].mass(e.c);
        const std::int64_t wfix = (2 * d_mass * kWeightScale + d_area) / (2 * d_area);
        for (int k = 0; k < bins; ++k) {
            const std::uint64_t outer = hist[std::size_t(l) * bins + k];
            const std::uint64_t inner = l + 1 < layers ? hist[std::size_t(l + 1) * bins + k] : 0;
            acc[k] += static_cast<std::int64_t>(outer - inner) * wfix;
        }
    }
    return unit_mass(acc);
}

double histogram_mse(const std::vector<double>& a, const std::vector<double>& b) {
    require(a.size() == b.size() && !a.empty(), "histogram_mse: size mismatch");
    double acc = 0;
    for (std::size_t i = 0; i < a.size(); ++i) acc += (a[i] - b[i]) * (a[i] - b[i]);
    return acc / static_cast<double>(a.size());
}

// ---------------------------------------------------------------- joint-IH median (motion.hpp)
void FrameWindow::validate() const {  // motion.cpp:12-19
    require(!frames.empty(), "FrameWindow: empty window");
    require(frames.size() % 2 == 1, "FrameWindow: window length must be odd");
    const int w = frames[0].width, h = frames[0].height;
    require(w > 0 && h > 0, "FrameWindow: empty frames");
    for (const auto& f : frames) require(f.width == w && f.height == h, "FrameWindow: frame dimensions differ");
}

struct MedianBackgroundIH::State {
    spct_ih joint{};
    std::unique_ptr<DevBuf> mem, frame, frame_old, ws, slide_ws;
    std::size_t ws_bytes = 0, slide_ws_bytes = 0;
};

MedianBackgroundIH::~MedianBackgroundIH() = default;
MedianBackgroundIH::MedianBackgroundIH(MedianBackgroundIH&&) noexcept = default;
MedianBackgroundIH& MedianBackgroundIH::operator=(MedianBackgroundIH&&) noexcept = default;

MedianBackgroundIH::MedianBackgroundIH(const FrameWindow& window, int bins, int m, int n)
    : bins_(bins), m_(m), n_(n) {
    window.validate();
    require(bins >= 1 && bins <= 256, "median_background_ih: bins must be in [1,256]");  // motion.cpp:38
    require(m >= 1 && n >= 1 && m % 2 == 1 && n % 2 == 1, "median_background_ih: kernel sides must be odd and positive");
    width_ = window.frames[0].width;
    height_ = window.frames[0].height;
    require(m <= width_ && n <= height_, "median_background_ih: kernel exceeds image");
    // the joint tensor is uint32: exact while every window count fits
    require(std::uint64_t(window.frames.size()) * width_ * height_ < (std::uint64_t(1) << 32),
            "median_background_ih: frames * H * W must be < 2^32");
    st_ = std::make_unique<State>();
    spct_ih& J = st_->joint;
    std::uint64_t bytes = 0;
    check(spct_cu_ih_layout(width_, height_, bins_, &J.row_pitch, &J.plane_pitch, &bytes));
    st_->mem = std::make_unique<DevBuf>(bytes);
    cuda(cudaMemset(st_->mem->p, 0, bytes), "memset");
    J.data = st_->mem->as<std::uint32_t>();
    J.bins = bins_;
    J.bin0 = 0;
    J.nbins_total = bins_;
    J.height = height_;
    J.width = width_;
    st_->frame = std::make_unique<DevBuf>(std::size_t(width_) * height_ * 2);
    spct_source s{};
    s.kind = SPCT_SRC_BINS_U16;
    s.width = width_;
    s.height = height_;
    s.nbins = bins_;
    check(spct_cu_ih_build_workspace(&s, 0, bins_, &st_->ws_bytes));
    st_->ws = std::make_unique<DevBuf>(st_->ws_bytes);
    st_->frame_old = std::make_unique<DevBuf>(std::size_t(width_) * height_ * 2);
    check(spct_cu_ih_slide_workspace(width_, height_, bins_, &st_->slide_ws_bytes));
    st_->slide_ws = std::make_unique<DevBuf>(st_->slide_ws_bytes);
    for (const auto& f : window.frames) {
        add_frame(f, +1);
        frames_.push_back(f);
    }
}

void MedianBackgroundIH::add_frame(const GrayImage& f, int sign) {  // motion.cpp:51-60
    for (auto v : f.data) require(v < bins_, "median_background_ih: frame value exceeds bin count");
    const std::vector<std::uint16_t> b(f.data.begin(), f.data.end());  // the frame's values are its bins
    upload(*st_->frame, b);
    spct_source s{};
    s.kind = SPCT_SRC_BINS_U16;
    s.plane[0] = st_->frame->p;
    s.pitch = width_;
    s.width = width_;
    s.height = height_;
    s.nbins = bins_;
    check(spct_cu_ih_accumulate(&s, &st_->joint, sign, st_->ws->p, st_->ws_bytes, nullptr));
    cuda(cudaDeviceSynchronize(), "median_background_ih");  // the staging buffer is reused
}

void MedianBackgroundIH::slide(const GrayImage& next) {  // motion.cpp:62-69
    require(next.width == width_ && next.height == height_, "median_background_ih: slide frame dimensions differ");
    for (auto v : next.data) require(v < bins_, "median_background_ih: frame value exceeds bin count");
    // both frames' bins on the device, then J += IH(next) - IH(front) in one pass
    // (the outgoing frame passed the same check when it entered)
    upload(*st_->frame, std::vector<std::uint16_t>(next.data.begin(), next.data.end()));
    const GrayImage& old = frames_.front();
    upload(*st_->frame_old, std::vector<std::uint16_t>(old.data.begin(), old.data.end()));
    spct_source sn{};
    sn.kind = SPCT_SRC_BINS_U16;
    sn.plane[0] = st_->frame->p;
    sn.pitch = width_;
    sn.width = width_;
    sn.height = height_;
    sn.nbins = bins_;
    spct_source so = sn;
    so.plane[0] = st_->frame_old->p;
    check(spct_cu_ih_slide(&sn, &so, &st_->joint, st_->slide_ws->p, st_->slide_ws_bytes, nullptr));
    cuda(cudaDeviceSynchronize(), "median_background_ih");  // the staging buffers are reused
    frames_.pop_front();
    frames_.push_back(next);
}

GrayImage MedianBackgroundIH::background() const {  // motion.cpp:71-99
    DevBuf out(std::size_t(width_) * height_);
    check(spct_cu_median_background(&st_->joint, static_cast<int>(frames_.size()), m_, n_, out.as<std::uint8_t>(),
                                    width_, nullptr));
    GrayImage g(width_, height_);
    cuda(cudaMemcpy(g.data.data(), out.p, g.data.size(), cudaMemcpyDeviceToHost), "D2H");
    return g;
}

GrayImage median_background_ih(const FrameWindow& window, int bins, int m, int n) {
    return MedianBackgroundIH(window, bins, m, n).background();
}

GrayImage median_background_sort(const FrameWindow& window) {  // motion.cpp:105-118
    window.validate();
    const int w = window.frames[0].width, h = window.frames[0].height;
    const std::size_t px = std::size_t(w) * h, nf = window.frames.size();
    DevBuf stack(px * (nf + 1));
    std::vector<const std::uint8_t*> ptrs(nf);
    for (std::size_t f = 0; f < nf; ++f) {
        ptrs[f] = stack.as<std::uint8_t>() + f * px;
        cuda(cudaMemcpy(stack.as<std::uint8_t>() + f * px, window.frames[f].data.data(), px, cudaMemcpyHostToDevice),
             "H2D");
    }
    std::uint8_t* out = stack.as<std::uint8_t>() + nf * px;
    check(spct_cu_median_sort(ptrs.data(), static_cast<int>(nf), w, h, w, out, w, nullptr));
    GrayImage g(w, h);
    cuda(cudaMemcpy(g.data.data(), out, px, cudaMemcpyDeviceToHost), "D2H");
    return g;
}

}  // namespace spct
