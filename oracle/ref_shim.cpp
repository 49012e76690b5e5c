// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (the sources under
// /root/reference/proj/src are compiled in place by oracle/Makefile into
// oracle/_ref/libspct_ref.so). Tests, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load it with ctypes to (a) pin the C
// restatement in oracle/spct_oracle.c and (b) time the reference CPU path.
//
// Every entry point returns 0 on success, 2 on spct::contract_error,
// 3 on spct::io_error, 1 on anything else — the CLI's exit-code mapping
// (reference proj/tools/spct_main.cpp:688-702).

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <cmath>

#include "spct/error.hpp"
#include "spct/features.hpp"
#include "spct/swih.hpp"
#include "spct/motion.hpp"
#include "spct/imagecore.hpp"
#include "spct/integral.hpp"
#include "spct/likelihood.hpp"

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const spct::contract_error& e) {
        g_last_error = e.what();
        return 2;
    } catch (const spct::io_error& e) {
        g_last_error = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 1;
    }
}

spct::BinMap make_binmap(const std::uint16_t* bins, int w, int h, int nbins) {
    spct::BinMap bm;
    bm.width = w;
    bm.height = h;
    bm.bins = nbins;
    if (w > 0 && h > 0) bm.data.assign(bins, bins + static_cast<std::size_t>(w) * h);
    return bm;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

// imagecore.cpp:17-24
int ref_to_grayscale(const std::uint8_t* r, const std::uint8_t* g, const std::uint8_t* b,
                     int w, int h, std::uint8_t* out) {
    return guarded([&] {
        spct::ColorImage img(w, h);
        const std::size_t n = static_cast<std::size_t>(w) * h;
        std::memcpy(img.r.data(), r, n);
        std::memcpy(img.g.data(), g, n);
        std::memcpy(img.b.data(), b, n);
        spct::GrayImage gi = spct::to_grayscale(img);
        std::memcpy(out, gi.data.data(), n);
    });
}

// imagecore.cpp:45-48
int ref_quantize_u8(const std::uint8_t* gray, int w, int h, int bins, double lo, double hi,
                    std::uint16_t* out) {
    return guarded([&] {
        spct::GrayImage img;
        img.width = w;
        img.height = h;
        if (w > 0 && h > 0) img.data.assign(gray, gray + static_cast<std::size_t>(w) * h);
        spct::BinMap bm = spct::quantize(img, bins, lo, hi);
        std::memcpy(out, bm.data.data(), bm.data.size() * sizeof(std::uint16_t));
    });
}

// imagecore.cpp:50-53
int ref_quantize_f64(const double* vals, int w, int h, int bins, double lo, double hi,
                     std::uint16_t* out) {
    return guarded([&] {
        spct::ScalarMap m;
        m.width = w;
        m.height = h;
        if (w > 0 && h > 0) m.data.assign(vals, vals + static_cast<std::size_t>(w) * h);
        spct::BinMap bm = spct::quantize(m, bins, lo, hi);
        std::memcpy(out, bm.data.data(), bm.data.size() * sizeof(std::uint16_t));
    });
}

// Opaque tensor handle: build_integral_histogram (integral.cpp:548-551).
int ref_ih_build(const std::uint16_t* bins, int w, int h, int nbins, int kind, int tile,
                 int threads, std::uint64_t budget, void** handle) {
    *handle = nullptr;
    return guarded([&] {
        spct::BinMap bm = make_binmap(bins, w, h, nbins);
        spct::ScanSchedule s{static_cast<spct::ScanScheduleKind>(kind), tile, threads};
        auto* t = new spct::IntegralHistogramTensor(spct::build_integral_histogram(bm, s, budget));
        *handle = t;
    });
}

// build_weighted_tensor (integral.cpp:553-559), for completeness of the oracle.
int ref_ih_build_weighted(const std::uint16_t* bins, const std::uint64_t* weights, int w, int h,
                          int nbins, int kind, int tile, int threads, std::uint64_t budget,
                          void** handle) {
    *handle = nullptr;
    return guarded([&] {
        spct::BinMap bm = make_binmap(bins, w, h, nbins);
        std::vector<std::uint64_t> wv(weights, weights + static_cast<std::size_t>(w) * h);
        spct::ScanSchedule s{static_cast<spct::ScanScheduleKind>(kind), tile, threads};
        auto* t = new spct::IntegralHistogramTensor(
            spct::build_weighted_tensor(bm, wv, s, budget));
        *handle = t;
    });
}

void ref_ih_free(void* handle) { delete static_cast<spct::IntegralHistogramTensor*>(handle); }

const std::uint64_t* ref_ih_data(void* handle) {
    return static_cast<spct::IntegralHistogramTensor*>(handle)->data.data();
}

std::uint64_t ref_ih_size(void* handle) {
    return static_cast<spct::IntegralHistogramTensor*>(handle)->data.size();
}

// region_histogram (integral.cpp:561-567)
int ref_region_histogram(void* handle, int x, int y, int w, int h, std::uint64_t* out) {
    return guarded([&] {
        auto& t = *static_cast<spct::IntegralHistogramTensor*>(handle);
        auto v = spct::region_histogram(t, spct::Rect{x, y, w, h});
        std::memcpy(out, v.data(), v.size() * sizeof(std::uint64_t));
    });
}

// region_count (integral.cpp:569-577)
int ref_region_count(void* handle, int bin, int x, int y, int w, int h, std::uint64_t* out) {
    return guarded([&] {
        auto& t = *static_cast<spct::IntegralHistogramTensor*>(handle);
        *out = spct::region_count(t, bin, spct::Rect{x, y, w, h});
    });
}

// hist_distance_map (likelihood.cpp:193-225); out has t.width*t.height doubles.
int ref_hist_distance_map(void* handle, const double* tmpl, int ntmpl, int kw, int kh, double p,
                          double* out) {
    return guarded([&] {
        auto& t = *static_cast<spct::IntegralHistogramTensor*>(handle);
        std::vector<double> th(tmpl, tmpl + ntmpl);
        spct::LikelihoodMap m = spct::hist_distance_map(t, th, kw, kh, p);
        std::memcpy(out, m.values.data(), m.values.size() * sizeof(double));
    });
}

// schedule_stats (integral.cpp:579-590)
int ref_schedule_stats(int w, int h, int tile, int scan_len, long long* iters, long long* tiles,
                       double* eff) {
    return guarded([&] {
        spct::ScheduleStats s = spct::schedule_stats(w, h, tile, scan_len);
        *iters = s.wavefront_iterations;
        *tiles = s.tile_count;
        *eff = s.scan_efficiency;
    });
}

// estimate_memory (integral.cpp:592-599)
int ref_estimate_memory(int w, int h, int bins, int elem, std::uint64_t* padded,
                        std::uint64_t* raw, int* degenerate) {
    return guarded([&] {
        spct::MemoryEstimate e = spct::estimate_memory(w, h, bins, elem);
        *padded = e.padded_bytes;
        *raw = e.raw_bytes;
        *degenerate = e.degenerate ? 1 : 0;
    });
}

// schedule_from_string (integral.cpp:63-69): returns kind or -1.
int ref_schedule_from_string(const char* s) {
    int kind = -1;
    guarded([&] { kind = static_cast<int>(spct::schedule_from_string(s)); });
    return kind;
}

// gradient_maps(GrayImage, sigma) (features.cpp:200-203) of the unmodified reference, then
// the binning of phog.cpp:15-20 (orientation_bin is file-local there; restated verbatim).
int ref_orientation_bins(const std::uint8_t* gray, int w, int h, double sigma, int bins, std::uint16_t* out) {
    return guarded([&] {
        spct::GrayImage img;
        img.width = w;
        img.height = h;
        img.data.assign(gray, gray + static_cast<std::size_t>(w) * h);
        const spct::GradientMaps g = spct::gradient_maps(img, sigma);
        for (std::size_t i = 0; i < g.orientation.data.size(); ++i) {
            int b = static_cast<int>(std::floor((g.orientation.data[i] + 90.0) * bins / 180.0));
            if (b < 0) b = 0;
            if (b >= bins) b = bins - 1;
            out[i] = static_cast<std::uint16_t>(b);
        }
    });
}

// Map consumers (likelihood.cpp:257-330).
namespace {
spct::LikelihoodMap make_map(const double* v, int w, int h) {
    spct::LikelihoodMap m;
    m.width = w;
    m.height = h;
    m.values.assign(v, v + static_cast<std::size_t>(w) * h);
    return m;
}
}  // namespace

int ref_fuse_maps(const double* const* maps, int nmaps, const double* weights, int nweights, int w, int h, double* out) {
    return guarded([&] {
        std::vector<spct::LikelihoodMap> ms;
        for (int m = 0; m < nmaps; ++m) ms.push_back(make_map(maps[m], w, h));
        std::vector<double> wv(weights, weights + nweights);
        const spct::LikelihoodMap f = spct::fuse_maps(ms, wv);
        std::memcpy(out, f.values.data(), f.values.size() * sizeof(double));
    });
}

int ref_find_peaks(const double* map, int w, int h, int* xs, int* ys, double* hs, int* ranks, int max_out, int* count) {
    return guarded([&] {
        const auto pk = spct::find_peaks(make_map(map, w, h));
        *count = static_cast<int>(pk.size());
        for (int i = 0; i < static_cast<int>(pk.size()) && i < max_out; ++i) {
            xs[i] = pk[i].x;
            ys[i] = pk[i].y;
            hs[i] = pk[i].height;
            ranks[i] = pk[i].rank;
        }
    });
}

int ref_score_map(const double* map, int w, int h, int gx, int gy, int gw, int gh, int* rank) {
    return guarded([&] { *rank = spct::score_map(make_map(map, w, h), spct::Rect{gx, gy, gw, gh}); });
}

// SWIH (swih.cpp:115-191): quadrant set + exact query, the brute-force oracle, normalised.
int ref_swlh_query_fixed(const std::uint16_t* bins, int w, int h, int nbins, int kw, int kh, const int* centres, int n,
                         std::int64_t* out) {
    return guarded([&] {
        spct::BinMap bm = make_binmap(bins, w, h, nbins);
        const spct::KernelSpec spec{kw, kh};
        const spct::WeightedQuadrantSet set = spct::build_quadrant_set(bm, spec);
        for (int i = 0; i < n; ++i) {
            const auto v = spct::swlh_query_fixed(set, centres[2 * i], centres[2 * i + 1], spec);
            std::memcpy(out + static_cast<std::size_t>(i) * nbins, v.data(), v.size() * sizeof(std::int64_t));
        }
    });
}

int ref_swlh_query(const std::uint16_t* bins, int w, int h, int nbins, int kw, int kh, const int* centres, int n,
                   double* out) {
    return guarded([&] {
        spct::BinMap bm = make_binmap(bins, w, h, nbins);
        const spct::KernelSpec spec{kw, kh};
        const spct::WeightedQuadrantSet set = spct::build_quadrant_set(bm, spec);
        for (int i = 0; i < n; ++i) {
            const auto v = spct::swlh_query(set, centres[2 * i], centres[2 * i + 1], spec);
            std::memcpy(out + static_cast<std::size_t>(i) * nbins, v.data(), v.size() * sizeof(double));
        }
    });
}

int ref_brute_force_swlh_fixed(const std::uint16_t* bins, int w, int h, int nbins, int kw, int kh, int cx, int cy,
                               std::int64_t* out) {
    return guarded([&] {
        const auto v = spct::brute_force_swlh_fixed(make_binmap(bins, w, h, nbins), cx, cy, spct::KernelSpec{kw, kh});
        std::memcpy(out, v.data(), v.size() * sizeof(std::int64_t));
    });
}

// MedianBackgroundIH (motion.cpp:35-99): construct on frames [0, nf), slide() through the
// rest, background(); and median_background_sort (motion.cpp:103-118).
namespace {
spct::GrayImage gray_of(const std::uint8_t* p, int w, int h) {
    spct::GrayImage g(w, h);
    std::memcpy(g.data.data(), p, static_cast<std::size_t>(w) * h);
    return g;
}
}  // namespace

int ref_median_bg_ih(const std::uint8_t* frames, int nf, int nslide, int w, int h, int bins, int m, int n,
                     std::uint8_t* out) {
    return guarded([&] {
        const std::size_t px = static_cast<std::size_t>(w) * h;
        spct::FrameWindow win;
        for (int f = 0; f < nf; ++f) win.frames.push_back(gray_of(frames + f * px, w, h));
        spct::MedianBackgroundIH bg(win, bins, m, n);
        for (int s = 0; s < nslide; ++s) bg.slide(gray_of(frames + (nf + s) * px, w, h));
        const spct::GrayImage o = bg.background();
        std::memcpy(out, o.data.data(), px);
    });
}

int ref_median_bg_sort(const std::uint8_t* frames, int nf, int w, int h, std::uint8_t* out) {
    return guarded([&] {
        const std::size_t px = static_cast<std::size_t>(w) * h;
        spct::FrameWindow win;
        for (int f = 0; f < nf; ++f) win.frames.push_back(gray_of(frames + f * px, w, h));
        const spct::GrayImage o = spct::median_background_sort(win);
        std::memcpy(out, o.data.data(), px);
    });
}

// dump_tensor / load_tensor (integral.cpp:619-659), the IHT1 wire format.
int ref_dump_tensor(void* handle, const char* path) {
    return guarded([&] { spct::dump_tensor(*static_cast<spct::IntegralHistogramTensor*>(handle), path); });
}

int ref_load_tensor(const char* path, void** out) {
    return guarded([&] { *out = new spct::IntegralHistogramTensor(spct::load_tensor(path)); });
}

}  // extern "C"
