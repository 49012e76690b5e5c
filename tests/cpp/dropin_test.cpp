// Drop-in check of the C++ API: reference-style test cases written against the
// unchanged spct:: signatures (cf. proj/tests/test_integral.cpp, test_likelihood.cpp,
// test_imagecore.cpp), compiled against include/spct/*.hpp and linked with
// libspct_b200.so instead of the reference library.  Run by tests/test_dropin_cpp.py
// on a GPU box; exits non-zero on the first failed check.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "spct/imagecore.hpp"
#include "spct/integral.hpp"
#include "spct/likelihood.hpp"
#include "spct/motion.hpp"
#include "spct/swih.hpp"

using namespace spct;

static int g_checks = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(cond)) {                                                               \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
            std::exit(1);                                                            \
        }                                                                            \
    } while (0)
#define CHECK_THROWS_AS(expr, E)      \
    do {                              \
        bool thrown = false;          \
        try {                         \
            (void)(expr);             \
        } catch (const E&) {          \
            thrown = true;            \
        }                             \
        CHECK(thrown);                \
    } while (0)

static BinMap random_binmap(int w, int h, int bins, unsigned seed) {
    std::mt19937 rng(seed);
    std::uniform_int_distribution<int> d(0, bins - 1);
    BinMap bm(w, h, bins);
    for (auto& v : bm.data) v = static_cast<std::uint16_t>(d(rng));
    return bm;
}

// Plain sequential recurrence (integral.cpp:348-361) as the in-test oracle.
static std::vector<std::uint64_t> seq_tensor(const BinMap& bm) {
    const std::size_t rs = bm.width + 1, ps = rs * (bm.height + 1);
    std::vector<std::uint64_t> t(ps * bm.bins, 0);
    for (int k = 0; k < bm.bins; ++k)
        for (int y = 1; y <= bm.height; ++y)
            for (int x = 1; x <= bm.width; ++x)
                t[k * ps + y * rs + x] = t[k * ps + y * rs + x - 1] + t[k * ps + (y - 1) * rs + x] -
                                         t[k * ps + (y - 1) * rs + x - 1] + (bm.at(x - 1, y - 1) == k);
    return t;
}

int main() {
    {  // hand-computed 2x2 prefix planes (test_integral.cpp:40-57)
        BinMap bm(2, 2, 2);
        bm.at(0, 0) = 0;
        bm.at(1, 0) = 1;
        bm.at(0, 1) = 1;
        bm.at(1, 1) = 0;
        auto t = build_integral_histogram(bm);
        CHECK(t.at(0, 2, 2) == 2);
        CHECK(t.at(1, 2, 2) == 2);
        CHECK(t.at(0, 1, 1) == 1);
        CHECK(t.at(1, 1, 1) == 0);
        for (int k = 0; k < 2; ++k)
            for (int i = 0; i < 3; ++i) {
                CHECK(t.at(k, 0, i) == 0);
                CHECK(t.at(k, i, 0) == 0);
            }
    }
    {  // all schedules produce identical tensors, equal to the recurrence (test_integral.cpp:72-87)
        const int sizes[][2] = {{1, 1}, {5, 3}, {33, 31}, {64, 64}, {70, 129}, {256, 40}};
        unsigned seed = 1000;
        for (auto& s : sizes) {
            BinMap bm = random_binmap(s[0], s[1], 16, seed++);
            auto want = seq_tensor(bm);
            for (auto kind : {ScanScheduleKind::Sequential, ScanScheduleKind::ScanTransposeScan,
                              ScanScheduleKind::CrossWeaveTiled, ScanScheduleKind::WavefrontTiled}) {
                auto t = build_integral_histogram(bm, {kind, 64, 4});
                CHECK(t.data == want);
                CHECK(t.data.size() == want.size());
            }
        }
    }
    {  // region histogram vs brute force, degenerate and out-of-range rects (test_integral.cpp:89-132)
        BinMap bm = random_binmap(200, 150, 32, 7);
        auto t = build_integral_histogram(bm, {ScanScheduleKind::WavefrontTiled, 32, 4});
        std::mt19937 rng(8);
        for (int i = 0; i < 50; ++i) {
            int x1 = rng() % 200, y1 = rng() % 150;
            Rect r{x1, y1, static_cast<int>(rng() % (200 - x1 + 1)), static_cast<int>(rng() % (150 - y1 + 1))};
            auto hist = region_histogram(t, r);
            std::uint64_t total = 0;
            for (int k = 0; k < 32; ++k) {
                std::uint64_t n = 0;
                for (int y = r.y; y < r.bottom(); ++y)
                    for (int x = r.x; x < r.right(); ++x) n += bm.at(x, y) == k;
                CHECK(hist[k] == n);
                CHECK(region_count(t, k, r) == n);
                total += hist[k];
            }
            CHECK(total == static_cast<std::uint64_t>(r.area()));
        }
        auto z = region_histogram(t, Rect{3, 3, 0, 0});
        for (auto v : z) CHECK(v == 0);
        CHECK_THROWS_AS(region_histogram(t, Rect{195, 145, 8, 8}), contract_error);
        CHECK_THROWS_AS(region_histogram(t, Rect{-1, 0, 2, 2}), contract_error);
        CHECK_THROWS_AS(region_count(t, 40, Rect{0, 0, 1, 1}), contract_error);
    }
    {  // build contract violations (test_integral.cpp:190-206)
        BinMap bm = random_binmap(16, 16, 4, 3);
        BinMap bad = bm;
        bad.data[7] = 4;
        CHECK_THROWS_AS(build_integral_histogram(bad), contract_error);
        CHECK_THROWS_AS(build_integral_histogram(bm, {}, 64), contract_error);
        CHECK_THROWS_AS(build_integral_histogram(BinMap{}), contract_error);
        CHECK_THROWS_AS(build_integral_histogram(bm, {ScanScheduleKind::WavefrontTiled, 32, 0}), contract_error);
        CHECK(schedule_from_string("wavefront") == ScanScheduleKind::WavefrontTiled);
        CHECK_THROWS_AS(schedule_from_string("bogus"), contract_error);
    }
    {  // quantize / grayscale (test_imagecore.cpp:48-50, 88-106)
        GrayImage img(4, 1);
        img.data = {0, 64, 128, 255};
        BinMap bm = quantize(img, 32, 0.0, 256.0);
        CHECK(bm.at(0, 0) == 0 && bm.at(1, 0) == 8 && bm.at(2, 0) == 16 && bm.at(3, 0) == 31);
        BinMap c = quantize(img, 4, 100.0, 200.0);
        CHECK(c.at(0, 0) == 0 && c.at(3, 0) == 3);
        CHECK_THROWS_AS(quantize(img, 0), contract_error);
        CHECK_THROWS_AS(quantize(img, 70000), contract_error);
        CHECK_THROWS_AS(quantize(img, 8, 10.0, 10.0), contract_error);
        ColorImage col(2, 1);
        col.r = {10, 255};
        col.g = {20, 255};
        col.b = {40, 255};
        GrayImage g = to_grayscale(col);
        CHECK(g.data[0] == 23 && g.data[1] == 255);
    }
    {  // hist distance: identity, disjoint, hand fixture (test_likelihood.cpp:156-194)
        GrayImage img(12, 10);
        std::mt19937 rng(3);
        std::uniform_int_distribution<int> d(0, 255);
        for (auto& p : img.data) p = static_cast<std::uint8_t>(d(rng));
        BinMap bm = quantize(img, 8);
        auto t = build_integral_histogram(bm);
        Rect win{4, 3, 5, 4};
        std::vector<double> th(8, 0.0);
        for (int y = win.y; y < win.bottom(); ++y)
            for (int x = win.x; x < win.right(); ++x) th[bm.at(x, y)] += 1.0;
        for (double& v : th) v /= win.area();
        LikelihoodMap map = hist_distance_map(t, th, win.w, win.h, 1.0);
        CHECK(std::abs(map.at(win.x + 2, win.y + 1) - 1.0) <= 1e-12);
        GrayImage dark(9, 9, 10);
        auto td = build_integral_histogram(quantize(dark, 4));
        std::vector<double> bright(4, 0.0);
        bright[3] = 1.0;
        for (double v : hist_distance_map(td, bright, 3, 3, 1.0).values) CHECK(std::abs(v) <= 1e-12);
        GrayImage six(2, 3);
        six.data = {0, 100, 100, 200, 200, 200};
        auto t6 = build_integral_histogram(quantize(six, 3));
        LikelihoodMap h6 = hist_distance_map(t6, {0.4, 0.4, 0.2}, 2, 3, 1.0);
        CHECK(std::abs(h6.at(0, 1) - 0.7) <= 1e-12);
        CHECK_THROWS_AS(hist_distance_map(t6, {0.4, 0.4, 0.2}, 2, 3, 0.5), contract_error);
        CHECK_THROWS_AS(hist_distance_map(t6, {0.5, 0.5}, 2, 3, 1.0), contract_error);
        // exact mode (tensor re-read, reference operation order) agrees with the default
        set_exact_maps(true);
        LikelihoodMap mx = hist_distance_map(t, th, win.w, win.h, 1.0);
        set_exact_maps(false);
        for (std::size_t i = 0; i < mx.values.size(); ++i)
            CHECK(std::abs(mx.values[i] - map.values[i]) <= 1e-5 * std::abs(mx.values[i]) + 1e-12);
        // the fused frame path agrees with build + hist_distance_map
        IntegralHistogramTensor tf;
        LikelihoodMap mf = likelihood_from_frame(img, 8, th, win.w, win.h, 1.0, &tf);
        CHECK(tf.data == t.data);
        for (std::size_t i = 0; i < mf.values.size(); ++i)
            CHECK(std::abs(mf.values[i] - map.values[i]) <= 1e-5 * std::abs(map.values[i]) + 1e-12);
        // a window too large for the fused sweep (kw > 128): the map comes from the stored
        // tensor in the default mode too, no contract error
        GrayImage big(240, 180);
        for (auto& p : big.data) p = static_cast<std::uint8_t>(d(rng));
        auto tb = build_integral_histogram(quantize(big, 6));
        std::vector<double> flat(6, 1.0 / 6);
        LikelihoodMap lb = hist_distance_map(tb, flat, 200, 150, 1.0);
        set_exact_maps(true);
        LikelihoodMap lbx = hist_distance_map(tb, flat, 200, 150, 1.0);
        set_exact_maps(false);
        CHECK(lb.values == lbx.values && lb.width == 240 && lb.height == 180);
    }
    {  // map consumers (test_likelihood.cpp:296-362, test_tracker.cpp:150-176)
        LikelihoodMap a;
        a.width = 4;
        a.height = 3;
        a.values.assign(12, 0.2);
        LikelihoodMap b = a;
        for (double& v : b.values) v = 0.8;
        CHECK(fuse_maps({a}).values == a.values);
        for (double v : fuse_maps({a, b}).values) CHECK(std::abs(v - 0.5) <= 1e-12);
        CHECK_THROWS_AS((void)fuse_maps({a, b}, {1.0}), contract_error);
        LikelihoodMap m;
        m.width = 30;
        m.height = 24;
        m.values.assign(720, 0.0);
        for (int y = 8; y < 13; ++y)
            for (int x = 10; x < 15; ++x) m.at(x, y) = 1.0 - 0.15 * (std::abs(x - 12) + std::abs(y - 10));
        auto peaks = find_peaks(m);
        CHECK(!peaks.empty() && peaks.front().rank == 1);
        CHECK(score_map(m, Rect{9, 7, 8, 8}) == 1);
        CHECK_THROWS_AS((void)score_map(m, Rect{28, 20, 5, 5}), contract_error);
        LikelihoodMap imp;
        imp.width = imp.height = 12;
        imp.values.assign(144, 0.0);
        imp.at(5, 7) = 1.0;
        CamshiftResult r = camshift_refine(imp, 3.0, 3.0, 9, 9);
        CHECK(!r.zero_mass && std::abs(r.cx - 5.0) <= 1e-12 && std::abs(r.cy - 7.0) <= 1e-12 && r.iterations >= 1);
    }
    {  // IHT1 round trip (test_integral.cpp:208-238)
        BinMap bm(33, 31, 16);
        for (std::size_t i = 0; i < bm.data.size(); ++i) bm.data[i] = static_cast<std::uint16_t>((i * 7 + i / 33) % 16);
        auto t = build_integral_histogram(bm);
        const std::string path = "/tmp/spct_dropin_t.iht";
        dump_tensor(t, path);
        std::FILE* f = std::fopen(path.c_str(), "rb");
        char head[4] = {};
        CHECK(f && std::fread(head, 1, 4, f) == 4);
        if (f) std::fclose(f);
        CHECK(std::string(head, 4) == "IHT1");
        auto t2 = load_tensor(path);
        CHECK(t2.bins == 16 && t2.height == 31 && t2.width == 33);
        CHECK(t2.data == t.data);
        CHECK_THROWS_AS(load_tensor("/nonexistent/t.iht"), io_error);
        std::remove(path.c_str());
    }
    {  // analytics (test_integral.cpp:155-188)
        auto s = schedule_stats(1024, 1024, 32, 1024);
        CHECK(s.wavefront_iterations == 63 && s.tile_count == 1024);
        CHECK(s.scan_efficiency > 0.29 && s.scan_efficiency < 0.31);
        auto e = estimate_memory(512, 512, 32, 8);
        CHECK(e.padded_bytes == 32ull * 513 * 513 * 8 && e.raw_bytes == 64ull * 1024 * 1024);
        CHECK(estimate_memory(100, 100, 0, 8).degenerate);
        CHECK_THROWS_AS(estimate_memory(-1, 4, 4, 4), contract_error);
    }
    {  // weighted IH vs direct accumulation (test_swih.cpp:78-96)
        BinMap bm = random_binmap(21, 14, 6, 55);
        auto fields = quadrant_weight_fields(21, 14, {5, 7});
        for (const auto& f : fields) {
            auto t = build_weighted_ih(bm, f);
            std::mt19937 rng(2);
            for (int trial = 0; trial < 40; ++trial) {
                int x1 = static_cast<int>(rng() % 21), y1 = static_cast<int>(rng() % 14);
                Rect r{x1, y1, static_cast<int>(rng() % (21 - x1 + 1)), static_cast<int>(rng() % (14 - y1 + 1))};
                std::vector<std::uint64_t> want(6, 0);
                for (int y = r.y; y < r.bottom(); ++y)
                    for (int x = r.x; x < r.right(); ++x) want[bm.at(x, y)] += quantize_weight(f.at(x, y));
                CHECK(region_histogram(t, r) == want);
            }
        }
        CHECK_THROWS_AS(build_weighted_tensor(bm, std::vector<std::uint64_t>(5, 1)), contract_error);
        // a dumped weighted tensor (16.16 sums beyond 2^32) loads back with uint64 cells
        std::vector<std::uint64_t> big(bm.data.size());
        for (std::size_t i = 0; i < big.size(); ++i) big[i] = (std::uint64_t(1) << 31) + i * 65536;
        auto wt = build_weighted_tensor(bm, big);
        const std::string wpath = "/tmp/spct_dropin_w.iht";
        dump_tensor(wt, wpath);
        auto wl = load_tensor(wpath);
        CHECK(wl.bins == 6 && wl.height == 14 && wl.width == 21);
        CHECK(wl.data == wt.data);
        CHECK(wl.at(0, 14, 21) + wl.at(1, 14, 21) > (std::uint64_t(1) << 32));
        CHECK(region_histogram(wl, Rect{3, 2, 9, 7}) == region_histogram(wt, Rect{3, 2, 9, 7}));
        std::remove(wpath.c_str());
    }
    {  // swlh query bit-exact against the brute force (test_swih.cpp:98-114)
        std::mt19937 rng(606);
        const KernelSpec kernels[] = {{1, 1}, {2, 2}, {3, 3}, {4, 4}, {5, 3}, {1, 7}, {8, 1}, {9, 9}, {6, 10}};
        for (const auto& spec : kernels) {
            BinMap bm = random_binmap(40, 36, 8, rng());
            auto set = build_quadrant_set(bm, spec);
            KernelExtents e = kernel_extents(spec);
            for (int trial = 0; trial < 25; ++trial) {
                int cx = e.sxl + static_cast<int>(rng() % (40 - spec.kw + 1));
                int cy = e.syt + static_cast<int>(rng() % (36 - spec.kh + 1));
                CHECK(swlh_query_fixed(set, cx, cy, spec) == brute_force_swlh_fixed(bm, cx, cy, spec));
            }
        }
        BinMap u(12, 12, 4);
        for (auto& v : u.data) v = 2;
        auto h = swlh_query(build_quadrant_set(u, {5, 5}), 6, 6, {5, 5});
        CHECK(h[2] == 1.0 && h[0] == 0.0);
        BinMap bm = random_binmap(10, 10, 4, 5);
        auto set = build_quadrant_set(bm, {5, 5});
        CHECK_THROWS_AS(swlh_query(set, 0, 5, {5, 5}), contract_error);
        CHECK_THROWS_AS(swlh_query(set, 5, 9, {5, 5}), contract_error);
        CHECK_THROWS_AS(swlh_query(set, 5, 5, KernelSpec{3, 3}), contract_error);
    }
    {  // wedding cake (test_swih.cpp:143-183): one layer = the plain local histogram
        BinMap bm = random_binmap(120, 100, 16, 20257);
        auto plain = build_integral_histogram(bm);
        KernelSpec spec{9, 7};
        auto cake = wedding_cake_swlh(plain, 30, 30, spec, 1);
        KernelExtents e = kernel_extents(spec);
        auto counts = region_histogram(plain, Rect{30 - e.sxl, 30 - e.syt, spec.kw, spec.kh});
        for (int k = 0; k < 16; ++k) CHECK(std::abs(cake[k] - counts[k] / 63.0) <= 1e-12);
        double prev = -1;
        for (int layers : {2, 4}) {
            const double mse = histogram_mse(wedding_cake_swlh(plain, 60, 50, {31, 41}, layers),
                                             brute_force_swlh(bm, 60, 50, {31, 41}));
            CHECK(mse > 0.0);
            if (prev >= 0) CHECK(mse <= prev);
            prev = mse;
        }
        CHECK_THROWS_AS(wedding_cake_swlh(plain, 30, 30, spec, 0), contract_error);
    }
    {  // temporal medians (test_motion.cpp:96-195)
        std::mt19937 rng(77);
        auto window = [&](int w, int h, int bins, int count) {
            FrameWindow win;
            std::uniform_int_distribution<int> d(0, bins - 1);
            for (int f = 0; f < count; ++f) {
                GrayImage g(w, h);
                for (auto& v : g.data) v = static_cast<std::uint8_t>(d(rng));
                win.frames.push_back(g);
            }
            return win;
        };
        FrameWindow win = window(13, 10, 256, 9);
        GrayImage bg = median_background_sort(win);
        for (int y = 0; y < 10; ++y)
            for (int x = 0; x < 13; ++x) {
                std::vector<int> vals;
                for (const auto& f : win.frames) vals.push_back(f.at(x, y));
                std::sort(vals.begin(), vals.end());
                CHECK(bg.at(x, y) == vals[4]);
            }
        // 1x1 kernel, 256 bins: the IH median is the sorting median (test_motion.cpp:148-155)
        CHECK(median_background_ih(win, 256, 1, 1).data == bg.data);
        // sliding equals rebuilding (test_motion.cpp:166-185); brute-force spatiotemporal median
        FrameWindow all = window(23, 17, 16, 9);
        FrameWindow first{std::vector<GrayImage>(all.frames.begin(), all.frames.begin() + 5)};
        MedianBackgroundIH model(first, 16, 5, 3);
        for (int i = 5; i < 9; ++i) {
            model.slide(all.frames[i]);
            FrameWindow cur{std::vector<GrayImage>(all.frames.begin() + i - 4, all.frames.begin() + i + 1)};
            const GrayImage got = model.background();
            CHECK(got.data == median_background_ih(cur, 16, 5, 3).data);
            for (int y = 0; y < 17; ++y)
                for (int x = 0; x < 23; ++x) {
                    std::vector<int> vals;
                    for (const auto& f : cur.frames)
                        for (int yy = std::max(0, y - 1); yy < std::min(17, y + 2); ++yy)
                            for (int xx = std::max(0, x - 2); xx < std::min(23, x + 3); ++xx) vals.push_back(f.at(xx, yy));
                    std::sort(vals.begin(), vals.end());
                    const int med = vals[(vals.size() - 1) / 2];
                    CHECK(got.at(x, y) == (2 * med + 1) * 128 / 16);
                }
        }
        CHECK_THROWS_AS(MedianBackgroundIH(first, 8, 3, 3), contract_error);   // value >= bins
        CHECK_THROWS_AS(MedianBackgroundIH(first, 16, 2, 3), contract_error);  // even side
        CHECK_THROWS_AS(model.slide(GrayImage(5, 5)), contract_error);
        FrameWindow even{std::vector<GrayImage>(all.frames.begin(), all.frames.begin() + 4)};
        CHECK_THROWS_AS(median_background_sort(even), contract_error);
        CHECK_THROWS_AS(median_background_sort(FrameWindow{}), contract_error);
    }
    std::printf("dropin_test: %d checks passed\n", g_checks);
    return 0;
}
