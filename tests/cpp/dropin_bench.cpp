// Wall time of the C++ drop-in calls a reference caller makes per frame (host frame in,
// host-visible results out): quantize -> build_integral_histogram -> hist_distance_map,
// and region_histogram.  Usage: dropin_bench [side] [bins] [frames]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "spct/imagecore.hpp"
#include "spct/integral.hpp"
#include "spct/likelihood.hpp"

using namespace spct;
using clk = std::chrono::steady_clock;

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 4096, bins = argc > 2 ? std::atoi(argv[2]) : 128;
    const int frames = argc > 3 ? std::atoi(argv[3]) : 5;
    GrayImage img(n, n);
    std::mt19937 rng(1);
    for (auto& v : img.data) v = static_cast<std::uint8_t>(rng() & 255);
    BinMap bm = quantize(img, bins);
    std::vector<double> tmpl(bins, 0.0);
    for (int y = n / 2 - 32; y < n / 2 + 32; ++y)
        for (int x = n / 2 - 32; x < n / 2 + 32; ++x) tmpl[bm.at(x, y)] += 1.0 / 4096;
    double tb = 0, tm = 0, tq = 0;
    for (int f = 0; f <= frames; ++f) {
        auto a = clk::now();
        auto t = build_integral_histogram(bm, {}, ~0ull);
        auto b = clk::now();
        auto m = hist_distance_map(t, tmpl, 64, 64, 1.0);
        auto c = clk::now();
        std::uint64_t s = 0;
        for (int i = 0; i < 100; ++i) s += region_histogram(t, Rect{(i * 7) % (n - 64), (i * 5) % (n - 64), 64, 64})[0];
        auto d = clk::now();
        if (f == 0) continue;  // warm-up
        tb += std::chrono::duration<double, std::milli>(b - a).count();
        tm += std::chrono::duration<double, std::milli>(c - b).count();
        tq += std::chrono::duration<double, std::milli>(d - c).count();
        if (s == 42 && m.values.empty()) std::printf(" ");
    }
    std::printf("%dx%d, %d bins: build %.3f ms, hist_distance_map %.3f ms, 100 region queries %.3f ms (per frame)\n",
                n, n, bins, tb / frames, tm / frames, tq / frames);
    // the host-side floor of the API's result: allocating and zeroing the W x H map vector
    double tv = 0;
    for (int f = 0; f < frames; ++f) {
        auto a = clk::now();
        std::vector<double> v(std::size_t(n) * n);
        auto b = clk::now();
        tv += std::chrono::duration<double, std::milli>(b - a).count();
        if (v[7] != 0.0) std::printf(" ");
    }
    std::printf("  (std::vector<double>(W*H) alone: %.3f ms)\n", tv / frames);
    // the reusing overload (non-reference extension)
    auto t = build_integral_histogram(bm, {}, ~0ull);
    LikelihoodMap m;
    hist_match_map_into(t, tmpl, 64, 64, HistMetric::Minkowski, 1.0, m);
    auto a = clk::now();
    for (int f = 0; f < frames; ++f) hist_match_map_into(t, tmpl, 64, 64, HistMetric::Minkowski, 1.0, m);
    auto b = clk::now();
    std::printf("  hist_match_map_into (map storage reused): %.3f ms\n",
                std::chrono::duration<double, std::milli>(b - a).count() / frames);
    return 0;
}
