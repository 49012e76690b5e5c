// Wall time of the C++ drop-in calls a reference caller makes per frame (host frame in,
// host-visible results out): quantize -> build_integral_histogram -> hist_distance_map
// (likelihood.hpp:59-61, integral.hpp:98-100: the reference signatures, results returned by
// value), the one-call fused likelihood_from_frame, the map-reusing hist_match_map_into,
// and region_histogram.  Usage: dropin_bench [side] [bins] [frames] [--json]
// bench.py runs it and reports the JSON line as `dropin_e2e`.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "spct/imagecore.hpp"
#include "spct/integral.hpp"
#include "spct/likelihood.hpp"

using namespace spct;
using clk = std::chrono::steady_clock;

static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

int main(int argc, char** argv) {
    bool json = false;
    int pos[3] = {4096, 128, 5}, np = 0;
    for (int i = 1; i < argc; ++i) {
        if (std::strcmp(argv[i], "--json") == 0) json = true;
        else if (np < 3) pos[np++] = std::atoi(argv[i]);
    }
    const int n = pos[0], bins = pos[1], frames = pos[2];
    GrayImage img(n, n);
    std::mt19937 rng(1);
    for (auto& v : img.data) v = static_cast<std::uint8_t>(rng() & 255);
    BinMap bm = quantize(img, bins);
    std::vector<double> tmpl(bins, 0.0);
    for (int y = n / 2 - 32; y < n / 2 + 32; ++y)
        for (int x = n / 2 - 32; x < n / 2 + 32; ++x) tmpl[bm.at(x, y)] += 1.0 / 4096;
    double tq = 0, tb = 0, tm = 0, tr = 0, tf = 0;
    double checksum = 0;
    for (int f = 0; f <= frames; ++f) {
        auto a = clk::now();
        BinMap q = quantize(img, bins);
        auto b = clk::now();
        auto t = build_integral_histogram(q, {}, ~0ull);
        auto c = clk::now();
        auto m = hist_distance_map(t, tmpl, 64, 64, 1.0);
        auto d = clk::now();
        std::uint64_t s = 0;
        for (int i = 0; i < 100; ++i) s += region_histogram(t, Rect{(i * 7) % (n - 64), (i * 5) % (n - 64), 64, 64})[0];
        auto e = clk::now();
        auto mf = likelihood_from_frame(img, bins, tmpl, 64, 64, 1.0, nullptr, ~0ull);
        auto g = clk::now();
        checksum += m.values[std::size_t(n / 2) * n + n / 2] + mf.values[7] + double(s);
        if (f == 0) continue;  // warm-up
        tq += ms(a, b);
        tb += ms(b, c);
        tm += ms(c, d);
        tr += ms(d, e);
        tf += ms(e, g);
    }
    tq /= frames, tb /= frames, tm /= frames, tr /= frames, tf /= frames;
    // the host-side floor of the API's result: allocating and zeroing the W x H map vector
    double tv = 0;
    for (int f = 0; f < frames; ++f) {
        auto a = clk::now();
        std::vector<double> v(std::size_t(n) * n);
        auto b = clk::now();
        tv += ms(a, b);
        checksum += v[7];
    }
    tv /= frames;
    // the reusing overload (non-reference extension)
    auto t = build_integral_histogram(bm, {}, ~0ull);
    LikelihoodMap m;
    hist_match_map_into(t, tmpl, 64, 64, HistMetric::Minkowski, 1.0, m);
    auto a = clk::now();
    for (int f = 0; f < frames; ++f) hist_match_map_into(t, tmpl, 64, 64, HistMetric::Minkowski, 1.0, m);
    const double ti = ms(a, clk::now()) / frames;
    const double binpx = double(bins) * n * n;
    if (json) {
        std::printf(
            "{\"side\": %d, \"bins\": %d, \"frames\": %d, \"quantize_ms\": %.4f, \"build_ms\": %.4f, "
            "\"hist_distance_map_ms\": %.4f, \"region_histogram_x100_ms\": %.4f, \"likelihood_from_frame_ms\": %.4f, "
            "\"hist_match_map_into_ms\": %.4f, \"vector_alloc_floor_ms\": %.4f, "
            "\"value\": %.3f, \"value_fused\": %.3f, \"checksum\": %.6g}\n",
            n, bins, frames, tq, tb, tm, tr, tf, ti, tv, binpx / ((tb + tm) * 1e-3) / 1e9, binpx / (tf * 1e-3) / 1e9,
            checksum);
        return 0;
    }
    std::printf("%dx%d, %d bins: quantize %.3f ms, build %.3f ms, hist_distance_map %.3f ms, 100 region queries %.3f ms,"
                " likelihood_from_frame %.3f ms (per frame)\n", n, n, bins, tq, tb, tm, tr, tf);
    std::printf("  (std::vector<double>(W*H) alone: %.3f ms)\n", tv);
    std::printf("  hist_match_map_into (map storage reused): %.3f ms\n", ti);
    return 0;
}
