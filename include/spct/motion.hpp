// Drop-in for the joint-IH temporal median of the reference's spct/motion.hpp
// (MedianBackgroundIH, median_background_ih, median_background_sort): the joint integral
// histogram stays in HBM and is updated by device accumulate sweeps; results are
// bit-identical to the reference (motion.cpp:35-118).  The rest of motion.hpp (masks,
// morphology, flux, GAC) is outside the B200 path.
#pragma once

#include <cstdint>
#include <deque>
#include <memory>
#include <vector>

#include "spct/spct.hpp"

namespace spct {

struct FrameWindow {
    std::vector<GrayImage> frames;  // odd count, uniform dims
    int center() const { return static_cast<int>(frames.size()) / 2; }
    void validate() const;
};

class MedianBackgroundIH {
public:
    MedianBackgroundIH(const FrameWindow& window, int bins, int m, int n);
    ~MedianBackgroundIH();
    MedianBackgroundIH(MedianBackgroundIH&&) noexcept;
    MedianBackgroundIH& operator=(MedianBackgroundIH&&) noexcept;

    void slide(const GrayImage& next);
    GrayImage background() const;
    int bins() const { return bins_; }

private:
    struct State;
    void add_frame(const GrayImage& f, int sign);
    int bins_, m_, n_;
    int width_ = 0, height_ = 0;
    std::deque<GrayImage> frames_;
    std::unique_ptr<State> st_;  // device joint tensor + workspace
};

GrayImage median_background_ih(const FrameWindow& window, int bins, int m, int n);
GrayImage median_background_sort(const FrameWindow& window);

}  // namespace spct
