"""B200-native (sm_100a) integral histograms and sliding-window likelihood maps.

The hot path of arxiv/paper_1711_01656 (pixel -> bin quantisation -> per-bin 2-D
inclusive-scan integral histogram -> sliding-window histogram matching ->
likelihood map), built as hand-written CUDA kernels behind a C-ABI
(include/spct_cuda.h, libspct_b200.so).  ``api`` mirrors the reference
interface in Python; include/spct/spct.hpp mirrors it in C++.
"""
from . import _capi, profiling
from ._capi import ContractError, SpctError, lib
from .api import (DEFAULT_BUDGET, IntegralHistogramTensor, ScanSchedule, build_and_match, build_and_match_map,
                  build_integral_histogram, dump_tensor, estimate_memory, load_tensor, hist_distance_map, hist_finalize,
                  hist_match_map, hist_partial, orientation_bins, quantize, region_count, region_histogram,
                  region_histograms, schedule_from_string, schedule_stats, to_grayscale)
from .channels import CHANNELS, channel_sources, likelihood_channels
from .consumers import camshift_batch, camshift_refine, find_peaks, fuse_maps, score_map
from . import motion, swih

__all__ = [
    "ContractError", "SpctError", "lib", "DEFAULT_BUDGET", "IntegralHistogramTensor", "ScanSchedule",
    "build_and_match", "build_and_match_map", "build_integral_histogram", "estimate_memory", "hist_distance_map",
    "hist_finalize", "hist_match_map", "hist_partial", "quantize", "region_count", "region_histogram",
    "region_histograms", "schedule_from_string", "schedule_stats", "to_grayscale", "orientation_bins",
    "CHANNELS", "channel_sources", "likelihood_channels", "dump_tensor", "load_tensor",
    "fuse_maps", "find_peaks", "score_map", "camshift_refine", "camshift_batch", "swih", "motion",
]
