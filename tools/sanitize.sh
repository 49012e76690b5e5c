#!/bin/bash
# compute-sanitizer over a representative subset of the GPU parity tests (small sizes).
mkdir -p gpurun_out
SEL='fused_wide_staging or multi_matches_single or channels or fused_integral_template or fused_map_direct or fused_general_template or fused_bands or fused_uniform or near_zero or multi_matches or ih_bit_exact_binmap or ih_band_carries or ih_bin_slab or maps_vs_oracle or iht1_dump or find_peaks or swlh or weighted or median_background or orientation_bins or tracking_batch or camshift or score or fuse_maps or tensor or loaded or extension or recover'
for tool in memcheck racecheck synccheck; do
  timeout 2400 /usr/local/cuda/bin/compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_tensor_maps.py -m gpu -x -q -k "$SEL" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool: rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
