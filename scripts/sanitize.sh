#!/bin/bash
# compute-sanitizer passes over wrapped-ring shapes of the tiled kernel
# (int32 INF / INF-free, f64, sum-product) and the streaming / generic
# kernels.  Output: gpurun_out/sanitize_<tool>.log
set -u
mkdir -p gpurun_out
SEL='test_ring_wraps_bucket_kernel or test_large_domain_lane_split or test_small_domain_random_descriptors_forced_stream or test_stream_broadcast_digit or test_stream_blocked_high_digits'
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python -m pytest tests/test_gpu_ringwrap.py tests/test_gpu_stream.py -q -x -k "$SEL" -p no:cacheprovider \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Error" gpurun_out/sanitize_$tool.log | tail -4
done
