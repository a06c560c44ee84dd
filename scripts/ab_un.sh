mkdir -p gpurun_out
for UN in 2 4 8; do
  GBE_KERNEL_POLICY=stream GBE_STREAM_UN=$UN DETAIL_JSON=gpurun_out/ab_un${UN}_c5_-1.json python scripts/bench_detail.py c5 -1 > /dev/null 2>&1
done
GBE_KERNEL_POLICY=stream DETAIL_JSON=gpurun_out/ab_stream_c5_-1.json python scripts/bench_detail.py c5 -1 > /dev/null 2>&1
GBE_KERNEL_POLICY=tiled DETAIL_JSON=gpurun_out/ab_tiled_c5_-1.json python scripts/bench_detail.py c5 -1 > /dev/null 2>&1
