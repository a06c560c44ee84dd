# A/B of streaming-kernel knobs on C5 (per-bucket times, resident inputs)
set -u
for E in "X=0" "GBE_STREAM_V4=0" "GBE_STREAM_V4=8" "GBE_STREAM_UN=8" "GBE_STREAM_PF=1" "GBE_KERNEL_POLICY=stream"; do
  echo "== $E"
  env $E timeout 300 python scripts/bench_detail.py c5 2>&1 | sed -n 1,10p
done
