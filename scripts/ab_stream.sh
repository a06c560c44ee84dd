# A/B of the kernel variants per bucket (development tool): per-task JSON
# of one resident solve per policy -> gpurun_out/ab_<policy>_<wl>.json
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -m gpu -q -x > gpurun_out/pytest_stream.log 2>&1; tail -2 gpurun_out/pytest_stream.log
for WL in "c5 -1" "c5 16" "c4 -1" "c2 -1"; do
  set -- $WL
  for POL in tiled stream; do
    GBE_KERNEL_POLICY=$POL DETAIL_JSON=gpurun_out/ab_${POL}_$1_$2.json python scripts/bench_detail.py $1 $2 > gpurun_out/ab_${POL}_$1_$2.txt 2>&1
  done
  DETAIL_JSON=gpurun_out/ab_auto_$1_$2.json python scripts/bench_detail.py $1 $2 > gpurun_out/ab_auto_$1_$2.txt 2>&1
done
