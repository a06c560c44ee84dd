set -u
mkdir -p gpurun_out
for E in "X=0" "GBE_FAST_NO_HTILE=1" "GBE_KERNEL_POLICY=tiled"; do echo "== C4 $E"; env $E timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 2,7p; done
