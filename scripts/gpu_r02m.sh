set -u
mkdir -p gpurun_out
for E in "X=0" "GBE_TILE_ORDER=1" "GBE_STREAM_PF=0" "GBE_TILE_ORDER=1 GBE_STREAM_PF=0" "GBE_TILE_ORDER=1 GBE_STREAM_PER_SM=2" "GBE_TILE_ORDER=1 GBE_STREAM_PER_SM=4 GBE_STREAM_PF=0"; do echo "== C4-d4 $E"; env $E timeout 300 python scripts/bench_detail.py c4d4 2>&1 | sed -n 2,5p; done
for E in "X=0" "GBE_TILE_ORDER=1"; do echo "== C4 $E"; env $E timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 2,6p; echo "== C5 $E"; env $E timeout 300 python scripts/bench_detail.py c5 2>&1 | sed -n 2,5p; done
