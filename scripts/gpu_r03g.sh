set -u
mkdir -p gpurun_out
O=gpurun_out/sweep_r03g.txt; : > $O
run() { local wl=$1; shift; env "$@" timeout 300 python scripts/sweep_one.py $wl "$*" >> $O 2>&1 || echo "$wl [$*] FAILED" >> $O; }
for wl in c5 c4d4; do run $wl GBE_KERNEL_POLICY=stream; run $wl GBE_KERNEL_POLICY=stream GBE_STREAM_STAGE=1; run $wl GBE_KERNEL_POLICY=stream GBE_STREAM_STAGE=1 GBE_STREAM_STAGE_KB=200; run $wl GBE_KERNEL_POLICY=stream GBE_STREAM_STAGE=1 GBE_STREAM_STAGE_KB=50; done
cat $O
