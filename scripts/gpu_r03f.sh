set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x -k "staged" > gpurun_out/pytest_r03f.log 2>&1; tail -5 gpurun_out/pytest_r03f.log
O=gpurun_out/sweep_r03f.txt; : > $O
run() { local wl=$1; shift; env "$@" timeout 300 python scripts/sweep_one.py $wl "$*" >> $O 2>&1 || echo "$wl [$*] FAILED" >> $O; }
for wl in c5 c4d4; do run $wl X=0; run $wl GBE_STREAM_STAGE=1; run $wl GBE_STREAM_STAGE=1 GBE_STREAM_STAGE_KB=200; run $wl GBE_STREAM_STAGE=1 GBE_STREAM_STAGE_KB=60; done
run c4 X=0
cat $O
