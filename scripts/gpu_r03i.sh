set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stream.py -q -x > gpurun_out/pytest_r03i.log 2>&1; tail -3 gpurun_out/pytest_r03i.log
O=gpurun_out/sweep_r03i.txt; : > $O
run() { local wl=$1; shift; env "$@" timeout 300 python scripts/sweep_one.py $wl "$*" >> $O 2>&1 || echo "$wl [$*] FAILED" >> $O; }
for wl in c5 c4d4 c4; do run $wl X=0; done
run c5 GBE_STREAM_HALF=0
cat $O
