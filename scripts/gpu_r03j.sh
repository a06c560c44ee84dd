set -u
mkdir -p gpurun_out
GBE_STREAM_KU=4 GBE_KERNEL_POLICY=stream timeout 900 python -m pytest tests/test_gpu_stream.py -q -x -k "small_domain or whole_solve_stream" > gpurun_out/pytest_r03j.log 2>&1; tail -3 gpurun_out/pytest_r03j.log
O=gpurun_out/sweep_r03j.txt; : > $O
run() { local wl=$1; shift; env "$@" timeout 300 python scripts/sweep_one.py $wl "$*" >> $O 2>&1 || echo "$wl [$*] FAILED" >> $O; }
for wl in c5 c4d4; do run $wl GBE_KERNEL_POLICY=stream; run $wl GBE_KERNEL_POLICY=stream GBE_STREAM_KU=4; run $wl GBE_STREAM_KU=4; done
cat $O
