set -u
mkdir -p gpurun_out
O=gpurun_out/sweep_r03q.txt; : > $O
run() { local wl=$1; shift; env "$@" timeout 300 python scripts/sweep_one.py $wl "$*" >> $O 2>&1 || echo "$wl [$*] FAILED" >> $O; }
run c4d4 X=0; run c5 X=0; run c4 X=0; SWEEP_IB=16 run c5 X=0
cat $O
timeout 1500 python -m pytest tests/test_gpu_stream.py tests/test_gpu_merge.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r03q.log 2>&1; tail -3 gpurun_out/pytest_r03q.log
