set -u
mkdir -p gpurun_out
O=gpurun_out/sweep_r03l.txt; : > $O
run() { local wl=$1; shift; env "$@" timeout 300 python scripts/sweep_one.py $wl "$*" >> $O 2>&1 || echo "$wl [$*] FAILED" >> $O; }
for wl in c4 c4d4 c5; do run $wl X=0; run $wl GBE_FAST_BANKTIE=0; done
SWEEP_IB=16 run c3 X=0; SWEEP_IB=16 run c3 GBE_FAST_BANKTIE=0
cat $O
timeout 900 python -m pytest tests/test_gpu_ringwrap.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r03l.log 2>&1; tail -3 gpurun_out/pytest_r03l.log
