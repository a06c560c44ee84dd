set -u
mkdir -p gpurun_out
O=gpurun_out/sweep_r03d.txt; : > $O
run() { local wl=$1; shift; env "$@" timeout 300 python scripts/sweep_one.py $wl "$*" >> $O 2>&1 || echo "$wl [$*] FAILED" >> $O; }
for wl in c5 c4d4 c4; do run $wl X=0; run $wl GBE_STREAM_WAVES=1; done
cat $O
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r03d.log 2>&1; tail -2 gpurun_out/pytest_r03d.log
export GBE_KERNEL_POLICY=stream
WL=c5 KREGEX=bk_stream PROF_VARIANT=2 bash scripts/gpu_prof.sh r03d 57
WL=c4d4 KREGEX=bk_stream PROF_VARIANT=2 bash scripts/gpu_prof.sh r03d 0
cat gpurun_out/ncu_r03d_x57.txt gpurun_out/ncu_r03d_x0.txt
