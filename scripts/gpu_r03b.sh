# knob sweep: per-bucket kernel times of C4 and C5 under each setting, plus an
# ncu --set full of C5's largest streaming bucket (memory-unit breakdown)
set -u
mkdir -p gpurun_out
O=gpurun_out/sweep_r03b.txt; : > $O
run() { local wl=$1; shift; env "$@" timeout 300 python scripts/sweep_one.py $wl "$*" >> $O 2>&1 || echo "$wl [$*] FAILED" >> $O; }
for E in "X=0" "GBE_FAST_NOUT=2" "GBE_FAST_WANT_STAGES=2" "GBE_FAST_WANT_STAGES=6" "GBE_FAST_PLMAX=729" "GBE_FAST_STAGES=6" "GBE_MERGE_CAP_LOG2=24" "GBE_MERGE_CAP_LOG2=28" "GBE_NO_MERGE=1" "GBE_FAST_QPERM=1"; do run c4 $E; done
for E in "X=0" "GBE_KERNEL_POLICY=tiled" "GBE_STREAM_PER_SM=2" "GBE_STREAM_PER_SM=4" "GBE_STREAM_PF=0" "GBE_STREAM_PF=1" "GBE_STREAM_V4=0" "GBE_STREAM_UN=2" "GBE_NO_MERGE=1"; do run c5 $E; done
cat $O
WL=c5 KREGEX=bk_stream PROF_VARIANT=2 bash scripts/gpu_prof.sh r03b 57
cat gpurun_out/ncu_r03b_x57.txt | head -60
