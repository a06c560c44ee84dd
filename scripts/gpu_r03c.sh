# ncu --set full of the largest streaming buckets: C5 x57 (f64 d=4) and C4-d4 x0 (int32 d=4, blocked high digits)
set -u
mkdir -p gpurun_out
export GBE_KERNEL_POLICY=stream
WL=c5 KREGEX=bk_stream PROF_VARIANT=2 bash scripts/gpu_prof.sh r03c 57
WL=c4d4 KREGEX=bk_stream PROF_VARIANT=2 bash scripts/gpu_prof.sh r03c 0
cat gpurun_out/ncu_r03c_x57.txt gpurun_out/ncu_r03c_x0.txt
