set -u
mkdir -p gpurun_out
timeout 300 python scripts/dbg_spill.py 2>&1 | tail -8
bash scripts/gpu_prof.sh r02d 57 9
WL=c5 KREGEX=bk_stream PROF_VARIANT=2 GBE_KERNEL_POLICY=stream bash scripts/gpu_prof.sh r02c5 57
ls -la gpurun_out/ | tail
