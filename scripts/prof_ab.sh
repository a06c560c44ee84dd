mkdir -p gpurun_out
GBE_KERNEL_POLICY=stream PROF_VARIANT=2 KREGEX=bk_stream WL=c5 bash scripts/gpu_prof.sh r02s 77 57
