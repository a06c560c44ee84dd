set -u
mkdir -p gpurun_out
make -j8 all > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_spill.py -q -x > gpurun_out/pytest_spill_r02c.log 2>&1; tail -5 gpurun_out/pytest_spill_r02c.log
KEEP=1 bash scripts/gpu_prof.sh r02c 57 9
WL=c5 KREGEX=bk_stream PROF_VARIANT=2 KEEP=1 bash scripts/gpu_prof.sh r02c5 57
ls -la gpurun_out/*.ncu-rep
