# ncu --set full captures of chosen bucket launches of one C4 DPOP solve.
# usage: bash scripts/gpu_prof.sh TAG VAR [VAR...]
set -u
TAG=$1; shift
mkdir -p gpurun_out
for V in "$@"; do
  IDX=$(python scripts/profile_step.py --which-fast --var $V | tail -1)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:bk_fast -s $IDX -c 1 -o gpurun_out/prof_${TAG}_x$V python scripts/profile_step.py > gpurun_out/ncu_${TAG}_x$V.log 2>&1
  tail -1 gpurun_out/ncu_${TAG}_x$V.log
done
