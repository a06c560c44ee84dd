# ncu --set full captures of chosen bucket launches of one C4 DPOP solve,
# summarised on the box (reports are too large to bring back together).
# usage: [WL=c4|c5|c2|c5sp] bash scripts/gpu_prof.sh TAG VAR [VAR...]   (KEEP=1 keeps the .ncu-rep)
set -u
TAG=$1; shift
WL=${WL:-c4}
KREGEX=${KREGEX:-bk_fast}   # bk_stream for the streaming kernel (GBE_KERNEL_POLICY=stream)
mkdir -p gpurun_out
for V in "$@"; do
  IDX=$(python scripts/profile_step.py --workload $WL --warm 0 --no-autotune --which-fast --var $V | tail -1)
  R=gpurun_out/prof_${TAG}_x$V
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s $IDX -c 1 -o $R python scripts/profile_step.py --workload $WL --warm 0 --no-autotune > gpurun_out/ncu_${TAG}_x$V.log 2>&1
  python scripts/ncu_summary.py $R.ncu-rep > gpurun_out/ncu_${TAG}_x$V.txt 2>&1
  ncu -i $R.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}_x$V.csv 2>/dev/null
  [ -z "${KEEP:-}" ] && rm -f $R.ncu-rep
  head -3 gpurun_out/ncu_${TAG}_x$V.txt
done
