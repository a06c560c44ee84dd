set -u
mkdir -p gpurun_out
O=gpurun_out/sweep_r03p.txt; : > $O
run() { local wl=$1; shift; env "$@" timeout 300 python scripts/sweep_one.py $wl "$*" >> $O 2>&1 || echo "$wl [$*] FAILED" >> $O; }
for E in "X=0" "GBE_FAST_STAGES=12"; do run c5 $E; run c4d4 $E; SWEEP_IB=16 run c3 $E; run c4 $E; done
cat $O
