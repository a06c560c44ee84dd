set -u
mkdir -p gpurun_out
O=gpurun_out/sweep_r03h.txt; : > $O
run() { local wl=$1; shift; env "$@" timeout 300 python scripts/sweep_one.py $wl "$*" >> $O 2>&1 || echo "$wl [$*] FAILED" >> $O; }
for E in "X=0" "GBE_STREAM_PLMAX=2048" "GBE_STREAM_PLMAX=1024" "GBE_STREAM_PLMAX=512" "GBE_STREAM_PLMAX=256"; do run c5 $E; done
for E in "X=0" "GBE_STREAM_PLMAX=1024" "GBE_STREAM_PLMAX=512"; do run c4d4 $E; done
cat $O
# DRAM bytes of C5 x57 (streaming, prefetch off) at two warp-tile caps
export GBE_KERNEL_POLICY=stream GBE_STREAM_PF=0 PROF_VARIANT=2
for PLM in 4096 1024; do
  IDX=$(GBE_STREAM_PLMAX=$PLM python scripts/profile_step.py --workload c5 --which-fast --var 57 | tail -1)
  GBE_STREAM_PLMAX=$PLM PROF_VARIANT=2 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct --clock-control none --profile-from-start off -k regex:bk_stream -s $IDX -c 1 python scripts/profile_step.py --workload c5 2>&1 | grep -E "dram__|gpu__time|hit_rate" | sed "s/^/PL$PLM /"
done
unset GBE_KERNEL_POLICY GBE_STREAM_PF PROF_VARIANT
KEEP= bash scripts/gpu_prof.sh r03 57 9
WL=c5 KREGEX=bk_stream PROF_VARIANT=2 bash scripts/gpu_prof.sh r03c5 57
head -30 gpurun_out/ncu_r03_x57.txt gpurun_out/ncu_r03_x9.txt gpurun_out/ncu_r03c5_x57.txt
