set -u
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r04c.csv python scripts/profile_step.py > gpurun_out/launches_r04c.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_r04c.csv > gpurun_out/launches_r04c.txt 2>&1; head -16 gpurun_out/launches_r04c.txt
WL=c4d4 KREGEX=bk_stream PROF_VARIANT=2 bash scripts/gpu_prof.sh r04c 0
head -14 gpurun_out/ncu_r04c_x0.txt
