#!/bin/bash
# Standard GPU pass: tests, smoke, bench line, launch list, ncu capture of the
# largest bucket kernel (summarised on the box).  Outputs land in gpurun_out/
# (copy summaries to profiles/).
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json; tail -2 gpurun_out/bench_$TAG.err
if [ "${2:-}" = "prof" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python scripts/profile_step.py > /dev/null 2>&1
  python scripts/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1; cat gpurun_out/launches_$TAG.txt
  KEEP= bash scripts/gpu_prof.sh $TAG 57
fi
