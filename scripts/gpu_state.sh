#!/bin/bash
# Full state pass: every GPU test (no -x), smoke, bench line, all configs,
# per-bucket C4/C5 breakdowns, launch list + ncu of the largest C4 bucket.
# Outputs in gpurun_out/ (tag $1).
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -5 gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; head -c 600 gpurun_out/bench_$TAG.json; echo; tail -2 gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; head -c 300 gpurun_out/bench_ref_$TAG.json; echo
timeout 1500 python scripts/bench_configs.py c1 c2 c3 c4 c4d4 c5 c5sp count c4host c4spill > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; cut -c1-300 gpurun_out/configs_$TAG.jsonl; tail -3 gpurun_out/configs_$TAG.err
for w in c4 c5 c4d4; do DETAIL_JSON=gpurun_out/detail_${w}_$TAG.json timeout 300 python scripts/bench_detail.py $w > gpurun_out/detail_${w}_$TAG.txt 2>&1; head -12 gpurun_out/detail_${w}_$TAG.txt; done
if [ "${2:-}" = "prof" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$TAG.csv python scripts/profile_step.py > /dev/null 2>&1
  python scripts/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1; head -20 gpurun_out/launches_$TAG.txt
  bash scripts/gpu_prof.sh $TAG 57 9
fi
