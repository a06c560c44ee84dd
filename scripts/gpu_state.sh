#!/bin/bash
# Full state pass: every GPU test (no -x), all configs, per-bucket C4/C5
# breakdowns.  Outputs in gpurun_out/ (tag $1).
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -5 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python scripts/bench_configs.py c1 c2 c3 c4 c5 c5sp count > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; cat gpurun_out/configs_$TAG.jsonl | cut -c1-400; tail -3 gpurun_out/configs_$TAG.err
for w in c4 c5; do DETAIL_JSON=gpurun_out/detail_${w}_$TAG.json timeout 300 python scripts/bench_detail.py $w > gpurun_out/detail_${w}_$TAG.txt 2>&1; head -30 gpurun_out/detail_${w}_$TAG.txt; done
