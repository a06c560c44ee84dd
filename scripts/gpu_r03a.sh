set -u
mkdir -p gpurun_out
bash scripts/gpu_round.sh r03a
for c in c4 c5 c4d4; do echo "== $c"; timeout 300 python scripts/bench_detail.py $c > gpurun_out/detail_${c}_r03a.txt 2>&1; sed -n 1,12p gpurun_out/detail_${c}_r03a.txt; done
