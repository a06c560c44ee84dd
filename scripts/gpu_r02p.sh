set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_spill.py -q -x > gpurun_out/pytest_r02p.log 2>&1; tail -2 gpurun_out/pytest_r02p.log; grep -E "^E " gpurun_out/pytest_r02p.log | head -5
for E in "X=0" "GBE_STREAM_PF=0"; do echo "== C4-d4 $E"; env $E timeout 300 python scripts/bench_detail.py c4d4 2>&1 | sed -n 2,6p; done
echo "== C4"; timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 2,4p
echo "== C5"; timeout 300 python scripts/bench_detail.py c5 2>&1 | sed -n 2,5p
