set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_merge.py tests/test_gpu_parity.py tests/test_gpu_stream.py -q -x > gpurun_out/pytest_r02q.log 2>&1; tail -2 gpurun_out/pytest_r02q.log; grep -E "^E " gpurun_out/pytest_r02q.log | head -5
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "c4 or c2" > gpurun_out/pytest_r02q2.log 2>&1; tail -2 gpurun_out/pytest_r02q2.log
for E in "X=0" "GBE_STREAM_HXUN=4"; do echo "== C4-d4 $E"; env $E timeout 300 python scripts/bench_detail.py c4d4 2>&1 | sed -n 2,6p; done
echo "== C4"; timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 2,6p
echo "== C5"; timeout 300 python scripts/bench_detail.py c5 2>&1 | sed -n 2,5p
echo "== C3 i16"; timeout 300 python scripts/bench_detail.py c3 16 2>&1 | sed -n 2,4p
