set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_htile.py -q -x -s > gpurun_out/pytest_r02s.log 2>&1; tail -15 gpurun_out/pytest_r02s.log; grep -E "^E " gpurun_out/pytest_r02s.log | head
DETAIL_JSON=gpurun_out/detail_c4_r02s.json timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 2,9p
python scripts/show_detail.py gpurun_out/detail_c4_r02s.json 3
echo "== NO_HTILE"; GBE_FAST_NO_HTILE=1 timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 2,5p
