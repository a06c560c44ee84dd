set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_spill.py tests/test_gpu_hostargs.py -q -x > gpurun_out/pytest_spill_r02e.log 2>&1; tail -3 gpurun_out/pytest_spill_r02e.log
DETAIL_JSON=gpurun_out/detail_c4_r02e.json timeout 300 python scripts/bench_detail.py c4 > /dev/null 2>&1
python scripts/show_detail.py gpurun_out/detail_c4_r02e.json 8
bash scripts/sanitize.sh
