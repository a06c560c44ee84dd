set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spill.py tests/test_gpu_ringwrap.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_r02f.log 2>&1; tail -3 gpurun_out/pytest_r02f.log
for E in "X=0" "GBE_FAST_NO_QPERM=1"; do echo "== C4 $E"; env $E timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 1,9p; done
bash scripts/ab_c5.sh
