set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_htile.py tests/test_gpu_ringwrap.py -q -x > gpurun_out/pytest_r02u.log 2>&1; tail -2 gpurun_out/pytest_r02u.log; grep -E "^E " gpurun_out/pytest_r02u.log | head -5
for E in "X=0" "GBE_FAST_STORE_DEPTH=3" "GBE_FAST_NO_HTILE=1" "GBE_FAST_NO_HTILE=1 GBE_FAST_STORE_DEPTH=2"; do echo "== C4 $E"; env $E timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 2,7p; done
