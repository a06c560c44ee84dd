set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ringwrap.py tests/test_gpu_parity.py tests/test_gpu_merge.py -q -x > gpurun_out/pytest_r02g.log 2>&1; tail -2 gpurun_out/pytest_r02g.log
for E in "X=0" "GBE_FAST_NOUT=2" "GBE_FAST_NOUT=1"; do echo "== C4 $E"; env $E timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 1,9p; done
echo "== C5"; timeout 300 python scripts/bench_detail.py c5 2>&1 | sed -n 1,8p
