set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/pytest_r02h.log 2>&1; tail -3 gpurun_out/pytest_r02h.log; grep -E "^E " gpurun_out/pytest_r02h.log | head -5
for E in "X=0" "GBE_STREAM_NO_BD=1"; do echo "== C5 $E"; env $E timeout 300 python scripts/bench_detail.py c5 2>&1 | sed -n 1,12p; done
for E in "X=0" "GBE_KERNEL_POLICY=stream"; do echo "== C4 $E"; env $E timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 1,8p; done
