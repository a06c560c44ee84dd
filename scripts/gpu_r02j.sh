set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/pytest_r02j.log 2>&1; tail -2 gpurun_out/pytest_r02j.log
for E in "X=0" "GBE_STREAM_V4=0"; do echo "== C5 $E"; env $E timeout 300 python scripts/bench_detail.py c5 2>&1 | sed -n 1,7p; done
for E in "GBE_FAST_WANT_STAGES=6" "GBE_FAST_WANT_STAGES=8" "GBE_FAST_PLMAX=729"; do echo "== C4 $E"; env $E timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 1,9p; done
timeout 600 python scripts/bench_domains.py > gpurun_out/domains_r02j.jsonl 2>&1; cat gpurun_out/domains_r02j.jsonl
