set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_merge.py tests/test_gpu_parity.py tests/test_gpu_ringwrap.py -q -x > gpurun_out/pytest_r02x.log 2>&1; tail -2 gpurun_out/pytest_r02x.log
for E in "X=0" "GBE_MERGE_GENERIC=1"; do echo "== C4 $E"; env $E timeout 300 python scripts/bench_detail.py c4 2>&1 | sed -n 2,7p; done
echo "== C4-d4"; timeout 300 python scripts/bench_detail.py c4d4 2>&1 | sed -n 2,4p
timeout 600 python bench.py --steps 10 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
