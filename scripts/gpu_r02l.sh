set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -q -x > gpurun_out/pytest_r02l.log 2>&1; tail -2 gpurun_out/pytest_r02l.log
timeout 600 python scripts/bench_domains.py > gpurun_out/domains_r02l.jsonl 2>&1; cut -c1-160 gpurun_out/domains_r02l.jsonl
GBE_STREAM_UNL=1 timeout 600 python scripts/bench_domains.py 2>&1 | cut -c1-120
for E in "X=0" "GBE_KERNEL_POLICY=tiled"; do echo "== C4-d4 $E"; env $E timeout 300 python scripts/bench_detail.py c4d4 2>&1 | sed -n 1,6p; done
WL=c4d4 KREGEX=bk_stream PROF_VARIANT=2 GBE_KERNEL_POLICY=stream bash scripts/gpu_prof.sh r02l 0
