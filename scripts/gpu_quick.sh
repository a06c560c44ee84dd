# development pass: per-bucket timing of C4, bench line, GPU tests
set -u
mkdir -p gpurun_out
python scripts/bench_detail.py c4 2>&1 | head -12
if [ -n "${AB:-}" ]; then env $AB python scripts/bench_detail.py c4 2>&1 | head -8; fi
python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
if [ "${1:-}" != "notest" ]; then python -m pytest tests -m gpu -x -q > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log; fi
