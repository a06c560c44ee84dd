# tuning-knob sweep on C4 (kernel sums, timing mode)
for e in "X=1" "GBE_FAST_NOUT=2" "GBE_FAST_WANT_STAGES=2" "GBE_FAST_WANT_STAGES=6" "GBE_FAST_PLMAX=729"; do
  echo "== $e"; env $e timeout 120 python scripts/bench_detail.py c4 2>&1 | grep "kernel sum" | head -1
done
