# merge-threshold A/B on C3 MBE(16) and C4 (kernel sums, timing mode)
for m in 22 27 30; do echo "== merge min 2^$m"; GBE_MERGE_MIN_LOG2=$m python scripts/bench_detail.py c3 16 2>&1 | sed -n 1,2p; GBE_MERGE_MIN_LOG2=$m python scripts/bench_detail.py c4 2>&1 | sed -n 1,2p; done
