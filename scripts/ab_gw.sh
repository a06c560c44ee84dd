# group-width A/B across configs (kernel sums, timing mode)
for L in libgbe_a.so libgbe_b.so; do for e in "X=1" "GBE_FAST_GW4=1"; do echo "== $L $e"; for w in c4 "c3 16" c5 c2; do env $e GBE_LIB=$PWD/paper_1608_05288_b200/$L python scripts/bench_detail.py $w 2>&1 | grep "kernel sum" | head -1; done; done; done
