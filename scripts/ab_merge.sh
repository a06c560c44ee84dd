# merge-policy A/B (kernel sums, timing mode): C4-alt, C3 MBE(16), C4
for v in 32 128 512; do echo "== cap C/$v"; for w in c4alt "c3 16" c4; do GBE_MERGE_CAP_DIV=$v python scripts/bench_detail.py $w 2>&1 | grep "kernel sum" | head -1; done; done
