# A/B of alternative libgbe builds on C4 (per-bucket times)
for L in "$@"; do echo "== $L"; GBE_LIB=$PWD/paper_1608_05288_b200/$L python scripts/bench_detail.py c4 2>&1 | sed -n 2,6p; done
