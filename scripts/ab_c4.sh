for cfg in "GBE_FAST_NOUT=2" "GBE_FAST_WANT_STAGES=6" "GBE_FAST_WANT_STAGES=8" "GBE_FAST_PLMAX=2187"; do echo "== $cfg"; env $cfg python scripts/bench_detail.py c4 2>&1 | sed -n 2,7p; done
