for r in 1 2; do for v in old new; do echo "== $v $(EFGP_LIB=$PWD/libv_$v.so python tools/spread_sweep.py --N 4e8 | sed 's/.*pts_per_s": //')"; done; done
