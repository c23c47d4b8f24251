# A/B of two builds of libefgp.so on the c5 spreading (two interleaved rounds):
#   cp build_A.so libv_old.so; cp build_B.so libv_new.so; gpurun -- bash tools/ab_spread.sh
for r in 1 2; do for v in old new; do echo "== $v $(EFGP_LIB=$PWD/libv_$v.so python tools/spread_sweep.py --N 4e8 | sed 's/.*pts_per_s": //')"; done; done
