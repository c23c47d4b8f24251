# A/B of library builds on the c5 spreading: bash tools/ab_lib.sh N lib1 lib2 ...  (interleaved, 2 rounds)
N=${1:-1e9}; shift
for r in 1 2; do for v in "$@"; do echo "== $v $(EFGP_LIB=$PWD/$v python tools/spread_once.py --N $N --fits 3 | tail -1)"; done; done
