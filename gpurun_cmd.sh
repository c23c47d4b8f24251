timeout 300 python tools/spread_sweep.py --N 2e8 --variants '[{}, {"weights":"mixed"}]' 2>&1
timeout 300 python tools/interp_once.py --q 1e9 2>&1 | tail -3
