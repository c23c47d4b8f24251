timeout 300 python tools/spread_sweep.py --N 2e8 --variants '[{}, {"weights":"mixed"}, {"weights":"fp32"}]' 2>&1
