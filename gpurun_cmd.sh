timeout 300 python tools/spread_sweep.py --N 2e8 --variants '[{}, {"EFGP_SORTED_DEBUG": 1}]' 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -p no:cacheprovider -x -k "sorted or strategies or invalid" 2>&1 | tail -2
