timeout 400 python tools/spread_sweep.py --N 4e8 --variants '[{}, {"weights": "mixed"}]' 2>&1 | sed 's/.*"weights": "\([a-z0-9]*\)".*"chunk": \([0-9]*\).*pts_per_s": \([0-9.e+]*\).*/\1 chunk=\2 pts\/s=\3/'
timeout 300 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -p no:cacheprovider -x -k "sorted or strategies or c5" 2>&1 | tail -1
