timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 400 -p no:cacheprovider -k "variance" 2>&1 | tail -15
