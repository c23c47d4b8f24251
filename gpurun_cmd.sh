timeout 600 python -m pytest tests -m gpu -q --timeout 120 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/spread_sweep.py --N 2e8 --variants '[{}, {"weights":"mixed"}, {"EFGP_SORTED_CHUNK": 8388608}, {"weights":"mixed", "EFGP_SORTED_CHUNK": 8388608}]' > gpurun_out/sweep.log 2>&1; cat gpurun_out/sweep.log
