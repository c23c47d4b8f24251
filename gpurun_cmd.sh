nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
timeout 600 python bench.py --steps 3 --warmup 3 --weights mixed --no-e2e --no-cpu-baseline --no-interp-n > gpurun_out/bench_mixed.log 2>&1; tail -1 gpurun_out/bench_mixed.log
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-interp-n > gpurun_out/bench_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-interp-n > gpurun_out/ncu_launch.log 2>&1
python tools/spread_once.py --N 2e7 --fits 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spread_fused" -s 1 -c 1 -o gpurun_out/prof_fused_v3 python tools/spread_once.py --N 2e7 --fits 2 > gpurun_out/ncu2.log 2>&1
tail -1 gpurun_out/ncu2.log
