# The round-end evidence run (one gpurun call): GPU suite, smoke, bench, per-config table (plain and
# preconditioned), the bench launch list, one ncu --set full capture of K9.  bash tools/final_gpu_run.sh
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/f_gpu_suite.log 2>&1; echo suite_exit=$? >> gpurun_out/f_gpu_suite.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/f_smoke.log
python bench.py > gpurun_out/f_bench.jsonl 2> gpurun_out/f_bench.err; echo bench_exit=$? >> gpurun_out/f_bench.err
python tools/bench_configs.py > gpurun_out/f_configs.jsonl 2> gpurun_out/f_configs.err
python tools/bench_configs.py --precond auto > gpurun_out/f_configs_auto.jsonl 2> gpurun_out/f_configs_auto.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-interp-n --no-variance --no-hetero --no-precond --no-spread-variants --no-cpu-baseline > gpurun_out/f_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_interp2_copies -c 1 -o gpurun_out/f_k9_full python tools/interp_ab.py --q 2e8 --reps 1 --variants c4 > gpurun_out/f_k9_ncu.log 2>&1
