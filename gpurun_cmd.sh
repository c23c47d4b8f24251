for CH in 4194304 16777216 67108864; do
python tools/spread_once.py --N 1.34e8 --fits 2 --weights mixed > gpurun_out/plain_$CH.log 2>&1
EFGP_SORTED_CHUNK=$CH ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ch$CH.csv -k regex:"k_bin5|k_tiles4" python tools/spread_once.py --N 1.34e8 --fits 1 --weights mixed > gpurun_out/ncu_$CH.log 2>&1
done
for W in fp64 fp32; do EFGP_SORTED_CHUNK=16777216 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_w$W.csv -k regex:"k_bin5|k_tiles4" python tools/spread_once.py --N 1.34e8 --fits 1 --weights $W > gpurun_out/ncu_w$W.log 2>&1; done
