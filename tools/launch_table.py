"""Per-kernel mean of an ncu --metrics CSV launch list (time in us, DRAM bytes in MB).
    python tools/launch_table.py gpurun_out/launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
sc = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3,
      "Mbyte": 1, "Gbyte": 1e3}
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg[r[ki][:48]][r[mi]].append(float(r[vi].replace(",", "")) * sc.get(r[ui], 1.0))
for k, d in sorted(agg.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", [0]))):
    t = d.get("gpu__time_duration.sum", [0])
    line = f"{k:50s} n={len(t):3d} mean_us={sum(t) / len(t):9.1f}"
    for m, lab in (("dram__bytes_read.sum", "rd_MB"), ("dram__bytes_write.sum", "wr_MB")):
        if m in d:
            line += f" {lab}={sum(d[m]) / len(d[m]):8.1f}"
    print(line)
