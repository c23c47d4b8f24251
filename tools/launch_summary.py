"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name.

    python tools/launch_summary.py gpurun_out/launches.csv [--top 12]
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 12
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        try:
            agg[r[ki].split("(")[0][:60]].append(float(r[vi].replace(",", "")))
        except (ValueError, IndexError):
            pass
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))[:top]:
        print(f"{100 * sum(v) / tot:5.1f}%  n={len(v):5d}  total={sum(v) / 1e6:8.3f} ms  mean={sum(v) / len(v) / 1e3:8.2f} us  {k}")


if __name__ == "__main__":
    main()
