"""Aggregate ncu warp-stall samples of one kernel by CUDA source line (needs -lineinfo).

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep k_tiles3 [--top 40]
"""
import csv
import io
import os
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
    rows, fname, hdr, total = [], "?", None, 0
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0] or r[0] in ("Function Name",):
            continue
        try:
            w = int(r[4] or 0)
            e = int(r[7] or 0)
        except (ValueError, IndexError):
            continue
        total += w
        rows.append((w, e, f"{fname}:{r[0]}", r[1].strip()[:100]))
    rows.sort(key=lambda t: -t[0])
    for w, e, loc, src in rows[:top]:
        print(f"{100.0 * w / max(total, 1):6.2f}%  inst={e:9d}  {loc:26s} {src}")


if __name__ == "__main__":
    main()
