"""bench.py's reference arm (the oracle on the host cores) prints the contract's JSON line on CPU:
metric, unit, value, the same workload as the GPU arm, cpu_baseline and e2e objects."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--oracle-points", "5e3"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["metric"].startswith("EFGP fit+predict") and d["unit"] == "points/s"
    assert d["config"]["workload"].startswith("c5: 2D Matern-1.5") and d["config"]["N"] == 10 ** 9
    assert d["config"]["sample"]["N"] == 5000
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
