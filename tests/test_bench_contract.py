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


def test_gpus_flag_spawns_ranks_with_index_shards():
    # `bench.py --gpus 2` started as one process re-launches itself under torch.distributed.run with
    # two ranks (127.0.0.1); each rank derives its shard with efgp_data.shard_range:
    # contiguous, disjoint, covering [0, N) and [0, q).  --dry-run keeps the ranks on CPU (gloo).
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                        "--N", "1000003", "--q", "777"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                       env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout           # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["N"] == 1000003
    sh = sorted(d["shards"], key=lambda s: s["rank"])
    assert [s["rank"] for s in sh] == [0, 1]
    assert sh[0]["points"][0] == 0 and sh[0]["points"][1] == sh[1]["points"][0] and sh[1]["points"][1] == 1000003
    assert sh[0]["targets"][0] == 0 and sh[0]["targets"][1] == sh[1]["targets"][0] and sh[1]["targets"][1] == 777
    assert abs((sh[0]["points"][1] - sh[0]["points"][0]) - (sh[1]["points"][1] - sh[1]["points"][0])) <= 1
