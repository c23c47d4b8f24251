"""Two ranks on two GPUs through the library's own NCCL communicator:
runs only where 2 GPUs are visible (the round's GPU boxes have one; the 8-GPU scaling box runs it)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_fit_matches_single_handle():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533",
                        os.path.join(ROOT, "tests", "_multirank_worker.py")],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("MULTIRANK ")][-1]
    res = json.loads(line[len("MULTIRANK "):])
    assert all(o["comm_size"] == 2 and o["N"] == 200_003 for o in res)
    assert res[0]["iters"] == res[1]["iters"]                 # replicated CG
    assert res[0]["v_rel"] < 1e-12 and res[0]["mu_rel"] < 1e-8
    assert all(o["bad_fit"] != "ok" for o in res)             # both ranks report the failure, none hangs
