"""Worker of tests/test_gpu_multirank.py (one process per GPU, launched by torch.distributed.run).

Each rank fits its index shard of the same c5-shaped data through the library's own NCCL
communicator (efgp_comm_init; the partial modes are summed inside efgp_fit), then rank 0 compares
the multi-rank mu with a single-handle fit of all points.  Second part: rank 1 gets an invalid
coordinate; every rank must return an error (none may hang in the collective)."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from efgp_data import CONFIGS, generate, shard_range  # noqa: E402
from paper_2210_10210_b200 import EFGP, EFGPError  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=dev)
    c = CONFIGS["c5"]
    N = 200_003
    x, y, xt = generate(c, N=N, q=500)
    a, b = shard_range(N, rank, world)
    g = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, cg_tol=1e-10)
    g.comm_init()
    g.fit(torch.from_numpy(x[a:b]).to(dev), torch.from_numpy(y[a:b]).to(dev))
    inf = g.info()
    mu = g.predict(torch.from_numpy(xt).to(dev)).cpu().numpy()
    out = {"rank": rank, "comm_size": inf["comm_size"], "N": inf["N"], "iters": inf["iters"]}
    if rank == 0:
        g1 = EFGP(c.kernel, c.ell, c.sigma, c.eps, c.d, c.nu, cg_tol=1e-10)
        g1.fit(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev))
        ref = g1.predict(torch.from_numpy(xt).to(dev)).cpu().numpy()
        out["mu_rel"] = float(np.linalg.norm(mu - ref) / np.linalg.norm(ref))
        out["v_rel"] = float(np.linalg.norm(g.vector("v") - g1.vector("v")) / np.linalg.norm(g1.vector("v")))
        g1.close()
    # failure on one rank: all ranks error out together
    xb = x[a:b].copy()
    if rank == 1:
        xb[17, 0] = 1.5
    try:
        g.fit(torch.from_numpy(xb).to(dev), torch.from_numpy(y[a:b]).to(dev))
        out["bad_fit"] = "ok"
    except EFGPError as exc:
        out["bad_fit"] = str(exc)[:120]
    g.close()
    allv = [None] * world
    dist.all_gather_object(allv, out)
    if rank == 0:
        print("MULTIRANK " + json.dumps(allv), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
