"""N > 1 orchestration on CPU (gloo, world_size 2): the multi-GPU decomposition of DESIGN.md §8.

Each rank takes its index shard (efgp_data.shard_range), computes partial modes, the binding's
EFGP.fit_distributed sums them (and N) with ONE all_reduce and hands the sum to fit_solve.  On CPU
the two device calls are stood in for by the oracle (test-only injection), so what is tested is the
binding's host logic: shard ranges, the all_reduce payload and the call sequence.  The result must
equal the single-process oracle fit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from efgp_data import CONFIGS, generate, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _CPUStandIn:
    """Replaces EFGP.fit_local / fit_solve with the oracle's sums (test infrastructure only)."""

    def __init__(self, cfg, h, m):
        self.cfg, self.h, self.m = cfg, h, m
        self.D = O.spectral_weights(cfg.kernel, cfg.ell, cfg.d, h, m, cfg.nu)
        self._torch = torch

    def fit_local(self, x, y):
        v = O.toeplitz_vector(x.numpy(), self.h, self.m)
        fy = O.rhs_Fy(x.numpy(), y.numpy(), self.h, self.m)
        flat = np.concatenate([v.ravel(), fy.ravel()])
        return torch.from_numpy(np.stack([flat.real, flat.imag], -1).ravel().copy())

    def fit_solve(self, modes, N_total):
        z = modes.numpy()[0::2] + 1j * modes.numpy()[1::2]
        nv = (4 * self.m + 1) ** self.cfg.d
        v = z[:nv].reshape((4 * self.m + 1,) * self.cfg.d)
        b = self.D * z[nv:].reshape((2 * self.m + 1,) * self.cfg.d)
        self.N_total = N_total
        self.beta, self.iters, _ = O.cg(lambda p: O.system_apply(v, self.D, self.cfg.sigma ** 2, p), b, 1e-12, 100000)

        return self


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2210_10210_b200.efgp import EFGP
    c = CONFIGS["c5"]
    N = 3001
    x, y, _ = generate(c, N=N, q=1)
    a, b = shard_range(N, rank, world)
    h, m = 0.62, 8
    stand = _CPUStandIn(c, h, m)
    # the binding's own fit_distributed, bound to the stand-in
    EFGP.fit_distributed(stand, torch.from_numpy(x[a:b]), torch.from_numpy(y[a:b]))
    out[rank] = (stand.N_total, stand.beta.copy())
    dist.destroy_process_group()


def test_fit_distributed_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    c = CONFIGS["c5"]
    x, y, _ = generate(c, N=3001, q=1)
    ref = O.efgp_fit(x, y, c.kernel, c.ell, c.sigma, c.eps, nu=c.nu, h=0.62, m=8, cg_tol=1e-12, max_iter=100000)
    for r in range(2):
        N_total, beta = out[r]
        assert N_total == 3001
        np.testing.assert_allclose(beta, ref.beta, rtol=1e-9, atol=1e-12 * np.abs(ref.beta).max())


def test_shard_ranges_partition():
    for N in (1, 7, 1000, 10 ** 9 + 3):
        for G in (1, 2, 3, 8):
            r = [shard_range(N, g, G) for g in range(G)]
            assert r[0][0] == 0 and r[-1][1] == N
            assert all(r[i][1] == r[i + 1][0] for i in range(G - 1))
            assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1
