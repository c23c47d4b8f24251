"""The five BASELINE.json workloads as seeded synthetic input recipes (DESIGN.md
"Input recipe").  Input generation only: no EFGP arithmetic lives here.

Each config gives kernel hyper-parameters, sizes and a generator of (x, y, targets) for any index
range [start, stop), so that shards (multi-GPU) and chunks (streaming oracle checks) regenerate
exactly the same records.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import philox

MIX_MEANS = np.array([[0.3, 0.3], [0.7, 0.5], [0.5, 0.8]])


@dataclass(frozen=True)
class Config:
    name: str
    kernel: str          # "se" | "matern"
    nu: float
    ell: float
    sigma: float
    eps: float
    d: int
    N: int
    q: int
    seed: int
    points: str          # "uniform" | "mixture"
    targets: str         # "equispaced" | "uniform"
    func: str            # test-function id
    noise: float

    @property
    def id(self) -> int:
        return int(self.name[1:])


CONFIGS = {
    "c1": Config("c1", "se", 0.0, 0.1, 0.1, 1e-6, 1, 10_000, 1_000, 0, "uniform", "equispaced", "f1", 0.1),
    "c2": Config("c2", "matern", 1.5, 0.1, 0.1, 1e-4, 2, 1_000_000, 10_000, 1, "uniform", "uniform", "f2", 0.1),
    "c3": Config("c3", "se", 0.0, 0.05, 0.3, 1e-6, 2, 10_000_000, 100_000, 2, "mixture", "uniform", "f3", 0.3),
    "c4": Config("c4", "matern", 0.5, 0.2, 0.1, 1e-3, 3, 10_000_000, 100_000, 3, "uniform", "uniform", "f4", 0.1),
    "c5": Config("c5", "matern", 1.5, 0.1, 0.1, 1e-3, 2, 1_000_000_000, 1_000_000, 4, "uniform", "uniform", "f2", 0.1),
}


def test_function(func: str, x: np.ndarray) -> np.ndarray:
    """Noise-free signal of each config (BASELINE.json configs)."""
    if func == "f1":
        return np.sin(6 * math.pi * x[:, 0]) + np.cos(2 * math.pi * x[:, 0]) ** 2
    if func == "f2":
        return np.sin(6 * math.pi * x[:, 0]) * np.cos(4 * math.pi * x[:, 1])
    if func == "f3":
        r2 = (x[:, 0] - 0.5) ** 2 + (x[:, 1] - 0.5) ** 2
        return np.exp(-r2 / 0.02)
    if func == "f4":
        return (np.sin(4 * math.pi * x[:, 0]) * np.sin(4 * math.pi * x[:, 1])
                * np.sin(4 * math.pi * x[:, 2]))
    raise ValueError(func)


def points(cfg: Config, start: int = 0, stop: int | None = None) -> np.ndarray:
    """Training points x_n, n in [start, stop), shape (n, d), row-major fp64 in [0, 1]^d."""
    stop = cfg.N if stop is None else stop
    idx = np.arange(start, stop, dtype=np.uint64)
    if cfg.points == "uniform":
        return np.stack([philox.uniform(cfg.seed, philox.STREAM_POINTS, idx, k) for k in range(cfg.d)], axis=1)
    # c3: equal-weight 3-component mixture, sd 0.1, clipped (clamped) to [0, 1]^2 (reading G13)
    comp = np.floor(3.0 * philox.uniform(cfg.seed, philox.STREAM_COMPONENT, idx, 0)).astype(np.int64)
    comp = np.minimum(comp, 2)
    off = np.stack([philox.normal(cfg.seed, philox.STREAM_POINTS, idx, 2 * k) for k in range(cfg.d)], axis=1)
    return np.clip(MIX_MEANS[comp] + 0.1 * off, 0.0, 1.0)


def observations(cfg: Config, x: np.ndarray, start: int = 0) -> np.ndarray:
    """y_n = f(x_n) + noise * N(0, 1), noise from stream 1 of the same record index."""
    idx = np.arange(start, start + len(x), dtype=np.uint64)
    return test_function(cfg.func, x) + cfg.noise * philox.normal(cfg.seed, philox.STREAM_NOISE, idx, 0)


def targets(cfg: Config, start: int = 0, stop: int | None = None) -> np.ndarray:
    """Targets x*: c1 equispaced t_i = i/(q-1) incl. endpoints (reading G8); else iid uniform
    from stream 2."""
    stop = cfg.q if stop is None else stop
    if cfg.targets == "equispaced":
        return (np.arange(start, stop, dtype=np.float64) / (cfg.q - 1))[:, None]
    idx = np.arange(start, stop, dtype=np.uint64)
    return np.stack([philox.uniform(cfg.seed, philox.STREAM_TARGETS, idx, k) for k in range(cfg.d)], axis=1)


def generate(cfg: Config, N: int | None = None, q: int | None = None, start: int = 0):
    """(x, y, xt) for the first N points (from `start`) and first q targets; defaults = full config."""
    N = cfg.N if N is None else N
    q = cfg.q if q is None else q
    x = points(cfg, start, start + N)
    y = observations(cfg, x, start)
    return x, y, targets(cfg, 0, q)


def shard_range(N: int, rank: int, world: int):
    """Rank g holds record indices [g N / G, (g+1) N / G)."""
    return (rank * N) // world, ((rank + 1) * N) // world
