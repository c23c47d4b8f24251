"""Shared helpers for the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

import oracle as O
from efgp_data import CONFIGS, generate


def rel(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def model(cfg, **kw):
    from paper_2210_10210_b200 import EFGP
    return EFGP(cfg.kernel, cfg.ell, cfg.sigma, cfg.eps, cfg.d, cfg.nu, **kw)


def gpu_v_full(m_, model_):
    from paper_2210_10210_b200 import half_to_full
    inf = model_.info()
    return half_to_full(model_.vector("v"), inf["m"], inf["d"], K=2 * inf["m"])


def gpu_rhs_full(model_):
    from paper_2210_10210_b200 import half_to_full
    inf = model_.info()
    return half_to_full(model_.vector("rhs"), inf["m"], inf["d"])


def gpu_beta_full(model_):
    from paper_2210_10210_b200 import half_to_full
    inf = model_.info()
    return half_to_full(model_.vector("beta"), inf["m"], inf["d"])


__all__ = ["rel", "dev", "model", "gpu_v_full", "gpu_rhs_full", "gpu_beta_full", "O", "CONFIGS", "generate"]
