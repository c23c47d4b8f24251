"""Device-side input generator (efgp_data/csrc/efgp_datagen.cu): the same Philox streams and config
recipes as efgp_data.configs, written straight into CUDA tensors.  Input generation only."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "efgp_datagen.cu")
LIB = os.path.join(HERE, "libefgp_datagen.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
               "-Xcompiler", "-fPIC", "-shared", SRC, "-o", LIB]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(r.stdout + r.stderr)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} missing: run __graft_entry__.build()")
        _lib = C.CDLL(LIB)
        _lib.efgp_datagen_points.restype = C.c_int
        _lib.efgp_datagen_points.argtypes = [C.c_int, C.c_uint32, C.c_int, C.c_int64, C.c_int64, C.c_double,
                                             C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.efgp_datagen_targets.restype = C.c_int
        _lib.efgp_datagen_targets.argtypes = [C.c_uint32, C.c_int, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
    return _lib


def generate_points(cfg, start: int, count: int, x=None, y=None, device=None):
    """(x, y) CUDA float64 tensors for records [start, start+count) of config cfg."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    if x is None:
        x = torch.empty((count, cfg.d), dtype=torch.float64, device=dev)
    if y is None:
        y = torch.empty(count, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    err = _load().efgp_datagen_points(cfg.id, cfg.seed, cfg.d, start, count, cfg.noise, C.c_void_p(x.data_ptr()),
                                      C.c_void_p(y.data_ptr()), C.c_void_p(st))
    if err:
        raise RuntimeError(f"datagen CUDA error {err}")
    return x, y


def generate_targets(cfg, start: int, count: int, out=None, device=None):
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    if cfg.targets == "equispaced":   # tiny: take the host recipe verbatim (same rounding)
        from .configs import targets
        return torch.from_numpy(targets(cfg, start, start + count)).to(dev)
    if out is None:
        out = torch.empty((count, cfg.d), dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    err = _load().efgp_datagen_targets(cfg.seed, cfg.d, start, count, C.c_void_p(out.data_ptr()), C.c_void_p(st))
    if err:
        raise RuntimeError(f"datagen CUDA error {err}")
    return out
