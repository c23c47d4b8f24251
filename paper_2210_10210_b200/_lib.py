"""ctypes loader for libefgp.so (argument marshalling only; no computation happens in Python).

The product path has no CPU fallback: if the shared library is missing this raises at import of
the binding, and efgp_setup itself fails with EFGP_ERR_CUDA when no device is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EFGP_LIB", os.path.join(HERE, "libefgp.so"))  # override: A/B builds

FALLBACK_NAMES = {0: "none", 1: "unaligned", 2: "coresidency", 3: "too_many_points"}
EFGP_OK, EFGP_ERR_NOCONVERGE, EFGP_ERR_INVALID, EFGP_ERR_RESOURCE, EFGP_ERR_CUDA, EFGP_ERR_NCCL = range(6)
STATUS_NAMES = {0: "EFGP_OK", 1: "EFGP_ERR_NOCONVERGE", 2: "EFGP_ERR_INVALID", 3: "EFGP_ERR_RESOURCE",
                4: "EFGP_ERR_CUDA", 5: "EFGP_ERR_NCCL"}


class Options(C.Structure):
    _fields_ = [("h", C.c_double), ("m", C.c_int64), ("cg_tol", C.c_double), ("max_iter", C.c_int64),
                ("nufft_tol", C.c_double), ("matern_rescale", C.c_int), ("spread_method", C.c_int),
                ("graph_iters", C.c_int), ("spread_weights", C.c_int), ("precond", C.c_int),
                ("hetero_method", C.c_int), ("stream", C.c_void_p)]


class Info(C.Structure):
    _fields_ = [("h", C.c_double), ("m", C.c_int64), ("M", C.c_int64), ("d", C.c_int64), ("N", C.c_int64),
                ("iters", C.c_int64), ("rel_resid", C.c_double), ("cg_tol", C.c_double),
                ("max_iter", C.c_int64), ("nf1", C.c_int64), ("nf2", C.c_int64), ("L", C.c_int64),
                ("w", C.c_int64), ("beta_es", C.c_double), ("nufft_tol", C.c_double),
                ("spread_method", C.c_int), ("t_spread_ms", C.c_double), ("t_modes_ms", C.c_double),
                ("t_solve_ms", C.c_double), ("t_predict_ms", C.c_double), ("sorted_t1", C.c_int64),
                ("sorted_t2", C.c_int64), ("sorted_chunk", C.c_int64), ("sorted_round", C.c_int64),
                ("spread_precision", C.c_int64), ("t_var_ms", C.c_double), ("var_iters_max", C.c_int64),
                ("var_batch", C.c_int64), ("hetero_sorted", C.c_int64),
                ("precond", C.c_int64), ("comm_size", C.c_int64), ("spread_fallback", C.c_int64),
                ("cg_persist_split", C.c_int64), ("cg_dft2", C.c_int64)]


# every symbol include/efgp.h declares, with (restype, argtypes)
SIGNATURES = {
    "efgp_abi_version": (C.c_int, []),
    "efgp_default_options": (None, [C.POINTER(Options)]),
    "efgp_setup": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                             C.c_int, C.POINTER(Options)]),
    "efgp_fit": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    "efgp_fit_hetero": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    "efgp_modes_count": (C.c_int64, [C.c_void_p]),
    "efgp_comm_unique_id": (C.c_int, [C.c_void_p]),
    "efgp_comm_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "efgp_fit_local": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "efgp_fit_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "efgp_predict": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "efgp_predict_var": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "efgp_weights_count": (C.c_int64, [C.c_void_p]),
    "efgp_get_weights": (C.c_int, [C.c_void_p, C.c_void_p]),
    "efgp_load_weights": (C.c_int, [C.c_void_p, C.c_void_p]),
    "efgp_copy_vector": (C.c_int64, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]),
    "efgp_get_info": (C.c_int, [C.c_void_p, C.POINTER(Info)]),
    "efgp_get_residual_history": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]),
    "efgp_debug_trace": (C.c_int64, [C.c_void_p, C.c_void_p, C.c_int64]),
    "efgp_last_error": (C.c_char_p, [C.c_void_p]),
    "efgp_destroy": (None, [C.c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libefgp.so (built in-tree by paper_2210_10210_b200.build); raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libefgp.so not found at {path}: run `python -m paper_2210_10210_b200.build` "
                           "(the EFGP product path has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
