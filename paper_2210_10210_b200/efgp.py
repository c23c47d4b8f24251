"""Thin Python binding over the C ABI in include/efgp.h (argument marshalling only).

Every step of the EFGP path (spreading, FFTs, deconvolution, Toeplitz CG, interpolation) runs in
libefgp.so's sm_100a kernels and cuFFT.  PyTorch supplies device memory, streams and (for
multi-GPU) the process group used for the one allreduce of partial modes.
"""
from __future__ import annotations

import ctypes as C
import math
import warnings

import numpy as np

from . import _lib as L

_KERNELS = {"se": 0, "matern": 1}
_RESCALE = {"B": 0, "none": 0, "A": 1, "l2": 1, "P": 2, "printed": 2}
_SPREAD = {"auto": 0, "global": 1, "smem": 2, "sorted": 3, "cellsort": 4}
SPREAD_NAMES = {v: k for k, v in _SPREAD.items()}


class EFGPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{L.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _ptr_and_keep(a, dtype=np.float64):
    """(pointer, keep-alive object) for a torch tensor (CUDA or CPU) or a numpy array."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64:
                raise TypeError("EFGP expects float64 tensors")
            if not a.is_contiguous():
                a = a.contiguous()
            return a.data_ptr(), a
    except ImportError:  # pragma: no cover
        pass
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr.ctypes.data, arr


def half_to_full(half: np.ndarray, m: int, d: int, K: int | None = None) -> np.ndarray:
    """Expand a Hermitian-half mode vector (interleaved re/im, j_d >= 0; include/efgp.h layout) to
    the full (2K+1,)*d complex array indexed by j + K, using x_{-j} = conj(x_j)."""
    K = m if K is None else K
    z = half[0::2] + 1j * half[1::2]
    z = z.reshape((2 * K + 1,) * (d - 1) + (K + 1,))
    full = np.zeros((2 * K + 1,) * d, dtype=np.complex128)
    full[..., K:] = z
    neg = np.conj(z[(slice(None, None, -1),) * (d - 1) + (slice(K, 0, -1),)])
    full[..., :K] = neg
    return full


def full_to_half(full: np.ndarray) -> np.ndarray:
    """Inverse of half_to_full for a (2K+1,)*d Hermitian array: interleaved re/im of j_d >= 0."""
    K = (full.shape[0] - 1) // 2
    z = np.ascontiguousarray(full[..., K:]).reshape(-1)
    out = np.empty(2 * z.size)
    out[0::2], out[1::2] = z.real, z.imag
    return out


class EFGP:
    """EFGP regression on one GPU (or one rank of a multi-GPU job).

    kernel: "se" or "matern" (nu >= 1/2); ell, sigma, eps as in the paper (Alg a1); d in {1,2,3}.
    Optional overrides: h and m (both), cg_tol (default eps), max_iter, nufft_tol (default eps/10),
    matern_rescale ("A" true L2 norm, "B" none, "P" printed), spread ("auto"/"global"/"smem"/"sorted"), weights ("fp64"/"fp32"/"mixed": SORTED spreading arithmetic, include/efgp.h).
    """

    def __init__(self, kernel: str, ell: float, sigma: float, eps: float, d: int, nu: float = 0.0, *,
                 h: float | None = None, m: int | None = None, cg_tol: float | None = None,
                 max_iter: int | None = None, nufft_tol: float | None = None, matern_rescale: str = "A",
                 spread: str = "auto", weights: str = "fp64", graph_iters: int | None = None, stream=None, device=None,
                 precond: str | None = None, hetero: str = "auto"):
        import torch
        self._lib = L.load()
        self._torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        opt = L.Options()
        self._lib.efgp_default_options(C.byref(opt))
        if (h is None) != (m is None):
            raise ValueError("h and m must be given together")
        if m is not None:
            opt.h, opt.m = float(h), int(m)
        if cg_tol is not None:
            opt.cg_tol = float(cg_tol)
        if max_iter is not None:
            opt.max_iter = int(max_iter)
        if nufft_tol is not None:
            opt.nufft_tol = float(nufft_tol)
        opt.matern_rescale = _RESCALE[matern_rescale]
        opt.spread_method = _SPREAD[spread]
        opt.spread_weights = {"fp64": 0, "fp32": 1, "mixed": 2}[weights]
        opt.precond = {None: 0, "none": 0, "kron": 1, "auto": 2, "jacobi": 3}[precond]  # NEXT-4 (G12, G12b)
        opt.hetero_method = {"auto": 0, "toeplitz": 1, "nufft": 2}[hetero]  # NEXT-3 (G11, G11b)
        if graph_iters is not None:
            opt.graph_iters = int(graph_iters)
        opt.stream = C.c_void_p(stream.cuda_stream)
        self.kernel, self.ell, self.sigma, self.eps, self.d, self.nu = kernel, ell, sigma, eps, d, nu
        self._h = C.c_void_p()
        with torch.cuda.device(self.device):
            st = self._lib.efgp_setup(C.byref(self._h), _KERNELS[kernel], float(nu), float(ell), float(sigma),
                                      float(eps), int(d), C.byref(opt))
        if st != L.EFGP_OK:
            msg = self._err()
            self.close()
            raise EFGPError(st, msg)
        self.last_status = L.EFGP_OK

    # ------------------------------------------------------------------ helpers
    def _err(self) -> str:
        if not self._h:
            return "no handle"
        s = self._lib.efgp_last_error(self._h)
        return s.decode() if s else ""

    def _check(self, st: int, allow_noconverge: bool = True):
        self.last_status = st
        if st == L.EFGP_OK:
            return
        if st == L.EFGP_ERR_NOCONVERGE and allow_noconverge:
            warnings.warn(f"EFGP: {self._err()}", RuntimeWarning)
            return
        raise EFGPError(st, self._err())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.efgp_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ fit / predict
    def fit(self, x, y):
        """Alg a1 steps 2-4 on this process's points (device or host arrays, fp64, x (N, d))."""
        N = int(x.shape[0])
        px, kx = _ptr_and_keep(x)
        py, ky = _ptr_and_keep(y)
        with self._torch.cuda.device(self.device):
            self._check(self._lib.efgp_fit(self._h, C.c_void_p(px), C.c_void_p(py), N))
        return self

    def fit_hetero(self, x, y, noise_sd):
        """NEXT-3: fit with per-point noise standard deviations noise_sd (N,) (reading G11): solves
        (Phi^* S^-1 Phi + I) beta = Phi^* S^-1 y.  Default solver (hetero="auto"/"toeplitz", reading
        G11b): the weighted Toeplitz system D T(v^w) D + I (v^w from strengths 1/sigma_n^2, one extra
        type-1 pass) with the FFT Toeplitz CG; hetero="nufft": one type-2 + one type-1 NUFFT per CG
        iteration (the BBMM-style product of P:2762-2763)."""
        N = int(x.shape[0])
        px, kx = _ptr_and_keep(x)
        py, ky = _ptr_and_keep(y)
        ps, ks = _ptr_and_keep(noise_sd)
        with self._torch.cuda.device(self.device):
            self._check(self._lib.efgp_fit_hetero(self._h, C.c_void_p(px), C.c_void_p(py), C.c_void_p(ps), N))
        return self

    def modes_count(self) -> int:
        return int(self._lib.efgp_modes_count(self._h))

    def fit_local(self, x, y, modes=None):
        """Spread this rank's shard; returns the device tensor of partial modes (to be summed)."""
        torch = self._torch
        if modes is None:
            modes = torch.empty(self.modes_count(), dtype=torch.float64, device=self.device)
        px, kx = _ptr_and_keep(x)
        py, ky = _ptr_and_keep(y)
        with torch.cuda.device(self.device):
            self._check(self._lib.efgp_fit_local(self._h, C.c_void_p(px), C.c_void_p(py), int(x.shape[0]),
                                                 C.c_void_p(modes.data_ptr())), allow_noconverge=False)
        return modes

    def fit_solve(self, modes, N_total: int):
        with self._torch.cuda.device(self.device):
            self._check(self._lib.efgp_fit_solve(self._h, C.c_void_p(modes.data_ptr()), int(N_total)))
        return self

    def comm_init(self, group=None):
        """Give the library its own NCCL communicator over the torch.distributed group (a 1-rank
        communicator without torch.distributed).  Afterwards fit()/fit_hetero() take this rank's
        shard and sum the partial modes over ranks inside the library (include/efgp.h)."""
        import torch.distributed as dist
        on = dist.is_available() and dist.is_initialized()
        world = dist.get_world_size(group) if on else 1
        rank = dist.get_rank(group) if on else 0
        uid = (C.c_char * 128)()
        if rank == 0:
            self._check(self._lib.efgp_comm_unique_id(uid), allow_noconverge=False)
        if world > 1:
            obj = [bytes(uid)]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(obj, src=src, group=group)
            C.memmove(uid, obj[0], 128)
        with self._torch.cuda.device(self.device):
            self._check(self._lib.efgp_comm_init(self._h, uid, world, rank), allow_noconverge=False)
        return self

    def fit_distributed(self, x, y, group=None):
        """Multi-GPU fit: local spreading, ONE allreduce of the partial modes
        over the process group, replicated CG.  x, y: this rank's shard."""
        import torch.distributed as dist
        torch = self._torch
        modes = self.fit_local(x, y)
        n = torch.tensor([float(x.shape[0])], dtype=torch.float64, device=modes.device)
        dist.all_reduce(modes, group=group)
        dist.all_reduce(n, group=group)
        return self.fit_solve(modes, int(round(n.item())))

    def predict(self, xt, out=None):
        """Posterior mean at targets xt (q, d).  Device tensor in -> device tensor out."""
        torch = self._torch
        q = int(xt.shape[0])
        if out is None:
            dev = xt.device if isinstance(xt, torch.Tensor) else torch.device("cpu")
            out = torch.empty(q, dtype=torch.float64, device=dev)
        px, kx = _ptr_and_keep(xt)
        with torch.cuda.device(self.device):
            self._check(self._lib.efgp_predict(self._h, C.c_void_p(px), q, C.c_void_p(out.data_ptr())),
                        allow_noconverge=False)
        return out

    def predict_var(self, xt, out=None):
        """Posterior variance at targets xt (q, d) (NEXT-2, eqs eta/sws).  Device in -> device out."""
        torch = self._torch
        q = int(xt.shape[0])
        if out is None:
            dev = xt.device if isinstance(xt, torch.Tensor) else torch.device("cpu")
            out = torch.empty(q, dtype=torch.float64, device=dev)
        px, kx = _ptr_and_keep(xt)
        with torch.cuda.device(self.device):
            # EFGP_ERR_NOCONVERGE (a target's CG hit max_iter) warns, as fit does
            self._check(self._lib.efgp_predict_var(self._h, C.c_void_p(px), q, C.c_void_p(out.data_ptr())))
        return out

    # ------------------------------------------------------------------ state
    def info(self) -> dict:
        inf = L.Info()
        self._check(self._lib.efgp_get_info(self._h, C.byref(inf)), allow_noconverge=False)
        d = {k: getattr(inf, k) for k, _ in L.Info._fields_}
        d["spread_method"] = SPREAD_NAMES.get(d["spread_method"], d["spread_method"])
        d["spread_fallback"] = L.FALLBACK_NAMES.get(d["spread_fallback"], d["spread_fallback"])
        return d

    def residual_history(self) -> np.ndarray:
        n = C.c_int64()
        self._lib.efgp_get_residual_history(self._h, None, 0, C.byref(n))
        out = np.empty(n.value)
        self._check(self._lib.efgp_get_residual_history(self._h, out.ctypes.data_as(C.c_void_p), n.value,
                                                         C.byref(n)), allow_noconverge=False)
        return out

    def vector(self, which: str) -> np.ndarray:
        """Hermitian-half vector of the last fit as interleaved doubles: "v", "rhs" or "beta"."""
        idx = {"v": 0, "rhs": 1, "beta": 2}[which]
        cap = self.modes_count()
        buf = np.empty(cap)
        n = self._lib.efgp_copy_vector(self._h, idx, buf.ctypes.data_as(C.c_void_p), cap)
        if n < 0:
            raise EFGPError(L.EFGP_ERR_INVALID, "copy_vector failed")
        return buf[:n].copy()

    def weights(self) -> np.ndarray:
        out = np.empty(int(self._lib.efgp_weights_count(self._h)))
        self._check(self._lib.efgp_get_weights(self._h, out.ctypes.data_as(C.c_void_p)), allow_noconverge=False)
        return out

    def load_weights(self, beta_half) -> "EFGP":
        """Load a Hermitian-half weight vector (numpy array or torch tensor, host or device)."""
        ptr, keep = _ptr_and_keep(beta_half)
        n = keep.numel() if hasattr(keep, "numel") else keep.size
        if n != int(self._lib.efgp_weights_count(self._h)):
            raise ValueError("weights length mismatch")
        with self._torch.cuda.device(self.device):
            self._check(self._lib.efgp_load_weights(self._h, C.c_void_p(ptr)), allow_noconverge=False)
        return self
