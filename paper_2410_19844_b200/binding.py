"""Thin Python binding of the C ABI in include/sos_b200.h.

Argument marshalling only: torch is used for device memory and the current
CUDA stream; every arithmetic step runs in libsos_b200.so.  If the library is
missing or no sm_100 device is present, calls raise -- there is no fallback.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsos_b200.so")

SOS_OPT_GD = 0
SOS_OPT_ADAM = 1

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64


class SosError(RuntimeError):
    pass


class _OptParams(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("lr", ctypes.c_float), ("beta1", ctypes.c_float),
                ("beta2", ctypes.c_float), ("eps", ctypes.c_float)]


class _PlanOpts(ctypes.Structure):
    _fields_ = [("split", ctypes.c_int), ("vtq_from_update", ctypes.c_int), ("vtq_in_aux", ctypes.c_int),
                ("rmax_direct", ctypes.c_int), ("narrow_tiles", ctypes.c_int), ("tile_w", ctypes.c_int),
                ("r_headroom", ctypes.c_int), ("tiny", ctypes.c_int)]


_lib = None

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "sos_last_error": [],
    "sos_version": [],
    "sos_build_index": [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)],
    "sos_index_destroy": [_vp],
    "sos_index_dims": [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
    "sos_index_alpha": [_vp, _vp, _vp],
    "sos_index_beta": [_vp, _vp, _vp],
    "sos_index_pair_ranks": [_vp, _vp, _vp, _i64, _vp, _vp],
    "sos_plan_create": [_vp, _i64, ctypes.POINTER(_vp)],
    "sos_plan_create_ex": [_vp, _i64, ctypes.POINTER(_PlanOpts), ctypes.POINTER(_vp)],
    "sos_plan_destroy": [_vp],
    "sos_plan_launch_count": [_vp],
    "sos_plan_timing": [_vp, ctypes.c_int],
    "sos_plan_timing_read": [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64)],
    "sos_forward": [_vp, _vp, _vp, _vp],
    "sos_backward": [_vp, _vp, _vp, _vp, _vp],
    "sos_loss_grad": [_vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "sos_opt_init": [_vp, ctypes.POINTER(_OptParams), _vp],
    "sos_opt_set_lr": [_vp, ctypes.c_float],
    "sos_opt_set_stop": [_vp, ctypes.c_double],
    "sos_step": [_vp, _vp, _vp, _vp, _vp],
    "sos_descend": [_vp, _vp, _vp, _i64, _vp, _vp],
    "sos_solve_host": [_vp, _vp, _vp, _i64, _vp],
}
_RESTYPES = {"sos_last_error": ctypes.c_char_p, "sos_plan_launch_count": _i64}


def load(path: str = LIB_PATH):
    """Load libsos_b200.so (raises if it is missing -- no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise SosError(f"{path} not built; run `python -m paper_2410_19844_b200.build`")
        L = ctypes.CDLL(path)
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise SosError(f"libsos_b200 error {rc}: {load().sos_last_error().decode()}")


def _stream():
    return _vp(torch.cuda.current_stream().cuda_stream)


def _dev_f32(t: torch.Tensor, name: str, numel: Optional[int] = None) -> torch.Tensor:
    if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise SosError(f"{name} must be a contiguous float32 CUDA tensor")
    if numel is not None and t.numel() != numel:
        raise SosError(f"{name} must have {numel} elements, got {t.numel()}")
    return t


def _dev_f64_out(t: torch.Tensor, name: str, min_numel: int) -> torch.Tensor:
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise SosError(f"{name} must be a contiguous float64 CUDA tensor")
    if t.numel() < min_numel:
        raise SosError(f"{name} needs at least {min_numel} elements, got {t.numel()}")
    return t


class SosIndex:
    """Monomial index for n variables, half-degree d."""

    def __init__(self, n: int, d: int):
        L = load()
        h = _vp()
        _check(L.sos_build_index(n, d, ctypes.byref(h)))
        self._h = h
        self.n, self.d = n, d
        N, M = _i64(), _i64()
        _check(L.sos_index_dims(h, ctypes.byref(N), ctypes.byref(M)))
        self.N, self.M = N.value, M.value

    def close(self):
        if getattr(self, "_h", None):
            load().sos_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def alpha(self) -> torch.Tensor:
        out = torch.empty((self.N, self.n), dtype=torch.uint8, device="cuda")
        _check(load().sos_index_alpha(self._h, _vp(out.data_ptr()), _stream()))
        return out

    def beta(self) -> torch.Tensor:
        out = torch.empty((self.M, self.n), dtype=torch.uint8, device="cuda")
        _check(load().sos_index_beta(self._h, _vp(out.data_ptr()), _stream()))
        return out

    def pair_ranks(self, i: torch.Tensor, j: torch.Tensor) -> torch.Tensor:
        if i.numel() != j.numel():
            raise SosError(f"i and j must have the same length, got {i.numel()} and {j.numel()}")
        i = i.to(device="cuda", dtype=torch.int64).contiguous()
        j = j.to(device="cuda", dtype=torch.int64).contiguous()
        out = torch.empty(i.numel(), dtype=torch.int32, device="cuda")
        _check(load().sos_index_pair_ranks(self._h, _vp(i.data_ptr()), _vp(j.data_ptr()), i.numel(),
                                           _vp(out.data_ptr()), _stream()))
        return out


class SosPlan:
    """Workspaces for one (index, r); the hot-path calls of the C ABI.

    Keyword options (sos_plan_opts: None = the library's choice by size, else
    True / False): split, vtq_from_update, vtq_in_aux, rmax_direct,
    narrow_tiles, r_headroom, tiny; tile_w (None, or a multiple of 16 in [16, 160]) -- implementation
    variants of the same step."""

    OPTS = ("split", "vtq_from_update", "vtq_in_aux", "rmax_direct", "narrow_tiles", "tile_w", "r_headroom", "tiny")

    def __init__(self, index: SosIndex, r: int, **opts):
        bad = set(opts) - set(self.OPTS)
        if bad:
            raise SosError(f"unknown plan options {sorted(bad)}")
        self.index = index
        self.r = r
        h = _vp()
        o = _PlanOpts(*[-1 if opts.get(k) is None else (int(opts[k]) if k == "tile_w" else int(bool(opts[k])))
                        for k in self.OPTS])
        _check(load().sos_plan_create_ex(index._h, r, ctypes.byref(o), ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            load().sos_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch_count(self) -> int:
        return int(load().sos_plan_launch_count(self._h))

    KERNELS = ("vmax", "pack_v", "gemm_fwd", "residual", "rmax", "pack_r", "gemm_bwd", "update", "mid", "tiny")

    def timing(self, enable: bool):
        """Start (clears old records) / stop per-kernel CUDA-event timing."""
        _check(load().sos_plan_timing(self._h, 1 if enable else 0))

    def timing_read(self) -> dict:
        """{kernel name: (total ms, launches)} over the recorded launches."""
        out = {}
        for k, name in enumerate(self.KERNELS):
            ms, cnt = ctypes.c_double(), _i64()
            _check(load().sos_plan_timing_read(self._h, k, ctypes.byref(ms), ctypes.byref(cnt)))
            out[name] = (ms.value, cnt.value)
        return out

    def _V(self, V):
        _dev_f32(V, "V")
        if tuple(V.shape) != (self.index.N, self.r):
            raise SosError(f"V must be {self.index.N} x {self.r}, got {tuple(V.shape)}")
        return V

    def forward(self, V: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        self._V(V)
        coef = out if out is not None else torch.empty(self.index.M, dtype=torch.float32, device="cuda")
        _dev_f32(coef, "out", self.index.M)
        _check(load().sos_forward(self._h, _vp(V.data_ptr()), _vp(coef.data_ptr()), _stream()))
        return coef

    def backward(self, V: torch.Tensor, res: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        self._V(V)
        _dev_f32(res, "res", self.index.M)
        grad = out if out is not None else torch.empty_like(V)
        _dev_f32(grad, "out", V.numel())
        _check(load().sos_backward(self._h, _vp(V.data_ptr()), _vp(res.data_ptr()), _vp(grad.data_ptr()), _stream()))
        return grad

    def loss_grad(self, V: torch.Tensor, p: torch.Tensor, want_grad: bool = True,
                  want_res: bool = False) -> Tuple[torch.Tensor, Optional[torch.Tensor], Optional[torch.Tensor]]:
        self._V(V)
        _dev_f32(p, "p", self.index.M)
        loss = torch.empty(1, dtype=torch.float64, device="cuda")
        grad = torch.empty_like(V) if want_grad else None
        res = torch.empty(self.index.M, dtype=torch.float32, device="cuda") if want_res else None
        _check(load().sos_loss_grad(self._h, _vp(V.data_ptr()), _vp(p.data_ptr()), _vp(loss.data_ptr()),
                                    _vp(grad.data_ptr()) if grad is not None else None,
                                    _vp(res.data_ptr()) if res is not None else None, _stream()))
        return loss, grad, res

    def opt_init(self, kind: str = "adam", lr: float = 1e-3, beta1: float = 0.9, beta2: float = 0.999,
                 eps: float = 1e-8):
        prm = _OptParams({"gd": SOS_OPT_GD, "adam": SOS_OPT_ADAM}[kind], lr, beta1, beta2, eps)
        _check(load().sos_opt_init(self._h, ctypes.byref(prm), _stream()))

    def set_lr(self, lr: float):
        """New learning rate for the next steps; optimiser state is kept."""
        _check(load().sos_opt_set_lr(self._h, lr))

    def set_stop(self, rel_tol: float):
        """Device-side stopping rule: once ||coef - p||^2 <= rel_tol ||p||^2,
        step() leaves V unchanged (0 disables)."""
        _check(load().sos_opt_set_stop(self._h, rel_tol))

    def step(self, V: torch.Tensor, p: torch.Tensor, loss_out: Optional[torch.Tensor] = None) -> torch.Tensor:
        self._V(V)
        _dev_f32(p, "p", self.index.M)
        loss = loss_out if loss_out is not None else torch.empty(1, dtype=torch.float64, device="cuda")
        _dev_f64_out(loss, "loss_out", 1)
        _check(load().sos_step(self._h, _vp(V.data_ptr()), _vp(p.data_ptr()), _vp(loss.data_ptr()), _stream()))
        return loss

    def descend(self, V: torch.Tensor, p: torch.Tensor, steps: int,
                losses_out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """`steps` descent steps in one call (V in place); returns the fp64 device
        tensor of the per-step losses L(V_t)."""
        self._V(V)
        _dev_f32(p, "p", self.index.M)
        losses = losses_out if losses_out is not None else torch.empty(max(steps, 1), dtype=torch.float64,
                                                                          device="cuda")
        _dev_f64_out(losses, "losses_out", steps)
        _check(load().sos_descend(self._h, _vp(V.data_ptr()), _vp(p.data_ptr()), steps, _vp(losses.data_ptr()),
                                  _stream()))
        return losses[:steps]

    def solve_host(self, V: np.ndarray, p: np.ndarray, steps: int) -> np.ndarray:
        """Host-buffer descent (V updated in place); returns per-step losses."""
        if not (V.dtype == np.float32 and V.flags.c_contiguous and V.shape == (self.index.N, self.r)):
            raise SosError(f"V must be a C-contiguous float32 array of shape {(self.index.N, self.r)}")
        if not (p.dtype == np.float32 and p.flags.c_contiguous and p.shape == (self.index.M,)):
            raise SosError(f"p must be a C-contiguous float32 array of shape {(self.index.M,)}")
        losses = np.empty(max(steps, 1), dtype=np.float64)
        _check(load().sos_solve_host(self._h, V.ctypes.data_as(_vp), p.ctypes.data_as(_vp), steps,
                                     losses.ctypes.data_as(_vp)))
        return losses[:steps]
