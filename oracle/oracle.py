"""fp64 CPU oracle for the SOS hot path -- ctypes wrapper around sos_oracle.c.

TEST INFRASTRUCTURE ONLY: only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product package ``paper_2410_19844_b200`` never imports it.

Every function follows the plain definition in PAPER.md (see the citations in
``sos_oracle.c``): colex-ordered monomial bases built by enumeration + sort,
pair ranks by binary search, coefficients of m_d V V^T m_d^T by explicit pair
loops (Eq. 2), the gradient of Eq. 2 written out, and plain
GD / Adam updates.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sos_oracle.c")
_LIB = os.path.join(_HERE, "_sos_oracle.so")

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile sos_oracle.c with gcc (plain -O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.or_index_create.restype = _vp
        L.or_index_create.argtypes = [ctypes.c_int, ctypes.c_int]
        L.or_index_destroy.argtypes = [_vp]
        L.or_index_N.restype = _i64
        L.or_index_N.argtypes = [_vp]
        L.or_index_M.restype = _i64
        L.or_index_M.argtypes = [_vp]
        L.or_basis_count.restype = _i64
        L.or_basis_count.argtypes = [ctypes.c_int, ctypes.c_int]
        L.or_index_alpha.argtypes = [_vp, _vp]
        L.or_index_beta.argtypes = [_vp, _vp]
        L.or_rank2d.argtypes = [_vp, _vp, _i64, _vp]
        L.or_pair_ranks.argtypes = [_vp, _vp, _i64, _vp]
        L.or_forward.argtypes = [_vp, _vp, _i64, _vp]
        L.or_forward_rows.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp]
        L.or_coef_sample.argtypes = [_vp, _vp, _i64, _vp, _i64, _vp]
        L.or_grad_rows.argtypes = [_vp, _vp, _i64, _vp, _vp, _i64, _vp]
        L.or_loss_grad.restype = ctypes.c_double
        L.or_loss_grad.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp, _vp]
        L.or_gd_update.argtypes = [_vp, _vp, _i64, ctypes.c_double]
        L.or_adam_update.argtypes = [_vp, _vp, _vp, _vp, _i64, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, _i64]
        L.or_descent.argtypes = [_vp, _vp, _i64, _vp, ctypes.c_int, _i64, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_double, _vp]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def basis_count(n: int, D: int) -> int:
    """Number of degree-D monomials in n variables, counted by enumeration."""
    return int(lib().or_basis_count(n, D))


def host_threads() -> int:
    """Host cores this process may run on (the threaded helpers' default)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _row_blocks(N: int, threads: int, block: int = 16):
    """Static, deterministic split of rows 0..N-1 over `threads` workers:
    worker t takes row blocks t, t + threads, ... (balances the pair loop)."""
    starts = list(range(0, N, block))
    return [[(s, min(N, s + block)) for s in starts[t::threads]] for t in range(threads)]


class OracleIndex:
    """Monomial bases m_d (N entries) and degree-2d basis (M entries), colex order."""

    def __init__(self, n: int, d: int):
        self.n, self.d = n, d
        self._h = lib().or_index_create(n, d)
        if not self._h:
            raise ValueError(f"bad (n,d)=({n},{d})")
        self.N = int(lib().or_index_N(self._h))
        self.M = int(lib().or_index_M(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.or_index_destroy(h)
            self._h = None

    # ---- tables -------------------------------------------------------
    def alpha(self) -> np.ndarray:
        out = np.empty((self.N, self.n), dtype=np.uint8)
        lib().or_index_alpha(self._h, _ptr(out))
        return out

    def beta(self) -> np.ndarray:
        out = np.empty((self.M, self.n), dtype=np.uint8)
        lib().or_index_beta(self._h, _ptr(out))
        return out

    def rank2d(self, ex: np.ndarray) -> np.ndarray:
        ex = np.ascontiguousarray(ex, dtype=np.uint8).reshape(-1, self.n)
        out = np.empty(ex.shape[0], dtype=np.int64)
        lib().or_rank2d(self._h, _ptr(ex), ex.shape[0], _ptr(out))
        return out

    def pair_ranks(self, rows=None) -> np.ndarray:
        rows = np.arange(self.N, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty((rows.shape[0], self.N), dtype=np.uint32)
        lib().or_pair_ranks(self._h, _ptr(rows), rows.shape[0], _ptr(out))
        return out

    # ---- forward / loss / gradient -------------------------------------
    def forward(self, V) -> np.ndarray:
        V = _f64(V)
        assert V.shape[0] == self.N
        out = np.empty(self.M, dtype=np.float64)
        lib().or_forward(self._h, _ptr(V), V.shape[1], _ptr(out))
        return out

    def forward_threaded(self, V, threads: int | None = None, rows: tuple | None = None) -> np.ndarray:
        """forward() with the pair loop's rows split over host threads
        (or_forward_rows per row range; the ctypes calls release the GIL).
        Equal to forward() up to the order of the fp64 additions.  rows=(i0, i1)
        restricts the loop to those rows (a partial sum; bench.py times it)."""
        V = _f64(V)
        assert V.shape[0] == self.N
        i0, i1 = rows if rows is not None else (0, self.N)
        T = max(1, min(threads or host_threads(), i1 - i0))
        block = max(1, min(16, (i1 - i0) // (2 * T)))  # >= 2 blocks per thread when the range allows
        parts = [[(a + i0, b + i0) for a, b in part] for part in _row_blocks(i1 - i0, T, block)]

        def work(blocks):
            acc = np.zeros(self.M, dtype=np.float64)
            for i0, i1 in blocks:
                lib().or_forward_rows(self._h, _ptr(V), V.shape[1], i0, i1, _ptr(acc))
            return acc

        with ThreadPoolExecutor(T) as ex:
            accs = list(ex.map(work, parts))
        out = accs[0]
        for a in accs[1:]:
            out += a
        return out

    def grad_rows_threaded(self, V, res, rows, threads: int | None = None) -> np.ndarray:
        """grad_rows() with the rows split over host threads (same C routine per row)."""
        V = _f64(V)
        res = _f64(res)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty((rows.shape[0], V.shape[1]), dtype=np.float64)
        T = max(1, min(threads or host_threads(), rows.shape[0]))
        chunks = [c for c in np.array_split(np.arange(rows.shape[0]), T) if c.size]

        def work(idx):
            sub = np.ascontiguousarray(rows[idx])
            g = np.empty((sub.shape[0], V.shape[1]), dtype=np.float64)
            lib().or_grad_rows(self._h, _ptr(V), V.shape[1], _ptr(res), _ptr(sub), sub.shape[0], _ptr(g))
            out[idx] = g

        with ThreadPoolExecutor(T) as ex:
            list(ex.map(work, chunks))
        return out

    def loss_grad_threaded(self, V, p, want_grad: bool = True, threads: int | None = None):
        """loss_grad() on host threads: same definitions (Eq. 2 and its gradient 4RV)."""
        V = _f64(V)
        p = _f64(p)
        coef = self.forward_threaded(V, threads)
        res = coef - p
        loss = float(np.sum(res * res))
        grad = self.grad_rows_threaded(V, res, np.arange(self.N), threads) if want_grad else None
        return loss, grad, coef, res

    def descent_threaded(self, V0, p, kind: str, steps: int, lr: float, b1: float = 0.9, b2: float = 0.999,
                         eps: float = 1e-8, threads: int | None = None, final_loss: bool = True,
                         grads_out: list | None = None):
        """The loop of or_descent (losses[t] = L(V_t) before update t, then
        GD or Adam with step index t+1), each loss/gradient evaluated on host
        threads and each update by the oracle's own or_gd_update /
        or_adam_update.  Returns (V_steps, losses): V_steps[t] = V_t; the
        last loss L(V_steps) only with final_loss.  grads_out (a list), if
        given, receives each step's gradient."""
        V = _f64(V0).copy()
        p = _f64(p)
        m = np.zeros_like(V)
        v = np.zeros_like(V)
        Vs, losses = [V.copy()], []
        for t in range(steps):
            loss, g, _, _ = self.loss_grad_threaded(V, p, True, threads)
            losses.append(loss)
            if grads_out is not None:
                grads_out.append(g.copy())
            if kind == "gd":
                lib().or_gd_update(_ptr(V), _ptr(g), V.size, lr)
            else:
                lib().or_adam_update(_ptr(V), _ptr(g), _ptr(m), _ptr(v), V.size, lr, b1, b2, eps, t + 1)
            Vs.append(V.copy())
        if final_loss:
            losses.append(self.loss_grad_threaded(V, p, False, threads)[0])
        return Vs, np.array(losses)

    def coef_sample(self, V, betas) -> np.ndarray:
        V = _f64(V)
        betas = np.ascontiguousarray(betas, dtype=np.int64)
        out = np.empty(betas.shape[0], dtype=np.float64)
        lib().or_coef_sample(self._h, _ptr(V), V.shape[1], _ptr(betas), betas.shape[0], _ptr(out))
        return out

    def grad_rows(self, V, res, rows) -> np.ndarray:
        """rows of dL/dV = 4 R V for a given residual vector res (length M)."""
        V = _f64(V)
        res = _f64(res)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty((rows.shape[0], V.shape[1]), dtype=np.float64)
        lib().or_grad_rows(self._h, _ptr(V), V.shape[1], _ptr(res), _ptr(rows), rows.shape[0], _ptr(out))
        return out

    def loss_grad(self, V, p, want_grad: bool = True):
        V = _f64(V)
        p = _f64(p)
        grad = np.empty_like(V) if want_grad else None
        coef = np.empty(self.M, dtype=np.float64)
        res = np.empty(self.M, dtype=np.float64)
        loss = lib().or_loss_grad(self._h, _ptr(V), V.shape[1], _ptr(p),
                                  _ptr(grad) if want_grad else None, _ptr(coef), _ptr(res))
        return float(loss), grad, coef, res

    def descent(self, V0, p, kind: str, steps: int, lr: float,
                b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8):
        V = _f64(V0).copy()
        p = _f64(p)
        losses = np.empty(steps + 1, dtype=np.float64)
        k = {"gd": 0, "adam": 1}[kind]
        lib().or_descent(self._h, _ptr(V), V.shape[1], _ptr(p), k, steps, lr, b1, b2, eps, _ptr(losses))
        return V, losses


def gd_update(V, g, lr):
    V = _f64(V).copy()
    g = _f64(g)
    lib().or_gd_update(_ptr(V), _ptr(g), V.size, lr)
    return V


def adam_update(V, g, m, v, lr, b1, b2, eps, t):
    V = _f64(V).copy()
    m = _f64(m).copy()
    v = _f64(v).copy()
    g = _f64(g)
    lib().or_adam_update(_ptr(V), _ptr(g), _ptr(m), _ptr(v), V.size, lr, b1, b2, eps, t)
    return V, m, v
