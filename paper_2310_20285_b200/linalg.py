"""Low-rank roots and the small symmetric eigensolve (mirror of ncgp/linalg.py).

``LowRankRoot`` keeps Q on the device as a (rank, dim) column block (each
column of Q contiguous), which is the layout the gemv / Gram / rotation
kernels read at full HBM bandwidth.  ``.columns`` returns the reference's
(dim, rank) host array lazily.

``sym_eigh_truncated`` (linalg.py:65-86) is K7: a <= ~600 x 600 fp64
eigensolve run on the host with LAPACK, as SURVEY.md 7 hard part 8 allows
(it is latency-bound and must be computed identically on every rank).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .device import is_device, resolve_dtype, to_device, to_host
from .exceptions import CgBreakdown, DimensionMismatch, InvalidInput, NotPositiveDefinite


class LowRankRoot:
    """Root Q of the PSD operator Q Q' (linalg.py:19-40)."""

    def __init__(self, columns=None, *, block: torch.Tensor = None,
                 kblock: torch.Tensor = None):
        self._kblock = kblock              # optional (rank, dim) device K^ Q
        if block is not None:
            self._block = block            # (rank, dim) device
            self._host = None
        else:
            cols = columns if is_device(columns) else np.asarray(columns, dtype=np.float64)
            if cols.ndim != 2:
                raise DimensionMismatch("root columns must be a (dim, rank) matrix")
            self._block = None
            self._host = cols

    @staticmethod
    def zero(dim: int, dtype=None) -> "LowRankRoot":
        return LowRankRoot(np.zeros((dim, 0)))

    @property
    def dim(self) -> int:
        return self._block.shape[1] if self._block is not None else self._host.shape[0]

    @property
    def rank(self) -> int:
        return self._block.shape[0] if self._block is not None else self._host.shape[1]

    def kblock(self, dtype=None):
        """K^ Q as a (rank, dim) device block when known, else None."""
        kb = self._kblock
        if kb is None:
            return None
        dt = resolve_dtype(dtype)
        return kb if kb.dtype == dt else kb.to(dt)

    def block(self, dtype=None) -> torch.Tensor:
        """(rank, dim) device column block in ``dtype``.  Each precision is
        derived from the most precise copy held (the host fp64 columns or
        the device block the root was built with), never from a rounded one."""
        dt = resolve_dtype(dtype)
        b = self._block
        if b is not None and b.dtype == dt:
            return b
        cache = self.__dict__.setdefault("_blocks", {})
        if dt in cache:
            return cache[dt]
        src = self._host
        if src is not None and not is_device(src):
            out = to_device(np.ascontiguousarray(src.T), dt)
        elif src is not None:
            out = src.t().to(dt).contiguous()
        else:
            out = b.to(dt)
        if b is None:
            self._block = out
        else:
            cache[dt] = out
        return out

    @property
    def columns(self) -> np.ndarray:
        """Q as a host (dim, rank) float64 array (reference layout)."""
        if self._host is None or is_device(self._host):
            src = self._block if self._block is not None else self._host.t()
            self._host = to_host(src).T.copy()
        return self._host


@dataclass(frozen=True)
class EigenPairs:
    vectors: np.ndarray  # (n, r)
    values: np.ndarray   # (r,)


def apply_lowrank(root: LowRankRoot, w, dtype=None):
    """Q (Q' w) without densifying (linalg.py:51-62); device gemv pair."""
    dev = is_device(w)
    dt = resolve_dtype(w.dtype if dev else dtype)
    t = to_device(w, dt)
    if t.shape[0] != root.dim:
        raise DimensionMismatch(
            f"operand has leading dimension {t.shape[0]}, expected {root.dim}")
    if root.rank == 0:
        out = torch.zeros_like(t)
    else:
        Q = root.block(dt)
        if t.dim() == 1:
            out = K.gemv_n(Q, K.gemv_t(Q, t), None, 1.0)
        else:
            cols = [K.gemv_n(Q, K.gemv_t(Q, t[:, j].contiguous()), None, 1.0)
                    for j in range(t.shape[1])]
            out = torch.stack(cols, dim=1)
    return out if dev else to_host(out)


def sym_eigh_truncated(M, rank_bound: int) -> EigenPairs:
    """Symmetrise, eigendecompose, keep the ``rank_bound`` largest pairs
    (linalg.py:65-86).  Host LAPACK, fp64."""
    M = to_host(M) if is_device(M) else np.asarray(M, dtype=np.float64)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise DimensionMismatch(f"expected a square matrix, got shape {M.shape}")
    if not np.isfinite(M).all():
        raise InvalidInput("matrix contains non-finite entries")
    n = M.shape[0]
    if not 0 <= rank_bound <= n:
        raise DimensionMismatch(f"rank bound {rank_bound} outside [0, {n}]")
    if n == 0 or rank_bound == 0:
        return EigenPairs(np.zeros((n, 0)), np.zeros(0))
    vals, vecs = np.linalg.eigh(0.5 * (M + M.T))
    order = np.argsort(vals)[::-1][:rank_bound]
    return EigenPairs(np.ascontiguousarray(vecs[:, order]), vals[order])


def _spd_factor(A: torch.Tensor) -> torch.Tensor:
    L, info = torch.linalg.cholesky_ex(A)
    code = int(info.item())
    if code > 0:
        raise NotPositiveDefinite(code)
    return L


def dense_spd_solve(A, b):
    """Solve A x = b for SPD A by Cholesky (linalg.py:89-96), on the device
    through cuSOLVER (torch.linalg); NotPositiveDefinite carries the order of
    the first non-positive leading minor.  numpy in, numpy out."""
    dev = is_device(A)
    At = to_device(A, A.dtype if dev else torch.float64)
    bt = to_device(b, At.dtype)
    if At.dim() != 2 or At.shape[0] != At.shape[1]:
        raise DimensionMismatch(f"expected a square matrix, got shape {tuple(At.shape)}")
    if bt.shape[0] != At.shape[0]:
        raise DimensionMismatch(
            f"right-hand side length {bt.shape[0]} != system size {At.shape[0]}")
    L = _spd_factor(At)
    x = torch.cholesky_solve(bt.reshape(bt.shape[0], -1), L).reshape(bt.shape)
    return x if dev else to_host(x)


def cholesky_inverse_root(A):
    """Upper-triangular Q with Q Q' = inv(A): the inverse transpose of the
    lower Cholesky factor (linalg.py:119-132), on the device."""
    dev = is_device(A)
    At = to_device(A, A.dtype if dev else torch.float64)
    L = _spd_factor(At)
    eye = torch.eye(At.shape[0], dtype=At.dtype, device=At.device)
    Q = torch.linalg.solve_triangular(L, eye, upper=False).t().contiguous()
    return Q if dev else to_host(Q)


def cg_reference(apply_A, b, iters: int):
    """Textbook conjugate gradients from zero (linalg.py:135-162), device
    vectors with fp64 dot products (K6 ``dots``); ``apply_A`` takes and
    returns device vectors.  Non-positive curvature raises CgBreakdown."""
    dev = is_device(b)
    bt = to_device(b, b.dtype if dev else torch.float64)
    x = torch.zeros_like(bt)
    r = bt.clone()
    rs = float(K.dots([(r, r)]).item())
    if rs == 0.0:
        return x if dev else to_host(x)
    p = r.clone()
    for k in range(iters):
        Ap = apply_A(p)
        curv = float(K.dots([(p, Ap)]).item())
        if curv <= 0.0:
            raise CgBreakdown(k, curv)
        alpha = rs / curv
        x = K.lincomb(1.0, x, alpha, p)
        r = K.lincomb(1.0, r, -alpha, Ap)
        rs_new = float(K.dots([(r, r)]).item())
        if rs_new == 0.0:
            break
        p = K.lincomb(1.0, r, rs_new / rs, p)
        rs = rs_new
    return x if dev else to_host(x)
