"""Thin Python wrappers over the C ABI (include/ncgp_b200.h).

Conventions: every tensor is a CUDA tensor of the working dtype.  A "column
block" of k vectors of length n is a (k, n) tensor whose rows are
contiguous (stride (ld, 1)); it is what the C ABI calls column b at
``ptr + b * ld``.  Reductions return fp64 device tensors.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading
from typing import Optional, Sequence, Tuple

import torch

from . import _native
from .device import code, ptr, require_cuda, stream, workspace

N = _native

# Cross-process sum of the fp64 partial reductions (dots, Q' z, Gram) when the
# solver state is row-sharded (parallel.sharded_state): a callable that sums a
# device tensor in place over the ranks, or None.  Thread-local, so that
# in-process ranks (parallel.ThreadComm) can each install their own.
_reduce_state = threading.local()


def set_reducer(fn, shard=None) -> None:
    """``shard``: (first global CN entry of this rank's shard, global dim), for
    the code that needs global indices (the unit-vector policy)."""
    _reduce_state.fn = fn
    _reduce_state.shard = shard


def get_shard():
    return getattr(_reduce_state, "shard", None)


def get_reducer():
    return getattr(_reduce_state, "fn", None)


def allreduce_partial(t: torch.Tensor) -> torch.Tensor:
    """Sum a rank-local partial result over the ranks (in place); the identity
    unless a reducer is installed."""
    fn = getattr(_reduce_state, "fn", None)
    if fn is not None:
        fn(t)
    return t


def _rows(t: torch.Tensor) -> Tuple[torch.Tensor, int]:
    """Return a (k, n) view with unit inner stride and its leading dim."""
    if t.dim() == 1:
        t = t.unsqueeze(0)
    if t.stride(-1) != 1:
        t = t.contiguous()
    return t, (t.stride(0) if t.shape[0] > 1 else t.shape[1])


# --------------------------------------------------------------------- K1

class Epi:
    """Fused epilogue of a K1 apply (``ncgp_kop_epilogue``)::

        out  = alpha * K V + beta * base + gamma * W^-1 V
        out2 = K V

    ``noise`` is ``None``, ``("softmax", pi)`` with pi the (n, C) cached
    probabilities, or ``("diag", d)`` with d the CN diagonal of W^-1.  ``base``
    and ``out2`` are (n_rows, w) tensors (rows of the full operator).  With
    ``row0`` > 0 they (and the noise state) are a row shard whose first row is
    the operator's global row ``row0``: the C ABI indexes them by global rows
    and only touches the rows of the apply's range, so the shard is passed as
    (its pointer - row0 rows).
    """

    __slots__ = ("alpha", "beta", "base", "gamma", "noise", "out2", "row0")

    def __init__(self, alpha=1.0, beta=1.0, base=None, gamma=0.0, noise=None, out2=None,
                 row0: int = 0):
        self.alpha, self.beta, self.base = float(alpha), float(beta), base
        self.gamma, self.noise, self.out2 = float(gamma), noise, out2
        self.row0 = int(row0)

    def native(self, c0: int, es: int, w: int = 0) -> "N.Epilogue":
        """``w``: width of the apply (the noise state's row length; needed
        only with ``row0``)."""
        e = N.Epilogue()
        e.alpha, e.beta, e.gamma = self.alpha, self.beta, self.gamma
        r0 = self.row0
        if self.base is not None:
            e.ldb = self.base.stride(0) if self.base.dim() == 2 else 1
            e.base = self.base.data_ptr() + (c0 - r0 * e.ldb) * es
        if self.noise is not None and self.gamma != 0.0:
            kind, st = self.noise
            e.noise = {"softmax": N.NOISE_SOFTMAX, "diag": N.NOISE_DIAG}[kind]
            if r0 and w <= 0:
                raise N.DimensionMismatch("a sharded noise state needs the apply's width")
            e.noise_state = st.data_ptr() - r0 * w * st.element_size()
        if self.out2 is not None:
            e.ld2 = self.out2.stride(0) if self.out2.dim() == 2 else 1
            e.out2 = self.out2.data_ptr() + (c0 - r0 * e.ld2) * es
        return e


class KernelOperator:
    """Device kernel operator for one stationary kernel spec:
    ``apply(V) = K(X_rows, X_cols) @ V`` without materialising K.

    Replaces the tile loop of prior_matvec (gp.py:144-172) and the dense
    cross_covariance products (gp.py:175-196, posterior.py:52-84).
    """

    def __init__(self, family: str, lengthscale: float, outputscale: float,
                 X_rows: torch.Tensor, X_cols: Optional[torch.Tensor] = None,
                 w_max: int = 32, impl: str = "auto"):
        require_cuda()
        self.family = family
        self.fam_code = {"rbf": N.RBF, "matern32": N.MATERN32}[family]
        self.lengthscale = float(lengthscale)
        self.outputscale = float(outputscale)
        self.X_rows = X_rows.contiguous()
        self.X_cols = self.X_rows if X_cols is None else X_cols.contiguous()
        if self.X_rows.dim() != 2 or self.X_cols.dim() != 2 or \
                self.X_rows.shape[1] != self.X_cols.shape[1]:
            raise N.DimensionMismatch("kernel inputs must be (n, d) with equal d")
        if self.X_rows.dtype != self.X_cols.dtype:
            raise N.DimensionMismatch("row and column inputs must share a dtype")
        self.dtype = self.X_rows.dtype
        self.n_rows, self.d = self.X_rows.shape
        self.n_cols = self.X_cols.shape[0]
        # up to 32 RHS columns per K1 launch; 32 < w_max <= 128 selects the
        # wide-RHS kernel (K2) for wide products and the posterior variance
        self.w_max = int(max(1, min(w_max, 128)))
        impl_code = {"auto": N.KOP_AUTO, "tcgen05": N.KOP_TCGEN05, "simt": N.KOP_SIMT}[impl]
        dt = code(self.dtype)
        nbytes = N.query("ncgp_kop_workspace_bytes", impl_code, dt, self.n_rows, self.n_cols,
                         self.d, self.w_max)
        self._ws = torch.empty(max(int(nbytes), 256), dtype=torch.uint8,
                               device=self.X_rows.device)
        h = N._vp()
        N.call("ncgp_kop_create", N.ctypes.byref(h), impl_code, self.fam_code,
               self.lengthscale, self.outputscale, dt, ptr(self.X_rows), self.n_rows,
               ptr(self.X_cols), self.n_cols, self.d, self.w_max, ptr(self._ws),
               self._ws.numel(), stream())
        self._h = h
        env = os.environ.get("NCGP_SYM", "")
        self._sym_mode0 = 0 if env.startswith("0") else (1 if env.startswith("1") else -1)
        self.impl = {N.KOP_TCGEN05: "tcgen05", N.KOP_SIMT: "simt"}[
            N.query("ncgp_kop_impl", h)]

    def set_sym(self, mode: int) -> None:
        """Symmetric-kernel policy (``ncgp_kop_set_sym``): -1 default, 0 plain
        kernel only, 1 symmetric kernel whenever it fits."""
        N.call("ncgp_kop_set_sym", self._h, int(mode))
        self._sym_mode = int(mode)

    @contextlib.contextmanager
    def sym_mode(self, mode: int):
        """Temporarily force the symmetric-kernel policy (tests, A/B timing)."""
        old = getattr(self, "_sym_mode", self._sym_mode0)
        self.set_sym(mode)
        try:
            yield self
        finally:
            self.set_sym(old)

    @property
    def last_variant(self) -> str:
        """Kernel variant of the last apply: "plain", "symmetric", "wide" or "none"."""
        return {0: "plain", 1: "symmetric", 2: "symmetric", 3: "wide",
                4: "symmetric"}.get(self.last_variant_code, "none")

    @property
    def last_variant_code(self) -> int:
        """ncgp_kop_last_variant: 0 plain, 1 symmetric pair kernel, 2 symmetric
        single-CTA kernel, 3 wide-RHS kernel, 4 blocked symmetric kernel, -1 none yet."""
        return int(N.query("ncgp_kop_last_variant", self._h))

    def apply(self, V: torch.Tensor, out: Optional[torch.Tensor] = None,
              row_begin: int = 0, row_end: Optional[int] = None,
              peers: Optional[Sequence[torch.Tensor]] = None,
              epi: Optional[Epi] = None, out_row0: int = 0) -> torch.Tensor:
        """K(X_rows[row_begin:row_end], X_cols) @ V for V of shape (n_cols, w).

        ``out_row0``: ``out`` is a row shard whose first row is global row
        ``out_row0`` (it must cover [row_begin, row_end)); by default ``out``
        has all n_rows rows.

        ``peers``: further (n_rows, w) buffers with ``out``'s strides (other
        ranks' gather buffers mapped into this process) that receive the same
        rows from the same kernel (``ncgp_kop_apply_multi``).  ``epi``: a
        fused :class:`Epi` (``ncgp_kop_apply_ex``); a noise term needs the
        whole row in one block (w <= w_max)."""
        vec = V.dim() == 1
        if vec:
            V = V.unsqueeze(1)
        if V.shape[0] != self.n_cols:
            raise N.DimensionMismatch(f"operand has {V.shape[0]} rows, expected {self.n_cols}")
        if V.dtype != self.dtype:
            raise N.DimensionMismatch(f"operand dtype {V.dtype} != operator dtype {self.dtype}")
        if V.stride(1) != 1:
            V = V.contiguous()
        w = V.shape[1]
        row_end = self.n_rows if row_end is None else row_end
        if out is None:
            out = torch.empty((row_end - out_row0 if out_row0 else self.n_rows, w),
                              dtype=self.dtype, device=V.device)
        elif out.dim() == 1:
            out = out.view(-1, 1)
        if out_row0 and not (out_row0 <= row_begin and row_end <= out_row0 + out.shape[0]):
            raise N.DimensionMismatch("output shard does not cover the row range")
        ldv = V.stride(0) if V.shape[0] > 1 else w
        ldo = out.stride(0) if out.shape[0] > 1 else w
        bases = [out.data_ptr() - out_row0 * ldo * V.element_size()]
        for p in peers or ():
            p = p.view(-1, 1) if p.dim() == 1 else p
            if tuple(p.shape) != tuple(out.shape) or p.stride() != out.stride() or \
                    p.dtype != out.dtype:
                raise N.DimensionMismatch("peer buffer shape / strides differ from the output")
            bases.append(p.data_ptr())
        es = V.element_size()
        if epi is not None:
            if len(bases) != 1:
                raise N.DimensionMismatch("a fused epilogue does not combine with peer outputs")
            if epi.noise is not None and epi.gamma != 0.0 and w > self.w_max:
                raise N.DimensionMismatch(f"a noise epilogue needs w <= {self.w_max}, got {w}")
            if epi.row0 > row_begin:
                raise N.DimensionMismatch("epilogue shard starts after the first row of the range")
            for t in (epi.base, epi.out2):
                if t is not None and (t.dtype != self.dtype or
                                      epi.row0 + t.shape[0] < min(row_end, self.n_rows) or
                                      (t.dim() == 2 and t.stride(1) != 1)):
                    raise N.DimensionMismatch("epilogue base / out2 must be (>= n_rows, w) rows")
        for c0 in range(0, w, self.w_max):
            c1 = min(w, c0 + self.w_max)
            if epi is not None:
                e = epi.native(c0, es, c1 - c0)
                N.call("ncgp_kop_apply_ex", self._h, V.data_ptr() + c0 * es, ldv, c1 - c0,
                       bases[0] + c0 * es, ldo, row_begin, row_end, ctypes.byref(e),
                       stream())
            elif len(bases) == 1:
                N.call("ncgp_kop_apply", self._h, V.data_ptr() + c0 * es, ldv, c1 - c0,
                       bases[0] + c0 * es, ldo, row_begin, row_end, stream())
            else:
                arr = (ctypes.c_void_p * len(bases))(*[b + c0 * es for b in bases])
                N.call("ncgp_kop_apply_multi", self._h, V.data_ptr() + c0 * es, ldv, c1 - c0,
                       arr, len(bases), ldo, row_begin, row_end, stream())
        return out[:, 0] if vec else out

    __call__ = apply

    def posterior_var(self, W: torch.Tensor, C: int, R: int, s2: torch.Tensor,
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """K2 (``ncgp_kop_posterior_var``): var[t, c] = max(s2[c] -
        sum_r (K(X_rows, X_cols) W[:, c R + r])[t]^2, 0) for the class-major
        root W (n_cols, C R), without materialising K W.  Raises
        :class:`_native.Unsupported` unless this is a tcgen05 operator
        created with w_max > 32 (callers fall back to the product path)."""
        if W.shape[0] != self.n_cols or W.dim() != 2 or W.shape[1] != C * R:
            raise N.DimensionMismatch(f"root block {tuple(W.shape)} != ({self.n_cols}, {C * R})")
        if W.dtype != self.dtype or W.stride(1) != 1:
            W = W.to(self.dtype).contiguous()
        s2 = s2.to(device=W.device, dtype=torch.float64).contiguous()
        if out is None:
            out = torch.empty((self.n_rows, C), dtype=self.dtype, device=W.device)
        ldw = W.stride(0) if W.shape[0] > 1 else W.shape[1]
        ldo = out.stride(0) if out.shape[0] > 1 else C
        N.call("ncgp_kop_posterior_var", self._h, W.data_ptr(), ldw, C, R, s2.data_ptr(),
               out.data_ptr(), ldo, stream())
        return out

    # ---- the symmetric K(X, X) kernel split across processes (parallel.py)
    def sym_acc_elems(self, w: int) -> int:
        """int64 elements of the per-process accumulator of a split symmetric
        apply of width ``w`` (<= w_max), or 0 when the full apply would not
        use a symmetric kernel (then shard rows instead)."""
        if not 1 <= w <= self.w_max:
            return 0
        return int(N.query("ncgp_kop_sym_acc_elems", self._h, w))

    def sym_partial(self, V: torch.Tensor, part: int, nparts: int, acc: torch.Tensor) -> None:
        """Part ``part`` of ``nparts`` of the triangular work list into ``acc``
        (int64, ``sym_acc_elems(w)`` elements; zeroed by the call).  The
        parts' accumulators sum exactly (integers): any split gives the same
        bits after :meth:`sym_finalize`."""
        if V.dim() == 1:
            V = V.unsqueeze(1)
        if V.shape[0] != self.n_cols or V.dtype != self.dtype:
            raise N.DimensionMismatch("operand shape / dtype do not match the operator")
        if V.stride(1) != 1:
            V = V.contiguous()
        w = V.shape[1]
        if acc.dtype != torch.int64 or not acc.is_contiguous():
            raise N.DimensionMismatch("accumulator must be a contiguous int64 tensor")
        ldv = V.stride(0) if V.shape[0] > 1 else w
        N.call("ncgp_kop_sym_partial", self._h, V.data_ptr(), ldv, w, part, nparts, acc.data_ptr(),
               acc.numel(), stream())

    def sym_finalize(self, acc: torch.Tensor, w: int, out: Optional[torch.Tensor] = None,
                     V: Optional[torch.Tensor] = None, epi: Optional[Epi] = None,
                     row_begin: int = 0, row_end: Optional[int] = None) -> torch.Tensor:
        """The (n_rows, w) product from the summed accumulators, through the
        fused epilogue ``epi`` (its noise term reads the operand ``V``).  With
        a row range, only those rows are finalised and ``out`` (and ``epi``'s
        tensors, ``epi.row0 == row_begin``) are the (row_end - row_begin)-row
        shard (``ncgp_kop_sym_finalize_rows``)."""
        row_end = self.n_rows if row_end is None else row_end
        if row_begin or row_end != self.n_rows:
            if out is None:
                out = torch.empty((row_end - row_begin, w), dtype=self.dtype, device=acc.device)
            if out.shape[0] < row_end - row_begin:
                raise N.DimensionMismatch("output shard is shorter than the row range")
            if epi is not None and epi.row0 != row_begin:
                raise N.DimensionMismatch("epilogue shard must start at row_begin")
            ldo = out.stride(0) if out.shape[0] > 1 else w
            vp, ldv = None, w
            if V is not None:  # the full operand (the noise term reads rows of the range)
                V = V.unsqueeze(1) if V.dim() == 1 else V
                vp, ldv = V.data_ptr(), (V.stride(0) if V.shape[0] > 1 else w)
            e = ctypes.byref(epi.native(0, out.element_size(), w)) if epi is not None else None
            N.call("ncgp_kop_sym_finalize_rows", self._h, acc.data_ptr(), acc.numel(), vp, ldv, w,
                   out.data_ptr() - row_begin * ldo * out.element_size(), ldo, e, row_begin,
                   row_end, stream())
            return out
        if epi is not None and epi.row0:
            raise N.DimensionMismatch("a sharded epilogue needs the matching row range")
        if out is None:
            out = torch.empty((self.n_rows, w), dtype=self.dtype, device=acc.device)
        ldo = out.stride(0) if out.shape[0] > 1 else w
        vp, ldv = None, w
        if V is not None:
            V = V.unsqueeze(1) if V.dim() == 1 else V
            vp, ldv = V.data_ptr(), (V.stride(0) if V.shape[0] > 1 else w)
        e = ctypes.byref(epi.native(0, out.element_size())) if epi is not None else None
        N.call("ncgp_kop_sym_finalize", self._h, acc.data_ptr(), acc.numel(), vp, ldv, w,
               out.data_ptr(), ldo, e, stream())
        return out

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                N.query("ncgp_kop_destroy", h)
            except Exception:
                pass
            self._h = None

    def __del__(self):
        self.close()


# --------------------------------------------------------------------- K3-K5

def softmax_stats(f: torch.Tensor, labels: Optional[torch.Tensor], n: int, C: int,
                  want_grad=True, want_yhat=True):
    pi = torch.empty((n, C), dtype=f.dtype, device=f.device)
    grad = torch.empty(n * C, dtype=f.dtype, device=f.device) if want_grad else None
    yhat = torch.empty(n * C, dtype=f.dtype, device=f.device) if want_yhat else None
    N.call("ncgp_softmax_stats", code(f), ptr(f), ptr(labels), n, C, ptr(pi), ptr(grad),
           ptr(yhat), stream())
    return pi, grad, yhat


def softmax_winv(pi: torch.Tensor, n: int, C: int, V: torch.Tensor,
                 base: Optional[torch.Tensor] = None, alpha: float = 1.0, beta: float = 1.0,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """beta*base + alpha*W^+ V on a column block V (k, n*C) (or a vector)."""
    vec = V.dim() == 1
    Vr, ldv = _rows(V)
    k = Vr.shape[0]
    if out is None:
        out = torch.empty_like(Vr)
    Or, ldo = _rows(out)
    Br, ldb = _rows(base) if base is not None else (None, 0)
    N.call("ncgp_softmax_winv", code(pi), ptr(pi), n, C, ptr(Vr), ldv, k, ptr(Br), ldb,
           float(alpha), float(beta), ptr(Or), ldo, stream())
    return Or[0] if vec else Or


def softmax_w(pi: torch.Tensor, n: int, C: int, V: torch.Tensor) -> torch.Tensor:
    vec = V.dim() == 1
    Vr, ldv = _rows(V)
    out = torch.empty_like(Vr)
    N.call("ncgp_softmax_w", code(pi), ptr(pi), n, C, ptr(Vr), ldv, Vr.shape[0], ptr(out),
           out.stride(0) if out.shape[0] > 1 else out.shape[1], stream())
    return out[0] if vec else out


def bernoulli_stats(f: torch.Tensor, labels: Optional[torch.Tensor]):
    n = f.numel()
    winv = torch.empty_like(f)
    w = torch.empty_like(f)
    grad = torch.empty_like(f) if labels is not None else None
    yhat = torch.empty_like(f) if labels is not None else None
    N.call("ncgp_bernoulli_stats", code(f), ptr(f), ptr(labels), n, ptr(winv), ptr(w),
           ptr(grad), ptr(yhat), stream())
    return winv, w, grad, yhat


def poisson_stats(f: torch.Tensor, counts: Optional[torch.Tensor]):
    """(W^-1 diag, W diag, grad, pseudo targets) of the Poisson log link."""
    winv = torch.empty_like(f)
    w = torch.empty_like(f)
    grad = torch.empty_like(f) if counts is not None else None
    yhat = torch.empty_like(f) if counts is not None else None
    N.call("ncgp_poisson_stats", code(f), ptr(f), ptr(counts), f.numel(), ptr(winv), ptr(w),
           ptr(grad), ptr(yhat), stream())
    return winv, w, grad, yhat


def diag_apply(dvec: torch.Tensor, V: torch.Tensor, base: Optional[torch.Tensor] = None,
               alpha: float = 1.0, beta: float = 1.0,
               out: Optional[torch.Tensor] = None) -> torch.Tensor:
    vec = V.dim() == 1
    Vr, ldv = _rows(V)
    if out is None:
        out = torch.empty_like(Vr)
    Or, ldo = _rows(out)
    Br, ldb = _rows(base) if base is not None else (None, 0)
    N.call("ncgp_diag_apply", code(dvec), ptr(dvec), dvec.numel(), ptr(Vr), ldv, Vr.shape[0],
           ptr(Br), ldb, float(alpha), float(beta), ptr(Or), ldo, stream())
    return Or[0] if vec else Or


# --------------------------------------------------------------------- K6

def _reduce_ws(n: int, k: int) -> torch.Tensor:
    nbytes = N.query("ncgp_reduce_workspace_bytes", n, k)
    return workspace().get("reduce", nbytes)


def dots(pairs: Sequence[Tuple[torch.Tensor, torch.Tensor]],
         out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """fp64 device vector of x_p . y_p (deterministic order), <= 4 pairs."""
    x0 = pairs[0][0]
    n = x0.numel()
    if out is None:
        out = torch.empty(len(pairs), dtype=torch.float64, device=x0.device)
    ws = _reduce_ws(n, len(pairs))
    xs = N.ptr_array([ptr(x) for x, _ in pairs])
    ys = N.ptr_array([ptr(y) for _, y in pairs])
    N.call("ncgp_dots", code(x0), n, len(pairs), xs, ys, ptr(out), ptr(ws), ws.numel(),
           stream())
    return allreduce_partial(out)


def gemv_t(Q: torch.Tensor, z: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Q' z for a column block Q (k, n): fp64 (k,)."""
    Qr, ldq = _rows(Q)
    k, n = Qr.shape
    if out is None:
        out = torch.empty(k, dtype=torch.float64, device=z.device)
    if k == 0:
        return out
    ws = _reduce_ws(n, k)
    N.call("ncgp_gemv_t", code(z), ptr(Qr), ldq, k, ptr(z), n, ptr(out), ptr(ws), ws.numel(),
           stream())
    return allreduce_partial(out)


def gemv_n(Q: torch.Tensor, y: torch.Tensor, s: Optional[torch.Tensor], alpha: float,
           out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """s + alpha * Q y for a column block Q (k, n) and fp64 y (k,)."""
    Qr, ldq = _rows(Q)
    k, n = Qr.shape
    if out is None:
        out = torch.empty(n, dtype=Qr.dtype, device=Qr.device)
    N.call("ncgp_gemv_n", code(out), ptr(Qr), ldq, k, ptr(y), ptr(s), float(alpha), ptr(out),
           n, stream())
    return out


def lincomb(a: float, x: torch.Tensor, b: float = 0.0, y: Optional[torch.Tensor] = None,
            c: float = 0.0, z: Optional[torch.Tensor] = None,
            out: Optional[torch.Tensor] = None) -> torch.Tensor:
    if out is None:
        out = torch.empty_like(x)
    N.call("ncgp_lincomb", code(x), x.numel(), float(a), ptr(x), float(b), ptr(y), float(c),
           ptr(z), ptr(out), stream())
    return out


def gram(S: torch.Tensor, Y: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """fp64 (ka, kb) matrix of S_a . Y_b for column blocks S (ka, n), Y (kb, n)."""
    Sr, lds = _rows(S)
    Yr, ldy = _rows(Y)
    ka, n = Sr.shape
    kb = Yr.shape[0]
    if out is None:
        out = torch.empty((ka, kb), dtype=torch.float64, device=Sr.device)
    if ka == 0 or kb == 0:
        return out
    nbytes = N.query("ncgp_gram_workspace_bytes", n, ka, kb)
    ws = workspace().get("gram", nbytes)
    N.call("ncgp_gram", code(Sr), ptr(Sr), lds, ka, ptr(Yr), ldy, kb, n, ptr(out),
           out.stride(0), ptr(ws), ws.numel(), stream())
    if get_reducer() is not None:  # ``out`` may be a strided block of the Gram matrix
        tmp = out.contiguous()
        allreduce_partial(tmp)
        if tmp.data_ptr() != out.data_ptr():
            out.copy_(tmp)
    return out


def rotate(S: torch.Tensor, U: torch.Tensor, out: Optional[torch.Tensor] = None,
           native: bool = False) -> torch.Tensor:
    """Column block S U: S (kb, n), U fp64 (kb, kc) -> (kc, n).

    A plain dense GEMM (the virtual solver run's rotation, solver.py:311-330),
    so it goes to cuBLAS (``Uᵀ S`` in the buffers' dtype, full fp32 / fp64
    precision -- TF32 is off for torch matmuls -- and deterministic):
    ~4x faster than ``ncgp_rotate``, which reads S once per 16 output rows
    (cfg4: 20 ms per call).  ``native=True`` keeps the C-ABI kernel (the
    path a non-Python host binds)."""
    Sr, lds = _rows(S)
    kb, n = Sr.shape
    U = U.to(device=Sr.device, dtype=torch.float64).contiguous()
    kc = U.shape[1]
    if out is None:
        out = torch.empty((kc, n), dtype=Sr.dtype, device=Sr.device)
    if kc == 0:
        return out
    if not native and Sr.dtype in (torch.float32, torch.float64):
        tf32 = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = False  # full precision even if a caller enabled TF32
        try:
            torch.mm(U.t().to(Sr.dtype), Sr, out=out)
        finally:
            torch.backends.cuda.matmul.allow_tf32 = tf32
        return out
    N.call("ncgp_rotate", code(Sr), ptr(Sr), lds, kb, ptr(U), U.stride(0), kc, ptr(out),
           out.stride(0) if kc > 1 else n, n, stream())
    return out


def marginal_var(A: torch.Tensor, C: int, R: int, s2: torch.Tensor,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
    nt = A.shape[0]
    if out is None:
        out = torch.empty((nt, C), dtype=A.dtype, device=A.device)
    N.call("ncgp_marginal_var", code(A), ptr(A), A.stride(0), nt, C, R, ptr(s2), ptr(out),
           stream())
    return out
