"""Posterior evaluation at test inputs (mirror of ncgp/posterior.py).

The belief (v, Q) stays on the device.  ``posterior_mean`` (posterior.py:52-64)
and ``posterior_marginal_var`` (posterior.py:67-84) apply the fused
cross-kernel operator K(X*, X) to v and to the class-gathered root
[Q_0 | ... | Q_{C-1}] instead of densifying the (N*·C) x (N·C) block matrix
the reference builds per chunk (gp.py:175-196), so they run at cfg4/cfg5
scale where the reference cannot.  ``probit_predict`` (posterior.py:104-121)
is O(N*·C) host arithmetic, as SURVEY.md 8(a) a9 allows.
"""

from __future__ import annotations

import math
from typing import Optional

import numpy as np
import torch

from . import kernels as K
from .device import is_device, resolve_dtype, to_device, to_host
from .exceptions import DimensionMismatch, InvalidInput
from .gp import MultiOutputPrior
from .linalg import LowRankRoot


class PosteriorBelief:
    """Representer weights and precision root (posterior.py:26-49).

    ``weights`` and ``root.columns`` are served as host float64 arrays on
    demand; ``weights_device`` / ``root.block()`` are the device copies.
    """

    def __init__(self, prior: MultiOutputPrior, train_inputs, weights, root: LowRankRoot,
                 newton_step: int = 0, solver_iterations: int = 0):
        self.prior = prior
        self.train_inputs = np.asarray(train_inputs, dtype=np.float64) \
            if not is_device(train_inputs) else train_inputs
        dim = self.train_inputs.shape[0] * prior.num_outputs
        if tuple(weights.shape) != (dim,):
            raise DimensionMismatch(f"weights have length {weights.shape[0]}, expected {dim}")
        if root.dim != dim:
            raise DimensionMismatch(f"root has dimension {root.dim}, expected {dim}")
        self._weights = weights
        self.root = root
        self.newton_step = newton_step
        self.solver_iterations = solver_iterations

    @property
    def weights(self) -> np.ndarray:
        if is_device(self._weights):
            return to_host(self._weights)
        return np.asarray(self._weights, dtype=np.float64)

    def weights_device(self, dtype=None) -> torch.Tensor:
        dt = resolve_dtype(dtype if dtype is not None else
                           (self._weights.dtype if is_device(self._weights) else None))
        return to_device(self._weights, dt)

    @property
    def dtype(self) -> torch.dtype:
        if is_device(self._weights):
            return self._weights.dtype
        return resolve_dtype(None)

    @classmethod
    def prior_only(cls, prior, train_inputs):
        dim = np.asarray(train_inputs).shape[0] * prior.num_outputs
        return cls(prior, train_inputs, np.zeros(dim), LowRankRoot.zero(dim))


def _cross_ops(belief: PosteriorBelief, X_test, dt, w_max=32):
    """One K(X*, X) operator per unique spec with its output indices."""
    Xr = to_device(X_test, dt)
    Xc = to_device(belief.train_inputs, dt)
    if Xr.dim() != 2 or Xr.shape[1] != Xc.shape[1]:
        raise DimensionMismatch(f"incompatible input shapes {tuple(Xr.shape)} vs "
                                f"{tuple(Xc.shape)}")
    return [(_wide_or_plain(spec, Xr, Xc, w_max), cols)
            for spec, cols in belief.prior.spec_groups()]


def _wide_or_plain(spec, Xr, Xc, w_max):
    """The cross operator; w_max > 32 asks for the wide-RHS kernel (K2),
    which exists for the fp32 tcgen05 path at D <= ~50 -- otherwise the
    32-column operator (the product path loops RHS blocks)."""
    try:
        return K.KernelOperator(spec.family, spec.lengthscale, spec.outputscale, Xr, Xc,
                                w_max=w_max)
    except (K.N.Unsupported, K.N.InvalidInput):
        if w_max <= 32:
            raise
        return K.KernelOperator(spec.family, spec.lengthscale, spec.outputscale, Xr, Xc,
                                w_max=32)


def posterior_mean(belief: PosteriorBelief, X_test, chunk: int = 512, dtype=None):
    """m_c + K(X*, X) v per test point and output, (N_test, C)."""
    dt = resolve_dtype(dtype if dtype is not None else belief.dtype)
    C = belief.prior.num_outputs
    n = belief.train_inputs.shape[0]
    V = belief.weights_device(dt).view(n, C)
    nt = X_test.shape[0]
    out = torch.empty((nt, C), dtype=dt, device=V.device)
    for op, cols in _cross_ops(belief, X_test, dt):
        if len(cols) == C:
            op.apply(V, out=out)
        else:
            idx = torch.tensor(cols, device=V.device)
            out[:, cols] = op.apply(V.index_select(1, idx).contiguous())
    K.allreduce_partial(out)  # row-sharded belief: this rank's columns of K(X*, X) only
    res = to_host(out) + np.asarray(belief.prior.mean, dtype=np.float64)[None, :]
    return res


def posterior_marginal_var(belief: PosteriorBelief, X_test, chunk: int = 512, dtype=None):
    """sigma_c^2 - sum_r (K_c(X*, X) Q[c::C, r])^2, clamped at 0, (N_test, C)."""
    dt = resolve_dtype(dtype if dtype is not None else belief.dtype)
    C = belief.prior.num_outputs
    n = belief.train_inputs.shape[0]
    nt = X_test.shape[0]
    s2 = torch.tensor(belief.prior.marginal_prior_variance(), dtype=torch.float64)
    R = belief.root.rank
    if R == 0:
        return np.tile(s2.numpy(), (nt, 1)).astype(np.float64)
    Qb = belief.root.block(dt)                         # (R, n*C)
    # W[j, c*R + r] = Q_r[j*C + c]
    W = Qb.view(R, n, C).permute(1, 2, 0).contiguous().view(n, C * R)
    dev = W.device
    var = torch.empty((nt, C), dtype=dt, device=dev)
    s2d = s2.to(dev)
    # K2: the fused cross-kernel posterior (ncgp_kop_posterior_var): each
    # kernel tile once per 128 root columns, square-reduce in the kernel's
    # fp64 reduction pass, A never stored
    # (a row-sharded belief holds a column slice of K(X*, X): the partial
    # products must be summed over the ranks before squaring, so it takes the
    # product path below)
    if dt == torch.float32 and C * R > 32 and K.get_reducer() is None:
        done = True
        for op, cols in _cross_ops(belief, X_test, dt, w_max=128):
            if op.impl != "tcgen05" or op.w_max <= 32:
                done = False
                break
            if len(cols) == C:
                op.posterior_var(W, C, R, s2d, out=var)
            else:
                idx = torch.tensor(cols, device=dev)
                Wg = W.view(n, C, R).index_select(1, idx).reshape(n, len(cols) * R).contiguous()
                var[:, cols] = op.posterior_var(Wg, len(cols), R, s2d[idx])
        if done:
            return to_host(var)
    # bound the (rows x C*R) intermediate to ~256 MiB
    rows = max(128, min(nt, int(2 ** 28 // max(1, C * R * W.element_size()))) // 128 * 128)
    for t0 in range(0, nt, rows):
        t1 = min(nt, t0 + rows)
        A = torch.empty((t1 - t0, C * R), dtype=dt, device=dev)
        for op, cols in _cross_ops(belief, X_test[t0:t1], dt):
            if len(cols) == C:
                op.apply(W, out=A)
            else:
                for c in cols:
                    op.apply(W[:, c * R:(c + 1) * R], out=A[:, c * R:(c + 1) * R])
        K.allreduce_partial(A)
        K.marginal_var(A, C, R, s2d, out=var[t0:t1])
    return to_host(var)


def posterior_covariance(belief: PosteriorBelief, X_test, dtype=None) -> np.ndarray:
    """Full predictive covariance over (point, output) pairs, CN layout,
    K(X*, X*) - A A' with A = K(X*, X) Q (posterior.py:87-101); dense in
    the test dimension, limited to 1000 test points like the reference.
    Both products run on K1 (identity blocks for K(X*, X*), the root block
    for A); the (N* C)^2 assembly is a device GEMM."""
    Xt = np.asarray(X_test, dtype=np.float64)
    if Xt.shape[0] > 1000:
        raise InvalidInput("full covariance limited to 1000 test points")
    dt = resolve_dtype(dtype if dtype is not None else belief.dtype)
    C = belief.prior.num_outputs
    nt, n = Xt.shape[0], belief.train_inputs.shape[0]
    Xr = to_device(Xt, dt)
    Xc = to_device(belief.train_inputs, dt)
    out = torch.zeros((nt * C, nt * C), dtype=dt, device=Xr.device)
    o4 = out.view(nt, C, nt, C)
    eye = torch.eye(nt, dtype=dt, device=Xr.device)
    R = belief.root.rank
    Qb = belief.root.block(dt) if R else None
    for spec, cols in belief.prior.spec_groups():
        op_tt = K.KernelOperator(spec.family, spec.lengthscale, spec.outputscale, Xr, w_max=32)
        with op_tt.sym_mode(0):
            Ktt = op_tt.apply(eye)
        for c in cols:
            o4[:, c, :, c] = Ktt
    if R:
        A = torch.empty((nt, C, R), dtype=dt, device=Xr.device)
        W = Qb.view(R, n, C).permute(1, 2, 0)                # W[j, c, r] = Q[j C + c, r]
        for op, cols in _cross_ops(belief, Xt, dt):
            for c in cols:
                A[:, c, :] = op.apply(W[:, c, :].contiguous())
        A2 = A.reshape(nt * C, R)
        out -= A2 @ A2.t()
    return to_host(out)


def probit_predict(mean, var) -> np.ndarray:
    """Moderated softmax / logistic probabilities (posterior.py:104-121)."""
    mean = np.atleast_2d(np.asarray(mean, dtype=np.float64))
    var = np.atleast_2d(np.asarray(var, dtype=np.float64))
    if mean.shape != var.shape:
        raise DimensionMismatch(f"mean {mean.shape} vs var {var.shape}")
    if (var < 0).any():
        raise InvalidInput("variances must be nonnegative")
    z = mean / np.sqrt(1.0 + (math.pi / 8.0) * var)
    if mean.shape[1] == 1:
        from scipy.special import expit
        p = expit(z[:, 0])
        return np.column_stack([1.0 - p, p])
    e = np.exp(z - z.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


from .metrics import (PredictiveSummary, mc_predict, metric_accuracy, metric_ece,  # noqa: E402
                      metric_nll, poisson_predictive_density)
