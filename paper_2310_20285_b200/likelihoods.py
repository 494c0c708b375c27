"""Log-concave observation models on the device (mirror of ncgp/likelihoods.py).

The public contract is the reference's ``Likelihood`` (likelihoods.py:44-78):
``log_lik``, ``grad_log_lik``, ``w_matvec``, ``w_inv_matvec(f, v, counter)``,
``w_inv_dense_blocks``, ``subset`` -- each accepting numpy arrays (returned
as numpy) or CUDA tensors (returned as CUDA tensors).  Products with W and
W^-1 / W^+ run in libncgp_b200 (K3-K5).

For the Newton loop, :meth:`Likelihood.noise_state` evaluates the per-point
statistics ONCE per Newton step (the reference recomputes pi inside every
``w_inv_matvec`` call, likelihoods.py:259) and returns a :class:`NoiseState`
whose ``apply`` is the cached W^-1 operator and whose ``pseudo_targets`` is
f + W^-1 grad (outer.py:129-131).
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import kernels as K
from .device import is_device, labels_to_device, resolve_dtype, to_device, to_host
from .exceptions import DimensionMismatch, InvalidInput

PROB_FLOOR = 1e-12  # likelihoods.py:22


class OpCount:
    """Scalar-operation tally (likelihoods.py:25-32)."""

    def __init__(self):
        self.total = 0

    def add(self, n):
        self.total += int(n)


def _latent(f, dim, dtype=None) -> torch.Tensor:
    t = to_device(f, dtype if dtype is not None else
                  (f.dtype if isinstance(f, torch.Tensor) else None))
    if t.dim() != 1 or t.shape[0] != dim:
        raise DimensionMismatch(f"latent length {t.shape[0]} != {dim}")
    if not bool(torch.isfinite(t).all()):
        raise InvalidInput("latent vector contains non-finite entries")
    return t


def _block(v, dim, dtype):
    """Operand -> ((k, dim) column block, was_vector, was_device)."""
    dev = is_device(v)
    t = to_device(v, dtype, contiguous=False)
    if t.shape[0] != dim:
        raise DimensionMismatch(f"operand length {t.shape[0]} != {dim}")
    if t.dim() == 1:
        return t.contiguous().unsqueeze(0), True, dev
    return t.t().contiguous(), False, dev


def _unblock(out: torch.Tensor, vec: bool, dev: bool):
    res = out[0] if vec else out.t()
    return res if dev else to_host(res)


class NoiseState:
    """Per-Newton-step device state: cached W^-1 (or W^+) at a fixed f.

    ``fused`` is the same operator in the form K1's fused epilogue takes
    (``("softmax", pi)`` or ``("diag", d)``, see :class:`kernels.Epi`)."""

    def __init__(self, apply_fn, yhat: torch.Tensor, grad: torch.Tensor, fused=None):
        self._apply = apply_fn
        self.pseudo_targets = yhat
        self.grad = grad
        self.fused = fused

    def apply(self, V: torch.Tensor, base: Optional[torch.Tensor] = None, alpha: float = 1.0,
              beta: float = 1.0, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """beta*base + alpha*W^-1 V for a vector or (k, dim) column block."""
        return self._apply(V, base, alpha, beta, out)

    __call__ = apply


class Likelihood:
    """Contract shared by all observation models (likelihoods.py:44-78)."""

    num_outputs = 1
    newton_is_exact = False

    def __init__(self, targets):
        self.targets = np.asarray(targets)
        self.n_points = self.targets.shape[0]
        self._dev_cache = {}

    @property
    def dim(self):
        return self.n_points * self.num_outputs

    def _labels_dev(self):
        t = self._dev_cache.get("labels")
        if t is None:
            t = labels_to_device(self.targets)
            self._dev_cache["labels"] = t
        return t

    def _dtype_of(self, *xs):
        for x in xs:
            if isinstance(x, torch.Tensor):
                return x.dtype
        return resolve_dtype(None)

    # -- device state for the Newton loop
    def noise_state(self, f: torch.Tensor) -> NoiseState:
        raise NotImplementedError

    # -- reference contract
    def log_lik(self, f) -> float:
        raise NotImplementedError

    def grad_log_lik(self, f):
        dt = self._dtype_of(f)
        st = self.noise_state(_latent(f, self.dim, dt))
        return st.grad if is_device(f) else to_host(st.grad)

    def w_inv_matvec(self, f, v, counter=None):
        dt = self._dtype_of(f, v)
        st = self.noise_state(_latent(f, self.dim, dt))
        B, vec, dev = _block(v, self.dim, dt)
        if counter is not None:
            self._count(counter, B.shape[0])
        return _unblock(st.apply(B), vec, dev)

    def w_matvec(self, f, v):
        raise NotImplementedError

    def w_inv_dense_blocks(self, f) -> np.ndarray:
        raise NotImplementedError

    def subset(self, indices) -> "Likelihood":
        raise NotImplementedError

    def _count(self, counter, k):
        pass


class _DiagonalLikelihood(Likelihood):
    """Single-output models with diagonal W (likelihoods.py:132-156)."""

    def _diag_pair(self, f: torch.Tensor):
        """(W^-1 diag, W diag, grad, pseudo targets) on the device."""
        raise NotImplementedError

    def noise_state(self, f):
        winv, _, grad, yhat = self._diag_pair(f)
        return NoiseState(lambda V, base, a, b, out: K.diag_apply(winv, V, base, a, b, out),
                          yhat, grad, fused=("diag", winv))

    def w_matvec(self, f, v):
        dt = self._dtype_of(f, v)
        _, w, _, _ = self._diag_pair(_latent(f, self.dim, dt))
        B, vec, dev = _block(v, self.dim, dt)
        return _unblock(K.diag_apply(w, B), vec, dev)

    def w_inv_dense_blocks(self, f):
        winv, _, _, _ = self._diag_pair(_latent(f, self.dim, torch.float64))
        return to_host(winv).reshape(-1, 1, 1)


class GaussianLikelihood(Likelihood):
    """Gaussian observations with fixed noise (likelihoods.py:81-129)."""

    newton_is_exact = True

    def __init__(self, targets, noise_variances, num_outputs=1):
        super().__init__(np.asarray(targets, dtype=np.float64))
        self.num_outputs = int(num_outputs)
        self.n_points = self.targets.shape[0] // self.num_outputs
        lam = np.broadcast_to(np.asarray(noise_variances, dtype=np.float64),
                              self.targets.shape).copy()
        if (lam <= 0).any():
            raise InvalidInput("noise variances must be positive")
        self.noise_variances = lam

    def _dev(self, name, arr, dt):
        key = (name, dt)
        t = self._dev_cache.get(key)
        if t is None:
            t = to_device(arr, dt)
            self._dev_cache[key] = t
        return t

    def log_lik(self, f):
        f = to_host(_latent(f, self.dim, torch.float64))
        r = f - self.targets
        lam = self.noise_variances
        return float(-0.5 * np.sum(r * r / lam + np.log(2.0 * np.pi * lam)))

    def noise_state(self, f):
        lam = self._dev("lam", self.noise_variances, f.dtype)
        y = self._dev("y", self.targets, f.dtype)
        grad = K.diag_apply(self._dev("ilam", 1.0 / self.noise_variances, f.dtype),
                            K.lincomb(1.0, y, -1.0, f))
        return NoiseState(lambda V, base, a, b, out: K.diag_apply(lam, V, base, a, b, out),
                          y.clone(), grad, fused=("diag", lam))

    def w_matvec(self, f, v):
        dt = self._dtype_of(f, v)
        B, vec, dev = _block(v, self.dim, dt)
        return _unblock(K.diag_apply(self._dev("ilam", 1.0 / self.noise_variances, dt), B),
                        vec, dev)

    def w_inv_dense_blocks(self, f):
        C = self.num_outputs
        blocks = np.zeros((self.n_points, C, C))
        idx = np.arange(C)
        blocks[:, idx, idx] = self.noise_variances.reshape(self.n_points, C)
        return blocks

    def subset(self, indices):
        base = np.asarray(indices, dtype=np.int64) * self.num_outputs
        flat = (base[:, None] + np.arange(self.num_outputs)[None, :]).ravel()
        return GaussianLikelihood(self.targets[flat], self.noise_variances[flat],
                                  self.num_outputs)


class PoissonLikelihood(_DiagonalLikelihood):
    """Poisson counts, log link (likelihoods.py:159-185)."""

    def __init__(self, counts):
        counts = np.asarray(counts)
        if (counts < 0).any():
            raise InvalidInput("Poisson counts must be nonnegative")
        super().__init__(np.asarray(counts, dtype=np.float64))
        from scipy.special import gammaln
        self._log_norm = float(np.sum(gammaln(self.targets + 1.0)))

    def log_lik(self, f):
        f = to_host(_latent(f, self.dim, torch.float64))
        return float(np.sum(self.targets * f - np.exp(f)) - self._log_norm)

    def _diag_pair(self, f):
        y = self._dev_cache.get(("y", f.dtype))
        if y is None:
            y = to_device(self.targets, f.dtype)
            self._dev_cache[("y", f.dtype)] = y
        return K.poisson_stats(f, y)

    def subset(self, indices):
        return PoissonLikelihood(self.targets[np.asarray(indices)])


class BernoulliLogisticLikelihood(_DiagonalLikelihood):
    """Binary labels through a logistic latent (likelihoods.py:188-215)."""

    def __init__(self, labels):
        labels = np.asarray(labels)
        if not np.isin(labels, (0, 1)).all():
            raise InvalidInput("binary labels must be in {0, 1}")
        super().__init__(np.asarray(labels, dtype=np.float64))

    def log_lik(self, f):
        f = to_host(_latent(f, self.dim, torch.float64))
        return float(np.sum(self.targets * f - np.logaddexp(0.0, f)))

    def _diag_pair(self, f):
        return K.bernoulli_stats(f, self._labels_dev())

    def subset(self, indices):
        return BernoulliLogisticLikelihood(self.targets[np.asarray(indices)])


class SoftmaxLikelihood(Likelihood):
    """Categorical labels through a softmax over C latents
    (likelihoods.py:218-282); W^+ is the explicit Moore-Penrose form."""

    def __init__(self, labels, num_classes):
        labels = np.asarray(labels)
        self.num_outputs = int(num_classes)
        if self.num_outputs < 2:
            raise InvalidInput("softmax needs at least two classes")
        if (labels < 0).any() or (labels >= self.num_outputs).any():
            raise InvalidInput(f"labels must lie in [0, {self.num_outputs})")
        super().__init__(np.asarray(labels, dtype=np.int64))

    def probabilities(self, f):
        dt = self._dtype_of(f)
        pi, _, _ = K.softmax_stats(_latent(f, self.dim, dt), None, self.n_points,
                                   self.num_outputs, want_grad=False, want_yhat=False)
        return pi if is_device(f) else to_host(pi)

    def log_lik(self, f):
        F = to_host(_latent(f, self.dim, torch.float64)).reshape(self.n_points,
                                                                 self.num_outputs)
        fmax = F.max(axis=1)
        lse = fmax + np.log(np.exp(F - fmax[:, None]).sum(axis=1))
        return float(np.sum(F[np.arange(self.n_points), self.targets] - lse))

    def noise_state(self, f):
        n, C = self.n_points, self.num_outputs
        pi, grad, yhat = K.softmax_stats(f, self._labels_dev(), n, C)
        st = NoiseState(lambda V, base, a, b, out: K.softmax_winv(pi, n, C, V, base, a, b, out),
                        yhat, grad, fused=("softmax", pi))
        st.pi = pi
        return st

    def w_matvec(self, f, v):
        dt = self._dtype_of(f, v)
        n, C = self.n_points, self.num_outputs
        pi, _, _ = K.softmax_stats(_latent(f, self.dim, dt), None, n, C, False, False)
        B, vec, dev = _block(v, self.dim, dt)
        return _unblock(K.softmax_w(pi, n, C, B), vec, dev)

    def _count(self, counter, k):
        size = self.n_points * self.num_outputs
        counter.add(2 * size + 5 * size * k)   # likelihoods.py:306-313

    def w_inv_dense_blocks(self, f):
        C = self.num_outputs
        pi = np.clip(self.probabilities(np.asarray(to_host(f))), PROB_FLOOR, None)
        P = np.eye(C) - np.ones((C, C)) / C
        inv = np.zeros((self.n_points, C, C))
        idx = np.arange(C)
        inv[:, idx, idx] = 1.0 / pi
        return np.einsum("ij,njk,kl->nil", P, inv, P)

    def subset(self, indices):
        return SoftmaxLikelihood(self.targets[np.asarray(indices)], self.num_outputs)


def make_likelihood(family: str, dataset, noise_variance: float = 1.0) -> Likelihood:
    """Observation model matching a dataset's domain (likelihoods.py:319-338)."""
    y = dataset.targets
    table = {"gaussian": ("real", lambda: GaussianLikelihood(np.asarray(y, dtype=np.float64),
                                                             noise_variance)),
             "poisson": ("counts", lambda: PoissonLikelihood(y)),
             "bernoulli_logistic": ("binary", lambda: BernoulliLogisticLikelihood(y)),
             "softmax": ("class-index", lambda: SoftmaxLikelihood(y, dataset.num_classes))}
    if family not in table:
        raise InvalidInput(f"unknown likelihood family {family!r}")
    domain, build = table[family]
    if dataset.domain != domain:
        raise InvalidInput(f"{family} likelihood expects {domain} targets")
    return build()
