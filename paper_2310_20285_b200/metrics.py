"""Predictive summaries and evaluation metrics (mirror of the reference's
posterior.py:125-271).

These act on the (N_test, C) latent moments that ``posterior_mean`` /
``posterior_marginal_var`` return, i.e. O(N_test C S) host arithmetic
outside the hot path, like ``probit_predict``.  The
Monte-Carlo streams follow the reference's contract: one Philox stream per
(seed, point, output), Box-Muller normals, so every result is independent
of evaluation order and equal to the reference's for the same moments.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
from scipy.special import expit, gammaln

from .exceptions import DimensionMismatch, InvalidInput

NLL_PROB_FLOOR = 1e-300  # posterior.py:24


@dataclass(frozen=True)
class PredictiveSummary:
    """Latent moments plus likelihood-mapped predictions (posterior.py:125-133)."""

    mean: np.ndarray
    variance: np.ndarray
    class_probabilities: Optional[np.ndarray] = None
    rate_median: Optional[np.ndarray] = None
    rate_lower: Optional[np.ndarray] = None
    rate_upper: Optional[np.ndarray] = None


def _stream_normals(seed: int, point: int, output: int, count: int) -> np.ndarray:
    """``count`` standard normals of the (point, output) Philox stream
    (posterior.py:136-153): uniforms u, then Box-Muller on (1 - u_a, u_b)."""
    gen = np.random.Generator(np.random.Philox(key=int(seed) & (2 ** 64 - 1),
                                               counter=[0, 0, int(output), int(point)]))
    half = (count + 1) // 2
    u = gen.random(2 * half)
    r = np.sqrt(-2.0 * np.log(1.0 - u[:half]))
    t = 2.0 * np.pi * u[half:]
    return np.concatenate([r * np.cos(t), r * np.sin(t)])[:count]


def latent_samples(mean, var, seed: int, n_samples: int) -> np.ndarray:
    """(N, C, S) samples mean + sd z per point and output (posterior.py:156-165)."""
    mean = np.atleast_2d(np.asarray(mean, dtype=np.float64))
    sd = np.sqrt(np.atleast_2d(np.asarray(var, dtype=np.float64)))
    N, C = mean.shape
    out = np.empty((N, C, n_samples))
    for i in range(N):
        for c in range(C):
            out[i, c] = mean[i, c] + sd[i, c] * _stream_normals(seed, i, c, n_samples)
    return out


def _softmax_last(a: np.ndarray) -> np.ndarray:
    e = np.exp(a - a.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def mc_predict(mean, var, likelihood, n_samples: int, seed: int) -> PredictiveSummary:
    """Monte-Carlo push of the latent belief through the likelihood
    (posterior.py:168-202): class probabilities for Bernoulli / softmax,
    the rate median with a central 95 % band for Poisson."""
    from .likelihoods import (BernoulliLogisticLikelihood, GaussianLikelihood,
                              PoissonLikelihood, SoftmaxLikelihood)
    mean = np.atleast_2d(np.asarray(mean, dtype=np.float64))
    var = np.atleast_2d(np.asarray(var, dtype=np.float64))
    if mean.shape != var.shape:
        raise DimensionMismatch(f"mean {mean.shape} vs var {var.shape}")
    if n_samples < 1:
        raise InvalidInput("n_samples must be >= 1")
    s = latent_samples(mean, var, seed, n_samples)
    if isinstance(likelihood, PoissonLikelihood):
        lo, med, hi = np.percentile(np.exp(s[:, 0, :]), [2.5, 50.0, 97.5], axis=1)
        return PredictiveSummary(mean, var, rate_median=med, rate_lower=lo, rate_upper=hi)
    if isinstance(likelihood, BernoulliLogisticLikelihood):
        p = expit(s[:, 0, :]).mean(axis=1)
        return PredictiveSummary(mean, var, class_probabilities=np.column_stack([1.0 - p, p]))
    if isinstance(likelihood, SoftmaxLikelihood):
        probs = np.stack([_softmax_last(s[i].T).mean(axis=0) for i in range(s.shape[0])])
        return PredictiveSummary(mean, var, class_probabilities=probs)
    if isinstance(likelihood, GaussianLikelihood):
        return PredictiveSummary(mean, var)
    raise InvalidInput(f"no predictive mapping for {type(likelihood).__name__}")


def poisson_predictive_density(mean, var, targets, n_samples: int, seed: int) -> np.ndarray:
    """MC average of the Poisson pmf of each target over the same streams as
    :func:`mc_predict` (posterior.py:205-218)."""
    y = np.asarray(targets, dtype=np.float64)
    s = latent_samples(mean, var, seed, n_samples)[:, 0, :]
    return np.exp(y[:, None] * s - np.exp(s) - gammaln(y + 1.0)[:, None]).mean(axis=1)


def metric_nll(probabilities, targets=None) -> float:
    """Mean negative log probability of the targets (posterior.py:221-234):
    rows of class probabilities indexed by targets, or per-point densities."""
    p = np.asarray(probabilities, dtype=np.float64)
    if p.ndim != 1:
        if targets is None:
            raise InvalidInput("class targets required for probability rows")
        p = p[np.arange(p.shape[0]), np.asarray(targets, dtype=np.int64)]
    return float(-np.mean(np.log(np.maximum(p, NLL_PROB_FLOOR))))


def metric_accuracy(probabilities, targets) -> float:
    """Fraction whose arg-max class (lowest index on ties) is the target
    (posterior.py:237-244)."""
    probs = np.asarray(probabilities, dtype=np.float64)
    return float(np.mean(np.argmax(probs, axis=1) == np.asarray(targets, dtype=np.int64)))


def metric_ece(probabilities, targets, n_bins: int = 15) -> float:
    """Expected calibration error over equal-width confidence bins,
    left-open / right-closed (posterior.py:247-271)."""
    if n_bins < 1:
        raise InvalidInput("n_bins must be >= 1")
    probs = np.asarray(probabilities, dtype=np.float64)
    conf = probs.max(axis=1)
    hit = (probs.argmax(axis=1) == np.asarray(targets, dtype=np.int64)).astype(np.float64)
    b = np.clip(np.ceil(conf * n_bins).astype(np.int64) - 1, 0, n_bins - 1)
    total, ece = conf.shape[0], 0.0
    for k in range(n_bins):
        m = b == k
        cnt = int(m.sum())
        if cnt:
            ece += (cnt / total) * abs(hit[m].mean() - conf[m].mean())
    return float(ece)
