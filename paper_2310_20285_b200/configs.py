"""Seeded synthetic stand-ins for the five BASELINE.json configurations.

BASELINE.json names no public dataset for these configs; SURVEY.md 8(d)
fixes the generators restated here.  Everything is drawn on the host in
float64 with ``numpy.random.default_rng(seed)`` in a fixed order
(mixture means, component labels, inputs, label flips, then the test set
with the same recipe), so the GPU path and the CPU oracle see identical
arrays.

Returned dict keys: ``X`` (N, D), ``y`` (N,), ``X_test``, ``y_test``,
``C`` (latent outputs; 1 for Bernoulli), ``kernel`` ((family, l, s2)),
``likelihood`` ("bernoulli_logistic" | "softmax"), the solver schedule
(``steps``, ``inner``, ``policy``, ``recycle``, ``rank``, ``delta``) and
``dtype``.
"""

from __future__ import annotations

import numpy as np


def _mixture(rng, means, sigma, n):
    C, D = means.shape
    lab = rng.integers(0, C, size=n)
    X = means[lab] + sigma * rng.standard_normal((n, D))
    return X, lab


def cfg1(seed: int = 0, n: int = 1000, n_test: int = 500) -> dict:
    """Binary Bernoulli-logit, D=2, x ~ U[-3,3]^2, y = 1[sin x1 + cos x2 + e > 0]."""
    rng = np.random.default_rng(seed)

    def draw(m):
        X = rng.uniform(-3.0, 3.0, size=(m, 2))
        eps = 0.1 * rng.standard_normal(m)
        y = (np.sin(X[:, 0]) + np.cos(X[:, 1]) + eps > 0).astype(np.int64)
        return X, y

    X, y = draw(n)
    Xt, yt = draw(n_test)
    return dict(name="cfg1", X=X, y=y, X_test=Xt, y_test=yt, C=1,
                kernel=("rbf", 1.0, 1.0), likelihood="bernoulli_logistic",
                steps=5, inner=20, policy="unit", recycle=False, rank=None,
                delta=1e-12, dtype="float64")


def cfg2(seed: int = 0, n: int = 5000, n_test: int = 1000) -> dict:
    """3-class softmax; means on a circle of radius 2, sigma 0.8, D=2."""
    rng = np.random.default_rng(seed)
    ang = 2.0 * np.pi * np.arange(3) / 3.0
    means = 2.0 * np.column_stack([np.cos(ang), np.sin(ang)])
    X, y = _mixture(rng, means, 0.8, n)
    Xt, yt = _mixture(rng, means, 0.8, n_test)
    return dict(name="cfg2", X=X, y=y, X_test=Xt, y_test=yt, C=3,
                kernel=("rbf", 1.0, 2.0), likelihood="softmax",
                steps=10, inner=50, policy="residual", recycle=True,
                rank=None, delta=0.01, dtype="float32")


def cfg3(seed: int = 0, n: int = 1_000_000, d: int = 8, w: int = 32,
         family: str = "rbf") -> dict:
    """Kernel-operator microbenchmark K(X, X) S, X ~ N(0, I_8), S ~ N(0, 1)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    S = rng.standard_normal((n, w))
    return dict(name="cfg3" if family == "rbf" else "cfg3-matern", X=X, S=S,
                kernel=(family, 1.5, 1.0), dtype="float32")


def cfg4(seed: int = 0, n: int = 100_000, n_test: int = 10_000) -> dict:
    """10-class softmax, D=20, means ~ N(0, 4 I), sigma 1, Matern-3/2 l=3."""
    rng = np.random.default_rng(seed)
    means = 2.0 * rng.standard_normal((10, 20))
    X, y = _mixture(rng, means, 1.0, n)
    Xt, yt = _mixture(rng, means, 1.0, n_test)
    return dict(name="cfg4", X=X, y=y, X_test=Xt, y_test=yt, C=10,
                kernel=("matern32", 3.0, 1.0), likelihood="softmax",
                steps=8, inner=100, policy="residual", recycle=True,
                rank=200, delta=0.01, dtype="float32")


def cfg5(seed: int = 0, n: int = 1_000_000, n_test: int = 50_000) -> dict:
    """10-class softmax, D=50, means ~ N(0, 2 I), sigma 1, 5% label flips to a
    uniformly drawn *different* class, RBF l=5."""
    rng = np.random.default_rng(seed)
    means = np.sqrt(2.0) * rng.standard_normal((10, 50))
    X, y = _mixture(rng, means, 1.0, n)
    flip = rng.random(n) < 0.05
    shift = rng.integers(1, 10, size=n)
    y = np.where(flip, (y + shift) % 10, y)
    Xt, yt = _mixture(rng, means, 1.0, n_test)
    return dict(name="cfg5", X=X, y=y, X_test=Xt, y_test=yt, C=10,
                kernel=("rbf", 5.0, 1.0), likelihood="softmax",
                steps=6, inner=64, policy="residual", recycle=True,
                rank=256, delta=0.01, dtype="float32")


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}
