"""CPU oracle for the IterNCGP hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The shipped package
(``paper_2310_20285_b200``) never imports anything from ``oracle/``.

It restates, in plain numpy/float64, the algorithms of the reference
package ``ncgp`` (``/root/reference/pkg/src/ncgp``) that lie on the hot path
named in SURVEY.md section 8(a).  Every function cites the reference
``file:line`` it follows.  The restatement deliberately uses the *same*
numpy reductions as the reference (feature-by-feature squared distances,
numpy's pairwise ``sum`` over full rows, LAPACK ``eigh``), so on identical
inputs its outputs are bit-identical to the reference's; that property is
pinned by ``tests/test_oracle_golden.py`` against fixtures produced by the
real reference (``tests/golden/make_golden.py``).  Parity is therefore
*pinned*, not merely restated.

Kernel hyper-parameters are passed as plain ``(family, lengthscale,
outputscale)`` triples so the oracle does not depend on the product's types.
"""

from __future__ import annotations

import math
from typing import Callable, Optional, Sequence

import numpy as np

Spec = tuple  # (family: str, lengthscale: float, outputscale: float)

PROB_FLOOR = 1e-12          # likelihoods.py:22
ETA_RTOL = 1e-12            # solver.py:28
EIG_FLOOR_RTOL = 1e-10      # solver.py:33


def as_spec(spec) -> Spec:
    """Accept a triple or any object with family/lengthscale/outputscale."""
    if isinstance(spec, tuple):
        return spec
    return (spec.family, float(spec.lengthscale), float(spec.outputscale))


# --------------------------------------------------------------------------
# L1 operators: gp.py
# --------------------------------------------------------------------------

def sqdist(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Pairwise squared distances, one feature at a time (gp.py:101-113).

    The accumulation order over features is the reference's, so every entry
    is independent of the block shape.
    """
    acc = np.zeros((A.shape[0], B.shape[0]))
    for d in range(A.shape[1]):
        t = A[:, d, None] - B[None, :, d]
        t *= t
        acc += t
    return acc


def kernel_values(spec, d2: np.ndarray) -> np.ndarray:
    """Stationary kernel from squared distances (gp.py:78-98).

    RBF: s2 * exp(-d2 / (2 l^2)); Matern-3/2: s2 * (1 + a) e^-a with
    a = sqrt(3 d2) / l.  d2 is clamped at 0 first (gp.py:84).
    """
    fam, ell, s2 = as_spec(spec)
    d2 = np.maximum(d2, 0.0)
    if fam == "rbf":
        k = d2 / (-2.0 * ell ** 2)
        np.exp(k, out=k)
        k *= s2
        return k
    if fam != "matern32":
        raise ValueError(f"unknown kernel family {fam!r}")
    a = d2 * 3.0
    np.sqrt(a, out=a)
    a /= ell
    k = np.negative(a)
    np.exp(k, out=k)
    a += 1.0
    k *= a
    k *= s2
    return k


def kernel_pair(spec, x, y) -> float:
    """Single-pair kernel evaluation (gp.py:66-75)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    y = np.atleast_1d(np.asarray(y, dtype=np.float64))
    return float(kernel_values(spec, np.array([float(((x - y) ** 2).sum())]))[0])


def prior_matvec(specs: Sequence, X: np.ndarray, v: np.ndarray,
                 tile: int = 256) -> np.ndarray:
    """Tiled block-diagonal prior product K v, CN layout (gp.py:144-172).

    One Gram tile per *unique* spec per row tile (gp.py:165-170); each output
    row is reduced with numpy's pairwise sum over the full row (gp.py:171),
    which makes the result bit-identical for every tile size.
    """
    specs = [as_spec(s) for s in specs]
    X = np.asarray(X, dtype=np.float64)
    n, C = X.shape[0], len(specs)
    v = np.asarray(v, dtype=np.float64)
    if v.shape[0] != n * C:
        raise ValueError("dimension mismatch")
    per_output = v.reshape(n, C).T
    res = np.empty((C, n))
    for lo in range(0, n, tile):
        hi = min(lo + tile, n)
        d2 = sqdist(X[lo:hi], X)
        cache = {}
        for c, sp in enumerate(specs):
            if sp not in cache:
                cache[sp] = kernel_values(sp, d2)
            res[c, lo:hi] = (cache[sp] * per_output[c]).sum(axis=1)
    return res.T.ravel()


def kernel_matmul_rows(spec, X_rows: np.ndarray, X_cols: np.ndarray,
                       V: np.ndarray, tile: int = 64) -> np.ndarray:
    """K(X_rows, X_cols) @ V for one shared spec, V of shape (n_cols, w).

    This is exactly the reference tile body (gp.py:162-171) applied with all
    ``w`` right-hand columns sharing one spec -- the form SURVEY.md 8(a) a1
    uses for cfg3 (``v = S.ravel()`` with 32 identical-spec outputs).  Used
    as the row-sampled oracle at N >= 1e5.
    """
    X_rows = np.asarray(X_rows, dtype=np.float64)
    X_cols = np.asarray(X_cols, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    out = np.empty((X_rows.shape[0], V.shape[1]))
    Vt = np.ascontiguousarray(V.T)
    for lo in range(0, X_rows.shape[0], tile):
        hi = min(lo + tile, X_rows.shape[0])
        blk = kernel_values(spec, sqdist(X_rows[lo:hi], X_cols))
        for c in range(V.shape[1]):
            out[lo:hi, c] = (blk * Vt[c]).sum(axis=1)
    return out


def cross_covariance(specs: Sequence, X_train: np.ndarray,
                     X_test: np.ndarray) -> np.ndarray:
    """Dense (Nt*C) x (N*C) cross-covariance, CN both ways (gp.py:175-196)."""
    specs = [as_spec(s) for s in specs]
    X_train = np.asarray(X_train, dtype=np.float64)
    X_test = np.asarray(X_test, dtype=np.float64)
    nt, n, C = X_test.shape[0], X_train.shape[0], len(specs)
    d2 = sqdist(X_test, X_train)
    G = np.zeros((nt * C, n * C))
    cache = {}
    for c, sp in enumerate(specs):
        if sp not in cache:
            cache[sp] = kernel_values(sp, d2)
        G[c::C, c::C] = cache[sp]
    return G


def cn_to_nc(v: np.ndarray, n: int, C: int) -> np.ndarray:
    """CN -> NC permutation (gp.py:31-42)."""
    return np.asarray(v).reshape(n, C).T.ravel().copy()


def nc_to_cn(v: np.ndarray, n: int, C: int) -> np.ndarray:
    return np.asarray(v).reshape(C, n).T.ravel().copy()


# --------------------------------------------------------------------------
# L1 likelihoods: likelihoods.py
# --------------------------------------------------------------------------

def softmax_rows(F: np.ndarray) -> np.ndarray:
    """Max-subtracted row softmax (likelihoods.py:285-288)."""
    E = np.exp(F - F.max(axis=1, keepdims=True))
    return E / E.sum(axis=1, keepdims=True)


def softmax_probabilities(f: np.ndarray, C: int) -> np.ndarray:
    """pi_n per point, shape (N, C) (likelihoods.py:235-238)."""
    f = np.asarray(f, dtype=np.float64)
    return softmax_rows(f.reshape(-1, C))


def softmax_grad(f: np.ndarray, labels: np.ndarray, C: int) -> np.ndarray:
    """onehot(y) - pi, CN (likelihoods.py:247-250)."""
    G = -softmax_probabilities(f, C)
    G[np.arange(G.shape[0]), np.asarray(labels, dtype=np.int64)] += 1.0
    return G.ravel()


def softmax_pinv_apply(pi: np.ndarray, V: np.ndarray) -> np.ndarray:
    """Blockwise (I - 11'/C) diag(1/pi) (I - 11'/C) on (N, C, k) columns
    (likelihoods.py:291-310)."""
    inv = 1.0 / np.clip(pi, PROB_FLOOR, None)
    U = V - V.mean(axis=1, keepdims=True)
    U *= inv[..., None]
    U -= U.mean(axis=1, keepdims=True)
    return U


def softmax_w_inv_matvec(f: np.ndarray, v: np.ndarray, C: int) -> np.ndarray:
    """W(f)^+ v for a CN vector or (dim, k) matrix (likelihoods.py:258-262)."""
    pi = softmax_probabilities(f, C)
    v = np.asarray(v, dtype=np.float64)
    k = 1 if v.ndim == 1 else v.shape[1]
    return softmax_pinv_apply(pi, v.reshape(pi.shape[0], C, k)).reshape(v.shape)


def softmax_w_matvec(f: np.ndarray, v: np.ndarray, C: int) -> np.ndarray:
    """(diag pi_n - pi_n pi_n') v_n (likelihoods.py:252-256)."""
    pi = softmax_probabilities(f, C)
    v = np.asarray(v, dtype=np.float64)
    k = 1 if v.ndim == 1 else v.shape[1]
    Vb = v.reshape(pi.shape[0], C, k)
    out = pi[..., None] * Vb - pi[..., None] * (pi[:, None, :] @ Vb)
    return out.reshape(v.shape)


def _expit(x):
    from scipy.special import expit
    return expit(x)


def bernoulli_grad(f: np.ndarray, y: np.ndarray) -> np.ndarray:
    """y - sigma(f) (likelihoods.py:202-204)."""
    return np.asarray(y, dtype=np.float64) - _expit(np.asarray(f, dtype=np.float64))


def bernoulli_w_diag(f: np.ndarray) -> np.ndarray:
    """sigma (1 - sigma) (likelihoods.py:206-208)."""
    s = _expit(np.asarray(f, dtype=np.float64))
    return s * (1.0 - s)


def bernoulli_w_inv_diag(f: np.ndarray) -> np.ndarray:
    """1 / (s (1 - s)) with s clipped to [1e-12, 1-1e-12] (likelihoods.py:210-212)."""
    s = np.clip(_expit(np.asarray(f, dtype=np.float64)), PROB_FLOOR, 1.0 - PROB_FLOOR)
    return 1.0 / (s * (1.0 - s))


def diag_apply(w: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Diagonal product for a vector or matrix operand (likelihoods.py:149-153)."""
    v = np.asarray(v, dtype=np.float64)
    return v * (w if v.ndim == 1 else w[:, None])


class OracleLikelihood:
    """Minimal likelihood handle: 'bernoulli' (C=1) or 'softmax' (C>=2)."""

    def __init__(self, kind: str, labels, C: int = 1):
        self.kind = kind
        self.labels = np.asarray(labels)
        self.C = C if kind == "softmax" else 1
        self.n = self.labels.shape[0]

    @property
    def dim(self):
        return self.n * self.C

    def grad(self, f):
        if self.kind == "softmax":
            return softmax_grad(f, self.labels, self.C)
        return bernoulli_grad(f, self.labels)

    def w_inv(self, f, v):
        if self.kind == "softmax":
            return softmax_w_inv_matvec(f, v, self.C)
        return diag_apply(bernoulli_w_inv_diag(f), v)

    def w(self, f, v):
        if self.kind == "softmax":
            return softmax_w_matvec(f, v, self.C)
        return diag_apply(bernoulli_w_diag(f), v)


def pseudo_targets(lik: OracleLikelihood, f: np.ndarray) -> np.ndarray:
    """f + W^-1 grad (outer.py:129-131 / 460-462)."""
    return f + lik.w_inv(f, lik.grad(f))


# --------------------------------------------------------------------------
# L0 dense substrate: linalg.py
# --------------------------------------------------------------------------

def lowrank_apply(Q: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Q (Q' w) (linalg.py:51-62)."""
    if Q.shape[1] == 0:
        return np.zeros_like(np.asarray(w, dtype=np.float64))
    return Q @ (Q.T @ w)


def eigh_desc(M: np.ndarray, keep: int):
    """Symmetrise, eigh, sort descending, keep ``keep`` (linalg.py:65-86)."""
    n = M.shape[0]
    if n == 0 or keep == 0:
        return np.zeros((n, 0)), np.zeros(0)
    vals, vecs = np.linalg.eigh(0.5 * (M + M.T))
    order = np.argsort(vals)[::-1][:keep]
    return np.ascontiguousarray(vecs[:, order]), vals[order]


# --------------------------------------------------------------------------
# L2 inner solver: solver.py
# --------------------------------------------------------------------------

class Buffers:
    """Action / product column store (solver.py:60-107).

    Storage mirrors the reference exactly -- row-major (dim, capacity)
    arrays grown by doubling from 8 and exposed as column-prefix views --
    because BLAS picks different kernels (and rounding) for strided views.
    """

    def __init__(self, dim: int):
        self.dim = dim
        self.count = 0
        self._S = np.empty((dim, 0))
        self._T = np.empty((dim, 0))

    @property
    def S(self):
        return self._S[:, :self.count]

    @property
    def T(self):
        return self._T[:, :self.count]

    def append(self, s, t):
        if self.count == self._S.shape[1]:
            cap = max(8, 2 * self.count)
            for name in ("_S", "_T"):
                old = getattr(self, name)
                grown = np.empty((self.dim, cap))
                grown[:, :self.count] = old[:, :self.count]
                setattr(self, name, grown)
        self._S[:, self.count] = s
        self._T[:, self.count] = t
        self.count += 1

    def replace(self, S, T):
        self._S = np.array(S)
        self._T = np.array(T)
        self.count = S.shape[1]


def itergp_solve(apply_K: Callable, apply_Winv: Callable, rhs: np.ndarray,
                 policy: str, buffers: Buffers, max_iters: int,
                 abs_tol: float = 1e-5, rel_tol: float = 1e-5,
                 Q0: Optional[np.ndarray] = None, on_iter=None) -> dict:
    """Algorithm 2 (solver.py:203-291).

    Returns a dict with weights, root columns Q, iterations, termination,
    matvec count, residual norm and per-iteration (rnorm, alpha, eta).
    """
    dim = rhs.shape[0]
    Q0 = np.zeros((dim, 0)) if Q0 is None else np.asarray(Q0, dtype=np.float64)
    base = Q0.shape[1]
    store = np.empty((dim, base + max_iters))   # preallocated like solver.py:227-230
    store[:, :base] = Q0
    ncols = base
    v = lowrank_apply(Q0, rhs) if base else np.zeros(dim)
    fresh = base == 0
    matvecs = 0
    rnorm = float(np.linalg.norm(rhs))
    tol = max(abs_tol, rel_tol * float(np.linalg.norm(rhs)))
    records = []
    j = 0
    unit_next = 0
    term = "max_iters"
    while True:
        if j >= max_iters:
            term = "max_iters"
            break
        if fresh:
            r = rhs.copy()
        else:
            r = rhs - apply_K(v) - apply_Winv(v)
            matvecs += 1
        rnorm = float(np.linalg.norm(r))
        if rnorm < tol:
            term = "converged"
            break
        if policy == "unit":
            if unit_next >= dim:
                term = "max_iters"
                break
            s = np.zeros(dim)
            s[unit_next] = 1.0
            unit_next += 1
        else:
            s = r.copy()
        alpha = float(s @ r)
        t = apply_K(s)
        matvecs += 1
        buffers.append(s, t)
        z = t + apply_Winv(s)
        Qv = store[:, :ncols]
        d = s if ncols == 0 else s - Qv @ (Qv.T @ z)
        eta = float(z @ d)
        if eta <= ETA_RTOL * float(np.linalg.norm(s)) * float(np.linalg.norm(z)):
            term = "eta_breakdown"
            records.append((j + 1, rnorm, alpha, eta))
            break
        store[:, ncols] = d / np.sqrt(eta)
        ncols += 1
        v = v + (alpha / eta) * d
        fresh = False
        j += 1
        records.append((j, rnorm, alpha, eta))
        if on_iter is not None:
            on_iter(j, v, store[:, :ncols], matvecs)
    return dict(weights=v, Q=store[:, :ncols], iterations=j, termination=term,
                matvecs=matvecs, residual_norm=rnorm, records=records)


def virtual_solver_run(buffers: Buffers, apply_Winv: Callable,
                       rank_bound: Optional[int] = None) -> np.ndarray:
    """Algorithm 3 (solver.py:294-331); rotates ``buffers`` in place and
    returns the recycled root Q0."""
    if buffers.count == 0:
        return np.zeros((buffers.dim, 0))
    S, T = buffers.S, buffers.T
    M = S.T @ (T + apply_Winv(S))
    U, lam = eigh_desc(M, buffers.count)
    top = float(lam[0]) if lam.size else 0.0
    keep = lam > EIG_FLOOR_RTOL * max(top, 0.0)
    lam, U = lam[keep], U[:, keep]
    if rank_bound is not None and lam.shape[0] > rank_bound:
        lam, U = lam[:rank_bound], U[:, :rank_bound]
    S_new, T_new = S @ U, T @ U
    buffers.replace(S_new, T_new)
    if lam.size == 0:
        return np.zeros((buffers.dim, 0))
    return S_new / np.sqrt(lam)[None, :]


# --------------------------------------------------------------------------
# L3 outer loop: outer.py
# --------------------------------------------------------------------------

def relative_change_stop(g_new, g_old, delta) -> bool:
    """outer_stop (outer.py:140-146)."""
    nn = float(np.linalg.norm(g_new))
    diff = float(np.linalg.norm(g_new - g_old))
    if nn == 0.0:
        return diff == 0.0
    return diff / nn <= delta


def fit(specs: Sequence, X: np.ndarray, lik: OracleLikelihood,
        max_steps: int, schedule, recycle: bool = True,
        rank: Optional[int] = None, delta: float = 0.01,
        abs_tol: float = 1e-5, rel_tol: float = 1e-5,
        policy: str = "residual", means: Optional[Sequence[float]] = None,
        apply_K: Optional[Callable] = None) -> dict:
    """Algorithm 1 (outer.py:149-257), without hooks or clocks.

    ``apply_K`` overrides the prior product (default: :func:`prior_matvec`).
    Returns weights, root Q, f, per-step records and totals.
    """
    specs = [as_spec(s) for s in specs]
    n, C = X.shape[0], lik.C
    dim = n * C
    m = np.tile(np.asarray(means if means else [0.0] * C, dtype=np.float64), n)
    Kop = apply_K or (lambda w: prior_matvec(specs, X, w))
    buffers = Buffers(dim)
    f = m.copy()
    g_old = None
    total = 0
    steps = []
    out = None
    term = "max_steps"

    def budget(i):
        if isinstance(schedule, int):
            return schedule
        return int(list(schedule)[min(i, len(schedule) - 1)])

    for i in range(max_steps):
        yhat = pseudo_targets(lik, f)
        rhs = yhat - m
        f_now = f
        Winv = lambda w, _f=f_now: lik.w_inv(_f, w)
        if recycle:
            Q0 = virtual_solver_run(buffers, Winv, rank)
        else:
            buffers = Buffers(dim)
            Q0 = np.zeros((dim, 0))
        res = itergp_solve(Kop, Winv, rhs, policy, buffers, budget(i),
                           abs_tol, rel_tol, Q0=Q0)
        total += res["matvecs"] + 1
        f_new = Kop(res["weights"]) + m
        g_new = f_new - m
        steps.append(dict(step=i, iterations=res["iterations"],
                          cum_matvecs=total, residual_norm=res["residual_norm"],
                          termination=res["termination"],
                          yhat_norm=float(np.linalg.norm(yhat))))
        out = res
        f = f_new
        if res["termination"] == "eta_breakdown" and res["iterations"] == 0:
            term = "stalled"
            break
        if g_old is not None and relative_change_stop(g_new, g_old, delta):
            term = "converged"
            break
        g_old = g_new
    return dict(weights=out["weights"], Q=out["Q"], f=f, steps=steps,
                total_matvecs=total, termination=term)


# --------------------------------------------------------------------------
# L4 prediction: posterior.py
# --------------------------------------------------------------------------

def posterior_mean(specs, X_train, weights, X_test, means=None,
                   chunk: int = 512) -> np.ndarray:
    """m_c + K(X*, X) v, chunked (posterior.py:52-64)."""
    specs = [as_spec(s) for s in specs]
    C = len(specs)
    mc = np.asarray(means if means else [0.0] * C, dtype=np.float64)
    nt = X_test.shape[0]
    out = np.empty((nt, C))
    for lo in range(0, nt, chunk):
        hi = min(lo + chunk, nt)
        G = cross_covariance(specs, X_train, X_test[lo:hi])
        out[lo:hi] = (G @ weights).reshape(hi - lo, C) + mc
    return out


def posterior_marginal_var(specs, X_train, Q, X_test,
                           chunk: int = 512) -> np.ndarray:
    """sigma_c^2 - rowsum((K(X*,X) Q)^2), clamped at 0 (posterior.py:67-84)."""
    specs = [as_spec(s) for s in specs]
    C = len(specs)
    pv = np.array([s[2] for s in specs])
    nt = X_test.shape[0]
    out = np.empty((nt, C))
    for lo in range(0, nt, chunk):
        hi = min(lo + chunk, nt)
        blk = np.tile(pv, hi - lo).astype(np.float64)
        if Q.shape[1]:
            G = cross_covariance(specs, X_train, X_test[lo:hi])
            A = G @ Q
            blk -= np.sum(A * A, axis=1)
        out[lo:hi] = blk.reshape(hi - lo, C)
    return np.maximum(out, 0.0)


def probit_predict(mean: np.ndarray, var: np.ndarray) -> np.ndarray:
    """Moderated softmax / logistic (posterior.py:104-121)."""
    mean = np.atleast_2d(np.asarray(mean, dtype=np.float64))
    var = np.atleast_2d(np.asarray(var, dtype=np.float64))
    z = mean / np.sqrt(1.0 + (math.pi / 8.0) * var)
    if mean.shape[1] == 1:
        p = _expit(z[:, 0])
        return np.column_stack([1.0 - p, p])
    return softmax_rows(z)


# --------------------------------------------------------------------------
# Row-sampled cost model for the CPU baseline
# --------------------------------------------------------------------------

def time_tile_body(spec, X: np.ndarray, V: np.ndarray, rows: np.ndarray,
                   tile: int = 64):
    """Run the reference tile body on ``rows`` against all columns and return
    (result, seconds).  Used by bench.py's cpu_baseline leg only."""
    import time
    t0 = time.perf_counter()
    out = kernel_matmul_rows(spec, X[rows], X, V, tile=tile)
    return out, time.perf_counter() - t0
