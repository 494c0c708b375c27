"""Subset-of-Data baseline on the device (the
reference's ``sod_fit``, outer.py:268-333, and its dense step solver,
outer.py:336-370).

Exact dense Newton on a random data subset: the subset's (n_s C) x (n_s C)
prior covariance is materialised by the fused kernel-matmul (K1 applied to
identity blocks), the per-point W^-1 blocks are added on the device, and
each Newton step is a cuSOLVER Cholesky factorisation (potrf) and solve
(potrs) through ``torch.linalg`` -- a plain library factorisation, as
SURVEY.md 2.3 K7 allows for dense linear algebra.  The belief's root is
L^-T (upper triangular, outer.py:318-322), so the posterior functions of
:mod:`posterior` apply unchanged.
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels as K
from .device import resolve_dtype, to_device, to_host
from .exceptions import InvalidInput, NotPositiveDefinite
from .gp import Dataset, MultiOutputPrior
from .likelihoods import Likelihood
from .linalg import LowRankRoot
from .outer import (OUTER_CONVERGED, OUTER_MAX_STEPS, FitTrace, OuterConfig, StepRecord,
                    _SolverClock, outer_stop)
from .posterior import PosteriorBelief

SOD_JITTER = 1e-12  # outer.py:350-352


def draw_subset(n_points: int, subset_size: int, seed: int) -> np.ndarray:
    """Uniform draw without replacement from a Philox stream keyed by the
    seed, sorted (outer.py:279-283)."""
    if not 1 <= subset_size <= n_points:
        raise InvalidInput(f"subset size {subset_size} outside [1, {n_points}]")
    rng = np.random.Generator(np.random.Philox(key=seed))
    return np.sort(rng.choice(n_points, size=subset_size, replace=False))


def dense_prior_covariance(prior: MultiOutputPrior, X: torch.Tensor) -> torch.Tensor:
    """K(X, X) of the block-diagonal multi-output prior in CN layout,
    (n C) x (n C), built by K1 on identity blocks (gp.py:175-196)."""
    n, C = X.shape[0], prior.num_outputs
    Kd = torch.zeros((n * C, n * C), dtype=X.dtype, device=X.device)
    K4 = Kd.view(n, C, n, C)
    eye = torch.eye(n, dtype=X.dtype, device=X.device)
    for spec, cols in prior.spec_groups():
        op = K.KernelOperator(spec.family, spec.lengthscale, spec.outputscale, X, w_max=32)
        with op.sym_mode(0):  # plain kernel: symmetric products are not needed here
            Kx = op.apply(eye)
        Kx = 0.5 * (Kx + Kx.t())  # exact symmetry for the factorisation
        for c in cols:
            K4[:, c, :, c] = Kx
    return Kd


def _factor_solve(Khat: torch.Tensor, rhs: torch.Tensor):
    L, info = torch.linalg.cholesky_ex(Khat)
    code = int(info.item())
    if code > 0:
        raise NotPositiveDefinite(code)
    return L, torch.cholesky_solve(rhs.unsqueeze(1), L).squeeze(1)


def _solve_dense_step(K_sub: torch.Tensor, blocks: torch.Tensor, rhs: torch.Tensor):
    """Assemble K^ = K + blockdiag(W^-1 blocks) and Cholesky-solve; retry
    once with 1e-12 diagonal jitter (outer.py:336-358)."""
    n, C = blocks.shape[0], blocks.shape[1]

    def assemble():
        Kh = K_sub.clone()
        idx = torch.arange(n, device=Kh.device)
        Kh.view(n, C, n, C)[idx, :, idx, :] += blocks
        return Kh

    try:
        return _factor_solve(assemble(), rhs)
    except NotPositiveDefinite:
        Kh = assemble()
        Kh.diagonal().add_(SOD_JITTER)
        try:
            return _factor_solve(Kh, rhs)
        except NotPositiveDefinite as err:
            raise NotPositiveDefinite(
                err.dimension,
                f"dense system not positive definite (leading minor {err.dimension}), "
                f"even after 1e-12 diagonal jitter") from err


def sod_fit(prior: MultiOutputPrior, dataset: Dataset, likelihood: Likelihood,
            subset_size: int, seed: int, outer_config: OuterConfig, subset_indices=None,
            *, dtype=torch.float64):
    """Exact dense Newton on a data subset; returns (belief, trace) like
    outer.py:268-333.  ``subset_indices`` replaces the seeded draw with
    explicit point indices."""
    N = dataset.n_points
    if subset_indices is not None:
        idx = np.asarray(subset_indices, dtype=np.int64)
    else:
        idx = draw_subset(N, subset_size, seed)
    dt = resolve_dtype(dtype)
    X_sub = dataset.inputs[idx]
    lik = likelihood.subset(idx)
    ns, C = idx.shape[0], likelihood.num_outputs
    dim = ns * C

    clock = _SolverClock()
    trace = FitTrace()
    trace.factorization_size = dim
    trace.peak_buffer_entries = 2 * dim * dim

    Xd = to_device(X_sub, dt)
    K_sub = dense_prior_covariance(prior, Xd)
    mean_vec = to_device(prior.mean_vector(ns), dt)
    f = mean_vec.clone()
    g_old = None
    L = None
    weights = torch.zeros(dim, dtype=dt, device=Xd.device)
    trace.termination = OUTER_MAX_STEPS
    for i in range(outer_config.max_newton_steps):
        noise = lik.noise_state(f)
        yhat = noise.pseudo_targets
        rhs = yhat - mean_vec
        blocks = to_device(lik.w_inv_dense_blocks(f), dt)
        L, weights = _solve_dense_step(K_sub, blocks, rhs)
        g_new = K_sub @ weights
        f = g_new + mean_vec
        trace.steps.append(StepRecord(
            step=i, pseudo_target_norm=float(torch.linalg.vector_norm(yhat)),
            inner_iterations=0, cum_kernel_matvecs=i + 1, wallclock_s=clock.read(),
            residual_norm=0.0, inner_termination="dense"))
        if lik.newton_is_exact:
            trace.termination = OUTER_CONVERGED
            break
        if g_old is not None and outer_stop(g_new, g_old, outer_config.delta):
            trace.termination = OUTER_CONVERGED
            break
        g_old = g_new
    # root L^-T: triangular inverse on the device (dtrtri, outer.py:315-322)
    eye = torch.eye(dim, dtype=dt, device=Xd.device)
    Linv = torch.linalg.solve_triangular(L, eye, upper=False)
    belief = PosteriorBelief(prior=prior, train_inputs=X_sub, weights=weights,
                             root=LowRankRoot(block=Linv),  # columns = L^-T, block = L^-1
                             newton_step=len(trace.steps) - 1, solver_iterations=dim)
    trace.total_kernel_matvecs = len(trace.steps)
    trace.wallclock_s = clock.read()
    trace.belief = belief
    trace.latent = f
    trace.subset = idx
    return belief, trace
