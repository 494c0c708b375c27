"""Gaussian and Poisson likelihoods on the device against the reference's
own outputs (tests/golden/likelihoods_gp.npz from make_golden_r2.py):
the ``Likelihood`` contract (likelihoods.py:81-129 Gaussian, :159-185
Poisson) and small end-to-end fits through ``fit`` (outer.py:149-257),
including Gaussian's exact single Newton step (outer.py:244-247).
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2310_20285_b200 as P  # noqa: E402

F64, F32 = torch.float64, torch.float32


def rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dev(x, dt):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)


@pytest.mark.parametrize("dt,tol", [(F64, 1e-13), (F32, 1e-6)])
def test_gaussian_contract(dt, tol):
    g = golden("likelihoods_gp")
    lik = P.GaussianLikelihood(g["ga_y"], g["ga_lam"], num_outputs=int(g["ga_C"]))
    f = dev(g["ga_f"], dt)
    assert abs(lik.log_lik(g["ga_f"]) - float(g["ga_loglik"])) <= 1e-12 * abs(float(g["ga_loglik"]))
    assert rel(lik.grad_log_lik(f), g["ga_grad"]) < tol
    assert rel(lik.w_matvec(f, dev(g["ga_v"], dt)), g["ga_w_v"]) < tol
    assert rel(lik.w_matvec(f, dev(g["ga_V"], dt)), g["ga_w_V"]) < tol
    assert rel(lik.w_inv_matvec(f, dev(g["ga_v"], dt)), g["ga_winv_v"]) < tol
    assert rel(lik.w_inv_matvec(f, dev(g["ga_V"], dt)), g["ga_winv_V"]) < tol
    assert rel(P.pseudo_targets(lik, f), g["ga_yhat"]) < tol
    np.testing.assert_array_equal(lik.w_inv_dense_blocks(g["ga_f"]), g["ga_blocks"])
    # numpy in -> numpy out
    assert isinstance(lik.w_inv_matvec(g["ga_f"], g["ga_v"]), np.ndarray)


@pytest.mark.parametrize("dt,tol", [(F64, 1e-13), (F32, 1e-6)])
def test_poisson_contract(dt, tol):
    g = golden("likelihoods_gp")
    lik = P.PoissonLikelihood(g["po_y"])
    f = dev(g["po_f"], dt)
    assert abs(lik.log_lik(g["po_f"]) - float(g["po_loglik"])) <= 1e-12 * abs(float(g["po_loglik"]))
    assert rel(lik.grad_log_lik(f), g["po_grad"]) < tol
    assert rel(lik.w_matvec(f, dev(g["po_v"], dt)), g["po_w_v"]) < tol
    assert rel(lik.w_matvec(f, dev(g["po_V"], dt)), g["po_w_V"]) < tol
    assert rel(lik.w_inv_matvec(f, dev(g["po_v"], dt)), g["po_winv_v"]) < tol
    assert rel(lik.w_inv_matvec(f, dev(g["po_V"], dt)), g["po_winv_V"]) < tol
    assert rel(P.pseudo_targets(lik, f), g["po_yhat"]) < tol
    # per entry, including f = +-12 (e^12 and e^-12)
    np.testing.assert_allclose(lik.w_inv_matvec(f, dev(np.ones(50), dt)).cpu().numpy(),
                               np.exp(-g["po_f"]), rtol=tol * 10)


@pytest.mark.parametrize("dt", [F64, F32])
def test_gaussian_fit_exact_step(dt):
    """Gaussian regression: Newton is exact, so fit stops after one step
    (outer.py:244-247); posterior mean and variance against the reference."""
    g = golden("likelihoods_gp")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("matern32", 1.2, 1.5),), mean=(0.3,))
    ds = P.Dataset(g["gfit_X"], g["gfit_y"], "real")
    lik = P.GaussianLikelihood(g["gfit_y"], 0.05)
    belief, trace = P.fit(prior, ds, lik, P.OuterConfig(max_newton_steps=3, inner_schedule=30),
                          P.InnerConfig(max_iters=1), policy_kind="residual", dtype=dt)
    assert trace.termination == str(g["gfit_termination"]) == "converged"
    assert len(trace.steps) == 1
    assert trace.total_kernel_matvecs == int(g["gfit_total_matvecs"])
    tol = 1e-9 if dt == F64 else 1e-3
    if dt == F64:
        assert [s.inner_iterations for s in trace.steps] == list(g["gfit_iters"])
        assert rel(belief.weights, g["gfit_weights"]) < 1e-9
    assert rel(P.posterior_mean(belief, g["gfit_Xt"]), g["gfit_mean"]) < tol
    assert rel(P.posterior_marginal_var(belief, g["gfit_Xt"]), g["gfit_var"]) < tol


@pytest.mark.parametrize("dt", [F64, F32])
def test_poisson_fit(dt):
    g = golden("likelihoods_gp")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0),), mean=(1.0,))
    ds = P.Dataset(g["pfit_X"], g["pfit_y"], "counts")
    lik = P.PoissonLikelihood(g["pfit_y"])
    belief, trace = P.fit(prior, ds, lik,
                          P.OuterConfig(max_newton_steps=6, delta=1e-3, inner_schedule=25),
                          P.InnerConfig(max_iters=1), policy_kind="residual", dtype=dt)
    if dt == F64:
        assert [s.inner_iterations for s in trace.steps] == list(g["pfit_iters"])
        assert trace.termination == str(g["pfit_termination"])
        assert trace.total_kernel_matvecs == int(g["pfit_total_matvecs"])
        assert rel(belief.weights, g["pfit_weights"]) < 1e-8
    tol = 1e-8 if dt == F64 else 1e-3
    assert rel(P.posterior_mean(belief, g["pfit_Xt"]), g["pfit_mean"]) < tol
    assert rel(P.posterior_marginal_var(belief, g["pfit_Xt"]), g["pfit_var"]) < (tol if dt == F64 else 1e-2)
