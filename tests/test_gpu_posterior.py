"""K2, the fused cross-kernel posterior variance (``ncgp_kop_posterior_var``;
SURVEY.md 2.3 K2 row; replaces posterior_marginal_var, posterior.py:67-84,
and its dense cross_covariance, gp.py:175-196), and the wide-RHS products
(32 < w <= 128) that share its kernel.

Tolerances: the wide kernel keeps K1's 3-term fp16 splits and sums <= 2048
training points per fp32 partial, so its products match the fp64 oracle at
K1's 1e-5 of the entry scale, and the variance -- sigma^2 minus a sum of
squares -- at 1e-5 relative (north_star: 1e-3).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2310_20285_b200 as P  # noqa: E402
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402
from oracle import ncgp_oracle as O  # noqa: E402


def _op(spec, Xt, X, w_max=128, dt=torch.float32):
    return KernelOperator(*spec, torch.from_numpy(Xt).to("cuda", dt),
                          torch.from_numpy(X).to("cuda", dt), w_max=w_max)


@pytest.mark.parametrize("nt,n,d,w,spec", [
    (300, 2000, 3, 40, ("rbf", 1.0, 1.0)),
    (1000, 9000, 8, 128, ("matern32", 1.5, 2.0)),
    (257, 20000, 50, 77, ("rbf", 5.0, 1.0)),       # cfg5 shape (D = 50), ragged rows
    (9000, 3000, 20, 100, ("matern32", 3.0, 1.0)),  # > 4096 rows: three row blocks
])
def test_wide_product_matches_oracle(nt, n, d, w, spec):
    rng = np.random.default_rng(nt + n)
    X = rng.standard_normal((n, d))
    Xt = rng.standard_normal((nt, d))
    V = rng.standard_normal((n, w))
    op = _op(spec, Xt, X)
    assert op.impl == "tcgen05" and op.w_max == 128
    got = op.apply(torch.from_numpy(V).float().cuda()).double().cpu().numpy()
    assert op.last_variant == "wide"
    rows = np.unique(np.r_[0, nt - 1, rng.choice(nt, size=min(nt, 64), replace=False)])
    ref = O.kernel_matmul_rows(spec, Xt[rows], X, V)
    bound = O.kernel_matmul_rows(spec, Xt[rows], X, np.abs(V))
    err = np.abs(got[rows] - ref) / bound
    assert err.max() < 1e-5, err.max()
    # the same columns through 32-wide blocks of the plain kernel
    plain = _op(spec, Xt, X, w_max=32).apply(torch.from_numpy(V).float().cuda()).double().cpu()
    assert float((torch.from_numpy(got) - plain).norm() / plain.norm()) < 1e-5


@pytest.mark.parametrize("C,R,spec,d", [
    (3, 100, ("rbf", 1.0, 2.0), 2),     # 300 root columns: 3 passes, classes straddle passes
    (1, 20, ("rbf", 1.0, 1.0), 2),      # C R <= 32: the product path
    (10, 40, ("matern32", 3.0, 1.0), 20),
    (10, 13, ("rbf", 5.0, 1.0), 50),    # cfg5 shape
])
def test_posterior_var_matches_oracle(C, R, spec, d):
    rng = np.random.default_rng(C * R + d)
    n, nt = 3000, 700
    X = rng.standard_normal((n, d))
    Xt = rng.standard_normal((nt, d))
    Q = rng.standard_normal((n * C, R))
    # scale the root so that sum_r A^2 reaches 60 % of sigma^2 at most: an
    # unclamped posterior, var in [0.4, 1] sigma^2 (no catastrophic cancellation)
    G = O.cross_covariance([spec] * C, X, Xt)
    Q *= np.sqrt(0.6 * spec[2] / np.max(np.sum((G @ Q) ** 2, axis=1)))
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*spec),) * C)
    b = P.PosteriorBelief(prior, X, np.zeros(n * C), P.LowRankRoot(Q))
    ref = O.posterior_marginal_var([spec] * C, X, Q, Xt)
    assert ref.min() > 0
    got = P.posterior_marginal_var(b, Xt, dtype=torch.float32)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-4
    # fp64 (the CUDA-core product path) agrees with the oracle to rounding
    got64 = P.posterior_marginal_var(b, Xt, dtype=torch.float64)
    assert np.linalg.norm(got64 - ref) / np.linalg.norm(ref) < 1e-12


def test_posterior_var_kernel_direct_and_clamp():
    """The C ABI entry point: s2 per class, the max(., 0) clamp, a
    per-class spec group (subset of classes) through posterior_marginal_var."""
    rng = np.random.default_rng(3)
    n, nt, C, R = 2000, 300, 2, 80
    X = rng.standard_normal((n, 2))
    Xt = X[:nt] + 1e-3 * rng.standard_normal((nt, 2))
    Q = rng.standard_normal((n * C, R)) * 0.3     # large root: variance clamps to 0
    W = torch.from_numpy(Q.reshape(n, C, R).reshape(n, C * R)).float().cuda()
    op = _op(("rbf", 1.0, 1.5), Xt, X)
    s2 = torch.tensor([1.5, 1.5], dtype=torch.float64, device="cuda")
    var = op.posterior_var(W, C, R, s2).double().cpu().numpy()
    ref = O.posterior_marginal_var([("rbf", 1.0, 1.5)] * C, X, Q, Xt)
    assert (var >= 0).all() and (ref == 0).any()
    assert np.abs(var - ref).max() < 1e-4 * 1.5   # clamped entries included
    # mixed specs: K2 per spec group on the gathered classes
    specs = (P.KernelSpec("rbf", 1.0, 1.5), P.KernelSpec("matern32", 2.0, 0.7))
    b = P.PosteriorBelief(P.MultiOutputPrior(kernels=specs), X, np.zeros(n * C),
                          P.LowRankRoot(Q * 0.01))
    ref2 = O.posterior_marginal_var([("rbf", 1.0, 1.5), ("matern32", 2.0, 0.7)], X, Q * 0.01, Xt)
    got2 = P.posterior_marginal_var(b, Xt, dtype=torch.float32)
    assert np.linalg.norm(got2 - ref2) / np.linalg.norm(ref2) < 1e-5


def test_posterior_var_fit_cfg4s_matches_reference():
    """A fitted belief (golden cfg4 reduction, compressed root) through K2
    against the reference's own posterior variance."""
    from conftest import golden
    g = golden("fit_cfg4s")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("matern32", 3.0, 1.0),) * 10)
    b = P.PosteriorBelief(prior, g["X"], g["weights"], P.LowRankRoot(g["Q"]))
    var = P.posterior_marginal_var(b, g["X_test"], dtype=torch.float32)
    assert np.linalg.norm(var - g["var"]) / np.linalg.norm(g["var"]) < 1e-5
