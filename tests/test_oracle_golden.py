"""Pin the CPU oracle against fixtures produced by the real reference.

These run without a GPU.  The oracle restates the reference with the same
numpy reductions, so most comparisons are bit-exact; where a restatement
reorders an fp64 reduction the tolerance is written beside the assertion.
"""

import numpy as np
import pytest

from conftest import golden, specs_from
from oracle import ncgp_oracle as O


@pytest.mark.parametrize("name", ["matvec_cfg3_rbf", "matvec_cfg3_matern",
                                  "matvec_cfg4", "matvec_cfg5", "matvec_cfg2"])
def test_shared_spec_matvec_bit_exact(name):
    g = golden(name)
    spec = specs_from(g["specs"])[0]
    w = g["V"].shape[1]
    out = O.prior_matvec([spec] * w, g["X"], g["V"].ravel()).reshape(-1, w)
    np.testing.assert_array_equal(out, g["out"])
    # the row-sampled body used at full scale is the same arithmetic
    rows = np.array([0, 5, 17, g["X"].shape[0] - 1])
    part = O.kernel_matmul_rows(spec, g["X"][rows], g["X"], g["V"])
    np.testing.assert_array_equal(part, g["out"][rows])


def test_mixed_spec_matvec_and_tile_invariance():
    g = golden("matvec_mixed")
    specs = specs_from(g["specs"])
    np.testing.assert_array_equal(O.prior_matvec(specs, g["X"], g["v"]), g["out"])
    np.testing.assert_array_equal(O.prior_matvec(specs, g["X"], g["v"], tile=7),
                                  g["out_tile7"])
    np.testing.assert_array_equal(g["out"], g["out_tile7"])  # reference pin gp.py:106-110
    np.testing.assert_array_equal(O.cross_covariance(specs, g["X"], g["X"]), g["K"])
    np.testing.assert_allclose(g["K"] @ g["v"], g["out"], atol=1e-10)


def test_kernel_closed_forms():
    # test_gp.py:28-41 known answers
    assert O.kernel_pair(("rbf", 1.0, 1.0), [0.3, -1.2], [0.3, -1.2]) == pytest.approx(1.0)
    assert O.kernel_pair(("rbf", 1.0, 1.0), [0.0], [1.0]) == pytest.approx(np.exp(-0.5), abs=1e-12)
    a = np.sqrt(3) * 0.7
    assert O.kernel_pair(("matern32", 1.0, 2.0), [0.0], [0.7]) == pytest.approx(
        2.0 * (1 + a) * np.exp(-a), abs=1e-12)


@pytest.mark.parametrize("C", [3, 10])
def test_softmax_likelihood(C):
    g = golden("likelihoods")
    p = f"sm{C}_"
    f, y = g[p + "f"], g[p + "y"]
    np.testing.assert_array_equal(O.softmax_probabilities(f, C), g[p + "pi"])
    np.testing.assert_array_equal(O.softmax_grad(f, y, C), g[p + "grad"])
    np.testing.assert_array_equal(O.softmax_w_inv_matvec(f, g[p + "v"], C), g[p + "winv_v"])
    np.testing.assert_array_equal(O.softmax_w_inv_matvec(f, g[p + "V"], C), g[p + "winv_V"])
    np.testing.assert_array_equal(O.softmax_w_matvec(f, g[p + "v"], C), g[p + "w_v"])
    np.testing.assert_array_equal(O.softmax_w_matvec(f, g[p + "V"], C), g[p + "w_V"])
    lik = O.OracleLikelihood("softmax", y, C)
    np.testing.assert_array_equal(O.pseudo_targets(lik, f), g[p + "yhat"])


def test_bernoulli_likelihood():
    g = golden("likelihoods")
    f, y = g["be_f"], g["be_y"]
    lik = O.OracleLikelihood("bernoulli", y)
    np.testing.assert_array_equal(lik.grad(f), g["be_grad"])
    np.testing.assert_array_equal(lik.w_inv(f, g["be_v"]), g["be_winv_v"])
    np.testing.assert_array_equal(lik.w_inv(f, g["be_V"]), g["be_winv_V"])
    np.testing.assert_array_equal(lik.w(f, g["be_v"]), g["be_w_v"])
    np.testing.assert_array_equal(O.pseudo_targets(lik, f), g["be_yhat"])
    assert np.isfinite(g["be_winv_v"]).all()  # saturation clamp, test_likelihoods.py:200-203


def _solver_problem():
    g = golden("solver")
    specs = specs_from(g["specs"]) * 3
    lik = O.OracleLikelihood("softmax", g["y"], 3)
    AK = lambda w: O.prior_matvec(specs, g["X"], w)
    return g, lik, AK


def test_itergp_solve_matches_reference():
    g, lik, AK = _solver_problem()
    buf = O.Buffers(g["rhs"].shape[0])
    res = O.itergp_solve(AK, lambda w: lik.w_inv(g["f1"], w), g["rhs"], "residual",
                         buf, 12)
    assert res["iterations"] == int(g["r_iters"])
    assert res["matvecs"] == int(g["r_matvecs"])
    np.testing.assert_array_equal(res["weights"], g["r_weights"])
    np.testing.assert_array_equal(res["Q"], g["r_Q"])
    np.testing.assert_array_equal(buf.S, g["r_S"])
    np.testing.assert_array_equal(buf.T, g["r_T"])
    rec = np.array([list(r) for r in res["records"]])
    np.testing.assert_array_equal(rec, g["r_records"])
    bu = O.Buffers(g["rhs"].shape[0])
    ru = O.itergp_solve(AK, lambda w: lik.w_inv(g["f1"], w), g["rhs"], "unit", bu, 8)
    assert ru["iterations"] == int(g["u_iters"])
    np.testing.assert_array_equal(ru["weights"], g["u_weights"])
    np.testing.assert_array_equal(ru["Q"], g["u_Q"])


def test_virtual_solver_run_and_recycled_solve():
    g, lik, AK = _solver_problem()
    v = golden("solver_vsr")
    buf = O.Buffers(g["rhs"].shape[0])
    buf.replace(g["r_S"], g["r_T"])
    W2 = lambda w: lik.w_inv(g["f2"], w)
    Q0 = O.virtual_solver_run(buf, W2, 5)
    np.testing.assert_array_equal(Q0, v["Q0"])
    np.testing.assert_array_equal(buf.S, v["S_vsr"])
    np.testing.assert_array_equal(buf.T, v["T_vsr"])
    res = O.itergp_solve(AK, W2, g["rhs2"], "residual", buf, 6, Q0=Q0)
    assert res["iterations"] == int(g["r2_iters"])
    np.testing.assert_array_equal(res["weights"], g["r2_weights"])
    np.testing.assert_array_equal(res["Q"], g["r2_Q"])
    np.testing.assert_array_equal(buf.S, v["S_after"])


def test_fit_cfg1_and_prediction():
    g = golden("fit_cfg1")
    spec = ("rbf", 1.0, 1.0)
    lik = O.OracleLikelihood("bernoulli", g["y"])
    res = O.fit([spec], g["X"], lik, max_steps=5, schedule=20, recycle=False,
                delta=1e-12, policy="unit")
    assert [s["iterations"] for s in res["steps"]] == list(g["steps_iters"])
    assert res["total_matvecs"] == int(g["total_matvecs"])
    np.testing.assert_array_equal(res["weights"], g["weights"])
    np.testing.assert_array_equal(res["Q"], g["Q"])
    mean = O.posterior_mean([spec], g["X"], res["weights"], g["X_test"])
    var = O.posterior_marginal_var([spec], g["X"], res["Q"], g["X_test"])
    np.testing.assert_array_equal(mean, g["mean"])
    np.testing.assert_array_equal(var, g["var"])
    np.testing.assert_array_equal(O.probit_predict(mean, var), g["probs"])


def test_fit_cfg2_small_recycling():
    g = golden("fit_cfg2s")
    specs = [("rbf", 1.0, 2.0)] * 3
    lik = O.OracleLikelihood("softmax", g["y"], 3)
    res = O.fit(specs, g["X"], lik, max_steps=10, schedule=20, recycle=True,
                delta=0.01, policy="residual")
    assert [s["iterations"] for s in res["steps"]] == list(g["steps_iters"])
    assert res["total_matvecs"] == int(g["total_matvecs"])
    np.testing.assert_array_equal(res["weights"], g["weights"])
    np.testing.assert_array_equal(res["Q"], g["Q"])
    mean = O.posterior_mean(specs, g["X"], res["weights"], g["X_test"])
    np.testing.assert_array_equal(mean, g["mean"])


def test_fit_cfg4_small_compressed():
    g = golden("fit_cfg4s")
    specs = [("matern32", 3.0, 1.0)] * 10
    lik = O.OracleLikelihood("softmax", g["y"], 10)
    res = O.fit(specs, g["X"], lik, max_steps=3, schedule=8, recycle=True,
                rank=6, delta=0.01, policy="residual")
    assert [s["iterations"] for s in res["steps"]] == list(g["steps_iters"])
    np.testing.assert_array_equal(res["weights"], g["weights"])
    np.testing.assert_array_equal(res["Q"], g["Q"])
    var = O.posterior_marginal_var(specs, g["X"], res["Q"], g["X_test"])
    np.testing.assert_array_equal(var, g["var"])
