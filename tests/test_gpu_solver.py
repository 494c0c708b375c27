"""Likelihood kernels (K3-K5), solver kernels (K6/K7) and end-to-end fits on
the B200 against the reference's golden fixtures.

Parity protocol: operator-level results at 1e-12 (fp64) /
1e-5..1e-4 (fp32); a solver iteration from identical state at 1e-8 (fp64);
end-to-end latent mean at 1e-3 and predicted labels on >= 99.9 % of test
points; marginal variance at 1e-3 only on schedules where the oracle itself
is stable (cfg1; SURVEY.md measured 1 % self-sensitivity on cfg2).
"""

import numpy as np
import pytest

from conftest import golden, specs_from

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2310_20285_b200 as P  # noqa: E402
from oracle import ncgp_oracle as O  # noqa: E402

F64, F32 = torch.float64, torch.float32


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) /
                 max(np.linalg.norm(np.asarray(b)), 1e-300))


def dev(x, dt=F64):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)


@pytest.mark.parametrize("dt,tol", [(F64, 1e-12), (F32, 2e-5)])
@pytest.mark.parametrize("C", [3, 10])
def test_softmax_kernels(C, dt, tol):
    g = golden("likelihoods")
    p = f"sm{C}_"
    lik = P.SoftmaxLikelihood(g[p + "y"], C)
    f = dev(g[p + "f"], dt)
    assert rel(lik.probabilities(f).cpu().numpy(), g[p + "pi"]) < tol
    assert rel(lik.grad_log_lik(f).cpu().numpy(), g[p + "grad"]) < tol
    assert rel(lik.w_inv_matvec(f, dev(g[p + "v"], dt)).cpu().numpy(), g[p + "winv_v"]) < tol
    assert rel(lik.w_inv_matvec(f, dev(g[p + "V"], dt)).cpu().numpy(), g[p + "winv_V"]) < tol
    assert rel(lik.w_matvec(f, dev(g[p + "v"], dt)).cpu().numpy(), g[p + "w_v"]) < tol
    assert rel(lik.w_matvec(f, dev(g[p + "V"], dt)).cpu().numpy(), g[p + "w_V"]) < tol
    assert rel(P.pseudo_targets(lik, f).cpu().numpy(), g[p + "yhat"]) < tol
    # numpy in -> numpy out, like the reference
    out = lik.w_inv_matvec(g[p + "f"], g[p + "v"])
    assert isinstance(out, np.ndarray)


def test_softmax_pinv_annihilates_constants_and_counts():
    rng = np.random.default_rng(14)
    lik = P.SoftmaxLikelihood(rng.integers(0, 4, size=5), 4)
    f = rng.normal(size=20)
    out = lik.w_inv_matvec(f, np.tile(rng.normal(), 20))
    np.testing.assert_allclose(out, np.zeros(20), atol=1e-9)
    counter = P.OpCount()
    lik.w_inv_matvec(f, rng.normal(size=20), counter=counter)
    assert counter.total == 7 * 20  # test_likelihoods.py:187-198


@pytest.mark.parametrize("dt,tol", [(F64, 1e-12), (F32, 2e-5)])
def test_bernoulli_kernels(dt, tol):
    g = golden("likelihoods")
    lik = P.BernoulliLogisticLikelihood(g["be_y"])
    f = dev(g["be_f"], dt)
    assert rel(lik.grad_log_lik(f).cpu().numpy(), g["be_grad"]) < tol
    w = lik.w_inv_matvec(f, dev(g["be_v"], dt)).cpu().numpy()
    assert np.isfinite(w).all()
    yh = P.pseudo_targets(lik, f).cpu().numpy()
    assert rel(lik.w_matvec(f, dev(g["be_v"], dt)).cpu().numpy(), g["be_w_v"]) < tol
    if dt == F64:
        # the reference clamp verbatim (likelihoods.py:210-212): every entry,
        # the saturated f = +-500 and f = 40 included, to 1e-12
        assert rel(w, g["be_winv_v"]) < tol
        assert rel(yh, g["be_yhat"]) < tol
        np.testing.assert_allclose(w, g["be_winv_v"], rtol=1e-13)
        return
    # fp32: 1 - 1e-12 rounds to 1, so the floor is applied to s * sigma(-f)
    # (SURVEY.md 8(a) a12).  At f = 40 that gives W^-1 = 1e12 exactly, where the
    # fp64 reference gets 1 / ((1 - 1e-12) (1 - (1 - 1e-12))) = 1.0000221e12 from
    # the cancellation in 1 - (1 - 1e-12): a 2.2e-5 relative difference on that
    # one entry, larger than the fp32 bound the other entries meet.
    sat = np.abs(g["be_f"]) >= 40
    assert np.allclose(w[sat], g["be_winv_v"][sat], rtol=3e-5)
    assert rel(w[~sat], g["be_winv_v"][~sat]) < tol
    assert rel(yh[~sat], g["be_yhat"][~sat]) < tol


def _solver_setup(dt):
    g = golden("solver")
    spec = P.KernelSpec(*specs_from(g["specs"])[0])
    prior = P.MultiOutputPrior(kernels=(spec,) * 3)
    op = P.PriorOperator(prior, g["X"], dtype=dt)
    lik = P.SoftmaxLikelihood(g["y"], 3)
    return g, op, lik


def test_itergp_solve_matches_reference_fp64():
    g, op, lik = _solver_setup(F64)
    n1 = lik.noise_state(dev(g["f1"]))
    buf = P.SolverBuffers.empty(180, F64)
    out = P.itergp_solve(P.RegressionSystem(op, n1, dev(g["rhs"])),
                         P.make_policy("residual", 180), buf, P.InnerConfig(max_iters=12))
    assert out.iterations_run == int(g["r_iters"])
    assert out.kernel_matvecs == int(g["r_matvecs"])
    assert rel(out.weights.cpu().numpy(), g["r_weights"]) < 1e-8
    assert rel(out.root.columns, g["r_Q"]) < 1e-8
    assert rel(buf.actions.cpu().numpy(), g["r_S"]) < 1e-8
    assert rel(buf.products.cpu().numpy(), g["r_T"]) < 1e-8
    recs = np.array([[r.iteration, r.residual_norm, r.alpha, r.eta] for r in out.records])
    np.testing.assert_allclose(recs, g["r_records"], rtol=1e-7)
    # unit-vector policy
    bu = P.SolverBuffers.empty(180, F64)
    ou = P.itergp_solve(P.RegressionSystem(op, n1, dev(g["rhs"])), P.make_policy("unit", 180),
                        bu, P.InnerConfig(max_iters=8))
    assert ou.iterations_run == int(g["u_iters"])
    assert rel(ou.weights.cpu().numpy(), g["u_weights"]) < 1e-10
    assert rel(ou.root.columns, g["u_Q"]) < 1e-10


def test_virtual_solver_run_matches_reference_fp64():
    g, op, lik = _solver_setup(F64)
    v = golden("solver_vsr")
    buf = P.SolverBuffers.empty(180, F64)
    buf.replace(g["r_S"], g["r_T"])
    n2 = lik.noise_state(dev(g["f2"]))
    root, buf = P.virtual_solver_run(buf, n2, 5)
    Q0 = root.columns
    # eigenvector signs are arbitrary: compare sign-free quantities
    np.testing.assert_allclose(Q0 @ Q0.T, v["Q0"] @ v["Q0"].T, atol=1e-9)
    S = buf.actions.cpu().numpy()
    np.testing.assert_allclose(np.abs(S), np.abs(v["S_vsr"]), atol=1e-9)
    out = P.itergp_solve(P.RegressionSystem(op, n2, dev(g["rhs2"])),
                         P.make_policy("residual", 180), buf, P.InnerConfig(max_iters=6),
                         initial_root=root)
    assert out.iterations_run == int(g["r2_iters"])
    assert rel(out.weights.cpu().numpy(), g["r2_weights"]) < 1e-7


def test_solver_seam_with_dense_operators():
    """The RegressionSystem seam accepts arbitrary device callables (the seam
    the reference's own solver tests inject dense matrices through)."""
    rng = np.random.default_rng(2)
    A = rng.normal(size=(30, 30))
    Kd = dev(A @ A.T + 0.1 * np.eye(30))
    Wd = dev(np.diag(0.5 * (0.2 + rng.random(30))))
    rhs = rng.normal(size=30)
    Kn, Wn = Kd.cpu().numpy(), Wd.cpu().numpy()
    iters = {}
    P.itergp_solve(P.RegressionSystem(lambda v: Kd @ v, lambda v: Wd @ v, dev(rhs)),
                   P.make_policy("residual", 30), P.SolverBuffers.empty(30, F64),
                   P.InnerConfig(max_iters=12, abs_tol=1e-14, rel_tol=1e-14),
                   on_iteration=lambda j, w, root, m: iters.__setitem__(j, w.cpu().numpy()))
    for j in (1, 3, 7, 12):
        ref = O.itergp_solve(lambda v: Kn @ v, lambda v: Wn @ v, rhs, "residual",
                             O.Buffers(30), j, 1e-14, 1e-14)["weights"]
        np.testing.assert_allclose(iters[j], ref, atol=1e-8)


def test_fit_cfg1_fp64_matches_reference():
    g = golden("fit_cfg1")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0),))
    ds = P.Dataset(g["X"], g["y"], "binary")
    lik = P.BernoulliLogisticLikelihood(ds.targets)
    belief, trace = P.fit(prior, ds, lik,
                          P.OuterConfig(max_newton_steps=5, delta=1e-12, inner_schedule=20,
                                        recycle=False),
                          P.InnerConfig(max_iters=1), policy_kind="unit", dtype=F64)
    assert [s.inner_iterations for s in trace.steps] == list(g["steps_iters"])
    assert trace.total_kernel_matvecs == int(g["total_matvecs"])
    assert rel(belief.weights, g["weights"]) < 1e-9
    assert rel(belief.root.columns, g["Q"]) < 1e-9
    mean = P.posterior_mean(belief, g["X_test"])
    var = P.posterior_marginal_var(belief, g["X_test"])
    assert rel(mean, g["mean"]) < 1e-9
    assert rel(var, g["var"]) < 1e-9
    probs = P.probit_predict(mean, var)
    assert np.array_equal(probs.argmax(1), g["probs"].argmax(1))


def test_fit_cfg1_fp32_within_stated_tolerances():
    g = golden("fit_cfg1")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0),))
    ds = P.Dataset(g["X"], g["y"], "binary")
    lik = P.BernoulliLogisticLikelihood(ds.targets)
    belief, trace = P.fit(prior, ds, lik,
                          P.OuterConfig(max_newton_steps=5, delta=1e-12, inner_schedule=20,
                                        recycle=False),
                          P.InnerConfig(max_iters=1), policy_kind="unit", dtype=F32)
    mean = P.posterior_mean(belief, g["X_test"])
    var = P.posterior_marginal_var(belief, g["X_test"])
    assert rel(mean, g["mean"]) < 1e-3
    assert rel(var, g["var"]) < 1e-3
    agree = np.mean(P.probit_predict(mean, var).argmax(1) == g["probs"].argmax(1))
    assert agree >= 0.999


@pytest.mark.parametrize("dt", [F64, F32])
def test_fit_cfg2_small_recycling(dt):
    g = golden("fit_cfg2s")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * 3)
    ds = P.Dataset(g["X"], g["y"], "class-index", 3)
    lik = P.SoftmaxLikelihood(ds.targets, 3)
    belief, trace = P.fit(prior, ds, lik,
                          P.OuterConfig(max_newton_steps=10, delta=0.01, inner_schedule=20,
                                        recycle=True),
                          P.InnerConfig(max_iters=1), policy_kind="residual", dtype=dt)
    mean = P.posterior_mean(belief, g["X_test"])
    var = P.posterior_marginal_var(belief, g["X_test"])
    assert rel(mean, g["mean"]) < 1e-3
    probs = P.probit_predict(mean, var)
    assert np.mean(probs.argmax(1) == g["probs"].argmax(1)) >= 0.999
    if dt == F64:
        assert [s.inner_iterations for s in trace.steps] == list(g["steps_iters"])


def _spread():
    import json
    import os
    from conftest import GOLDEN
    return json.load(open(os.path.join(GOLDEN, "fit_cfg2_spread.json")))


@pytest.mark.parametrize("dt", [F64, F32])
def test_fit_cfg2_full_size(dt):
    """BASELINE cfg2 at its full size (N = 5000, C = 3, 1000 test points, RBF
    l = 1 s2 = 2, residual policy, 10 x 50, recycling) against the reference's
    own fit (tests/golden/fit_cfg2_full.npz, outer.py:149-257).

    Asserted: latent mean within 1e-3, >= 99.9 % identical
    labels.  The marginal variance is reported beside the reference's own
    spread: the same reference fit with its K products perturbed by 1e-14
    moves the variance by ~1e-2 (tests/golden/fit_cfg2_spread.json), so a
    1e-3 variance bound cannot hold for any implementation whose rounding
    differs; it is asserted at 3x that spread (fp64) and 10x (fp32)."""
    import json
    import os
    g = golden("fit_cfg2_full")
    sp = _spread()
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * 3)
    ds = P.Dataset(g["X"], g["y"], "class-index", 3)
    lik = P.SoftmaxLikelihood(ds.targets, 3)
    belief, trace = P.fit(prior, ds, lik,
                          P.OuterConfig(max_newton_steps=10, delta=0.01, inner_schedule=50,
                                        recycle=True),
                          P.InnerConfig(max_iters=1), policy_kind="residual", dtype=dt)
    mean = P.posterior_mean(belief, g["X_test"])
    var = P.posterior_marginal_var(belief, g["X_test"])
    probs = P.probit_predict(mean, var)
    report = {
        "dtype": str(dt), "steps_iters": [s.inner_iterations for s in trace.steps],
        "ref_steps_iters": [int(i) for i in g["steps_iters"]],
        "ref_spread_steps_iters": sp["steps_iters"],
        "total_matvecs": trace.total_kernel_matvecs, "ref_total_matvecs": int(g["total_matvecs"]),
        "weights_rel": rel(belief.weights, g["weights"]), "ref_spread_weights_rel": sp["weights_rel"],
        "mean_rel": rel(mean, g["mean"]), "ref_spread_mean_rel": sp["mean_rel"],
        "var_rel": rel(var, g["var"]), "ref_spread_var_rel": sp["var_rel"],
        "label_agreement": float(np.mean(probs.argmax(1) == g["probs"].argmax(1))),
        "test_accuracy": float(np.mean(probs.argmax(1) == g["y_test"])),
        "ref_test_accuracy": float(np.mean(g["probs"].argmax(1) == g["y_test"])),
        "wallclock_s": trace.wallclock_s, "ref_wallclock_s_cpu": float(g["wallclock_s"]),
    }
    out = os.environ.get("NCGP_REPORT_DIR")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"cfg2_full_{'f64' if dt == F64 else 'f32'}.json"), "w") as fh:
            json.dump(report, fh, indent=1)
    print(report)
    assert report["mean_rel"] < 1e-3, report
    assert report["label_agreement"] >= 0.999, report
    assert report["var_rel"] < (3.0 if dt == F64 else 10.0) * sp["var_rel"], report
    if dt == F64:
        # the reference's own 1e-14 spread moves 6 + 6 iterations ([.., 49, 50] -> [.., 43, 50])
        assert abs(sum(report["steps_iters"]) - sum(report["ref_steps_iters"])) <= 15, report
    # (fp32: the explicit residual r = rhs - K^ v cannot fall below the fp32
    # rounding of K^ v, ~1e-6 |rhs|, so the 1e-5 relative tolerance exit
    # (solver.py:252) rarely fires and every step runs its 50-iteration budget)


def test_fit_cfg4_small_compressed():
    g = golden("fit_cfg4s")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("matern32", 3.0, 1.0),) * 10)
    ds = P.Dataset(g["X"], g["y"], "class-index", 10)
    lik = P.SoftmaxLikelihood(ds.targets, 10)
    belief, trace = P.fit(prior, ds, lik,
                          P.OuterConfig(max_newton_steps=3, delta=0.01, inner_schedule=8,
                                        recycle=True, compression_rank=6),
                          P.InnerConfig(max_iters=1), policy_kind="residual", dtype=F64)
    assert [s.inner_iterations for s in trace.steps] == list(g["steps_iters"])
    assert rel(belief.weights, g["weights"]) < 1e-7
    var = P.posterior_marginal_var(belief, g["X_test"])
    assert rel(var, g["var"]) < 1e-6


def test_posterior_large_width_path():
    """Variance with C*R > 64 exercises the multi-pass cross operator."""
    rng = np.random.default_rng(9)
    n, C, R = 400, 3, 40
    X = rng.standard_normal((n, 2))
    Xt = rng.standard_normal((150, 2))
    Q = rng.standard_normal((n * C, R)) * 0.05
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * C)
    b = P.PosteriorBelief(prior, X, np.zeros(n * C), P.LowRankRoot(Q))
    specs = [("rbf", 1.0, 2.0)] * C
    ref = O.posterior_marginal_var(specs, X, Q, Xt)
    assert rel(P.posterior_marginal_var(b, Xt, dtype=F64), ref) < 1e-12


def test_sharded_operator_single_rank_equals_plain():
    from paper_2310_20285_b200.parallel import ShardedPriorOperator
    g = golden("fit_cfg2s")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * 3)
    plain = P.PriorOperator(prior, g["X"], dtype=F32)
    sharded = ShardedPriorOperator(prior, g["X"], dtype=F32)
    v = dev(np.random.default_rng(0).standard_normal(g["X"].shape[0] * 3), F32)
    assert torch.equal(plain(v), sharded(v))
    ds = P.Dataset(g["X"], g["y"], "class-index", 3)
    lik = P.SoftmaxLikelihood(ds.targets, 3)
    oc = P.OuterConfig(max_newton_steps=3, delta=0.01, inner_schedule=10, recycle=True)
    b1, _ = P.fit(prior, ds, lik, oc, P.InnerConfig(max_iters=1), dtype=F32)
    b2, _ = P.fit(prior, ds, lik, oc, P.InnerConfig(max_iters=1), dtype=F32, operator=sharded)
    np.testing.assert_array_equal(b1.weights, b2.weights)


def _cfg5_fixture():
    import json
    import os
    from conftest import GOLDEN
    p = os.path.join(GOLDEN, "cfg5_trajectory.json")
    return json.load(open(p)) if os.path.exists(p) else {}


@pytest.mark.parametrize("n,dt", [("1500", F64), ("5000", F64), ("1500", F32)])
def test_fit_cfg5_trajectory_matches_oracle(n, dt):
    """cfg5 at reduced N, fp64: the Newton trajectory (inner iterations,
    termination, |yhat| per step) and the mean-label accuracy follow the
    oracle's step for step -- including the divergence of the reference's
    undamped Newton iteration that cfg5 triggers from N ~ 5000 up
    (tests/golden/make_cfg5_trajectory.py).  fp32 (the tcgen05 path) is
    checked where the iteration converges (N = 1500)."""
    from paper_2310_20285_b200 import configs
    ref = _cfg5_fixture().get(n)
    if ref is None:
        pytest.skip("fixture tests/golden/cfg5_trajectory.json lacks N=" + n)
    c = configs.cfg5(n=int(n), n_test=2000)
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*c["kernel"]),) * 10)
    ds = P.Dataset(c["X"], c["y"], "class-index", 10)
    lik = P.SoftmaxLikelihood(ds.targets, 10)
    belief, trace = P.fit(prior, ds, lik,
                          P.OuterConfig(max_newton_steps=6, delta=0.01, inner_schedule=64,
                                        recycle=True, compression_rank=256),
                          P.InnerConfig(max_iters=1), policy_kind="residual", dtype=dt)
    got = [(s.inner_iterations, s.inner_termination, s.pseudo_target_norm) for s in trace.steps]
    want = [(s["iterations"], s["termination"], s["yhat_norm"]) for s in ref["steps"]]
    assert [g[:2] for g in got] == [w[:2] for w in want]
    for (_, _, a), (_, _, b) in zip(got, want):
        assert abs(a - b) <= 1e-2 * abs(b), (a, b)
    mean = P.posterior_mean(belief, c["X_test"][:500])
    acc = float(np.mean(mean.argmax(1) == c["y_test"][:500]))
    assert abs(acc - ref["accuracy_mean_500"]) <= 0.01


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_local_blocks_fill_gather_buffer(world):
    """The per-rank blocks the sharded operator writes into its (per * world)-row
    gather buffer (before the in-place all-gather) assemble the plain product
    bitwise (the multi-rank path itself is covered with gloo on CPU)."""
    from paper_2310_20285_b200.parallel import ShardedPriorOperator, row_partition
    rng = np.random.default_rng(1)
    n, C = 3000, 3
    X = rng.standard_normal((n, 2))
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * C)
    plain = P.PriorOperator(prior, X, dtype=F32)
    sharded = ShardedPriorOperator(prior, X, dtype=F32)
    V = dev(rng.standard_normal((n, C)), F32)
    per = row_partition(n, world, 0)[2]
    full = torch.full((per * world, C), float("nan"), dtype=F32, device="cuda")
    for r in range(world):
        r0, r1, _ = row_partition(n, world, r)
        sharded.sharded.local_apply(V, full, r0, r1)
    assert torch.equal(full[:n], plain(V.reshape(-1)).reshape(n, C))


def test_recurrence_residual_mode_matches_explicit():
    """Opt-in recurrence residual: one kernel product per
    inner iteration instead of two, same iterates up to rounding (fp64)."""
    g, op, lik = _solver_setup(F64)
    n1 = lik.noise_state(dev(g["f1"]))
    runs = {}
    for mode in ("explicit", "recurrence"):
        buf = P.SolverBuffers.empty(180, F64)
        runs[mode] = P.itergp_solve(P.RegressionSystem(op, n1, dev(g["rhs"])),
                                    P.make_policy("residual", 180), buf,
                                    P.InnerConfig(max_iters=12, residual=mode))
    e, r = runs["explicit"], runs["recurrence"]
    assert r.iterations_run == e.iterations_run == int(g["r_iters"])
    assert r.kernel_matvecs == r.iterations_run
    assert e.kernel_matvecs == int(g["r_matvecs"])
    assert rel(r.weights.cpu().numpy(), e.weights.cpu().numpy()) < 1e-9
    assert rel(r.root.columns, e.root.columns) < 1e-9
    # against the reference's own iterates (golden solver.npz)
    assert rel(r.weights.cpu().numpy(), g["r_weights"]) < 1e-8
    assert rel(r.root.columns, g["r_Q"]) < 1e-8
    # from a recycled belief: K^ Q0 comes from the virtual solver run, no products
    n2 = lik.noise_state(dev(g["f2"]))
    outs = {}
    for mode in ("explicit", "recurrence"):
        buf = P.SolverBuffers.empty(180, F64)
        buf.replace(g["r_S"], g["r_T"])
        root, buf = P.virtual_solver_run(buf, n2, 5, with_kq=mode == "recurrence")
        outs[mode] = P.itergp_solve(P.RegressionSystem(op, n2, dev(g["rhs2"])),
                                    P.make_policy("residual", 180), buf,
                                    P.InnerConfig(max_iters=6, residual=mode),
                                    initial_root=root)
    assert outs["recurrence"].kernel_matvecs == outs["recurrence"].iterations_run
    assert outs["recurrence"].iterations_run == int(g["r2_iters"])
    assert rel(outs["recurrence"].weights.cpu().numpy(),
               outs["explicit"].weights.cpu().numpy()) < 1e-8
    assert rel(outs["recurrence"].weights.cpu().numpy(), g["r2_weights"]) < 1e-7


def test_fit_recurrence_mode_cfg2_small():
    g = golden("fit_cfg2s")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * 3)
    ds = P.Dataset(g["X"], g["y"], "class-index", 3)
    lik = P.SoftmaxLikelihood(ds.targets, 3)
    oc = P.OuterConfig(max_newton_steps=10, delta=0.01, inner_schedule=20, recycle=True)
    be, te = P.fit(prior, ds, lik, oc, P.InnerConfig(max_iters=1), dtype=F64)
    br, tr = P.fit(prior, ds, lik, oc, P.InnerConfig(max_iters=1, residual="recurrence"),
                   dtype=F64)
    assert tr.total_kernel_matvecs < te.total_kernel_matvecs
    me, mr = P.posterior_mean(be, g["X_test"]), P.posterior_mean(br, g["X_test"])
    assert rel(mr, me) < 1e-3
    assert np.mean(mr.argmax(1) == me.argmax(1)) >= 0.999


def test_belief_artifact_device_round_trip(tmp_path):
    """A fitted belief (device weights and root block) saves to the same bytes
    as its host copy, and a device load predicts identically."""
    from paper_2310_20285_b200.artifact import load_belief, save_belief
    g = golden("fit_cfg2s")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * 3)
    ds = P.Dataset(g["X"], g["y"], "class-index", 3)
    lik = P.SoftmaxLikelihood(ds.targets, 3)
    belief, _ = P.fit(prior, ds, lik, P.OuterConfig(max_newton_steps=2, inner_schedule=10),
                      P.InnerConfig(max_iters=1), dtype=F64)
    echo = {"prior": {"kernel": {"family": "rbf", "lengthscale": 1.0, "outputscale": 2.0}}}
    p1, p2 = tmp_path / "dev.ncgp", tmp_path / "host.ncgp"
    save_belief(p1, belief, echo)
    host = P.PosteriorBelief(prior, g["X"], belief.weights, P.LowRankRoot(belief.root.columns),
                             belief.newton_step, belief.solver_iterations)
    save_belief(p2, host, echo)
    assert p1.read_bytes() == p2.read_bytes()
    b2, _ = load_belief(p1, device=True, dtype=F64)
    np.testing.assert_array_equal(P.posterior_mean(b2, g["X_test"]),
                                  P.posterior_mean(belief, g["X_test"]))
    np.testing.assert_allclose(P.posterior_marginal_var(b2, g["X_test"]),
                               P.posterior_marginal_var(belief, g["X_test"]), rtol=0, atol=0)


@pytest.mark.parametrize("case", ["cfg1", "cfg2s", "cfg4s"])
def test_fit_fp32_with_symmetric_kernel(case, monkeypatch):
    """fp32 fits whose K(X, X) products run on the symmetric kernel (forced
    on: the golden configs are below its default size threshold) stay within
    the stated tolerances of the reference: 1e-3 on the latent mean and
    marginal variance, >= 99.9 % identical predicted labels."""
    if case == "cfg1":
        g = golden("fit_cfg1")
        prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0),))
        ds = P.Dataset(g["X"], g["y"], "binary")
        lik = P.BernoulliLogisticLikelihood(ds.targets)
        outer = P.OuterConfig(max_newton_steps=5, delta=1e-12, inner_schedule=20, recycle=False)
        kind = "unit"
    elif case == "cfg2s":
        g = golden("fit_cfg2s")
        prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * 3)
        ds = P.Dataset(g["X"], g["y"], "class-index", 3)
        lik = P.SoftmaxLikelihood(ds.targets, 3)
        outer = P.OuterConfig(max_newton_steps=10, delta=0.01, inner_schedule=20, recycle=True)
        kind = "residual"
    else:
        g = golden("fit_cfg4s")
        prior = P.MultiOutputPrior(kernels=(P.KernelSpec("matern32", 3.0, 1.0),) * 10)
        ds = P.Dataset(g["X"], g["y"], "class-index", 10)
        lik = P.SoftmaxLikelihood(ds.targets, 10)
        outer = P.OuterConfig(max_newton_steps=3, delta=0.01, inner_schedule=8, recycle=True,
                              compression_rank=6)
        kind = "residual"
    from paper_2310_20285_b200.gp import PriorOperator

    def run(sym):
        monkeypatch.setenv("NCGP_SYM", sym)
        op = PriorOperator(prior, g["X"], dtype=F32)
        belief, trace = P.fit(prior, ds, lik, outer, P.InnerConfig(max_iters=1),
                              policy_kind=kind, dtype=F32, operator=op)
        assert op.groups[0][0].last_variant == ("symmetric" if sym == "1" else "plain")
        return P.posterior_mean(belief, g["X_test"]), P.posterior_marginal_var(belief, g["X_test"])

    mean, var = run("1")
    mean0, var0 = run("0")
    # against the reference (fp64 oracle fixture)
    assert rel(mean, g["mean"]) < 1e-3
    if case != "cfg2s":
        # (cfg2s in fp32 ends its last Newton step one inner iteration earlier
        # than the fp64 reference, with either kernel, and its variance moves
        # by ~1e-2: compared with the plain-kernel fp32 fit below)
        assert rel(var, g["var"]) < 1e-3
    # against the same fit on the plain kernel.  cfg2s's fp32 variance moves by
    # ~2e-3 under a 1e-6 perturbation of the products and by ~6e-3 under the
    # blocked kernel's ~1e-5 (the recycled belief drops eigenpairs at the
    # numerical floor); fp32 against the fp64 reference it moves by ~1e-2 with
    # either kernel (above), hence its looser bound
    assert rel(mean, mean0) < 1e-3
    assert rel(var, var0) < (1e-2 if case == "cfg2s" else 1e-3)
    ref_probs = g["probs"] if "probs" in g else P.probit_predict(g["mean"], g["var"])
    agree = np.mean(np.asarray(P.probit_predict(mean, var)).argmax(1) == np.asarray(ref_probs).argmax(1))
    assert agree >= 0.999
