"""Generate golden fixtures by running the REAL reference package ``ncgp``.

Run in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Each fixture stores the seeded inputs together with the reference's outputs
so the tests never need the reference (it does not travel to the GPU box).
The fixtures pin (i) the CPU oracle (``oracle/ncgp_oracle.py``, bit-exact)
and (ii) the CUDA path (within the tolerances written in the GPU tests).
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--out", default=HERE)
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    sys.path.insert(0, ROOT)
    import ncgp  # the reference
    from ncgp import (KernelSpec, MultiOutputPrior, Dataset, prior_matvec,
                      cross_covariance, SoftmaxLikelihood,
                      BernoulliLogisticLikelihood, SolverBuffers, InnerConfig,
                      OuterConfig, RegressionSystem, itergp_solve, make_policy,
                      virtual_solver_run, fit, posterior_mean,
                      posterior_marginal_var, probit_predict, pseudo_targets,
                      LowRankRoot)
    from paper_2310_20285_b200 import configs

    def save(name, **arrs):
        path = os.path.join(args.out, name + ".npz")
        np.savez_compressed(path, **arrs)
        print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")

    def fam_code(spec):
        return {"rbf": 0, "matern32": 1}[spec.family]

    def spec_arr(specs):
        return np.array([[fam_code(s), s.lengthscale, s.outputscale] for s in specs])

    # ---- A: small mixed-spec matvec (mirrors the shape of test_gp.py:79-89)
    rng = np.random.default_rng(0)
    X = rng.normal(size=(25, 2))
    specs = (KernelSpec("rbf", 0.8, 1.5), KernelSpec("matern32", 1.2, 0.7),
             KernelSpec("rbf", 0.5, 2.0))
    prior = MultiOutputPrior(kernels=specs)
    v = rng.normal(size=75)
    save("matvec_mixed", X=X, v=v, specs=spec_arr(specs),
         out=prior_matvec(prior, X, v),
         out_tile7=prior_matvec(prior, X, v, tile=7),
         K=cross_covariance(prior, X, X))

    # ---- B/C/D: config-shaped matvecs, shared spec across w outputs
    def shared(name, X, V, spec):
        w = V.shape[1]
        pr = MultiOutputPrior(kernels=(spec,) * w)
        out = prior_matvec(pr, X, V.ravel()).reshape(-1, w)
        save(name, X=X, V=V, specs=spec_arr((spec,)), out=out)

    rng = np.random.default_rng(1)
    X3 = rng.standard_normal((1000, 8))
    S3 = rng.standard_normal((1000, 32))
    shared("matvec_cfg3_rbf", X3, S3, KernelSpec("rbf", 1.5, 1.0))
    shared("matvec_cfg3_matern", X3, S3, KernelSpec("matern32", 1.5, 1.0))
    c4 = configs.cfg4(seed=3, n=700, n_test=10)
    shared("matvec_cfg4", c4["X"], np.random.default_rng(4).standard_normal((700, 10)),
           KernelSpec("matern32", 3.0, 1.0))
    c5 = configs.cfg5(seed=5, n=600, n_test=10)
    shared("matvec_cfg5", c5["X"], np.random.default_rng(6).standard_normal((600, 10)),
           KernelSpec("rbf", 5.0, 1.0))
    c2 = configs.cfg2(seed=7, n=333, n_test=10)
    shared("matvec_cfg2", c2["X"], np.random.default_rng(8).standard_normal((333, 3)),
           KernelSpec("rbf", 1.0, 2.0))

    # ---- E: likelihoods
    rng = np.random.default_rng(10)
    lik_arrs = {}
    for C, n in ((3, 50), (10, 40)):
        y = rng.integers(0, C, size=n)
        f = 2.0 * rng.normal(size=n * C)
        f[:C] = [30.0] + [-30.0] * (C - 1)   # saturated point
        lik = SoftmaxLikelihood(y, C)
        v = rng.normal(size=n * C)
        V = rng.normal(size=(n * C, 4))
        lik_arrs.update({
            f"sm{C}_y": y, f"sm{C}_f": f, f"sm{C}_v": v, f"sm{C}_V": V,
            f"sm{C}_pi": lik.probabilities(f), f"sm{C}_grad": lik.grad_log_lik(f),
            f"sm{C}_winv_v": lik.w_inv_matvec(f, v),
            f"sm{C}_winv_V": lik.w_inv_matvec(f, V),
            f"sm{C}_w_v": lik.w_matvec(f, v), f"sm{C}_w_V": lik.w_matvec(f, V),
            f"sm{C}_yhat": pseudo_targets(lik, f)})
    n = 64
    y = rng.integers(0, 2, size=n)
    f = 3.0 * rng.normal(size=n)
    f[0], f[1], f[2] = 500.0, -500.0, 40.0
    lik = BernoulliLogisticLikelihood(y)
    v = rng.normal(size=n)
    V = rng.normal(size=(n, 3))
    lik_arrs.update({"be_y": y, "be_f": f, "be_v": v, "be_V": V,
                     "be_grad": lik.grad_log_lik(f),
                     "be_winv_v": lik.w_inv_matvec(f, v),
                     "be_winv_V": lik.w_inv_matvec(f, V),
                     "be_w_v": lik.w_matvec(f, v),
                     "be_yhat": pseudo_targets(lik, f)})
    save("likelihoods", **lik_arrs)

    # ---- F: solver state (itergp_solve + virtual_solver_run)
    rng = np.random.default_rng(20)
    n, C = 60, 3
    Xs = rng.uniform(-2, 2, size=(n, 2))
    ys = rng.integers(0, C, size=n)
    spec = KernelSpec("rbf", 1.0, 2.0)
    pr = MultiOutputPrior(kernels=(spec,) * C)
    lik = SoftmaxLikelihood(ys, C)
    f1 = rng.normal(size=n * C)
    f2 = f1 + 0.3 * rng.normal(size=n * C)
    rhs = pseudo_targets(lik, f1)
    AK = lambda w: prior_matvec(pr, Xs, w)
    AN1 = lambda w: lik.w_inv_matvec(f1, w)
    AN2 = lambda w: lik.w_inv_matvec(f2, w)
    buf = SolverBuffers.empty(n * C)
    out_r = itergp_solve(RegressionSystem(AK, AN1, rhs), make_policy("residual", n * C),
                         buf, InnerConfig(max_iters=12))
    S_before, T_before = buf.actions.copy(), buf.products.copy()
    root0, buf2 = virtual_solver_run(buf, AN2, 5)
    S_vsr, T_vsr = buf2.actions.copy(), buf2.products.copy()
    rhs2 = pseudo_targets(lik, f2)
    out_r2 = itergp_solve(RegressionSystem(AK, AN2, rhs2), make_policy("residual", n * C),
                          buf2, InnerConfig(max_iters=6), initial_root=root0)
    bufu = SolverBuffers.empty(n * C)
    out_u = itergp_solve(RegressionSystem(AK, AN1, rhs), make_policy("unit", n * C),
                         bufu, InnerConfig(max_iters=8))
    save("solver", X=Xs, y=ys, specs=spec_arr((spec,)), f1=f1, f2=f2, rhs=rhs,
         rhs2=rhs2,
         r_weights=out_r.weights, r_Q=out_r.root.columns, r_S=S_before, r_T=T_before,
         r_iters=out_r.iterations_run, r_matvecs=out_r.kernel_matvecs,
         r_rnorm=out_r.residual_norm,
         r_records=np.array([[r.iteration, r.residual_norm, r.alpha, r.eta]
                             for r in out_r.records]),
         r2_weights=out_r2.weights, r2_Q=out_r2.root.columns,
         r2_iters=out_r2.iterations_run,
         u_weights=out_u.weights, u_Q=out_u.root.columns,
         u_iters=out_u.iterations_run)
    save("solver_vsr", S_vsr=S_vsr, T_vsr=T_vsr, Q0=root0.columns,
         S_after=buf2.actions.copy(), T_after=buf2.products.copy())

    # ---- G: cfg1 full fit (fp64 reference; delta tiny -> exactly 5 steps)
    c1 = configs.cfg1(seed=0)
    ds = Dataset(c1["X"], c1["y"], "binary")
    pr = MultiOutputPrior(kernels=(KernelSpec("rbf", 1.0, 1.0),))
    lik = BernoulliLogisticLikelihood(ds.targets)
    belief, trace = fit(pr, ds, lik,
                        OuterConfig(max_newton_steps=5, delta=1e-12,
                                    inner_schedule=20, recycle=False),
                        InnerConfig(max_iters=1), policy_kind="unit")
    mean = posterior_mean(belief, c1["X_test"])
    var = posterior_marginal_var(belief, c1["X_test"])
    save("fit_cfg1", X=c1["X"], y=c1["y"], X_test=c1["X_test"], y_test=c1["y_test"],
         weights=belief.weights, Q=belief.root.columns,
         steps_iters=np.array([s.inner_iterations for s in trace.steps]),
         steps_matvecs=np.array([s.cum_kernel_matvecs for s in trace.steps]),
         total_matvecs=trace.total_kernel_matvecs,
         mean=mean, var=var, probs=probit_predict(mean, var),
         train_mean=posterior_mean(belief, c1["X"]))

    # ---- H: cfg2 scaled down (softmax, residual, recycling)
    c2 = configs.cfg2(seed=0, n=400, n_test=200)
    ds = Dataset(c2["X"], c2["y"], "class-index", 3)
    pr = MultiOutputPrior(kernels=(KernelSpec("rbf", 1.0, 2.0),) * 3)
    lik = SoftmaxLikelihood(ds.targets, 3)
    belief, trace = fit(pr, ds, lik,
                        OuterConfig(max_newton_steps=10, delta=0.01,
                                    inner_schedule=20, recycle=True),
                        InnerConfig(max_iters=1), policy_kind="residual")
    mean = posterior_mean(belief, c2["X_test"])
    var = posterior_marginal_var(belief, c2["X_test"])
    save("fit_cfg2s", X=c2["X"], y=c2["y"], X_test=c2["X_test"], y_test=c2["y_test"],
         weights=belief.weights, Q=belief.root.columns,
         steps_iters=np.array([s.inner_iterations for s in trace.steps]),
         steps_matvecs=np.array([s.cum_kernel_matvecs for s in trace.steps]),
         total_matvecs=trace.total_kernel_matvecs,
         mean=mean, var=var, probs=probit_predict(mean, var))

    # ---- I: compressed recycling (rank bound) on a small cfg4-like problem
    c4 = configs.cfg4(seed=1, n=300, n_test=100)
    ds = Dataset(c4["X"], c4["y"], "class-index", 10)
    pr = MultiOutputPrior(kernels=(KernelSpec("matern32", 3.0, 1.0),) * 10)
    lik = SoftmaxLikelihood(ds.targets, 10)
    belief, trace = fit(pr, ds, lik,
                        OuterConfig(max_newton_steps=3, delta=0.01,
                                    inner_schedule=8, recycle=True,
                                    compression_rank=6),
                        InnerConfig(max_iters=1), policy_kind="residual")
    mean = posterior_mean(belief, c4["X_test"])
    var = posterior_marginal_var(belief, c4["X_test"])
    save("fit_cfg4s", X=c4["X"], y=c4["y"], X_test=c4["X_test"], y_test=c4["y_test"],
         weights=belief.weights, Q=belief.root.columns,
         steps_iters=np.array([s.inner_iterations for s in trace.steps]),
         total_matvecs=trace.total_kernel_matvecs, mean=mean, var=var)


if __name__ == "__main__":
    main()
