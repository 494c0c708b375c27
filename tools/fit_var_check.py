import os, sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2310_20285_b200 as P
from paper_2310_20285_b200.gp import PriorOperator
from conftest import golden
g = golden("fit_cfg2s")
def rel(a, b): a=np.asarray(a); b=np.asarray(b); return float(np.linalg.norm(a-b)/np.linalg.norm(b))
for sym in ("0", "1"):
    os.environ["NCGP_SYM"] = sym
    for dt in (torch.float32, torch.float64):
        prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * 3)
        ds = P.Dataset(g["X"], g["y"], "class-index", 3)
        lik = P.SoftmaxLikelihood(ds.targets, 3)
        op = PriorOperator(prior, g["X"], dtype=dt)
        belief, trace = P.fit(prior, ds, lik, P.OuterConfig(max_newton_steps=10, delta=0.01, inner_schedule=20, recycle=True),
                              P.InnerConfig(max_iters=1), policy_kind="residual", dtype=dt, operator=op)
        mean = P.posterior_mean(belief, g["X_test"]); var = P.posterior_marginal_var(belief, g["X_test"])
        print(sym, dt, op.groups[0][0].last_variant, "mean", rel(mean, g["mean"]), "var", rel(var, g["var"]), [s.inner_iterations for s in trace.steps])
