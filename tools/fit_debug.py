"""Per-Newton-step diagnostics of a cfg5-like fit."""
import sys, math
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2310_20285_b200 as P
from paper_2310_20285_b200 import configs
torch.cuda.set_device(0)
n = int(sys.argv[1]); dt = torch.float64 if sys.argv[2] == "f64" else torch.float32
c = configs.cfg5(n=n, n_test=2000)
prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*c["kernel"]),) * 10)
ds = P.Dataset(c["X"], c["y"], "class-index", 10)
lik = P.SoftmaxLikelihood(ds.targets, 10)
def on_step(i, belief, trace):
    w = belief.weights_device()
    Q = belief.root.block(dt)
    s = trace.steps[-1]
    print(f"step {i}: iters={s.inner_iterations} term={s.inner_termination} rnorm={s.residual_norm:.3e} "
          f"|yhat|={s.pseudo_target_norm:.3e} |v|={float(w.norm()):.3e} finite_v={bool(torch.isfinite(w).all())} "
          f"rank={Q.shape[0]} finite_Q={bool(torch.isfinite(Q).all())} maxQ={float(Q.abs().max()) if Q.numel() else 0:.3e}",
          flush=True)
belief, trace = P.fit(prior, ds, lik, P.OuterConfig(max_newton_steps=6, delta=0.01, inner_schedule=64,
                      recycle=True, compression_rank=256), P.InnerConfig(max_iters=1),
                      policy_kind="residual", dtype=dt, on_step=on_step)
mean = P.posterior_mean(belief, c["X_test"])
var = P.posterior_marginal_var(belief, c["X_test"])
print("mean finite", np.isfinite(mean).all(), "var finite", np.isfinite(var).all(), "var min/max", var.min(), var.max())
probs = P.probit_predict(mean, var)
print("acc", P.metric_accuracy(probs, c["y_test"]), "acc(mean only)", np.mean(mean.argmax(1) == c["y_test"]))
