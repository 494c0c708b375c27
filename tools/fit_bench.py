"""End-to-end IterNCGP fits on the BASELINE configs (synthetic, seeded).

Reports FitTrace.wallclock_s (the reference's fit-time definition, outer.py:
434-457; metric hooks excluded), K-product count, posterior timing and
test-set accuracy of the probit predictions.

usage: python tools/fit_bench.py cfg1 cfg2 cfg4 [cfg5] [--dtype float32]
"""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_20285_b200 as P
from paper_2310_20285_b200 import configs

ap = argparse.ArgumentParser()
ap.add_argument("cfgs", nargs="+")
ap.add_argument("--dtype", default=None)
ap.add_argument("--n", type=int, default=None, help="override N (smoke runs)")
ap.add_argument("--residual", default="explicit", choices=["explicit", "recurrence"],
                help="inner residual mode (recurrence: opt-in, one K product per iteration)")
args = ap.parse_args()
torch.cuda.set_device(0)
for name in args.cfgs:
    kw = {} if args.n is None else {"n": args.n}
    c = configs.CONFIGS[name](**kw)
    dt = torch.float64 if (args.dtype or c["dtype"]) == "float64" else torch.float32
    C = c["C"]
    spec = P.KernelSpec(*c["kernel"])
    prior = P.MultiOutputPrior(kernels=(spec,) * C)
    if c["likelihood"] == "softmax":
        ds = P.Dataset(c["X"], c["y"], "class-index", C)
        lik = P.SoftmaxLikelihood(ds.targets, C)
    else:
        ds = P.Dataset(c["X"], c["y"], "binary")
        lik = P.BernoulliLogisticLikelihood(ds.targets)
    oc = P.OuterConfig(max_newton_steps=c["steps"], delta=c["delta"], inner_schedule=c["inner"],
                       recycle=c["recycle"], compression_rank=c["rank"])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    belief, trace = P.fit(prior, ds, lik, oc, P.InnerConfig(max_iters=1, residual=args.residual),
                          policy_kind=c["policy"], dtype=dt)
    torch.cuda.synchronize()
    t_fit = time.perf_counter() - t0
    t1 = time.perf_counter()
    mean = P.posterior_mean(belief, c["X_test"])
    var = P.posterior_marginal_var(belief, c["X_test"])
    torch.cuda.synchronize()
    t_post = time.perf_counter() - t1
    probs = P.probit_predict(mean, var)
    acc = P.metric_accuracy(probs, c["y_test"])
    out = {"cfg": name, "n": int(c["X"].shape[0]), "C": C, "dtype": str(dt).split(".")[-1],
           "residual": args.residual,
           "fit_wallclock_s": round(trace.wallclock_s, 3), "fit_total_s": round(t_fit, 3),
           "steps": len(trace.steps), "inner_iters": [s.inner_iterations for s in trace.steps],
           "kernel_matvecs": trace.total_kernel_matvecs, "final_rank": belief.root.rank,
           "termination": trace.termination, "posterior_s": round(t_post, 3),
           "n_test": int(c["X_test"].shape[0]), "test_accuracy": round(acc, 4),
           "impl": "tcgen05" if dt == torch.float32 else "simt-fp64"}
    print(json.dumps(out), flush=True)
