"""Default kernel choice vs the plain kernel on the shapes the benchmarks and
fits use (regression check).  w_max = w, as PriorOperator builds them.
usage: python tools/perf_keys.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)
SHAPES = [("cfg3 RBF", 200_000, 8, 32, "rbf", 1.5), ("cfg3 Matern", 200_000, 8, 32, "matern32", 1.5),
          ("cfg4 Matern", 100_000, 20, 10, "matern32", 3.0), ("cfg5 RBF", 200_000, 50, 10, "rbf", 5.0),
          ("RBF w=10", 200_000, 8, 10, "rbf", 1.5), ("cfg2 RBF", 5_000, 2, 3, "rbf", 1.0)]


def timed(op, V, reps):
    op.apply(V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        op.apply(V)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, n, d, w, fam, ell in SHAPES:
    rng = np.random.default_rng(0)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    op = KernelOperator(fam, ell, 1.0, X, w_max=w)
    reps = 50 if n < 50_000 else 5
    os.environ["NCGP_SYM"] = "0"
    tp = timed(op, V, reps)
    os.environ.pop("NCGP_SYM")
    td = timed(op, V, reps)
    var = {0: "plain", 1: "symmetric (pairs)", 2: "symmetric (single CTA)"}[op.last_variant_code]
    print(f"{name:12s} n={n:7d} D={d:2d} w={w:2d}: plain {tp:8.3f} ms  default {td:8.3f} ms "
          f"[{var}]  x{tp / td:.2f}", flush=True)
