"""Single-CTA symmetric kernel vs the plain kernel over n (policy threshold)
and at cfg3 size.  usage: python tools/sym1_sweep.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)
os.environ["NCGP_SYM_CG"] = "1"


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


for n, d, w, fam in [(10_000, 8, 10, "rbf"), (20_000, 8, 10, "rbf"), (40_000, 8, 10, "rbf"), (70_000, 8, 10, "rbf"),
                     (20_000, 8, 32, "matern32"), (40_000, 8, 32, "matern32"), (70_000, 8, 32, "rbf"),
                     (1_000_000, 8, 32, "rbf"), (1_000_000, 8, 32, "matern32"), (1_000_000, 8, 10, "rbf")]:
    rng = np.random.default_rng(0)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    op = KernelOperator(fam, 1.5, 1.0, X, w_max=32)
    reps = 2 if n >= 1_000_000 else 10
    os.environ["NCGP_SYM"] = "0"
    tp = timed(op, V, reps)
    os.environ["NCGP_SYM"] = "1"
    ts = timed(op, V, reps)
    print(f"{fam:9s} n={n:8d} d={d} w={w:2d}: plain {tp:9.3f} ms  sym1 {ts:9.3f} ms  ({op.last_variant})  "
          f"speed-up {tp / ts:5.2f}", flush=True)
