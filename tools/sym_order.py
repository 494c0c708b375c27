"""Symmetric kernel: block-major vs pair-major work list at cfg3 scale.
usage: python tools/sym_order.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)
for n, d, w, fam, ell in [(1_000_000, 8, 32, "matern32", 1.5), (1_000_000, 8, 10, "rbf", 1.5),
                          (200_000, 8, 32, "matern32", 1.5), (100_000, 20, 10, "matern32", 3.0)]:
    rng = np.random.default_rng(0)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    line = f"{fam:9s} n={n} d={d} w={w}:"
    ref = None
    for order in ("block", "pair"):
        os.environ["NCGP_SYM_ORDER"] = order
        op = KernelOperator(fam, ell, 1.0, X, w_max=32)
        out = op.apply(V)
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(2):
            op.apply(V)
        e1.record()
        torch.cuda.synchronize()
        line += f"  {order} {e0.elapsed_time(e1) / 2:8.3f} ms ({op.last_variant})"
        del op
    line += f"  rel diff {float((out - ref).norm() / ref.norm()):.2e}"
    print(line, flush=True)
