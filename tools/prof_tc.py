"""Profiling driver: a few K(X,X)S products with the cfg3 shape at reduced N."""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200_000)
ap.add_argument("--d", type=int, default=8)
ap.add_argument("--w", type=int, default=32)
ap.add_argument("--family", default="rbf")
ap.add_argument("--impl", default="tcgen05")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
torch.cuda.set_device(0)
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((a.n, a.d))).float().cuda()
S = torch.from_numpy(rng.standard_normal((a.n, a.w))).float().cuda()
op = KernelOperator(a.family, 1.5, 1.0, X, w_max=a.w, impl=a.impl)
out = torch.empty((a.n, a.w), device="cuda")
for _ in range(a.iters):
    op.apply(S, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
op.apply(S, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
pairs = float(a.n) ** 2
print(f"n={a.n} {a.family} {op.impl}: {ms:.3f} ms  {pairs/ms/1e9:.3f} Tpairs/s  "
      f"{(2*a.d+2*a.w)*pairs/ms/1e9:.1f} TFLOP/s")
