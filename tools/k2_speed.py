"""K2 (wide kernel + fused square-reduce, posterior.py:67-84) against the
round-1 path (K1 over 32-column blocks of the class-gathered root, A stored,
then the square-reduce kernel) at the cfg5 posterior shape: 5e4 test points,
N = 1e6 training points, D = 50, C = 10 classes, root rank R.
usage: python tools/k2_speed.py [R] [n]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_20285_b200 import kernels as K  # noqa: E402
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
nt, d, C = 50_000, 50, 10
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).cuda()
Xt = torch.from_numpy(rng.standard_normal((nt, d)).astype(np.float32)).cuda()
W = torch.from_numpy(rng.standard_normal((n, C * R)).astype(np.float32)).cuda() * (1.0 / n ** 0.5)
s2 = torch.ones(C, dtype=torch.float64, device="cuda")
spec = ("rbf", 5.0, 1.0)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return out, a.elapsed_time(b)


op2 = KernelOperator(*spec, Xt, X, w_max=128)
v2, t2 = timed(lambda: op2.posterior_var(W, C, R, s2))
op1 = KernelOperator(*spec, Xt, X, w_max=32)
A = torch.empty((nt, C * R), dtype=torch.float32, device="cuda")


def k1_path():
    for c0 in range(0, C * R, 32):
        op1.apply(W[:, c0:c0 + 32], out=A[:, c0:c0 + 32])
    return K.marginal_var(A, C, R, s2)


v1, t1 = timed(k1_path)
err = float((v1.double() - v2.double()).norm() / v1.double().norm())
print(f"cfg5 posterior variance, {nt} test x {n} train, D={d}, C={C}, R={R}: "
      f"K2 {t2:.1f} ms, K1 32-column loop {t1:.1f} ms, speed-up {t1 / t2:.2f}x, rel diff {err:.1e}")
