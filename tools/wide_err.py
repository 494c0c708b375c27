"""Error of the wide-RHS kernel and the 32-wide plain kernel against the fp64
CUDA-core operator on the same inputs.  usage: python tools/wide_err.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

for nt, n, d, w, spec in ((1000, 9000, 8, 128, ("matern32", 1.5, 2.0)),
                          (257, 20000, 50, 77, ("rbf", 5.0, 1.0)),
                          (1000, 9000, 8, 128, ("rbf", 1.5, 2.0))):
    rng = np.random.default_rng(nt + n)
    X = torch.from_numpy(rng.standard_normal((n, d))).cuda()
    Xt = torch.from_numpy(rng.standard_normal((nt, d))).cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).cuda()
    ref = KernelOperator(*spec, Xt, X, w_max=32, impl="simt").apply(V)
    wide = KernelOperator(*spec, Xt.float(), X.float(), w_max=128)
    a = wide.apply(V.float()).double()
    plain = KernelOperator(*spec, Xt.float(), X.float(), w_max=32).apply(V.float()).double()
    e = lambda x: float((x - ref).norm() / ref.norm())
    col = lambda x: ((x - ref).norm(dim=0) / ref.norm(dim=0)).max().item()
    print(spec, nt, n, d, w, wide.last_variant, "wide", e(a), col(a), "plain", e(plain), col(plain))
