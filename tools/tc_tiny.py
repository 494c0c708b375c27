"""Tiny tcgen05-operator invocations (for compute-sanitizer runs)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
for (n, d, w, fam) in [(300, 2, 3, "rbf"), (1000, 8, 32, "rbf"), (700, 20, 10, "matern32"),
                       (600, 50, 32, "rbf")]:
    rng = np.random.default_rng(n)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    op = KernelOperator(fam, 1.0 * np.sqrt(d), 1.0, X, w_max=w, impl="tcgen05")
    out = op.apply(V)
    torch.cuda.synchronize()
    print(n, d, w, fam, float(out.abs().max()), flush=True)
