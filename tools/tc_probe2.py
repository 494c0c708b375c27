"""tcgen05 vs CUDA-core operator on cfg5-like shapes (D=50) incl. 32-wide RHS."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
from paper_2310_20285_b200 import configs
torch.cuda.set_device(0)
for (n, d, w) in [(4096, 50, 32), (4096, 50, 10), (30000, 50, 32), (30000, 50, 10), (2000, 20, 32)]:
    c = configs.cfg5(n=n, n_test=10) if d == 50 else configs.cfg4(n=n, n_test=10)
    X = torch.from_numpy(c["X"][:, :d]).float().cuda()
    rng = np.random.default_rng(1)
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    spec = c["kernel"]
    tc = KernelOperator(*spec, X, w_max=w, impl="tcgen05")
    si = KernelOperator(*spec, X, w_max=w, impl="simt")
    a = tc.apply(V).double(); b = si.apply(V).double()
    torch.cuda.synchronize()
    print(f"n={n} d={d} w={w}: rel={float((a-b).norm()/b.norm()):.3e} nan={bool(torch.isnan(a).any())} "
          f"max|a|={float(a.abs().max()):.3e} max|b|={float(b.abs().max()):.3e}", flush=True)
