"""Debug probe: tcgen05 operator vs the CUDA-core operator on small shapes."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)
for (n, d, w, fam) in [(128, 8, 32, "rbf"), (256, 8, 32, "rbf"), (1000, 8, 32, "rbf"),
                       (1000, 8, 32, "matern32"), (300, 2, 3, "rbf"), (4096, 50, 10, "rbf"),
                       (20000, 8, 32, "rbf")]:
    rng = np.random.default_rng(n + d)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    ell = 1.5 if d == 8 else (1.0 if d == 2 else 5.0)
    tc = KernelOperator(fam, ell, 1.0, X, w_max=w, impl="tcgen05")
    si = KernelOperator(fam, ell, 1.0, X, w_max=w, impl="simt")
    a = tc.apply(V).double()
    b = si.apply(V).double()
    torch.cuda.synchronize()
    err = float((a - b).norm() / b.norm())
    print(f"n={n} d={d} w={w} {fam}: rel={err:.3e} maxabs={float((a-b).abs().max()):.3e} "
          f"|b|={float(b.abs().max()):.3e}", flush=True)
