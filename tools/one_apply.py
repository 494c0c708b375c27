import os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
n, w, fam = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 8))).float().cuda()
V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
op = KernelOperator(fam, 1.5, 1.0, X, w_max=32)
for _ in range(3): op.apply(V)
torch.cuda.synchronize(); print(op.last_variant)
