"""Per-column and per-row-position error pattern of the wide kernel."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

nt, n, d, w = 1024, 9000, 8, 128
spec = ("rbf", 1.5, 2.0)
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, d))).cuda()
Xt = torch.from_numpy(rng.standard_normal((nt, d))).cuda()
V = torch.from_numpy(rng.standard_normal((n, w))).cuda()
ref = KernelOperator(*spec, Xt, X, w_max=32, impl="simt").apply(V)
a = KernelOperator(*spec, Xt.float(), X.float(), w_max=128).apply(V.float()).double()
p = KernelOperator(*spec, Xt.float(), X.float(), w_max=32).apply(V.float()).double()
for name, x in (("wide", a), ("plain", p)):
    ec = ((x - ref).norm(dim=0) / ref.norm(dim=0)).cpu().numpy()
    er = ((x - ref).norm(dim=1) / ref.norm(dim=1)).cpu().numpy()
    print(name, "cols 0-31 %.2e 32-63 %.2e 64-95 %.2e 96-127 %.2e" % tuple(ec.reshape(4, 32).mean(1)))
    print(name, "row mod 128: 0-31 %.2e 32-63 %.2e 64-95 %.2e 96-127 %.2e" % tuple(er.reshape(-1, 4, 32).mean((0, 2))))
    print(name, "row tile parity even %.2e odd %.2e" % (er.reshape(-1, 128)[0::2].mean(), er.reshape(-1, 128)[1::2].mean()))
# the same data with V rounded to fp16-exact values (no V_lo): isolates the P side
Vh = V.half().double()
ref2 = KernelOperator(*spec, Xt, X, w_max=32, impl="simt").apply(Vh)
a2 = KernelOperator(*spec, Xt.float(), X.float(), w_max=128).apply(Vh.float()).double()
p2 = KernelOperator(*spec, Xt.float(), X.float(), w_max=32).apply(Vh.float()).double()
print("V fp16-exact: wide %.2e plain %.2e" % (float((a2 - ref2).norm() / ref2.norm()), float((p2 - ref2).norm() / ref2.norm())))
