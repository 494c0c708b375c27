"""Operator accuracy check: fp32 K1 products against the fp64 operator per
entry (relative to |K||v|) and the bilinear forms u'Kv, v'Ku.  usage: python tools/sym_check.py"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
rng = np.random.default_rng(5)
X = rng.standard_normal((4096, 8))
Xd = torch.from_numpy(X).float().cuda()
a = rng.standard_normal((4096, 1)); b = rng.standard_normal((4096, 1))
op = KernelOperator("rbf", 1.5, 1.0, Xd, w_max=32)
op64 = KernelOperator("rbf", 1.5, 1.0, torch.from_numpy(X).cuda(), w_max=32)
for name, v in (("a", a), ("b", b)):
    g = op.apply(torch.from_numpy(v).float().cuda()).double().cpu().numpy()
    r = op64.apply(torch.from_numpy(v).cuda()).cpu().numpy()
    sc = op64.apply(torch.from_numpy(np.abs(v)).cuda()).cpu().numpy()
    print(name, "max |err|/scale", float(np.max(np.abs(g - r) / sc)), "rel norm", float(np.linalg.norm(g-r)/np.linalg.norm(r)))
Ka = op.apply(torch.from_numpy(a).float().cuda()).double().cpu().numpy()
Kb = op.apply(torch.from_numpy(b).float().cuda()).double().cpu().numpy()
Ka64 = op64.apply(torch.from_numpy(a).cuda()).cpu().numpy()
Kb64 = op64.apply(torch.from_numpy(b).cuda()).cpu().numpy()
af = a.astype(np.float32).astype(np.float64); bf = b.astype(np.float32).astype(np.float64)
print("uKv", float((af*Kb).sum()), "vKu", float((bf*Ka).sum()), "fp64 uKv", float((a*Kb64).sum()), float((b*Ka64).sum()))
