"""Timing of the symmetric kernel with parts removed (NCGP_SYM_DBG bits; wrong
results, timing only).  usage: python tools/sym_modes.py [n] [family]"""
import os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
fam = sys.argv[2] if len(sys.argv) > 2 else "rbf"
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 8))).float().cuda()
V = torch.from_numpy(rng.standard_normal((n, 32))).float().cuda()
op = KernelOperator(fam, 1.5, 1.0, X, w_max=32)
for sym, dbg, name in (("0", "0", "plain"), ("1", "0", "sym"), ("1", "1", "no D_T red"), ("1", "3", "no red at all"),
                       ("1", "9", "no D_T ld/red"), ("1", "4", "no transposed MMAs"), ("1", "13", "no T MMA, no D_T ld/red"),
                       ("1", "16", "no P smem stores"), ("1", "29", "no T path at all")):
    os.environ["NCGP_SYM"] = sym
    os.environ["NCGP_SYM_DBG"] = dbg
    op.apply(V); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); op.apply(V); e1.record(); torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1):8.3f} ms", flush=True)
