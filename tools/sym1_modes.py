"""K1-sym1 timing with parts removed (NCGP_SYM_DBG bits, wrong results):
1 no D_T reductions, 2 no O reductions, 4 no T MMAs, 8 no D_T drain at all,
16 no P stores.  usage: python tools/sym1_modes.py [n] [family] [w]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ["NCGP_SYM_CG"] = "1"
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
fam = sys.argv[2] if len(sys.argv) > 2 else "rbf"
w = int(sys.argv[3]) if len(sys.argv) > 3 else 32
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 8))).float().cuda()
V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
op = KernelOperator(fam, 1.5, 1.0, X, w_max=32)
for sym, dbg, name in (("0", "0", "plain"), ("1", "0", "sym1"), ("1", "1", "no D_T red"), ("1", "3", "no red"),
                       ("1", "8", "no D_T drain"), ("1", "16", "no P stores"), ("1", "4", "no T MMAs"),
                       ("1", "12", "no T MMAs, no D_T drain"), ("1", "28", "no T path, no P stores")):
    os.environ["NCGP_SYM"] = sym
    os.environ["NCGP_SYM_DBG"] = dbg
    op.apply(V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3):
        op.apply(V)
    e1.record()
    torch.cuda.synchronize()
    print(f"{fam} w={w} {name:28s} {e0.elapsed_time(e1) / 3:8.3f} ms", flush=True)
