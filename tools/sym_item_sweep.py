"""cfg3 product time against the symmetric work-list item length
(NCGP_SYM_ITEM, read when the operator is built).  usage: python tools/sym_item_sweep.py [family]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)
fam = sys.argv[1] if len(sys.argv) > 1 else "rbf"
n, w = 1_000_000, 32
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 8))).float().cuda()
V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
for L in ("128", "64", "256", "512", "128"):
    os.environ["NCGP_SYM_ITEM"] = L
    op = KernelOperator(fam, 1.5, 1.0, X, w_max=w)
    op.apply(V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(2):
        op.apply(V)
    e1.record()
    torch.cuda.synchronize()
    print(f"{fam} item {L:>4s}: {e0.elapsed_time(e1) / 2:8.2f} ms ({op.last_variant})", flush=True)
    del op
