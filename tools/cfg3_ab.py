"""cfg3 product: plain vs symmetric kernel, interleaved on one box (CUDA
events, L2 flushed before each timed product).  usage: python tools/cfg3_ab.py [family] [w]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)
fam = sys.argv[1] if len(sys.argv) > 1 else "rbf"
w = int(sys.argv[2]) if len(sys.argv) > 2 else 32
n = 1_000_000
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 8))).float().cuda()
V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
op = KernelOperator(fam, 1.5, 1.0, X, w_max=32)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
res = {"0": [], "1": []}
for rep in range(4):
    for sym in ("0", "1"):
        os.environ["NCGP_SYM"] = sym
        op.apply(V)
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        op.apply(V)
        e1.record()
        torch.cuda.synchronize()
        res[sym].append(e0.elapsed_time(e1))
print(f"{fam} w={w}: plain {np.round(res['0'], 1)} ms  symmetric {np.round(res['1'], 1)} ms  "
      f"ratio {np.median(res['0']) / np.median(res['1']):.3f}", flush=True)
