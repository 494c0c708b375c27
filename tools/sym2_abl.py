"""Time the blocked symmetric kernel (K1-sym2) under build-time ablations
(tools/ab/lib_ablN.so, NCGP_SYM2_ABL bits; results are wrong by design).
usage: python tools/sym2_abl.py n [libs...]   (run once per library via NCGP_LIB)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NCGP_SYM"] = "1"
os.environ["NCGP_SYM_CG"] = os.environ.get("NCGP_SYM_CG", "3")
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 32
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 8)).astype(np.float32)).cuda()
V = torch.from_numpy(rng.standard_normal((n, w)).astype(np.float32)).cuda()
op = KernelOperator("rbf", 1.5, 1.0, X, w_max=32)
op.apply(V)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    op.apply(V)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"{os.path.basename(os.environ.get('NCGP_LIB', 'default'))}: {min(ts):.3f} ms (variant {op.last_variant_code})")
