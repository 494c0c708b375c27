"""Apply one K(X, X) product `reps` times (ncu target).
usage: [PROF_WMAX=32] [PROF_ELL=1.5] python tools/prof_one.py n d w fam [cg] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402

n, d, w, fam = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
cg = sys.argv[5] if len(sys.argv) > 5 else "3"
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
os.environ["NCGP_SYM_CG"] = cg
os.environ["NCGP_SYM"] = "1"
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).cuda()
V = torch.from_numpy(rng.standard_normal((n, w)).astype(np.float32)).cuda()
op = KernelOperator(fam, float(os.environ.get("PROF_ELL", "1.5")), 1.0, X,
                    w_max=int(os.environ.get("PROF_WMAX", "32")))
for _ in range(reps):
    op.apply(V)
torch.cuda.synchronize()
print("variant", op.last_variant_code)
