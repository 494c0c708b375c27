"""Where the symmetric kernels overtake the plain kernel (policy thresholds of
sym_enabled): NCGP_SYM=0 against NCGP_SYM=1 over n.  usage: python tools/sym_threshold.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402


def timed(op, V, reps=30):
    op.apply(V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        op.apply(V)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for d, w, fam in ([(8, 10, "rbf"), (20, 10, "rbf"), (8, 10, "matern32"), (20, 10, "matern32")] if os.environ.get("THR_WMAX") else []) or [(8, 32, "rbf"), (8, 32, "matern32"), (8, 10, "rbf"), (20, 10, "matern32"), (20, 32, "matern32"),
                  (50, 10, "matern32"), (50, 10, "rbf")]:
    for n in (12_000, 16_000, 20_000, 25_000, 30_000, 38_000, 50_000, 65_000):
        rng = np.random.default_rng(0)
        X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
        V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
        res = {}
        for mode in ("0", "1", ""):
            if mode:
                os.environ["NCGP_SYM"] = mode
            else:
                os.environ.pop("NCGP_SYM", None)
            op = KernelOperator(fam, 3.0 if d >= 20 else 1.5, 1.0, X, w_max=int(os.environ.get("THR_WMAX", "32")))
            res[mode] = (timed(op, V), op.last_variant_code)
            del op
        print(f"{fam:9s} d={d:2d} w={w:2d} n={n:6d}: plain {res['0'][0]:7.3f}  sym[{res['1'][1]}] {res['1'][0]:7.3f}  "
              f"policy[{res[''][1]}] {res[''][0]:7.3f}  sym/plain {res['1'][0] / res['0'][0]:5.2f}", flush=True)
