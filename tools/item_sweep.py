"""Work-item length (column tiles per item) of the symmetric kernels K1-sym1 /
pair against problem size: time per product for NCGP_SYM_ITEM in {16..128}.
usage: python tools/item_sweep.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NCGP_SYM"] = "1"
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402


def timed(op, V, reps):
    op.apply(V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        op.apply(V)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


shapes = [(45_000, 8, 32, "matern32"), (60_000, 8, 10, "rbf"), (100_000, 20, 10, "matern32"),
          (150_000, 20, 10, "matern32"), (200_000, 8, 10, "rbf"), (200_000, 50, 10, "rbf"),
          (400_000, 20, 10, "matern32")]
for n, d, w, fam in shapes:
    rng = np.random.default_rng(0)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    row = []
    for item in (0, 16, 32, 64, 128):
        if item:
            os.environ["NCGP_SYM_ITEM"] = str(item)
        else:
            os.environ.pop("NCGP_SYM_ITEM", None)
        op = KernelOperator(fam, 3.0 if d >= 20 else 1.5, 1.0, X, w_max=w)
        row.append(f"{'auto' if not item else item}: {timed(op, V, 20 if n <= 200_000 else 5):8.3f}")
        code = op.last_variant_code
        del op
    print(f"{fam:9s} n={n:7d} d={d:2d} w={w:2d} (variant {code}) ms per product  " + "  ".join(row), flush=True)
