"""Single-CTA symmetric kernel (NCGP_SYM_CG=1) against the plain kernel and
the pair symmetric kernel: accuracy and timing.  usage: python tools/sym1_check.py [--big]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)


def timed(op, V, reps=3):
    op.apply(V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        op.apply(V)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


small = [(300, 3, 4, "rbf", 1.0), (1000, 2, 1, "matern32", 1.0), (3000, 8, 32, "rbf", 1.5),
         (5000, 20, 10, "matern32", 3.0), (20000, 8, 10, "rbf", 1.5)]
big = [(200_000, 8, 32, "rbf", 1.5), (200_000, 8, 32, "matern32", 1.5), (200_000, 8, 10, "rbf", 1.5),
       (100_000, 20, 10, "matern32", 3.0), (100_000, 20, 10, "rbf", 3.0)]
for n, d, w, fam, ell in (big if "--big" in sys.argv else small):
    rng = np.random.default_rng(n + d)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    res = {}
    for name, env in (("plain", {"NCGP_SYM": "0", "NCGP_SYM_CG": "2"}), ("pair", {"NCGP_SYM": "1", "NCGP_SYM_CG": "2"}),
                      ("cg1", {"NCGP_SYM": "1", "NCGP_SYM_CG": "1"})):
        os.environ.update(env)
        op = KernelOperator(fam, ell, 1.0, X, w_max=32)
        out = op.apply(V).double()
        torch.cuda.synchronize()
        t = timed(op, V) if "--big" in sys.argv else 0.0
        res[name] = (out, t, op.last_variant)
        del op
    ref = res["plain"][0]
    line = f"{fam:9s} n={n:6d} d={d:2d} w={w:2d}:"
    for name in ("plain", "pair", "cg1"):
        out, t, var = res[name]
        rel = float((out - ref).norm() / ref.norm())
        line += f"  {name} {t:8.3f} ms rel {rel:.1e}"
    print(line, flush=True)
