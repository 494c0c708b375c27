"""Timing of the symmetric kernel against the plain one under environment
variants (NCGP_SYM, NCGP_SYM_DBG, NCGP_SYM_ITEM, NCGP_RINGS).
usage: python tools/sym_exp.py [NCGP_SYM_DBG values ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)
KEYS = ("NCGP_SYM", "NCGP_RINGS", "NCGP_SYM_ITEM", "NCGP_SYM_DBG", "NCGP_SYM_NPB")


def timed(op, V, env, reps=3):
    for k in KEYS:
        os.environ.pop(k, None)
    os.environ.update(env)
    op.apply(V)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        op.apply(V)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cases = [(200_000, 8, 32, "rbf", 1.5), (200_000, 8, 32, "matern32", 1.5), (200_000, 8, 10, "rbf", 1.5),
         (200_000, 8, 10, "matern32", 1.5), (100_000, 20, 10, "matern32", 3.0), (100_000, 20, 10, "rbf", 3.0),
         (100_000, 24, 10, "rbf", 3.0), (5_000, 2, 3, "rbf", 1.0), (20_000, 8, 10, "rbf", 1.5), (50_000, 8, 32, "rbf", 1.5)]
# arguments: NCGP_SYM_DBG values, or npb=1 / npb=2
variants = [{"NCGP_SYM": "0"}, {"NCGP_SYM": "1"}] + [
    {"NCGP_SYM": "1", "NCGP_SYM_NPB": v[4:]} if v.startswith("npb=") else {"NCGP_SYM": "1", "NCGP_SYM_DBG": v}
    for v in sys.argv[1:] or ["64", "29"]]
if os.environ.get("SYM_EXP_CASES") == "large_d":
    cases = [(200_000, 50, 10, "rbf", 5.0), (200_000, 32, 10, "rbf", 5.0), (200_000, 50, 10, "matern32", 5.0),
             (200_000, 8, 10, "rbf", 1.5), (200_000, 8, 32, "matern32", 1.5)]
for n, d, w, fam, ell in cases:
    rng = np.random.default_rng(0)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    op = KernelOperator(fam, ell, 1.0, X, w_max=32)
    line = f"{fam:9s} n={n} d={d} w={w}:"
    for env in variants:
        line += f"  {'/'.join(env.values()):5s} {timed(op, V, env):7.3f}"
    print(line, flush=True)
