"""Symmetric K(X, X) kernel vs the plain kernel: accuracy against the fp64
operator and timing.  usage: python tools/sym_test.py [--time]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)


def run(n, d, w, fam, ell, timing=False):
    rng = np.random.default_rng(n + d + w)
    X = rng.standard_normal((n, d))
    V = rng.standard_normal((n, w))
    Xd = torch.from_numpy(X).float().cuda()
    Vd = torch.from_numpy(V).float().cuda()
    op = KernelOperator(fam, ell, 1.0, Xd, w_max=32)
    os.environ["NCGP_SYM"] = "0"
    ref = op.apply(Vd).double()
    os.environ["NCGP_SYM"] = "1"
    got = op.apply(Vd).double()
    torch.cuda.synchronize()
    line = f"{fam:8s} n={n:7d} d={d:2d} w={w:2d}"
    if n <= 20000:
        op64 = KernelOperator(fam, ell, 1.0, torch.from_numpy(X).cuda(), w_max=32)
        r64 = op64.apply(torch.from_numpy(V).cuda())
        sc = op64.apply(torch.from_numpy(np.abs(V)).cuda())
        e_sym = float(((got - r64).abs() / sc).max())
        e_pl = float(((ref - r64).abs() / sc).max())
        line += f"  max|err|/scale sym {e_sym:.2e} plain {e_pl:.2e}"
    rel = float((got - ref).norm() / ref.norm())
    line += f"  rel(sym, plain) {rel:.2e}"
    if timing:
        for flag in ("0", "1"):
            os.environ["NCGP_SYM"] = flag
            op.apply(Vd)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(3):
                op.apply(Vd)
            e1.record()
            torch.cuda.synchronize()
            line += f"  {'sym' if flag == '1' else 'plain'} {e0.elapsed_time(e1) / 3:.3f} ms"
    print(line, flush=True)


timing = "--time" in sys.argv
for n, d, w, fam, ell in [(300, 3, 4, "rbf", 1.0), (3000, 8, 32, "rbf", 1.5), (5000, 8, 10, "rbf", 1.5),
                          (20000, 8, 32, "rbf", 1.5), (20000, 20, 10, "matern32", 3.0),
                          (12345, 8, 32, "matern32", 1.5)]:
    run(n, d, w, fam, ell)
if timing and "--shapes" in sys.argv:
    for n, d, w, fam, ell in [(200_000, 8, 10, "rbf", 1.5), (200_000, 20, 10, "rbf", 3.0),
                              (200_000, 8, 16, "rbf", 1.5), (200_000, 20, 32, "rbf", 3.0),
                              (200_000, 20, 10, "matern32", 3.0), (200_000, 32, 10, "rbf", 5.0)]:
        run(n, d, w, fam, ell, True)
    sys.exit(0)
if timing:
    run(200_000, 8, 32, "rbf", 1.5, True)
    run(200_000, 8, 32, "matern32", 1.5, True)
    run(100_000, 20, 10, "matern32", 3.0, True)
    run(1_000_000, 8, 32, "rbf", 1.5, True)
