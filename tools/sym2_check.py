"""K1-sym2 (blocked symmetric kernel) against K1-sym1 and the plain kernel:
accuracy (vs plain, vs fp64 on sampled rows) and CUDA-event time per product.
usage: python tools/sym2_check.py [n d w fam] ..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402
from oracle import ncgp_oracle as O  # noqa: E402


def timed(op, V, reps=3):
    op.apply(V)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = op.apply(V)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return out, min(ts)


def case(n, d, w, fam, ell=1.5):
    rng = np.random.default_rng(n + d)
    X = rng.standard_normal((n, d)).astype(np.float32)
    V = rng.standard_normal((n, w)).astype(np.float32)
    Xd, Vd = torch.from_numpy(X).cuda(), torch.from_numpy(V).cuda()
    res = {}
    outs = {}
    for cg in (0, 1, 3):
        os.environ["NCGP_SYM_CG"] = str(max(cg, 1))
        os.environ["NCGP_SYM"] = "0" if cg == 0 else "1"
        op = KernelOperator(fam, ell, 1.0, Xd, w_max=32)
        out, ms = timed(op, Vd, 2 if n >= 500_000 else 3)
        outs[cg] = out.double()
        res[cg] = (ms, op.last_variant_code)
        del op
    os.environ.pop("NCGP_SYM_CG")
    os.environ.pop("NCGP_SYM")
    rows = np.linspace(0, n - 1, 6).astype(int)
    ref = O.kernel_matmul_rows((fam, ell, 1.0), X[rows].astype(np.float64), X.astype(np.float64),
                               V.astype(np.float64), tile=8)
    line = f"n={n} d={d} w={w} {fam}:"
    for cg, name in ((0, "plain"), (1, "sym1"), (3, "sym2")):
        got = outs[cg][torch.from_numpy(rows).cuda()].cpu().numpy()
        e64 = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        ep = float((outs[cg] - outs[0]).norm() / outs[0].norm())
        line += f"  {name}[{res[cg][1]}] {res[cg][0]:.2f} ms err64 {e64:.1e} vs_plain {ep:.1e}"
    print(line, flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    shapes = [(20000, 8, 32, "rbf"), (45000, 8, 32, "matern32"), (100000, 20, 10, "matern32"),
              (200000, 8, 32, "rbf"), (1000000, 8, 32, "rbf")]
    if args:
        shapes = [(int(args[i]), int(args[i + 1]), int(args[i + 2]), args[i + 3]) for i in range(0, len(args), 4)]
    for s in shapes:
        case(*s)
