"""CUDA-event time per product of every K1 flavour on one shape.
usage: python tools/flavours.py n d w fam [ell]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402

n, d, w, fam = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
ell = float(sys.argv[5]) if len(sys.argv) > 5 else 1.5
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).cuda()
V = torch.from_numpy(rng.standard_normal((n, w)).astype(np.float32)).cuda()
line = f"n={n} d={d} w={w} {fam}:"
ref = None
for name, env in (("plain", {"NCGP_SYM": "0"}), ("pair", {"NCGP_SYM": "1", "NCGP_SYM_CG": "2"}),
                  ("sym1", {"NCGP_SYM": "1", "NCGP_SYM_CG": "1"}), ("sym2", {"NCGP_SYM": "1", "NCGP_SYM_CG": "3"}),
                  ("default", {})):
    for k in ("NCGP_SYM", "NCGP_SYM_CG"):
        os.environ.pop(k, None)
    os.environ.update(env)
    try:
        op = KernelOperator(fam, ell, 1.0, X, w_max=int(os.environ.get("FLAV_WMAX", "32")))
        out = op.apply(V)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3 if n < 500_000 else 2):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = op.apply(V)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        o = out.double()
        if ref is None:
            ref = o
        err = float((o - ref).norm() / ref.norm())
        line += f"  {name}[{op.last_variant_code}] {min(ts):.2f} ms ({err:.0e})"
        del op
    except Exception as e:  # flavour not available for this shape
        line += f"  {name}: n/a ({type(e).__name__})"
print(line, flush=True)
