"""Runtime knobs of the symmetric pair kernel at the cfg5 product shape
(n = 1e6, D = 50, w = 10, RBF l = 5): NCGP_SYM_ITEM, NCGP_SYM_ORDER, NCGP_SYM_ATM,
NCGP_SYM_NPB.  Two interleaved passes (the GPU's power-capped clock drifts).
usage: python tools/pair_knobs.py [n]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 50)) + 1.0).float().cuda()
V = torch.from_numpy(rng.standard_normal((n, 10))).float().cuda()
KNOBS = ("NCGP_SYM_ITEM", "NCGP_SYM_ORDER", "NCGP_SYM_ATM", "NCGP_SYM_NPB")
configs = [{}, {"NCGP_SYM_ITEM": "64"}, {"NCGP_SYM_ITEM": "256"}, {"NCGP_SYM_ITEM": "512"},
           {"NCGP_SYM_ORDER": "pair"}, {"NCGP_SYM_ATM": "0"}, {"NCGP_SYM_NPB": "1"}, {"NCGP_SYM_NPB": "2"}]
res = {i: [] for i in range(len(configs))}
for rep in range(2):
    for i, env in enumerate(configs):
        for k in KNOBS:
            os.environ.pop(k, None)
        os.environ.update(env)
        op = KernelOperator("rbf", 5.0, 1.0, X, w_max=10)
        op.apply(V)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(2):
            op.apply(V)
        b.record()
        torch.cuda.synchronize()
        res[i].append((a.elapsed_time(b) / 2, op.last_variant_code))
        del op
for i, env in enumerate(configs):
    print(f"{str(env or 'default'):32s} " + "  ".join(f"{t:8.2f} ms [{c}]" for t, c in res[i]), flush=True)
