"""Symmetric-kernel diagnostics: which output row tiles differ from the plain
kernel.  usage: NCGP_SYM_ITEM=L python tools/sym_diag.py"""
import os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)


def diag(n, d, w, fam, ell, reps=1):
    rng = np.random.default_rng(1)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    op = KernelOperator(fam, ell, 1.0, X, w_max=32)
    os.environ["NCGP_SYM"] = "0"; ref = op.apply(V).double()
    os.environ["NCGP_SYM"] = "1"
    for _ in range(reps):
        got = op.apply(V).double()
        err = ((got - ref).abs().max(1).values / (ref.abs().max(1).values + 1e-9)).cpu().numpy()
        bad = np.where(err > 1e-3)[0]
        tiles = sorted(set((bad // 128).tolist()))
        print(f"item={os.environ.get('NCGP_SYM_ITEM', '128')} {fam} n={n} w={w} bad rows {len(bad)} "
              f"tiles {tiles[:24]}{' ...' if len(tiles) > 24 else ''}", flush=True)


diag(20000, 8, 32, "rbf", 1.5, reps=3)
diag(12345, 8, 32, "rbf", 1.5)
