import os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
for n, d, w, fam in [(1000, 2, 1, "matern32"), (1000, 2, 16, "matern32"), (300, 3, 4, "matern32"), (3000, 8, 8, "rbf"), (3000, 8, 32, "rbf"), (20000, 8, 10, "rbf")]:
    rng = np.random.default_rng(1)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    op = KernelOperator(fam, 1.5, 1.0, X, w_max=32)
    os.environ["NCGP_SYM"] = "0"; ref = op.apply(V).double()
    line = f"{fam} n={n} d={d} w={w}:"
    for npb in ("2", "1"):
        os.environ["NCGP_SYM"] = "1"; os.environ["NCGP_SYM_NPB"] = npb
        got = op.apply(V).double(); torch.cuda.synchronize()
        err = ((got - ref).norm(dim=1) / ref.norm(dim=1).clamp_min(1e-30)).cpu().numpy()
        bad = np.nonzero(err > 1e-4)[0]
        line += f"  npb={npb} rel {float((got-ref).norm()/ref.norm()):.2e} bad rows {len(bad)} {bad[:6]}"
    print(line, flush=True)
