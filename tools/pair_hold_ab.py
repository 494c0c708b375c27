import os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
for n, d, w, fam in [(200_000, 24, 32, "matern32"), (200_000, 32, 32, "matern32")]:
    rng = np.random.default_rng(0)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    op = KernelOperator(fam, 3.0, 1.0, X, w_max=32)
    res = {}
    for rep in range(3):
        for k, env in (("plain", {"NCGP_SYM": "0"}), ("hold", {}), ("nohold", {"NCGP_SYM_DBG": "64"})):
            for kk in ("NCGP_SYM", "NCGP_SYM_DBG"): os.environ.pop(kk, None)
            os.environ.update(env)
            op.apply(V); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); op.apply(V); e1.record(); torch.cuda.synchronize()
            res.setdefault(k, []).append(e0.elapsed_time(e1))
    print(fam, d, w, {k: round(float(np.median(v)), 3) for k, v in res.items()}, op.last_variant_code, flush=True)
