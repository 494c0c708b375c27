import os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
n, d, w = 100_000, 20, 10
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
def timed(op, reps=20):
    op.apply(V); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): op.apply(V)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for name, env in (("plain", {"NCGP_SYM": "0"}), ("cg1", {"NCGP_SYM_CG": "1"}), ("cg2", {"NCGP_SYM_CG": "2"}), ("cg2-noatm", {"NCGP_SYM_CG": "2", "NCGP_SYM_ATM": "0"})):
    for k in ("NCGP_SYM", "NCGP_SYM_CG", "NCGP_SYM_ATM"): os.environ.pop(k, None)
    os.environ.update(env)
    op = KernelOperator("matern32", 3.0, 1.0, X, w_max=10)
    t = timed(op)
    print(f"{name:10s} {t:7.3f} ms variant {op.last_variant_code}", flush=True)
