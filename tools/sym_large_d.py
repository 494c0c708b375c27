import os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
def timed(op, V, reps=3):
    op.apply(V); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): op.apply(V)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for n, d, w, fam, ell in [(200_000, 50, 10, "rbf", 5.0), (200_000, 50, 10, "matern32", 5.0), (200_000, 32, 10, "rbf", 5.0), (200_000, 8, 10, "rbf", 1.5)]:
    rng = np.random.default_rng(0)
    X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
    V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
    line = f"{fam} n={n} d={d} w={w}:"
    ref = None
    for name, env in (("plain", {"NCGP_SYM": "0"}), ("pair", {"NCGP_SYM": "1", "NCGP_SYM_CG": "2"}), ("cg1npb1", {"NCGP_SYM": "1", "NCGP_SYM1_NPB": "1"})):
        for k in ("NCGP_SYM", "NCGP_SYM_CG", "NCGP_SYM1_NPB"): os.environ.pop(k, None)
        os.environ.update(env)
        op = KernelOperator(fam, ell, 1.0, X, w_max=32)
        out = op.apply(V).double()
        if ref is None: ref = out
        t = timed(op, V)
        line += f"  {name} {t:7.3f} ms ({op.last_variant_code}) rel {float((out-ref).norm()/ref.norm()):.1e}"
        del op
    print(line, flush=True)
