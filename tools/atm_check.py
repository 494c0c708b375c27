import os, sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
n, d, w = int(sys.argv[1]), int(sys.argv[2]), 10
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, d))).float().cuda()
V = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
op = KernelOperator("rbf", 5.0, 1.0, X, w_max=16)
os.environ["NCGP_SYM"] = "0"; ref = op.apply(V).double(); torch.cuda.synchronize()
os.environ["NCGP_SYM"] = "1"
t0 = time.time()
try:
    got = op.apply(V).double(); torch.cuda.synchronize()
    print("variant", op.last_variant_code, "rel", float((got - ref).norm() / ref.norm()), "t", time.time() - t0)
except Exception as e:
    print("ERR after", time.time() - t0, "s:", str(e)[:300])
