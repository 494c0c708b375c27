"""Split the symmetric kernel's output into its normal (block (r, c >= 2a))
and transposed parts and check each against the fp64 operator per row tile.
usage: NCGP_SYM_ITEM=L python tools/sym_diag2.py n"""
import os, sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
d, w = 8, 32
rng = np.random.default_rng(1)
X = rng.standard_normal((n, d)); V = rng.standard_normal((n, w))
Xf = torch.from_numpy(X).float().cuda(); Vf = torch.from_numpy(V).float().cuda()
op = KernelOperator("rbf", 1.5, 1.0, Xf, w_max=32)
os.environ["NCGP_SYM"] = "1"
os.environ["NCGP_SYM_DBG"] = "1"; normal = op.apply(Vf).double().cpu().numpy()
os.environ["NCGP_SYM_DBG"] = "2"; trans = op.apply(Vf).double().cpu().numpy()
X64 = torch.from_numpy(X).cuda(); V64 = torch.from_numpy(V).cuda()
nb = (n + 127) // 128
bad_n, bad_t = [], []
for r in range(nb):
    r0, r1 = 128 * r, min(n, 128 * r + 128)
    a = r // 2
    c0 = 256 * a  # normal part: columns >= 2a * 128
    opn = KernelOperator("rbf", 1.5, 1.0, X64[r0:r1], X64[c0:], w_max=32)
    ref_n = opn.apply(V64[c0:]).cpu().numpy()
    full = KernelOperator("rbf", 1.5, 1.0, X64[r0:r1], X64, w_max=32).apply(V64).cpu().numpy()
    ref_t = full - ref_n
    en = np.abs(normal[r0:r1] - ref_n).max() / (np.abs(ref_n).max() + 1e-9)
    et = np.abs(trans[r0:r1] - ref_t).max() / (np.abs(full).max() + 1e-9)
    if en > 1e-4: bad_n.append((r, round(float(en), 3)))
    if et > 1e-4: bad_t.append((r, round(float(et), 3)))
print("item", os.environ.get("NCGP_SYM_ITEM", "128"), "n", n, "bad normal tiles", bad_n[:20])
print("bad transposed tiles", bad_t[:20])
