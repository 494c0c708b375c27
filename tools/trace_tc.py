"""Per-tile timeline of CTA 0 of the tcgen05 operator (debug hook)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2310_20285_b200 import _native
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
fam = sys.argv[2] if len(sys.argv) > 2 else "rbf"
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 8))).float().cuda()
S = torch.from_numpy(rng.standard_normal((n, 32))).float().cuda()
op = KernelOperator(fam, 1.5, 1.0, X, w_max=32, impl="tcgen05")
op.apply(S)
buf = torch.zeros(256 * 8, dtype=torch.int64, device="cuda")
lib = _native.load()
lib.ncgp_debug_set_trace.argtypes = [ctypes.c_void_p]
lib.ncgp_debug_set_trace(buf.data_ptr())
lib.ncgp_debug_set_mode(mode)
op.apply(S)
torch.cuda.synchronize()
lib.ncgp_debug_set_trace(None)
lib.ncgp_debug_set_mode(0)
t = buf.view(256, 8).cpu().numpy().astype(np.int64)
t0 = t[t > 0].min()
names = ["p_ready", "mma2_iss", "g1_iss", "e0_wait", "e0_go", "e1_wait", "e1_go", "e0_done"]
print("tile " + " ".join(f"{x:>9s}" for x in names))
for g in list(range(0, 12)) + list(range(100, 112)):
    print(f"{g:4d} " + " ".join(f"{(v - t0) if v else -1:9d}" for v in t[g]))
d = np.diff(t[20:250, 0])
print("p_ready interval: mean %.0f  median %.0f" % (d.mean(), np.median(d)))
e = t[20:250]
print("epi0 busy (go->done) mean %.0f ; epi0 wait (wait->go) mean %.0f ; epi1 wait mean %.0f" % (
    (e[:, 7] - e[:, 4]).mean(), (e[:, 4] - e[:, 3]).mean(), (e[:, 6] - e[:, 5]).mean()))
print("mma: p_ready->mma2_issued %.0f ; mma2_issued->g1_issued %.0f ; e0_done -> p_ready %.0f" % (
    (e[:, 1] - e[:, 0]).mean(), (e[:, 2] - e[:, 1]).mean(), (e[:, 0] - e[:, 7]).mean()))
print("g1_issued(g) -> e0_go(g+3) %.0f" % (t[23:253, 4] - t[20:250, 2]).mean())
