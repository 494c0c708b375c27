"""Per-tile timeline of CTA 0 of the blocked symmetric kernel (K1-sym2, debug hook).

usage: python tools/trace_sym2.py [n] [w]
Events (clock64, per tile step g; see kop_sym2_kernel):
  0/1/2 GEMM1 wait/go/issued  3/4/5/6 epilogue wait/s_full/S released/done
  7/8/9 GEMM2 wait/go/issued  10/11/12 T wait/go/issued  13/14 D_T drain start/done
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NCGP_SYM"] = "1"
os.environ.setdefault("NCGP_SYM_CG", "3")
from paper_2310_20285_b200 import _native  # noqa: E402
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 32
EV = 16
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 8))).float().cuda()
S = torch.from_numpy(rng.standard_normal((n, w))).float().cuda()
op = KernelOperator("rbf", 1.5, 1.0, X, w_max=32)
op.apply(S)
buf = torch.zeros(256 * EV + 4 * 4096, dtype=torch.int64, device="cuda")
lib = _native.load()
lib.ncgp_debug_set_trace.argtypes = [ctypes.c_void_p]
lib.ncgp_debug_set_trace(buf.data_ptr())
op.apply(S)
torch.cuda.synchronize()
lib.ncgp_debug_set_trace(None)
print("variant", op.last_variant_code)
t = buf.cpu().numpy()[:256 * EV].reshape(256, EV).astype(np.int64)
lo, hi = 32, 224
e = t[lo:hi]


def med(x):
    x = x[np.isfinite(x)]
    return f"{np.median(x):7.0f} (p90 {np.percentile(x, 90):7.0f})"


period = np.diff(t[lo:hi + 1, 9])
print("cycles per tile (GEMM2 issued to issued):", med(period.astype(float)))
rows = [("GEMM1 wait (S buffer / XA)", 1, 0), ("GEMM1 issue", 2, 1),
        ("epi wait s_full", 4, 3), ("epi s_full -> done", 6, 4),
        ("GEMM2 wait rdy (+V, O)", 8, 7), ("GEMM2 issue (24 MMAs + commits)", 9, 8),
        ("T wait rdy (+VI, D_T)", 11, 10), ("T issue", 12, 11)]
for name, a, b in rows:
    print(f"{name:34s}", med((e[:, a] - e[:, b]).astype(float)))
pt = e[:, 5] - e[:, 4]
print(f"{'epi s_full -> S released':34s}", med(np.where(e[:, 5] > 0, pt, np.nan).astype(float)))
print(f"{'epi S released -> done':34s}", med((e[:, 6] - e[:, 5]).astype(float)))
print(f"{'epi done(g-1) -> epi wait(g+1)':34s}", "(group idle between its tiles)", med((t[lo + 1:hi + 1, 3] - t[lo:hi, 6]).astype(float)))
print(f"{'GEMM1 issued -> epi s_full seen':34s}", med((e[:, 4] - e[:, 2]).astype(float)))
print(f"{'epi done -> GEMM2 go':34s}", med((e[:, 8] - e[:, 6]).astype(float)))
print(f"{'epi done -> T go':34s}", med((e[:, 11] - e[:, 6]).astype(float)))
print(f"{'S released(g-1) -> GEMM1 go(g)':34s}", med((e[:, 1] - t[lo - 1:hi - 1, 5]).astype(float)))
print(f"{'GEMM2 issued(g-2) -> epi S released(g)':34s}", med((e[:, 5] - t[lo - 2:hi - 2, 9]).astype(float)))
dr = e[:, 14] - e[:, 13]
print(f"{'D_T drain':34s}", med(np.where(e[:, 13] > 0, dr, np.nan).astype(float)))
np.set_printoptions(linewidth=200)
print("tiles 40..47 relative to GEMM2-issued of tile 40:")
print((t[40:48] - t[40, 9]))
