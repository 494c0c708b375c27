"""Per-tile timeline of cluster 0 of the symmetric K(X, X) kernel (debug hook).

usage: NCGP_SYM=1 [TRACE_D=8] [TRACE_W=32] python tools/trace_sym.py [n] [family]
Item 0 is row-tile pair 0 over column tiles 0..127 (transposed from tile 2).
Events (clock64 of CTA 0, row = tile step g):
  11 GEMM2 starts waiting rdy(g)    0 GEMM2 saw rdy(g)    1 GEMM2(g) issued
  9  GEMM1 saw g2done (S buffer free) for tile g           2 GEMM1(g) issued
  3/5 epilogue group wait start     4/6 saw s_full(g)   8 saw pt_free (before the first P store)   7/10 P(g) done
  12 T saw rdy(g)   13 T saw dt_empty   14 T(g) issued + committed
  15 correction drained D_T(g) (warp 0)
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ.setdefault("NCGP_SYM", "1")
from paper_2310_20285_b200 import _native
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
fam = sys.argv[2] if len(sys.argv) > 2 else "rbf"
EV = 16
rng = np.random.default_rng(0)
D = int(os.environ.get("TRACE_D", "8"))
X = torch.from_numpy(rng.standard_normal((n, D))).float().cuda()
W = int(os.environ.get("TRACE_W", "32"))
S = torch.from_numpy(rng.standard_normal((n, W))).float().cuda()
op = KernelOperator(fam, float(os.environ.get("TRACE_ELL", "1.5")), 1.0, X, w_max=W, impl="tcgen05")
op.apply(S)
buf = torch.zeros(256 * EV + 4 * 4096, dtype=torch.int64, device="cuda")
lib = _native.load()
lib.ncgp_debug_set_trace.argtypes = [ctypes.c_void_p]
lib.ncgp_debug_set_trace(buf.data_ptr())
op.apply(S)
torch.cuda.synchronize()
lib.ncgp_debug_set_trace(None)
allb = buf.cpu().numpy().astype(np.int64)
t = allb[:256 * EV].reshape(256, EV)
span = allb[256 * EV:].reshape(4096, 4)
span = span[span[:, 0] > 0]
t0 = span[:, 0].min()
ends = (span[:, 1] - t0) / 1e3
starts = (span[:, 0] - t0) / 1e3
print(f"CTAs {len(span)}: start max {starts.max():.1f} us, end min {ends.min():.1f} / median "
      f"{np.median(ends):.1f} / max {ends.max():.1f} us")
print("end-time deciles (us):", np.round(np.percentile(ends, np.arange(0, 101, 10)), 1))
lo, hi = 16, 112
e = t[lo:hi]


def st(x):
    return "mean %7.0f  med %7.0f" % (np.mean(x), np.median(x))


go = np.where(e[:, 4] > 0, e[:, 4], e[:, 6])
wt = np.where(e[:, 3] > 0, e[:, 3], e[:, 5])
done = np.where(e[:, 7] > 0, e[:, 7], e[:, 10])
print(f"n={n} {fam}: steps {lo}..{hi} of cluster 0 (item 0)")
print("step interval (GEMM2 saw rdy)   ", st(np.diff(e[:, 0])))
print("step interval (T issued)        ", st(np.diff(e[:, 14])))
print("GEMM2: wait rdy                 ", st(e[:, 0] - e[:, 11]))
print("GEMM2: issue                    ", st(e[:, 1] - e[:, 0]))
print("GEMM1(g): g2done seen -> issued ", st(e[:, 2] - e[:, 9]))
print("GEMM1(g+3) issued - GEMM2(g) iss", st(t[lo + 3:hi + 3, 2] - e[:, 1]))
print("EPI: wait s_full                ", st(go - wt))
print("EPI: go -> pt_free seen (chunk1)", st(e[:, 8] - go))
print("EPI: transform (go -> done)     ", st(done - go))
print("EPI: GEMM1 issued -> s_full seen", st(go - e[:, 2]))
print("P done -> GEMM2 saw rdy         ", st(e[:, 0] - done))
print("T: saw rdy - GEMM2 saw rdy      ", st(e[:, 12] - e[:, 0]))
print("T: wait dt_empty                ", st(e[:, 13] - e[:, 12]))
print("T: issue                        ", st(e[:, 14] - e[:, 13]))
print("T issued -> D_T drained         ", st(e[:, 15] - e[:, 14]))
print("D_T drained -> next T dt_empty  ", st(t[lo + 1:hi + 1, 13] - e[:, 15]))
base = e[0, 0]
np.set_printoptions(linewidth=200)
cols = [11, 0, 1, 2, 8, 4, 6, 7, 10, 12, 13, 14, 15]
print("raw (cycles from step %d GEMM2 rdy), columns %s" % (lo, cols))
for g in range(8):
    print(lo + g, [int(e[g, c] - base) if e[g, c] else None for c in cols])
