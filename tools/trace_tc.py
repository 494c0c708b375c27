"""Per-tile timeline of CTA 0 of the tcgen05 operator (debug hook).

usage: python tools/trace_tc.py [n] [family] [debug_mode]
Events (clock64 of CTA 0, one row per tile step g):
  0 p_ready  MMA warp saw p_full(g)        8 v_ready  MMA warp saw v_full(g)
  1 g2_iss   GEMM2(g) issued               2 g1_iss   GEMM1(g+3) issued
  9 xb_ready MMA warp saw xb_full(g) (before issuing GEMM1(g))
  3/5 eN_wait  epilogue WG N starts waiting s_full(g); 4/6 eN_go  it saw s_full(g)
  7/10 eN_done epilogue WG N arrived p_full(g)
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200 import _native
from paper_2310_20285_b200.kernels import KernelOperator

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
fam = sys.argv[2] if len(sys.argv) > 2 else "rbf"
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
EV = 16
rng = np.random.default_rng(0)
X = torch.from_numpy(rng.standard_normal((n, 8))).float().cuda()
W = int(os.environ.get("TRACE_W", "32"))
S = torch.from_numpy(rng.standard_normal((n, W))).float().cuda()
op = KernelOperator(fam, 1.5, 1.0, X, w_max=32, impl="tcgen05")
op.apply(S)
buf = torch.zeros(256 * EV + 4 * 4096, dtype=torch.int64, device="cuda")
lib = _native.load()
lib.ncgp_debug_set_trace.argtypes = [ctypes.c_void_p]
lib.ncgp_debug_set_trace(buf.data_ptr())
lib.ncgp_debug_set_mode(mode)
op.apply(S)
torch.cuda.synchronize()
lib.ncgp_debug_set_trace(None)
lib.ncgp_debug_set_mode(0)
allb = buf.cpu().numpy().astype(np.int64)
t = allb[:256 * EV].reshape(256, EV)
span = allb[256 * EV:].reshape(4096, 4)
span = span[span[:, 0] > 0]
t0 = span[:, 0].min()
ends = (span[:, 1] - t0) / 1e3
print(f"CTAs {len(span)}: end min {ends.min():.1f} / median {np.median(ends):.1f} / max {ends.max():.1f} us")
lo, hi = 40, 200
e = t[lo:hi]


def st(x):
    return "mean %6.0f  med %6.0f" % (np.mean(x), np.median(x))


# epilogue done / go for either WG
done = np.where(e[:, 7] > 0, e[:, 7], e[:, 10])
go = np.where(e[:, 4] > 0, e[:, 4], e[:, 6])
wt = np.where(e[:, 3] > 0, e[:, 3], e[:, 5])
print(f"n={n} {fam} mode={mode}: steps {lo}..{hi} of CTA 0")
print("step interval (p_ready)      ", st(np.diff(e[:, 0])))
print("MMA: p_ready -> v_ready      ", st(e[:, 8] - e[:, 0]))
print("MMA: v_ready -> g2 issued    ", st(e[:, 1] - e[:, 8]))
print("MMA: g2 issued -> xb_ready   ", st(t[lo + 3:hi + 3, 9] - e[:, 1]))
print("MMA: xb_ready -> g1 issued   ", st(e[:, 2] - t[lo + 3:hi + 3, 9]))
print("MMA: g1 issued -> next p_rdy ", st(t[lo + 1:hi + 1, 0] - e[:, 2]))
print("EPI: wait s_full             ", st(go - wt))
print("EPI: busy (go -> done)       ", st(done - go))
print("EPI: done -> MMA p_ready     ", st(e[:, 0] - done))
print("g1 issued(g) -> epi go(g+3)  ", st(t[lo + 3:hi + 3][:, [4, 6]].max(1) - e[:, 2]))

if len(sys.argv) > 4:  # raw per-step dump
    base = t[lo, 0]
    print(" g   g2_pre  rdy_seen  g2_iss  g1_iss | epiA_wait epiA_go epiA_done | epiB_wait epiB_go epiB_done")
    for g in range(lo, lo + int(sys.argv[4])):
        r = t[g]
        print("%3d %7d %8d %7d %7d | %8d %7d %8d | %8d %7d %8d" % (g, r[11] - base, r[0] - base, r[1] - base,
              r[2] - base, r[3] - base, r[4] - base, r[7] - base, r[5] - base, r[6] - base, r[10] - base))
