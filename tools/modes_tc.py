"""Time the tcgen05 operator with debug modes that remove pipeline parts."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2310_20285_b200 import _native
from paper_2310_20285_b200.kernels import KernelOperator
torch.cuda.set_device(0)
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200_000)
ap.add_argument("--d", type=int, default=8)
ap.add_argument("--w", type=int, default=32)
ap.add_argument("--ell", type=float, default=1.5)
ap.add_argument("--families", default="rbf,matern32")
args = ap.parse_args()
n = args.n
lib = _native.load()
for fam in args.families.split(","):
    rng = np.random.default_rng(0)
    X = torch.from_numpy(rng.standard_normal((n, args.d))).float().cuda()
    S = torch.from_numpy(rng.standard_normal((n, args.w))).float().cuda()
    op = KernelOperator(fam, args.ell, 1.0, X, w_max=args.w, impl="tcgen05")
    for mode, name in ((0, "full"), (1, "no epilogue TMEM/MUFU"), (2, "no GEMM2"), (3, "no GEMM1"), (5, "no copies, no epilogue"), (6, "no GEMMs (sync + epilogue)"),
                       (4, "no column copies"), (8, "no XB copies"), (9, "no V copies")):
        lib.ncgp_debug_set_mode(mode)
        op.apply(S); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); op.apply(S); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        tiles = ((n + 127) // 128) ** 2 / 148  # per SM
        print(f"{fam:8s} mode {mode} {name:24s}: {ms:7.3f} ms  {ms*1e-3*1.965e9/tiles:7.0f} clk/tile")
    lib.ncgp_debug_set_mode(0)
