"""Achieved HBM bandwidth of the bandwidth-bound path kernels (K3-K6) at cfg5
scale (N = 1e6 points, C = 10 classes, fp32), against MEASURED_PEAKS.json.

Algorithmic bytes per launch: every operand read once and
every result written once.  Times are CUDA-event averages after warm-up.  Run
it under `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum` for the DRAM bytes each kernel actually moved.

usage: python tools/bw_kernels.py [--json out.json]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200 import kernels as K

ap = argparse.ArgumentParser()
ap.add_argument("--json", default=None)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--n", type=int, default=1_000_000, help="points (C = 10 classes each)")
ap.add_argument("--no-flush", action="store_true", help="keep L2 warm between repetitions")
args = ap.parse_args()
torch.cuda.set_device(0)
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]

n, C, R = args.n, 10, 320 if args.n <= 1_000_000 else 16
dim = n * C
dt = torch.float32
g = torch.Generator(device="cuda").manual_seed(0)
f = torch.randn(dim, device="cuda", dtype=dt, generator=g)
labels = torch.randint(0, C, (n,), device="cuda", dtype=torch.int64, generator=g)
pi, _, _ = K.softmax_stats(f, labels, n, C)
s = torch.randn(dim, device="cuda", dtype=dt, generator=g)
t = torch.randn(dim, device="cuda", dtype=dt, generator=g)
V8 = torch.randn(8, dim, device="cuda", dtype=dt, generator=g)
Q = torch.randn(R, dim, device="cuda", dtype=dt, generator=g)
y = torch.randn(R, device="cuda", dtype=torch.float64, generator=g)
fb = torch.randn(dim, device="cuda", dtype=dt, generator=g)
lb = (torch.rand(dim, device="cuda", generator=g) > 0.5).to(torch.int64)
nt, Rv = 50_000, 256
A = torch.randn(nt, C * Rv, device="cuda", dtype=dt, generator=g)
s2 = torch.ones(C, device="cuda", dtype=torch.float64)
es = 4

cases = [
    ("softmax_stats (pi, grad, yhat)", lambda: K.softmax_stats(f, labels, n, C),
     dim * es + n * 8 + 3 * dim * es),
    ("softmax_winv  k=1, base (K^ s)", lambda: K.softmax_winv(pi, n, C, s, base=t),
     dim * es * 4),
    ("softmax_winv  k=8 block", lambda: K.softmax_winv(pi, n, C, V8),
     dim * es + 2 * 8 * dim * es),
    ("softmax_w     k=1", lambda: K.softmax_w(pi, n, C, s), 3 * dim * es),
    ("bernoulli_stats (N=1e7)", lambda: K.bernoulli_stats(fb, lb), dim * es + dim * 8 + 4 * dim * es),
    ("diag_apply    k=1, base", lambda: K.diag_apply(fb, s, base=t), 4 * dim * es),
    ("lincomb       a x + b y", lambda: K.lincomb(1.0, s, 0.5, t), 3 * dim * es),
    ("dots          4 pairs", lambda: K.dots([(s, t), (s, s), (t, t), (s, f)]), 3 * dim * es),
    ("gemv_t        Q'z, R=320", lambda: K.gemv_t(Q, s), (R + 1) * dim * es),
    ("gemv_n        s - Q y, R=320", lambda: K.gemv_n(Q, y, s, -1.0), (R + 2) * dim * es),
    ("marginal_var  5e4 x (C R=2560)", lambda: K.marginal_var(A, C, Rv, s2),
     A.numel() * es + nt * C * es),
]

flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
rows = []
for name, fn, nbytes in cases:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(args.reps):
        if not args.no_flush:
            flush.fill_(1)  # evict the operands from the 126 MB L2: HBM, not L2, bandwidth
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / args.reps
    gbs = nbytes / (ms * 1e-3) / 1e9
    rows.append({"kernel": name, "ms": round(ms, 4), "algorithmic_bytes": int(nbytes),
                 "achieved_gbs": round(gbs, 1), "frac_of_hbm_peak": round(gbs / peak, 3)})
    print(f"{name:34s} {ms:8.4f} ms  {gbs:7.0f} GB/s  {100 * gbs / peak:5.1f} % of {peak:.0f}",
          flush=True)
if args.json:
    json.dump({"hbm_peak_gbs": peak, "source": "MEASURED_PEAKS.json", "shape":
               {"n": n, "C": C, "R": R, "dtype": "fp32"},
               "l2": "warm" if args.no_flush else "flushed (256 MiB write) before every timed launch",
               "timing": "CUDA events around each launch, averaged", "kernels": rows},
              open(args.json, "w"), indent=1)
