"""HBM bandwidth of the solver's vector kernels at cfg5 scale (dim = N C = 1e7,
rank up to 320): gemv_t (Q' z), gemv_n (s - Q y), dots, lincomb, gram."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2310_20285_b200 import kernels as K

torch.cuda.set_device(0)
dim, R = 10_000_000, 320
Q = torch.randn(R, dim, device="cuda")
z = torch.randn(dim, device="cuda")
s = torch.randn(dim, device="cuda")
y = torch.randn(R, device="cuda", dtype=torch.float32)


def bench(name, fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{name:28s} {1e3 * dt:8.3f} ms  {nbytes / dt / 1e9:8.0f} GB/s", flush=True)


bench("gemv_t  Q'z  (R=320)", lambda: K.gemv_t(Q, z), Q.numel() * 4 + dim * 4)
bench("gemv_n  s-Qy (R=320)", lambda: K.gemv_n(Q, y, s, -1.0), Q.numel() * 4 + 2 * dim * 4)
bench("dots x4", lambda: K.dots([(z, s), (s, s), (z, z), (s, z)]), 2 * dim * 4)
bench("lincomb", lambda: K.lincomb(1.0, z, 0.5, s), 3 * dim * 4)
B = 64
S = Q[:B]
bench("gram 64x320 over dim", lambda: K.gram(Q, S), (Q.numel() + S.numel()) * 4)
