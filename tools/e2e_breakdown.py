"""Where the e2e (public API, host S in / host result out) time goes at cfg3."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_20285_b200 as P
from paper_2310_20285_b200 import configs

torch.cuda.set_device(0)
c = configs.cfg3()
X, S = c["X"], c["S"]
w = S.shape[1]
prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*c["kernel"]),) * w)
Xh = torch.from_numpy(X).to(torch.float32)
Sh = torch.from_numpy(S).to(torch.float32).pin_memory()
res = P.prior_matvec(prior, Xh, Sh.view(-1))
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    Sd = Sh.view(-1).to("cuda", non_blocking=False)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    out = P.prior_matvec(prior, Xh, Sd)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    host = out.to("cpu")
    t3 = time.perf_counter()
    pin = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
    t4 = time.perf_counter()
    pin.copy_(out)
    torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"H2D {1e3*(t1-t0):.1f} ms  kernel+API {1e3*(t2-t1):.1f} ms  D2H pageable {1e3*(t3-t2):.1f} ms"
          f"  pinned alloc {1e3*(t4-t3):.1f} ms  D2H pinned {1e3*(t5-t4):.1f} ms", flush=True)
    t0 = time.perf_counter()
    r = P.prior_matvec(prior, Xh, Sh.view(-1))
    t1 = time.perf_counter()
    print(f"full prior_matvec(host in/out) {1e3*(t1-t0):.1f} ms", flush=True)
