"""Per-call time of ShardedPriorOperator (gather reduce vs nccl) as rank 0 of
a fake world of W (collectives are identities / local copies), split into
upload, operator and download.  usage: python tools/e2e_split_probe.py W"""
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dist.is_initialized = lambda: True
dist.get_world_size = lambda group=None: W
dist.get_rank = lambda group=None: 0
dist.all_reduce = lambda t, op=None, group=None: t


def _gather(out, inp, group=None, **kw):
    per = inp.shape[0]
    for r in range(W):
        if out[r * per:(r + 1) * per].data_ptr() != inp.data_ptr():
            out[r * per:(r + 1) * per].copy_(inp)


dist.all_gather_into_tensor = _gather
sys.path.insert(0, ".")
import paper_2310_20285_b200 as P  # noqa: E402
from paper_2310_20285_b200.device import to_host_tensor  # noqa: E402
from paper_2310_20285_b200.parallel import ShardedPriorOperator  # noqa: E402

torch.cuda.set_device(0)
n, w = 1_000_000, 32
rng = np.random.default_rng(0)
X = rng.standard_normal((n, 8)).astype(np.float32)
S = torch.from_numpy(rng.standard_normal((n, w)).astype(np.float32)).pin_memory()
prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.5, 1.0),) * w)
for g in ("nccl", "reduce", "nccl", "reduce"):
    sop = ShardedPriorOperator(prior, X, dtype=torch.float32, gather=g)
    v = S.view(-1).to("cuda", non_blocking=True)
    r = sop(v)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        v = S.view(-1).to("cuda", non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        r = sop(v)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        h = to_host_tensor(r)
        t3 = time.perf_counter()
        ts.append((t1 - t0, t2 - t1, t3 - t2))
    m = np.min(np.array(ts), axis=0) * 1e3
    print(f"{g:6s} W={W}: upload {m[0]:.2f} ms  operator {m[1]:.2f} ms  download {m[2]:.2f} ms", flush=True)
    del sop
