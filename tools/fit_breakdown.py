"""Device-time breakdown of an IterNCGP fit (cfg4 / cfg5): K products
against the solver's vector work, the virtual solver run (Gram, host
eigensolve, rotations) and the likelihood statistics, from CUDA events on
the nvtx ranges (device.profile_ranges).  usage:
    python tools/fit_breakdown.py cfg4 [cfg5] > profiles/r02_fit_breakdown.json"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2310_20285_b200 as P
from paper_2310_20285_b200 import configs
from paper_2310_20285_b200.device import profile_ranges

out = {}
for name in sys.argv[1:] or ["cfg4"]:
    c = configs.CONFIGS[name]()
    C = c["C"]
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*c["kernel"]),) * C)
    ds = P.Dataset(c["X"], c["y"], "class-index", C)
    lik = P.SoftmaxLikelihood(ds.targets, C)
    op = P.PriorOperator(prior, c["X"], dtype=torch.float32)
    P.fit(prior, ds, lik, P.OuterConfig(max_newton_steps=1, inner_schedule=2), P.InnerConfig(max_iters=1),
          dtype=torch.float32, operator=op)
    oc = P.OuterConfig(max_newton_steps=c["steps"], delta=c["delta"], inner_schedule=c["inner"],
                       recycle=c["recycle"], compression_rank=c["rank"])
    torch.cuda.synchronize()
    with profile_ranges() as rt:
        t0 = time.perf_counter()
        belief, trace = P.fit(prior, ds, lik, oc, P.InnerConfig(max_iters=1), dtype=torch.float32,
                              operator=op)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    tot = rt.totals()
    groups = {}
    for k, (t, n) in tot.items():
        g = "K products" if k.startswith("K product") else \
            ("solver (host sync + control)" if k.startswith("itergp_solve") else k)
        s, m = groups.get(g, (0.0, 0))
        groups[g] = (s + t, m + n)
    kt = groups.get("K products", (0.0, 0))[0]
    rec = {"wallclock_s": round(trace.wallclock_s, 3), "measured_wall_s": round(wall, 3),
           "kernel_matvecs": trace.total_kernel_matvecs,
           "inner_iters": [s.inner_iterations for s in trace.steps],
           "k_product_variant": op.groups[0][0].last_variant,
           "device_time_s": {k: round(v[0], 4) for k, v in sorted(groups.items())},
           "calls": {k: v[1] for k, v in sorted(groups.items())},
           "k_share_of_wall": round(kt / wall, 4),
           "non_k_share_of_wall": round(1 - kt / wall, 4),
           "note": "exclusive CUDA-event time per nvtx range on the compute stream; "
                   "'solver (host sync + control)' is the itergp_solve time outside the "
                   "named sub-ranges (residual norm / breakdown syncs, W^-1, policy)"}
    out[name] = rec
    print(json.dumps({name: rec}), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
