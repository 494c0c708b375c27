"""Per-kernel GPU time breakdown of a short IterNCGP fit (torch.profiler /
CUPTI activity records; not a timing run).

usage: python tools/fit_profile.py cfg4 [--steps 2] [--inner 20]
"""
import argparse
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
import paper_2310_20285_b200 as P
from paper_2310_20285_b200 import configs

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--inner", type=int, default=20)
ap.add_argument("--residual", default="explicit")
args = ap.parse_args()
torch.cuda.set_device(0)
c = configs.CONFIGS[args.cfg]()
C = c["C"]
prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*c["kernel"]),) * C)
ds = P.Dataset(c["X"], c["y"], "class-index", C)
lik = P.SoftmaxLikelihood(ds.targets, C)
inner = P.InnerConfig(max_iters=1, residual=args.residual)
oc = P.OuterConfig(max_newton_steps=args.steps, delta=c["delta"], inner_schedule=args.inner,
                   recycle=c["recycle"], compression_rank=c["rank"])
P.fit(prior, ds, lik, P.OuterConfig(max_newton_steps=1, inner_schedule=2), inner,
      policy_kind=c["policy"], dtype=torch.float32)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    belief, trace = P.fit(prior, ds, lik, oc, inner, policy_kind=c["policy"], dtype=torch.float32)
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0, 0.0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        a = agg[ev.name[:90]]
        a[0] += 1
        a[1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
tot = sum(v[1] for v in agg.values())
print(f"{args.cfg}: fit wallclock {trace.wallclock_s:.3f} s, GPU busy {tot / 1e6:.3f} s, "
      f"{trace.total_kernel_matvecs} K products")
for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{100 * us / tot:6.2f} %  {us / 1e3:10.2f} ms  {n:6d}x  {name}")
