"""Per-rank time of the row-sharded fit (parallel.fit_sharded) at world size W,
measured on ONE GPU.

1. Record: the W ranks run together as threads (parallel.ThreadComm), and the
   result of every collective of the ranks to be timed is kept on the device.
2. Replay: each of those ranks runs ALONE, its collectives answered from the
   record (a device copy), so it follows exactly the W-rank computation -- its
   slice of every K product, its shard of every vector / Gram / rotation --
   with the GPU to itself.  FitTrace.wallclock_s of the replay is the rank's
   fit time on a GPU of its own, without the collectives' latency (NCCL over
   NVSwitch: an all-gather of N*C values and an all-reduce of the int64
   accumulators per product, a few small all-reduces per iteration).

usage: python tools/sharded_fit_replay.py cfg4 8 [ranks=0,7] [gather=auto] [out.json]
"""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_20285_b200 as P  # noqa: E402
from paper_2310_20285_b200 import configs  # noqa: E402
from paper_2310_20285_b200 import parallel as PP  # noqa: E402
from paper_2310_20285_b200.device import profile_ranges  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
ranks = [int(r) for r in (sys.argv[3] if len(sys.argv) > 3 else f"0,{W - 1}").split(",")]
gather = sys.argv[4] if len(sys.argv) > 4 else "auto"
out_path = sys.argv[5] if len(sys.argv) > 5 else None

c = configs.CONFIGS[name]()
C, dt = c["C"], torch.float32
prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*c["kernel"]),) * C)
ds = P.Dataset(c["X"], c["y"], "class-index", C)
lik = P.SoftmaxLikelihood(ds.targets, C)
inner = P.InnerConfig(max_iters=1)
oc = P.OuterConfig(max_newton_steps=c["steps"], delta=c["delta"], inner_schedule=c["inner"],
                   recycle=c["recycle"], compression_rank=c["rank"])
warm = P.OuterConfig(max_newton_steps=1, inner_schedule=2)


class Recording:
    """A communicator that keeps every collective's result."""

    def __init__(self, comm):
        self.comm, self.rank, self.world, self.log = comm, comm.rank, comm.world, []

    def all_reduce_(self, t):
        self.comm.all_reduce_(t)
        self.log.append(t.clone())
        return t

    def all_gather_(self, full, mine):
        self.comm.all_gather_(full, mine)
        self.log.append(full.clone())
        return full


class Replay:
    def __init__(self, rank, world, log):
        self.rank, self.world, self.log, self.i = rank, world, log, 0

    def _next(self, t):
        t.copy_(self.log[self.i].view_as(t))
        self.i += 1
        return t

    def all_reduce_(self, t):
        return self._next(t)

    def all_gather_(self, full, mine):
        return self._next(full)


def one_fit(comm, config):
    op = PP.ShardedStateOperator(prior, c["X"], comm, dtype=dt, gather=gather)
    belief, trace = PP.fit_sharded(prior, ds, lik, config, inner, c["policy"], comm=comm,
                                   dtype=dt, operator=op)
    torch.cuda.synchronize()
    return op, trace


# one GPU: the plain fit (after a warm-up fit, as bench.py does)
op1 = P.PriorOperator(prior, c["X"], dtype=dt)
P.fit(prior, ds, lik, warm, inner, policy_kind=c["policy"], dtype=dt, operator=op1)
_, t1 = P.fit(prior, ds, lik, oc, inner, policy_kind=c["policy"], dtype=dt, operator=op1)
torch.cuda.synchronize()
del op1
torch.cuda.empty_cache()
print(f"{name}: one GPU {t1.wallclock_s:.3f} s, {t1.total_kernel_matvecs} K products, "
      f"inner {[s.inner_iterations for s in t1.steps]}", flush=True)

comms = PP.ThreadComm.create(W)
recs = {r: Recording(comms[r]) for r in ranks}
traces, errs = {}, []


def body(r):
    try:
        torch.cuda.set_device(0)
        comm = recs.get(r, comms[r])
        one_fit(comms[r], warm)            # warm-up fit (not recorded)
        _, traces[r] = one_fit(comm, oc)
    except BaseException as e:  # noqa: BLE001
        errs.append(e)
        comms[r]._s.barrier.abort()


t0 = time.perf_counter()
ts = [threading.Thread(target=body, args=(r,)) for r in range(W)]
[t.start() for t in ts]
[t.join() for t in ts]
if errs:
    raise errs[0]
tr = traces[ranks[0]]
print(f"record: {W} ranks as threads in {time.perf_counter() - t0:.1f} s; "
      f"{tr.total_kernel_matvecs} K products, inner {[s.inner_iterations for s in tr.steps]}; "
      f"{sum(len(r.log) for r in recs.values())} collective results kept "
      f"({sum(t.numel() * t.element_size() for r in recs.values() for t in r.log) / 2**30:.1f} GiB)",
      flush=True)

res = {"config": name, "world": W, "gather": gather, "one_gpu_s": round(t1.wallclock_s, 3),
       "one_gpu_k_products": t1.total_kernel_matvecs,
       "sharded_k_products": tr.total_kernel_matvecs,
       "sharded_inner_iters": [s.inner_iterations for s in tr.steps], "ranks": {}}
for r in ranks:
    rp = Replay(r, W, recs[r].log)
    op, trace = one_fit(rp, oc)   # first replay doubles as the warm-up of this rank's operator
    rp.i = 0
    op, trace = one_fit(rp, oc)
    assert rp.i == len(rp.log), (rp.i, len(rp.log))
    assert [s.inner_iterations for s in trace.steps] == res["sharded_inner_iters"]
    eff = t1.wallclock_s / (W * trace.wallclock_s)
    # where the rank's time goes: CUDA-event time per nvtx range (a range's time
    # includes the stream's idle gaps while the host issues its launches)
    rp.i = 0
    with profile_ranges() as rt:
        _, tb = one_fit(rp, oc)
    groups = {}
    for k, (t, n) in rt.totals().items():
        g = "solver (host sync + control)" if k.startswith("itergp_solve") else k
        groups[g] = round(groups.get(g, 0.0) + t, 4)
    res["ranks"][str(r)] = {"rows": [op.r0, op.r1], "fit_s": round(trace.wallclock_s, 3),
                            "efficiency_vs_one_gpu": round(eff, 3), "gather": op.gather,
                            "range_time_s": dict(sorted(groups.items())),
                            "range_run_fit_s": round(tb.wallclock_s, 3)}
    print(f"rank {r} of {W} alone (rows {op.r0}:{op.r1}, gather={op.gather}): "
          f"{trace.wallclock_s:.3f} s -> efficiency {eff:.3f} (collective latency not included)",
          flush=True)
    del op, rp
    recs[r].log.clear()
    torch.cuda.empty_cache()
res["note"] = ("per-rank FitTrace.wallclock_s with the rank alone on the GPU and its collectives "
               "replayed from a recorded W-rank run (device copies); NCCL latency not included")
if out_path:
    with open(out_path, "w") as fh:
        json.dump(res, fh, indent=1)
print(json.dumps(res))
