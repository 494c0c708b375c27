#!/usr/bin/env python
"""Benchmark: fused kernel-operator product K(X, X) S on B200 (BASELINE cfg3)
and the IterNCGP fit time (cfg4, and cfg5 = N 1M, C 10).

BASELINE.json metric: "fused K^.S GFLOP/s (%roofline) and IterNCGP fit time,
N=1M C=10".  One step is one kernel-operator product over the cfg3 workload
(N = 1e6 points, D = 8, S of width 32, RBF l = 1.5; ``--workload
cfg3-matern`` for the Matern variant) with inputs resident in HBM.
Algorithmic FLOPs per (i, j) pair are F = 2D + 2w,
i.e. 80 at cfg3.  The same JSON line carries, under ``fit``, the end-to-end
fit time of cfg4 and cfg5 (``FitTrace.wallclock_s``, outer.py:103-126,
253-255), its K-product count and the reference CPU time extrapolated from
the reference tile body timed on sample rows.

Multi-GPU (torchrun): the symmetric kernel's work list split across ranks
with an int64 all-reduce (``--gather reduce``, the default when available),
or contiguous row blocks with the output all-gathered.  Total work is fixed
as N grows -> "strong" scaling.

``--impl reference`` times the reference algorithm's CPU implementation (the
numpy restatement in oracle/, bit-identical to the reference, run with all
host cores over row samples of the same workload).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P_MUFU_PER_SM_CLK = 16          # ex2 per clock per SM (cc 10.0 throughput table)
TF32_FALLBACK_TFLOPS = None


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return dict(hbm=d.get("hbm_gbs", 6552.0), bf16=d.get("bf16_tflops", 1668.4),
                    sm_max_mhz=d.get("sm_max_mhz", 1965.0), source="measured")
    return dict(hbm=6650.0, bf16=1590.0, sm_max_mhz=1965.0, source="fallback")


def workload(name):
    from paper_2310_20285_b200 import configs
    fam = "matern32" if name.endswith("matern") else "rbf"
    c = configs.cfg3(family=fam)
    return c


def product_config(c):
    """The workload-defining config, identical in both arms (``same_config``)."""
    X, S, spec = c["X"], c["S"], c["kernel"]
    n, d = X.shape
    w = S.shape[1]
    return {"workload": c["name"], "n": int(n), "d": int(d), "w": int(w), "kernel": list(spec),
            "flops_per_pair": 2 * d + 2 * w, "exp_per_pair": 1 if spec[0] == "rbf" else 2,
            "l2": "flushed (256 MiB write) before every timed GPU step; fresh random rows per "
                  "CPU step"}


def executed_per_pair(variant, d, w, n):
    """Executed tensor flops and evaluated-pair fraction of a K1 variant
    (DESIGN.md 3.1/3.1b): GEMM1 2 ka, GEMM2 2 (2 WP + WP) per evaluated
    pair, plus the symmetric kernels' transposed product on off-diagonal
    tiles (pair kernel: N = 2 WP per CTA pair, half of it discarded)."""
    ka = -(-(3 * d + 4) // 16) * 16
    wp = 16 if w <= 16 else 32
    nb = -(-n // 128)
    base = 2 * ka + 6 * wp
    if variant == 2:        # single-CTA symmetric kernel: row tile r covers [r, nb)
        ev = (nb + 1) / (2.0 * nb)
        tfrac = (nb - 1) / (nb + 1.0)
        return base + 6 * wp * tfrac, ev
    if variant == 4:        # blocked symmetric kernel: same tiles as variant 2; the
        ev = (nb + 1) / (2.0 * nb)   # transposed product P_hi^T [Vhi|Vlo] (fp16, N = 2 WP)
        tfrac = (nb - 1) / (nb + 1.0)  # + P_lo^T Vhi in E4M3 (N = WP at twice the rate)
        return base + 5 * wp * tfrac, ev
    if variant == 1:        # pair kernel: row-tile pair a covers [2a, nb)
        tiles = sum(nb - 2 * a for a in range((nb + 1) // 2))
        trans = sum(max(0, nb - 2 * a - 2) for a in range((nb + 1) // 2))
        ev = 2.0 * tiles / (nb * nb)
        return base + 12 * wp * trans / max(tiles, 1), ev
    return float(base), 1.0


class ClockSampler(threading.Thread):
    """Samples SM clock and clock-event reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        super().__init__(daemon=True)
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop_evt = threading.Event()
        self.ok = False

    def run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            while not self._stop_evt.is_set():
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
                time.sleep(0.1)
        except Exception as exc:  # NVML unavailable: report, do not fake
            self.error = repr(exc)

    def stop(self):
        self._stop_evt.set()
        self.join(timeout=2)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def cpu_reference_sample(spec, X, S, rows, processes):
    """Time the reference tile body (oracle restatement) on ``rows``."""
    from oracle import ncgp_oracle as O
    if processes <= 1:
        t0 = time.perf_counter()
        O.kernel_matmul_rows(spec, X[rows], X, S, tile=len(rows))
        return time.perf_counter() - t0
    import multiprocessing as mp
    chunks = np.array_split(rows, processes)
    ctx = mp.get_context("fork")
    global _SHARED
    _SHARED = (spec, X, S)
    with ctx.Pool(processes) as pool:
        pool.map(_cpu_chunk, [chunks[0][:1]] * processes)  # warm the workers
        t0 = time.perf_counter()
        pool.map(_cpu_chunk, chunks)
        return time.perf_counter() - t0


_SHARED = None


def _cpu_chunk(rows):
    from oracle import ncgp_oracle as O
    spec, X, S = _SHARED
    O.kernel_matmul_rows(spec, X[rows], X, S, tile=max(1, len(rows)))
    return 0


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    c = workload(args.workload)
    X, S, spec = c["X"], c["S"], c["kernel"]
    n, d = X.shape
    w = S.shape[1]
    F = 2 * d + 2 * w
    cores = os.cpu_count() or 1
    rows_per_step = 2 * cores
    rng = np.random.default_rng(1)
    times = []
    for it in range(args.warmup + args.steps):
        rows = np.sort(rng.choice(n, size=rows_per_step, replace=False))
        dt = cpu_reference_sample(spec, X, S, rows, cores)
        if it >= args.warmup:
            times.append(dt)
    pairs = rows_per_step * n
    value = F * pairs / statistics.mean(times) / 1e9
    line = {
        "impl": "reference", "metric": "fused K^.S GFLOP/s (cfg3 K(X,X)S)",
        "value": round(value, 4), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * statistics.mean(times), 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": product_config(c),
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores,
                         "kind": "port",
                         "sample": f"{rows_per_step} random rows x all {n} columns per step "
                                   f"(reference tile body gp.py:162-171, numpy fp64, "
                                   f"{cores} worker processes)"},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2310_20285_b200 as P
    from paper_2310_20285_b200 import _native
    from paper_2310_20285_b200.kernels import KernelOperator

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    c = workload(args.workload)
    X, S, spec = c["X"], c["S"], c["kernel"]
    n, d = X.shape
    w = S.shape[1]
    F = 2 * d + 2 * w
    E = 1 if spec[0] == "rbf" else 2
    Xd = torch.from_numpy(X).to(dev, torch.float32)
    Sd = torch.from_numpy(S).to(dev, torch.float32)
    op = KernelOperator(spec[0], spec[1], spec[2], Xd, w_max=w, impl=args.kop)
    from paper_2310_20285_b200.parallel import row_partition
    r0, r1, per = row_partition(n, world, rank)
    # nccl: each rank writes its rows straight into its slice of the gather
    # buffer and the all-gather runs in place.  fused: the gather buffers are
    # symmetric memory and K1 stores every row into all ranks' buffers
    # (parallel.RowShardedOperator implements both).
    # reduce: the symmetric kernel's triangular work list is split across the
    # ranks and an NCCL all-reduce sums the int64 fixed-point accumulators
    # (parallel.SymmetricSplitOperator; exact, so 1 and N GPUs give the same
    # bits); auto takes it when available.
    gather = args.gather
    if gather == "auto":
        gather = "reduce" if world > 1 and op.sym_acc_elems(w) > 0 else "nccl"
    reduce_ = world > 1 and gather == "reduce"
    acc = torch.empty(max(1, op.sym_acc_elems(w)), dtype=torch.int64, device=dev) if reduce_ else None
    fused = world > 1 and gather == "fused"
    peer_rows = None
    if fused:
        from paper_2310_20285_b200.parallel import TorchSymmetricMemory
        out_full, barrier, peers = TorchSymmetricMemory().alloc((per * world, w), torch.float32,
                                                                dev)
        peer_rows = [q[:n] for q in peers]
    else:
        out_full = torch.empty((per * world, w), dtype=torch.float32, device=dev)
    out_rows = out_full[:n]
    mine = out_full[rank * per:(rank + 1) * per]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def pre():
        if fused:
            barrier(0)

    def post():
        if fused:
            barrier(1)
        elif reduce_:
            dist.all_reduce(acc)
            op.sym_finalize(acc, w, out_rows)
        elif world > 1:
            dist.all_gather_into_tensor(out_full, mine)

    def kernel():
        if reduce_:
            op.sym_partial(Sd, rank, world, acc)
        else:
            op.apply(Sd, out=out_rows, row_begin=r0, row_end=r1, peers=peer_rows)

    def step():
        pre()
        kernel()
        post()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    launches0 = _native.launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kstarts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for k in range(args.steps):
        flush.zero_()  # evict L2 between timed steps (outside the events)
        starts[k].record(stream)
        pre()
        kstarts[k].record(stream)
        kernel()
        kends[k].record(stream)
        post()
        ends[k].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = _native.launch_count() - launches0
    clocks = sampler.stop()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    kern_ms = [s.elapsed_time(e) for s, e in zip(kstarts, kends)]
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms, sum(kern_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kern_total = float(t[0]), float(t[1])
    if os.environ.get("NCGP_BENCH_RANK_REPORT"):  # per-rank kernel time (tools/fake_dist_bench.py)
        print(json.dumps({"rank": rank, "kernel_ms": round(kern_total / args.steps, 3)}),
              file=sys.stderr, flush=True)
    pairs = float(n) * float(n)
    value = F * pairs * args.steps / (total_ms / 1e3) / 1e9

    # ---- e2e through the public API: pinned host S in, host result out.
    # One GPU: gp.prior_matvec (cached operator).  N GPUs: the row-sharded
    # operator (parallel.ShardedPriorOperator: local rows + in-place NCCL
    # all-gather) on every rank; max over ranks.
    from paper_2310_20285_b200.device import to_host_tensor
    Sh = torch.from_numpy(S).to(torch.float32).pin_memory()
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*spec),) * w)
    if world == 1:
        Xh = torch.from_numpy(X).to(torch.float32)
        call = lambda: P.prior_matvec(prior, Xh, Sh.view(-1))  # noqa: E731
    else:
        from paper_2310_20285_b200.parallel import ShardedPriorOperator
        sop = ShardedPriorOperator(prior, X.astype(np.float32), dtype=torch.float32,
                                   gather=gather)
        call = lambda: to_host_tensor(sop(Sh.view(-1).to(dev, non_blocking=True)))  # noqa: E731
    # builds + caches the operator; two results alive at once so the pinned
    # host allocator holds the blocks the timed calls cycle through
    warm = [call(), call()]
    del warm
    res = call()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(max(1, args.steps)):
        res = call()
    torch.cuda.synchronize()
    e2e_s = torch.tensor([(time.perf_counter() - t0) / max(1, args.steps)], dtype=torch.float64,
                         device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_np = None
    if world == 1:
        # the reference's own call shape: numpy fp64 X and v in, numpy fp64
        # out (gp.py:144-172), pageable host memory both ways
        Snp = np.ascontiguousarray(S).reshape(-1)
        call_np = lambda: P.prior_matvec(prior, X, Snp, dtype=torch.float32)  # noqa: E731
        call_np()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        k_np = max(1, min(3, args.steps))
        for _ in range(k_np):
            r_np = call_np()
        torch.cuda.synchronize()
        s_np = (time.perf_counter() - t0) / k_np
        e2e_np = {"value": round(F * pairs / s_np / 1e9, 3), "unit": "GFLOP/s",
                  "ms_per_call": round(1e3 * s_np, 2),
                  "h2d_bytes_per_step": int(Snp.nbytes), "d2h_bytes_per_step": int(r_np.nbytes),
                  "note": "gp.prior_matvec(prior, X, v) with numpy fp64 X and v (pageable), numpy "
                          "fp64 result: the reference's signature; the cached operator is "
                          "validated against a full copy of X every call"}
    e2e = {"value": round(F * pairs / float(e2e_s[0]) / 1e9, 3), "unit": "GFLOP/s",
           "h2d_bytes_per_step": int(Sh.numel() * 4),
           "d2h_bytes_per_step": int(res.numel() * res.element_size()),
           "note": "X resident in the cached operator; S (pinned fp32) uploaded and the "
                   "product downloaded every step" +
                   ("" if world == 1 else f" on each of the {world} ranks (row-sharded "
                                          "operator, " + ("rows stored into every rank's "
                                                          "symmetric-memory buffer by K1)"
                                                          if fused else "in-place all-gather)"))}
    if reduce_:
        e2e["note"] = ("X resident in the cached operator; S (pinned fp32) uploaded and the product "
                       f"downloaded every step on each of the {world} ranks (symmetric kernel's work "
                       "list split across ranks, int64 accumulators summed by an NCCL all-reduce)")

    # ---- roofline of the dominant kernel (the fused kernel-matmul)
    roofline = product_roofline(op, n, d, w, F, E, world, local_pairs=(
        float(n) * n / world if reduce_ else float(r1 - r0) * n), t_kernel=kern_total / args.steps / 1e3,
        dev=dev, workload_name=c["name"])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows = np.sort(np.random.default_rng(0).choice(n, size=args.cpu_rows, replace=False))
        cpu_s = cpu_reference_sample(spec, X, S, rows, 1)
        cpu = {"value": round(F * len(rows) * n / cpu_s / 1e9, 4), "unit": "GFLOP/s",
               "cores": 1, "kind": "port",
               "sample": f"{len(rows)} random rows x all {n} columns (reference tile body, "
                         f"numpy fp64, 1 core), {cpu_s:.1f} s"}

    line = None
    if rank == 0:
        line = {"metric": "fused K^.S GFLOP/s (cfg3 K(X,X)S)", "value": round(value, 3),
                "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": product_config(c),
                "parallelism": (f"symmetric work list split x{world}" if reduce_
                                else f"row-sharded x{world}"),
                "gather": gather if world > 1 else None,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_numpy_f64": e2e_np,
                "gpu_launches": int(launches), "clocks": clocks}
    del op, Xd, Sd, out_full, flush
    torch.cuda.empty_cache()
    # the metric's second half: IterNCGP fit time (cfg4, and cfg5 = N 1M C 10)
    if not args.no_fit:
        fits = {}
        for name in args.fits.split(","):
            if name:
                # cfg4 (~6 s, two host syncs per inner iteration: sensitive to host
                # noise) is timed three times and the median reported; cfg5 once
                fits[name] = measure_fit(name, args, rank, world, local_rank, warmup_fits=1,
                                         timed_fits=3 if name == "cfg4" else 1,
                                         cpu_extrapolate=not args.no_cpu_baseline)
        if line is not None:
            line["fit"] = fits
            line["gpu_launches"] = int(line["gpu_launches"]) + sum(
                int(f["gpu_launches"]) for f in fits.values())
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


def product_roofline(op, n, d, w, F, E, world, local_pairs, t_kernel, dev, workload_name):
    """Roofline of one K1 launch, two ways.

    - ``frac`` (BASELINE.md section 4 / SURVEY.md 8(d)): ALGORITHMIC flops F
      per pair over all local pairs, against t* = max(F / P_tensor, E /
      P_mufu) per pair.  For the symmetric kernels this can exceed 1 (they
      evaluate half of the kernel values), so it is not a bound there.
    - ``executed``: the work the kernel actually issues -- tensor flops of
      the 3-term fp16 GEMMs (kind::f16, against the measured dense bf16
      peak) and ex2 (+ sqrt) per evaluated pair (against 16 per clock per
      SM) -- the utilisation of each pipe; ``limiter`` is the busier one.
    """
    import torch
    pk = peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    mufu_rate = sms * P_MUFU_PER_SM_CLK * pk["sm_max_mhz"] * 1e6   # ex2 / s
    tensor_tflops = pk["bf16"] / 2.0                                 # tf32-class dense
    achieved = F * local_pairs / t_kernel / 1e12
    peak_tflops = min(tensor_tflops, F * mufu_rate / E / 1e12)
    variant = op.last_variant_code
    fx, ev = executed_per_pair(variant, d, w, n)
    pairs_eval = local_pairs * ev
    ten = fx * pairs_eval / t_kernel / 1e12
    mufu = E * pairs_eval / t_kernel
    executed = {"tensor": {"achieved": round(ten, 2), "peak": pk["bf16"], "unit": "TFLOP/s",
                           "frac": round(ten / pk["bf16"], 4),
                           "flops_per_evaluated_pair": round(fx, 2),
                           "basis": "kind::f16 MMAs (GEMM1 3-term split along K, GEMM2 "
                                    "P_hi [Vhi|Vlo] + P_lo Vhi, transposed product) against "
                                    f"the {pk['source']} dense bf16 peak"},
                "mufu": {"achieved": round(mufu / 1e12, 4), "peak": round(mufu_rate / 1e12, 4),
                         "unit": "Tex2/s", "frac": round(mufu / mufu_rate, 4),
                         "per_evaluated_pair": E},
                "evaluated_pair_fraction": round(ev, 4)}
    lim = "tensor pipe" if executed["tensor"]["frac"] >= executed["mufu"]["frac"] else "MUFU ex2"
    # DRAM traffic of the same kernel variant on the same workload: copied
    # from the committed ncu --set full capture (a number taken under a
    # profiler cannot be measured inside this run)
    traffic, traffic_src = None, None
    captures = {("cfg3", 2): "r02_summary.json", ("cfg3", 4): "r02f_summary.json"}
    prof = captures.get((workload_name, variant))
    if prof and world == 1 and os.path.exists(os.path.join(ROOT, "profiles", prof)):
        with open(os.path.join(ROOT, "profiles", prof)) as fh:
            traffic = json.load(fh).get("traffic_bytes_per_launch")
        traffic_src = f"copied from profiles/{prof} (ncu --set full of this kernel on this " \
                      "workload: dram__bytes_read.sum + dram__bytes_write.sum)"
    return {"bound": "tensor", "limiter": lim, "achieved": round(achieved, 3),
            "peak": round(peak_tflops, 3), "unit": "TFLOP/s",
            "frac": round(achieved / peak_tflops, 4), "traffic": traffic,
            "traffic_source": traffic_src, "executed": executed,
            "frac_executed": round(max(executed["tensor"]["frac"], executed["mufu"]["frac"]), 4),
            "peak_basis": f"algorithmic: min({pk['source']} bf16 {pk['bf16']}/2 TF/s, "
                          f"{sms} SM x {P_MUFU_PER_SM_CLK} ex2/clk x {pk['sm_max_mhz']} MHz x "
                          f"F/E={F}/{E}); bound 'tensor' = compute-bound (tensor pipe / MUFU), "
                          f"not HBM",
            "kernel_ms": round(1e3 * t_kernel, 3), "impl": op.impl,
            "variant": {0: "plain", 1: "symmetric (CTA pairs)", 2: "symmetric (single CTA)",
                        4: "symmetric (blocked, single CTA)"}.get(variant, "none")}


CPU_FIT_ROWS = {"cfg4": 64, "cfg5": 8}   # reference tile-body sample rows per K product


def measure_fit(name, args, rank, world, local_rank, warmup_fits=1, timed_fits=1,
                cpu_extrapolate=True):
    """End-to-end IterNCGP fit on a BASELINE config (synthetic, seeded):
    FitTrace.wallclock_s, the reference's fit-time definition (outer.py:103-126,
    253-255: solver clock, metric hooks excluded), max over ranks.  Warm-up
    fits use a 1-step schedule on the same data (operator packing, allocator,
    library load).  The posterior mean / marginal variance at the test
    points are timed separately.  The reference CPU time is
    extrapolated as BASELINE.md section 3 prescribes: the reference tile body
    (gp.py:162-171) timed on sample rows x all N columns at the config's
    shape, scaled to one K product, times the K-product count of this fit."""
    import torch
    import torch.distributed as dist
    import paper_2310_20285_b200 as P
    from paper_2310_20285_b200 import configs
    from paper_2310_20285_b200 import parallel as PP
    from paper_2310_20285_b200.parallel import ShardedPriorOperator

    torch.cuda.set_device(local_rank)
    c = configs.CONFIGS[name]()
    dt = torch.float32
    C = c["C"]
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*c["kernel"]),) * C)
    ds = P.Dataset(c["X"], c["y"], "class-index", C)
    lik = P.SoftmaxLikelihood(ds.targets, C)
    # N > 1: the solver state is row-sharded like the operator (
    # --state replicated keeps every rank's full copy of v, r, S, T, Q)
    sharded = world > 1 and args.state == "sharded"
    if sharded:
        comm = PP.TorchDistComm()
        op = PP.ShardedStateOperator(prior, c["X"], comm, dtype=dt, gather={
            "auto": "auto", "reduce": "reduce"}.get(args.gather, "rows"))

        def run_fit_(oc_):
            return PP.fit_sharded(prior, ds, lik, oc_, inner, c["policy"], comm=comm, dtype=dt,
                                  operator=op)
    else:
        op = ShardedPriorOperator(prior, c["X"], dtype=dt, gather=args.gather) if world > 1 else \
            P.PriorOperator(prior, c["X"], dtype=dt)

        def run_fit_(oc_):
            return P.fit(prior, ds, lik, oc_, inner, policy_kind=c["policy"], dtype=dt,
                         operator=op)
    inner = P.InnerConfig(max_iters=1, residual=args.residual)
    for _ in range(max(0, warmup_fits)):
        run_fit_(P.OuterConfig(max_newton_steps=1, inner_schedule=2))
    oc = P.OuterConfig(max_newton_steps=c["steps"], delta=c["delta"], inner_schedule=c["inner"],
                       recycle=c["recycle"], compression_rank=c["rank"])
    sampler = ClockSampler(local_rank)
    sampler.start()
    launches0 = _native_launches()
    times, trace, belief = [], None, None
    for _ in range(max(1, timed_fits)):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        belief, trace = run_fit_(oc)
        torch.cuda.synchronize()
        times.append(trace.wallclock_s)
    clocks = sampler.stop()
    launches = _native_launches() - launches0
    t = torch.tensor(times, dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)   # each fit: max over ranks
    times = sorted(float(x) for x in t.tolist())
    secs = times[len(times) // 2] if len(times) % 2 else \
        0.5 * (times[len(times) // 2 - 1] + times[len(times) // 2])   # median over the timed fits
    inner_kind = getattr(getattr(op, "inner", op), "groups", [[None]])[0][0]
    variant = inner_kind.last_variant if inner_kind is not None else None
    del op
    rec = None
    if sharded:  # every rank: its columns of K(X*, X) on its rows of v and Q, all-reduced
        Xt = c["X_test"]
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        with PP.sharded_state(comm, 0, 0):
            mean = P.posterior_mean(belief, Xt)
            t1 = time.perf_counter()
            var = P.posterior_marginal_var(belief, Xt)
        t2 = time.perf_counter()
    if rank == 0:
        Xt = c["X_test"]
        if not sharded:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            mean = P.posterior_mean(belief, Xt)
            t1 = time.perf_counter()
            var = P.posterior_marginal_var(belief, Xt)
            t2 = time.perf_counter()
        probs = P.probit_predict(mean, var)
        rec = {"metric": f"IterNCGP fit time ({name})", "value": round(secs, 3), "unit": "s",
               "higher_is_better": False, "wallclock_s": round(secs, 3),
               "timed_fits_s": [round(x, 3) for x in times],
               "kernel_matvecs": trace.total_kernel_matvecs,
               "inner_iters": [s.inner_iterations for s in trace.steps],
               "termination": trace.termination,
               "config": {"workload": f"fit-{name}", "n": int(c["X"].shape[0]), "C": C,
                          "d": int(c["X"].shape[1]), "kernel": list(c["kernel"]),
                          "schedule": [c["steps"], c["inner"]], "rank": c["rank"],
                          "policy": c["policy"], "recycle": c["recycle"],
                          "residual": args.residual,
                          "solver_state": ("row-sharded" if sharded else
                                           ("replicated" if world > 1 else "single"))},
               "k_product_variant": variant,
               "posterior": {"n_test": int(Xt.shape[0]), "root_rank": int(belief.root.rank),
                             "mean_s": round(t1 - t0, 3), "marginal_var_s": round(t2 - t1, 3),
                             "test_accuracy": round(float(np.mean(probs.argmax(1) == c["y_test"])), 4)},
               "gpu_launches": int(launches), "clocks": clocks}
        if cpu_extrapolate:
            rows_n = CPU_FIT_ROWS.get(name, 16)
            rng = np.random.default_rng(7)
            rows = np.sort(rng.choice(c["X"].shape[0], size=rows_n, replace=False))
            V = rng.standard_normal((c["X"].shape[0], C))
            t_rows = cpu_reference_sample(c["kernel"], c["X"], V, rows, 1)
            per_product = t_rows * c["X"].shape[0] / rows_n
            rec["cpu_baseline"] = {
                "value": round(per_product * trace.total_kernel_matvecs, 1), "unit": "s",
                "cores": 1, "kind": "port",
                "k_product_s": round(per_product, 2),
                "sample": f"reference tile body (gp.py:162-171, numpy fp64) on {rows_n} random rows "
                          f"x all {c['X'].shape[0]} columns, w={C}: {t_rows:.2f} s, scaled to one K "
                          f"product and multiplied by this fit's {trace.total_kernel_matvecs} K "
                          f"products (BASELINE.md 3); the vector work of the solver is not counted"}
    return rec


def run_fit(args, rank, world, local_rank):
    """``--workload fit-cfgN``: one JSON line with the fit time alone."""
    name = args.workload[len("fit-"):]
    rec = measure_fit(name, args, rank, world, local_rank, warmup_fits=args.warmup,
                      timed_fits=args.steps, cpu_extrapolate=not args.no_cpu_baseline)
    if rank == 0:
        line = dict(rec)
        line.update({"n_gpus": world, "steps": max(1, args.steps), "warmup": args.warmup,
                     "ms_per_step": round(1e3 * rec["value"], 1), "scaling": "strong",
                     "vs_baseline": None, "dtype": "f32", "data": "synthetic"})
        print(json.dumps(line), flush=True)
    return 0


def _native_launches():
    from paper_2310_20285_b200 import _native
    return _native.launch_count()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3",
                    choices=["cfg3", "cfg3-matern", "fit-cfg4", "fit-cfg5"],
                    help="cfg3*: the K(X,X)S product (BASELINE metric, default); fit-cfg*: "
                         "end-to-end IterNCGP fit time (the metric's second half)")
    ap.add_argument("--residual", default="explicit", choices=["explicit", "recurrence"],
                    help="fit workloads: inner residual mode (recurrence is opt-in)")
    ap.add_argument("--kop", default="auto", choices=["auto", "tcgen05", "simt"])
    ap.add_argument("--gather", default="auto", choices=["auto", "reduce", "nccl", "fused"],
                    help="N>1 exchange: reduce = the symmetric kernel's work list split across "
                         "ranks + NCCL all-reduce of the accumulators; nccl = row blocks + in-place "
                         "all-gather; fused = row blocks stored by K1 into every rank's "
                         "symmetric-memory buffer; auto = reduce when available, else nccl")
    ap.add_argument("--state", default="sharded", choices=["sharded", "replicated"],
                    help="N > 1 fits: row-shard the solver state with the operator "
                         "(SURVEY.md 8(e)) or replicate it on every rank")
    ap.add_argument("--cpu-rows", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fits", default="cfg4,cfg5",
                    help="product workloads: fit configs timed after the product (the metric's "
                         "second half, 'IterNCGP fit time N=1M C=10' = cfg5)")
    ap.add_argument("--no-fit", action="store_true", help="skip the fit records")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.workload.startswith("fit-"):
            return run_fit(args, rank, world, local_rank)
        return run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
