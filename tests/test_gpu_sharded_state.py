"""Row-sharded solver state on one B200.

The N-rank path is exercised on a single GPU with ``parallel.ThreadComm``:
``world`` Python threads, one per rank, each running the real sharded fit
(its own operator, its own row shard of every vector and column block, the
CUDA kernels of the C ABI) and meeting at host barriers for the collectives
-- no kernel waits on another rank's kernel.  The sharded fit must follow
the single-process fit: same inner iteration counts, weights / posterior
within the rounding of the differently-ordered fp64 partial sums.
"""

import threading

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2310_20285_b200 as P  # noqa: E402
from paper_2310_20285_b200 import kernels as K  # noqa: E402
from paper_2310_20285_b200 import parallel as PP  # noqa: E402

F64, F32 = torch.float64, torch.float32


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) /
                 max(np.linalg.norm(np.asarray(b)), 1e-300))


def run_ranks(world, fn):
    """fn(comm) on ``world`` threads; returns the per-rank results."""
    comms = PP.ThreadComm.create(world)
    out, err = [None] * world, [None] * world

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(comms[r])
        except BaseException as e:  # noqa: BLE001
            err[r] = e
            comms[r]._s.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return out


# ------------------------------------------------------------------ C ABI

def _sym_problem(n=45_056 + 100, d=4, w=10, seed=0):
    rng = np.random.default_rng(seed)
    X = torch.from_numpy(rng.standard_normal((n, d))).to("cuda", F32)
    V = torch.from_numpy(rng.standard_normal((n, w))).to("cuda", F32)
    return X, V


@pytest.mark.parametrize("w", [10, 32])
def test_sym_finalize_rows_is_a_slice_of_the_full_finalize(w):
    """ncgp_kop_sym_finalize_rows on a shard (output, base, noise state and
    raw-product tensors all shards) writes exactly the rows the full finalize
    writes."""
    X, V = _sym_problem(w=w)
    n = X.shape[0]
    op = K.KernelOperator("matern32", 1.3, 1.0, X, w_max=32)
    op.set_sym(1)
    if op.sym_acc_elems(w) == 0:
        pytest.skip("no symmetric kernel for this shape")
    acc = torch.empty(op.sym_acc_elems(w), dtype=torch.int64, device="cuda")
    op.sym_partial(V, 0, 1, acc)
    rng = np.random.default_rng(1)
    base = torch.from_numpy(rng.standard_normal((n, w))).to("cuda", F32)
    logits = torch.from_numpy(rng.standard_normal((n, w))).to("cuda", F32)
    pi = torch.softmax(logits, dim=1).contiguous()
    raw = torch.empty((n, w), dtype=F32, device="cuda")
    full = op.sym_finalize(acc, w, V=V, epi=K.Epi(-1.0, 1.0, base, -1.0, ("softmax", pi), raw))
    plain = op.sym_finalize(acc, w)
    for r0, r1 in [(0, 256), (256, 20_480), (20_480, n)]:
        raw_l = torch.full((r1 - r0, w), float("nan"), dtype=F32, device="cuda")
        out_l = op.sym_finalize(
            acc, w, V=V, row_begin=r0, row_end=r1,
            epi=K.Epi(-1.0, 1.0, base[r0:r1].contiguous(), -1.0,
                      ("softmax", pi[r0:r1].contiguous()), raw_l, row0=r0))
        assert torch.equal(out_l, full[r0:r1])
        assert torch.equal(raw_l, raw[r0:r1])
        assert torch.equal(op.sym_finalize(acc, w, row_begin=r0, row_end=r1), plain[r0:r1])
    with pytest.raises(K.N.DimensionMismatch):
        op.sym_finalize(acc, w, row_begin=256, row_end=n + 1)


@pytest.mark.parametrize("dt,impl", [(F32, "tcgen05"), (F64, "simt")])
def test_row_range_apply_into_a_shard(dt, impl):
    """apply(row_begin, row_end, out_row0) with shard-sized output and
    epilogue tensors equals the same rows of the full fused apply."""
    rng = np.random.default_rng(2)
    n, d, w = 3000, 5, 3
    X = torch.from_numpy(rng.standard_normal((n, d))).to("cuda", dt)
    V = torch.from_numpy(rng.standard_normal((n, w))).to("cuda", dt)
    base = torch.from_numpy(rng.standard_normal((n, w))).to("cuda", dt)
    dvec = torch.from_numpy(rng.uniform(0.5, 2.0, n * w)).to("cuda", dt)
    op = K.KernelOperator("rbf", 1.1, 2.0, X, w_max=32)
    assert op.impl == impl
    op.set_sym(0)
    raw = torch.empty((n, w), dtype=dt, device="cuda")
    full = op.apply(V, epi=K.Epi(1.0, 0.5, base, 1.0, ("diag", dvec), raw))
    for r0, r1 in [(0, 1024), (1024, 2560), (2560, n)]:
        raw_l = torch.empty((r1 - r0, w), dtype=dt, device="cuda")
        out_l = torch.empty((r1 - r0, w), dtype=dt, device="cuda")
        op.apply(V, out=out_l, row_begin=r0, row_end=r1, out_row0=r0,
                 epi=K.Epi(1.0, 0.5, base[r0:r1].contiguous(), 1.0,
                           ("diag", dvec[r0 * w:r1 * w].contiguous()), raw_l, row0=r0))
        assert torch.equal(out_l, full[r0:r1])
        assert torch.equal(raw_l, raw[r0:r1])


# ------------------------------------------------------------------ operator

@pytest.mark.parametrize("gather,world", [("rows", 2), ("rows", 3), ("reduce", 2), ("reduce", 4)])
def test_sharded_state_operator_matches_the_full_product(gather, world):
    rng = np.random.default_rng(3)
    n, d, C = (45_056 + 300, 4, 10) if gather == "reduce" else (2000, 3, 3)
    X = rng.standard_normal((n, d))
    v = torch.from_numpy(rng.standard_normal(n * C)).to("cuda", F32)
    m = torch.from_numpy(rng.standard_normal(n * C)).to("cuda", F32)
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("matern32", 1.3, 1.0),) * C)
    ref_op = P.PriorOperator(prior, X, dtype=F32)
    for kop, _ in ref_op.groups:
        kop.set_sym(1 if gather == "reduce" else 0)
    g_ref = torch.empty_like(v)
    f_ref = ref_op.apply_fused(v, K.Epi(beta=1.0, base=m, out2=g_ref))

    def rank(comm):
        op = PP.ShardedStateOperator(prior, X, comm, dtype=F32, gather=gather)
        for kop, _ in op.inner.groups:
            kop.set_sym(1 if gather == "reduce" else 0)
        v_l, m_l = op.shard(v), op.shard(m)
        g_l = torch.empty_like(v_l)
        f_l = op.apply_fused(v_l, K.Epi(beta=1.0, base=m_l, out2=g_l))
        kv_l = op.apply(v_l)
        return op.r0 * C, op.r1 * C, f_l, g_l, kv_l

    for a, b, f_l, g_l, kv_l in run_ranks(world, rank):
        # integer accumulators (reduce) and row-independent reductions (rows):
        # the shard is bitwise the one-process product
        assert torch.equal(f_l, f_ref[a:b])
        assert torch.equal(g_l, g_ref[a:b])
        assert torch.equal(kv_l, g_ref[a:b])


# ------------------------------------------------------------------ fits

def _gathered(results, key):
    return np.concatenate([r[key] for r in results])


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_fit_cfg1_unit_policy(world):
    """cfg1 (Bernoulli, unit-vector policy, fp64): the unit actions index the
    global vector, so rank r contributes e_j only for its own entries."""
    g = golden("fit_cfg1")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0),))
    ds = P.Dataset(g["X"], g["y"], "binary")
    lik = P.BernoulliLogisticLikelihood(ds.targets)
    oc = P.OuterConfig(max_newton_steps=5, delta=1e-12, inner_schedule=20, recycle=False)

    def rank(comm):
        belief, trace = PP.fit_sharded(prior, ds, lik, oc, P.InnerConfig(max_iters=1),
                                       "unit", comm=comm, dtype=F64)
        mean, var = PP.sharded_posterior(belief, g["X_test"], comm=comm)
        return {"w": belief.weights, "mean": mean, "var": var,
                "iters": [s.inner_iterations for s in trace.steps],
                "mv": trace.total_kernel_matvecs, "rank": belief.root.rank}

    res = run_ranks(world, rank)
    # the global dots are sums of per-rank partials: a different fp64 summation
    # order than one process (which meets the golden at 1e-9), hence 1e-8
    assert rel(_gathered(res, "w"), g["weights"]) < 1e-8
    for r in res:
        assert rel(r["mean"], g["mean"]) < 1e-8
        assert rel(r["var"], g["var"]) < 1e-8
        assert r["iters"] == list(g["steps_iters"])
        assert r["mv"] == int(g["total_matvecs"])


@pytest.mark.parametrize("dt,world", [(F64, 2), (F32, 2)])
def test_sharded_fit_cfg2_small_recycling(dt, world):
    """cfg2 reduction (softmax, residual policy, recycling: the virtual solver
    run's Gram is all-reduced, the eigenproblem solved on every rank)."""
    g = golden("fit_cfg2s")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * 3)
    ds = P.Dataset(g["X"], g["y"], "class-index", 3)
    lik = P.SoftmaxLikelihood(ds.targets, 3)
    oc = P.OuterConfig(max_newton_steps=10, delta=0.01, inner_schedule=20, recycle=True)
    b1, t1 = P.fit(prior, ds, lik, oc, P.InnerConfig(max_iters=1), policy_kind="residual",
                   dtype=dt)
    mean1 = P.posterior_mean(b1, g["X_test"])
    var1 = P.posterior_marginal_var(b1, g["X_test"])

    def rank(comm):
        belief, trace = PP.fit_sharded(prior, ds, lik, oc, P.InnerConfig(max_iters=1),
                                       "residual", comm=comm, dtype=dt)
        mean, var = PP.sharded_posterior(belief, g["X_test"], comm=comm)
        full = PP.gather_belief(belief, comm=comm)
        return {"w": belief.weights, "mean": mean, "var": var, "full_w": full.weights,
                "full_rank": full.root.rank, "full_n": full.train_inputs.shape[0],
                "iters": [s.inner_iterations for s in trace.steps],
                "norms": [s.pseudo_target_norm for s in trace.steps],
                "term": trace.termination}

    res = run_ranks(world, rank)
    # cfg2 amplifies rounding (6.5e-6 on the mean from summation order alone)
    tol = 1e-5 if dt == F64 else 2e-3
    assert rel(_gathered(res, "w"), b1.weights) < tol
    for r in res:
        assert rel(r["mean"], mean1) < tol
        assert rel(r["mean"], g["mean"]) < 1e-3
        # the root of a recycled cfg2 fit moves by ~1e-2 under rounding alone
        # (7.9e-3 in norm, 6e-2 max, from summation order)
        assert rel(r["var"], var1) < 3e-2
        assert rel(r["full_w"], b1.weights) < tol
        assert r["full_rank"] == b1.root.rank and r["full_n"] == ds.n_points
        assert r["term"] == t1.termination
        if dt == F64:
            assert r["iters"] == [s.inner_iterations for s in t1.steps]
            np.testing.assert_allclose(r["norms"], [s.pseudo_target_norm for s in t1.steps],
                                       rtol=1e-5)
    # every rank followed the same control flow
    assert all(r["iters"] == res[0]["iters"] for r in res)


def test_sharded_fit_cfg5_shape_three_ranks():
    """cfg5 at N = 1500 (C = 10, D = 50, compression to rank 256) on 3 ranks,
    fp64: the Newton trajectory of the one-process fit, step for step."""
    from paper_2310_20285_b200 import configs
    c = configs.cfg5(n=1500, n_test=500)
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*c["kernel"]),) * 10)
    ds = P.Dataset(c["X"], c["y"], "class-index", 10)
    lik = P.SoftmaxLikelihood(ds.targets, 10)
    oc = P.OuterConfig(max_newton_steps=4, delta=0.01, inner_schedule=32, recycle=True,
                       compression_rank=64)
    b1, t1 = P.fit(prior, ds, lik, oc, P.InnerConfig(max_iters=1), dtype=F64)
    mean1 = P.posterior_mean(b1, c["X_test"])

    def rank(comm):
        belief, trace = PP.fit_sharded(prior, ds, lik, oc, P.InnerConfig(max_iters=1),
                                       comm=comm, dtype=F64)
        mean, var = PP.sharded_posterior(belief, c["X_test"], comm=comm)
        return {"w": belief.weights, "mean": mean, "shard": trace.shard,
                "steps": [(s.inner_iterations, s.inner_termination) for s in trace.steps],
                "mv": trace.total_kernel_matvecs, "peak": trace.peak_buffer_entries}

    res = run_ranks(3, rank)
    assert [r["shard"] for r in res] == [(0, 512), (512, 1024), (1024, 1500)]
    assert rel(_gathered(res, "w"), b1.weights) < 1e-6
    for r in res:
        assert r["steps"] == [(s.inner_iterations, s.inner_termination) for s in t1.steps]
        assert r["mv"] == t1.total_kernel_matvecs
        assert r["peak"] == t1.peak_buffer_entries
        assert rel(r["mean"], mean1) < 1e-6


def test_world_one_is_the_plain_fit():
    g = golden("fit_cfg2s")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * 3)
    ds = P.Dataset(g["X"], g["y"], "class-index", 3)
    lik = P.SoftmaxLikelihood(ds.targets, 3)
    oc = P.OuterConfig(max_newton_steps=3, delta=0.01, inner_schedule=10, recycle=True)
    b1, _ = P.fit(prior, ds, lik, oc, P.InnerConfig(max_iters=1), dtype=F64)
    comm = PP.ThreadComm.create(1)[0]
    b2, _ = PP.fit_sharded(prior, ds, lik, oc, P.InnerConfig(max_iters=1), comm=comm, dtype=F64)
    np.testing.assert_array_equal(b1.weights, b2.weights)
    # default communicator: the torch.distributed world (not initialised here: one rank)
    b3, t3 = PP.fit_sharded(prior, ds, lik, oc, P.InnerConfig(max_iters=1), dtype=F64)
    np.testing.assert_array_equal(b1.weights, b3.weights)
    assert t3.shard == (0, ds.n_points)
    mean, var = PP.sharded_posterior(b3, g["X_test"])
    np.testing.assert_array_equal(mean, P.posterior_mean(b1, g["X_test"]))
    np.testing.assert_array_equal(var, P.posterior_marginal_var(b1, g["X_test"]))
    assert K.get_reducer() is None and K.get_shard() is None   # the context restored the hook
