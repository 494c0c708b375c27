"""K1 kernel-operator parity on the B200 against the reference's golden
vectors and the CPU oracle.

Tolerances (north_star): fp32 operator products within 1e-4 relative; the
fp64 path within 1e-12 (it replays the reference arithmetic per entry and
differs only in the order of the long j-sum).
"""

import os

import numpy as np
import pytest

from conftest import golden, specs_from

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2310_20285_b200 as P  # noqa: E402
from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402
from oracle import ncgp_oracle as O  # noqa: E402

SHARED = ["matvec_cfg3_rbf", "matvec_cfg3_matern", "matvec_cfg4", "matvec_cfg5", "matvec_cfg2"]


def scale_bound(spec, X, V):
    """Per-entry magnitude scale |K| |V| used for the elementwise bound."""
    return O.kernel_matmul_rows(spec, X, X, np.abs(V))


def op_for(spec, X, dtype, impl="auto", w=64):
    Xd = torch.from_numpy(np.ascontiguousarray(X)).to("cuda", dtype)
    return KernelOperator(spec[0], spec[1], spec[2], Xd, w_max=w, impl=impl), Xd


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", SHARED)
def test_fp64_operator_matches_reference(name):
    g = golden(name)
    spec = specs_from(g["specs"])[0]
    op, _ = op_for(spec, g["X"], torch.float64)
    assert op.impl == "simt"
    out = op.apply(torch.from_numpy(g["V"]).cuda()).cpu().numpy()
    bound = scale_bound(spec, g["X"], g["V"])
    assert np.all(np.abs(out - g["out"]) <= 1e-12 * bound + 1e-300)
    assert rel(out, g["out"]) < 1e-13


@pytest.mark.parametrize("impl", ["auto", "simt"])
@pytest.mark.parametrize("name", SHARED)
def test_fp32_operator_matches_reference(name, impl):
    g = golden(name)
    spec = specs_from(g["specs"])[0]
    op, _ = op_for(spec, g["X"], torch.float32, impl=impl)
    out = op.apply(torch.from_numpy(g["V"]).float().cuda()).double().cpu().numpy()
    bound = scale_bound(spec, g["X"], g["V"])
    # relative 1e-4 on operator products (north_star), per entry and in norm
    assert rel(out, g["out"]) < 1e-4, rel(out, g["out"])
    assert np.all(np.abs(out - g["out"]) <= 1e-4 * bound)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_prior_matvec_mixed_specs_and_dense(dtype):
    g = golden("matvec_mixed")
    specs = [P.KernelSpec(*s) for s in specs_from(g["specs"])]
    prior = P.MultiOutputPrior(kernels=tuple(specs))
    out = P.prior_matvec(prior, g["X"], g["v"], dtype=dtype)
    tol = 1e-12 if dtype == torch.float64 else 1e-5
    np.testing.assert_allclose(out, g["out"], rtol=0, atol=tol * np.abs(g["out"]).max())
    K = P.cross_covariance(prior, g["X"], g["X"], dtype=dtype)
    np.testing.assert_allclose(K, g["K"], rtol=0, atol=tol)


def test_zero_vector_gives_exact_zero():
    g = golden("matvec_cfg3_rbf")
    for dt in (torch.float32, torch.float64):
        op, _ = op_for(("rbf", 1.5, 1.0), g["X"], dt)
        out = op.apply(torch.zeros((g["X"].shape[0], 32), dtype=dt, device="cuda"))
        assert bool((out == 0).all())


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_row_sharding_is_bitwise_identical(dt):
    """1-vs-P shards: rows computed in separate launches equal the full launch."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((3000, 8))
    V = torch.from_numpy(rng.standard_normal((3000, 16))).to("cuda", dt)
    op, _ = op_for(("rbf", 1.5, 1.0), X, dt)
    full = op.apply(V)
    part = torch.empty_like(full)
    for r0, r1 in ((0, 1280), (1280, 2560), (2560, 3000)):
        op.apply(V, out=part, row_begin=r0, row_end=r1)
    assert torch.equal(full, part)
    again = op.apply(V)
    assert torch.equal(full, again)  # deterministic run to run


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
@pytest.mark.parametrize("n,d,w", [(1, 1, 1), (129, 3, 1), (257, 2, 33), (500, 50, 10),
                                   (1000, 20, 64), (131, 64, 7)])
def test_ragged_shapes_against_oracle(n, d, w, dt):
    rng = np.random.default_rng(n + d + w)
    X = rng.standard_normal((n, d))
    V = rng.standard_normal((n, w))
    for spec in (("rbf", 0.9 * np.sqrt(d), 1.3), ("matern32", 0.7 * np.sqrt(d), 0.8)):
        ref = O.kernel_matmul_rows(spec, X, X, V)
        op, _ = op_for(spec, X, dt)
        out = op.apply(torch.from_numpy(V).to("cuda", dt)).double().cpu().numpy()
        bound = O.kernel_matmul_rows(spec, X, X, np.abs(V))
        tol = 1e-12 if dt == torch.float64 else 1e-4
        assert np.all(np.abs(out - ref) <= tol * bound + 1e-30)


def test_cross_operator_rectangular():
    rng = np.random.default_rng(11)
    Xtr = rng.standard_normal((700, 5))
    Xte = rng.standard_normal((333, 5))
    V = rng.standard_normal((700, 12))
    spec = ("matern32", 2.0, 1.7)
    ref = O.kernel_matmul_rows(spec, Xte, Xtr, V)
    for dt, tol in ((torch.float64, 1e-12), (torch.float32, 1e-4)):
        op = KernelOperator(spec[0], spec[1], spec[2],
                            torch.from_numpy(Xte).to("cuda", dt),
                            torch.from_numpy(Xtr).to("cuda", dt), w_max=12)
        out = op.apply(torch.from_numpy(V).to("cuda", dt)).double().cpu().numpy()
        assert rel(out, ref) < tol


def test_linearity_and_symmetry_fp32():
    rng = np.random.default_rng(5)
    X = rng.standard_normal((4096, 8))
    op, _ = op_for(("rbf", 1.5, 1.0), X, torch.float32)
    a = torch.from_numpy(rng.standard_normal((4096, 1))).float().cuda()
    b = torch.from_numpy(rng.standard_normal((4096, 1))).float().cuda()
    Ka, Kb = op.apply(a), op.apply(b)
    Kab = op.apply(2.0 * a - 3.0 * b)
    assert float((Kab - (2 * Ka - 3 * Kb)).norm() / Kab.norm()) < 1e-5
    # u'Kv = v'Ku, up to the operator's per-entry error (<= 1e-6 of |K||v|,
    # measured 6e-7: tools/sym_check.py), summed against |u|: the bound is
    # 1e-6 |u|'K|v|.  uKv itself cancels heavily (|uKv| ~ 1e-3 |u|'K|v|).
    uKv = float((a.double() * Kb.double()).sum())
    vKu = float((b.double() * Ka.double()).sum())
    scale = float((a.abs().double() * op.apply(b.abs()).double()).sum())
    assert abs(uKv - vKu) <= 1e-6 * scale, (uKv, vKu, scale)


def test_errors_are_mapped():
    g = golden("matvec_mixed")
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0),) * 3)
    with pytest.raises(P.DimensionMismatch):
        P.prior_matvec(prior, g["X"], np.zeros(10))
    bad = g["X"].copy()
    bad[0, 0] = np.inf
    with pytest.raises(P.InvalidInput):
        P.prior_matvec(prior, bad, np.zeros(75))
    with pytest.raises(P.InvalidInput):
        P.prior_matvec(prior, g["X"], np.zeros(75), tile=0)


@pytest.mark.slow
@pytest.mark.parametrize("family", ["rbf", "matern32"])
def test_cfg3_full_size_row_sampled(family):
    """cfg3 shape (N=1e6, D=8, w=32) against the oracle on sampled rows."""
    from paper_2310_20285_b200 import configs
    c = configs.cfg3(family=family)
    X, S = c["X"], c["S"]
    spec = c["kernel"]
    op, _ = op_for(spec, X, torch.float32, w=32)
    out = op.apply(torch.from_numpy(S).float().cuda())
    rows = np.array([0, 1, 4097, 500_000, 999_999])
    got = out[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    ref = O.kernel_matmul_rows(spec, X[rows], X, S, tile=8)
    bound = O.kernel_matmul_rows(spec, X[rows], X, np.abs(S), tile=8)
    assert np.all(np.abs(got - ref) <= 1e-4 * bound)
    assert rel(got, ref) < 1e-4


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["cfg4", "cfg5"])
def test_fit_shape_full_size_row_sampled(cfg):
    """The operator a cfg4 / cfg5 fit applies (N=1e5, D=20, Matern / N=1e6,
    D=50, RBF; w = C = 10), at full size, against the oracle on sampled rows."""
    from paper_2310_20285_b200 import configs
    c = configs.CONFIGS[cfg](n_test=10)
    X = c["X"]
    n = X.shape[0]
    V = np.random.default_rng(5).standard_normal((n, c["C"]))
    spec = c["kernel"]
    op, _ = op_for(spec, X, torch.float32, w=c["C"])
    assert op.impl == "tcgen05"
    out = op.apply(torch.from_numpy(V).float().cuda())
    rows = np.array([0, 7, n // 3, n // 2 + 1, n - 1])
    got = out[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    ref = O.kernel_matmul_rows(spec, X[rows], X, V, tile=8)
    bound = O.kernel_matmul_rows(spec, X[rows], X, np.abs(V), tile=8)
    assert np.all(np.abs(got - ref) <= 1e-4 * bound)
    assert rel(got, ref) < 1e-4


def test_precision_guard_auto_falls_back_on_gpu():
    """Inputs spread beyond the tcgen05 split's precision range (scaled
    |x~|^2 > 256): AUTO switches to the CUDA-core operator (on the GPU, same
    results); an explicit tcgen05 request is refused."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((600, 4))
    X[0] *= 60.0  # one far point: (60 * 2)^2 / (2 l^2) >> 256 in log2 units
    V = rng.standard_normal((600, 5))
    spec = ("rbf", 1.0, 1.0)
    op, _ = op_for(spec, X, torch.float32, w=8)
    assert op.impl == "simt"
    out = op.apply(torch.from_numpy(V).float().cuda()).double().cpu().numpy()
    ref = O.kernel_matmul_rows(spec, X, X, V)
    assert rel(out, ref) < 1e-4
    with pytest.raises(P.NcgpError):
        op_for(spec, X, torch.float32, impl="tcgen05", w=8)


def test_prior_matvec_cache_sees_in_place_updates():
    """prior_matvec caches the packed operator per input array; an in-place
    update of that array must not return products of the stale inputs."""
    rng = np.random.default_rng(11)
    X = rng.standard_normal((300, 3))
    v = rng.standard_normal(300 * 2)
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0),) * 2)
    a = P.prior_matvec(prior, X, v, dtype=torch.float64)
    X *= 1.5  # same object, new contents
    b = P.prior_matvec(prior, X, v, dtype=torch.float64)
    ref = O.prior_matvec([("rbf", 1.0, 1.0)] * 2, X, v)
    assert rel(b, ref) < 1e-12 and rel(a, ref) > 1e-3


@pytest.mark.parametrize("impl", ["tcgen05", "simt"])
@pytest.mark.parametrize("n,w", [(3000, 16), (40_000, 40)])
def test_multi_destination_store_is_the_fused_gather(impl, n, w, monkeypatch):
    """ncgp_kop_apply_multi (the all-gather fused into K1's store): every
    destination receives bitwise the rows a plain apply writes, each shard
    only its own rows.  n=3000 takes the split-partial reduction path, n=40k
    the in-kernel store; w=40 loops two RHS column blocks.  (Full-range
    applies of K(X, X) may take the symmetric kernel, whose fp32 reductions
    are not bitwise comparable, so the plain kernel is pinned.)"""
    monkeypatch.setenv("NCGP_SYM", "0")
    rng = np.random.default_rng(5)
    X = rng.standard_normal((n, 8))
    V = torch.from_numpy(rng.standard_normal((n, w))).to("cuda", torch.float32)
    op, _ = op_for(("rbf", 1.5, 1.0), X, torch.float32, impl=impl, w=32)
    assert op.impl == impl
    ref = op.apply(V)
    bufs = [torch.full_like(ref, float("nan")) for _ in range(3)]
    cuts = [0, (n // 3) // 256 * 256, (2 * n // 3) // 256 * 256, n]
    for r0, r1 in zip(cuts[:-1], cuts[1:]):  # three "ranks", each storing to all buffers
        op.apply(V, out=bufs[0], row_begin=r0, row_end=r1, peers=bufs[1:])
    for b in bufs:
        assert torch.equal(b, ref)
    # one shard alone touches only its rows in every destination
    fresh = [torch.full_like(ref, float("nan")) for _ in range(2)]
    op.apply(V, out=fresh[0], row_begin=cuts[1], row_end=cuts[2], peers=fresh[1:])
    for b in fresh:
        assert torch.equal(b[cuts[1]:cuts[2]], ref[cuts[1]:cuts[2]])
        assert bool(torch.isnan(b[:cuts[1]]).all()) and bool(torch.isnan(b[cuts[2]:]).all())


def test_multi_destination_store_validates_peers():
    X = np.random.default_rng(0).standard_normal((300, 4))
    op, _ = op_for(("rbf", 1.0, 1.0), X, torch.float32)
    V = torch.ones((300, 4), device="cuda")
    out = torch.empty((300, 4), device="cuda")
    with pytest.raises(P.DimensionMismatch):
        op.apply(V, out=out, peers=[torch.empty((300, 5), device="cuda")])
    with pytest.raises(P.InvalidInput):
        op.apply(V, out=out, peers=[torch.empty_like(out) for _ in range(8)])  # 9 > 8 outputs


def test_prior_operator_peers_with_per_class_specs():
    """Mixed per-class specs go through the index_select path; peers still
    receive exactly the shard's rows."""
    g = golden("matvec_mixed")
    specs = [P.KernelSpec(*s) for s in specs_from(g["specs"])]
    prior = P.MultiOutputPrior(kernels=tuple(specs))
    from paper_2310_20285_b200.gp import PriorOperator
    op = PriorOperator(prior, g["X"], dtype=torch.float32)
    v = torch.from_numpy(g["v"]).float().cuda()
    ref = op.apply(v)
    n = op.n_rows
    out = torch.full_like(ref, float("nan"))
    peer = torch.full_like(ref, float("nan"))
    r1 = min(n, 256)
    op.apply(v, out=out, row_begin=0, row_end=r1, peers=[peer])
    op.apply(v, out=out, row_begin=r1, row_end=n, peers=[peer])
    assert torch.equal(out, ref) and torch.equal(peer, ref)


def test_fused_gather_symmetric_memory_single_rank(tmp_path):
    """torchrun world=1, NCCL: ShardedPriorOperator(gather='fused') goes
    through torch symmetric memory (rendezvous, peer mapping, device
    barriers) and matches the unsharded product bitwise; gather='reduce'
    (the symmetric kernel's split with an NCCL all-reduce) within 5e-5 (blocked kernel)."""
    import subprocess
    import sys
    script = tmp_path / "symm_run.py"
    script.write_text(
        "import os, sys, numpy as np, torch, torch.distributed as dist\n"
        f"sys.path.insert(0, {repr(str(__import__('pathlib').Path(__file__).resolve().parents[1]))})\n"
        "import paper_2310_20285_b200 as P\n"
        "from paper_2310_20285_b200.parallel import ShardedPriorOperator\n"
        "torch.cuda.set_device(0)\n"
        "dist.init_process_group('nccl')\n"
        "rng = np.random.default_rng(1)\n"
        "X = rng.standard_normal((5000, 8)).astype(np.float32)\n"
        "prior = P.MultiOutputPrior(kernels=(P.KernelSpec('rbf', 1.5, 1.0),) * 3)\n"
        "v = torch.from_numpy(rng.standard_normal(5000 * 3)).float().cuda()\n"
        "a = ShardedPriorOperator(prior, X, dtype=torch.float32, gather='fused')\n"
        "b = ShardedPriorOperator(prior, X, dtype=torch.float32, gather='nccl')\n"
        "ra = a(v); ra2 = a(2 * v); rb = b(v)\n"
        "torch.cuda.synchronize()\n"
        "assert torch.equal(ra, rb), float((ra - rb).abs().max())\n"
        "assert torch.equal(ra2, b(2 * v))\n"
        "os.environ['NCGP_SYM'] = '1'  # the symmetric kernel at this small n\n"
        "c = ShardedPriorOperator(prior, X, dtype=torch.float32, gather='reduce')\n"
        "rc = c(v)\n"
        "assert float((rc - rb).norm() / rb.norm()) < 5e-5\n"
        "dist.destroy_process_group()\n"
        "print('SYMM_OK')\n")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
                        "--master-port", "29631", str(script)],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0 and "SYMM_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("device_input", [False, True])
def test_prior_matvec_cache_sees_single_element_edit(device_input):
    """an in-place edit of ONE element of a large input
    (X[1, 0] at N = 1e5, which a strided content sample would miss) must
    invalidate prior_matvec's packed-operator cache."""
    rng = np.random.default_rng(12)
    n = 100_000
    X = rng.standard_normal((n, 8))
    v = rng.standard_normal(n)
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.5, 1.0),))
    Xin = torch.from_numpy(X).cuda() if device_input else X
    vin = torch.from_numpy(v).cuda() if device_input else v
    a = P.prior_matvec(prior, Xin, vin, dtype=torch.float64)
    if device_input:
        Xin[1, 0] += 0.75
        X = Xin.cpu().numpy()
    else:
        X[1, 0] += 0.75
    b = P.prior_matvec(prior, Xin, vin, dtype=torch.float64)
    a = a.cpu().numpy() if device_input else a
    b = b.cpu().numpy() if device_input else b
    rows = np.array([0, 1, 2, 77_777])
    ref = O.kernel_matmul_rows(("rbf", 1.5, 1.0), X[rows], X, v[:, None])[:, 0]
    scale = O.kernel_matmul_rows(("rbf", 1.5, 1.0), X[rows], X, np.abs(v)[:, None])[:, 0]
    assert np.all(np.abs(b[rows] - ref) <= 1e-12 * scale)
    assert abs(a[1] - ref[1]) > 1e-6 * scale[1]   # the stale product really differed
