"""K1 kernel-operator parity on the B200 against the reference's golden
vectors and the CPU oracle.

Tolerances (north_star): fp32 operator products within 1e-4 relative; the
fp64 path within 1e-12 (it replays the reference arithmetic per entry and
differs only in the order of the long j-sum).
"""

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
    # u'Kv = v'Ku
    uKv = float((a.double() * Kb.double()).sum())
    vKu = float((b.double() * Ka.double()).sum())
    assert abs(uKv - vKu) <= 1e-5 * (abs(uKv) + 1.0)


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
