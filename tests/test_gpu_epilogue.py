"""Fused K^ epilogues of K1 (``ncgp_kop_apply_ex``).

    out = alpha K V + beta base + gamma W^-1 V,   out2 = K V

Each kernel path (CUDA-core fp64, tcgen05 plain kernel with its in-kernel
store and with split-column partials, both symmetric kernels) is checked
against the unfused composition the reference performs (solver.py:249,
262-265; outer.py:134-137): the raw product out2 is bitwise the plain
apply, and out matches the composition within the output dtype's rounding
(1e-6 relative fp32, 1e-13 fp64).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2310_20285_b200 as P  # noqa: E402
from paper_2310_20285_b200 import kernels as K  # noqa: E402
from paper_2310_20285_b200.gp import PriorOperator  # noqa: E402


def _rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm())


CASES = [
    # n, d, C, dtype, sym mode, expected variant
    (2000, 2, 3, torch.float64, -1, "plain"),       # CUDA-core fp64 (split reduce pass)
    (3000, 8, 3, torch.float32, 0, "plain"),        # tcgen05, split-column partials
    (40_000, 8, 10, torch.float32, 0, "plain"),     # tcgen05, in-kernel row store
    (45_000, 8, 10, torch.float32, 1, "symmetric"), # single-CTA symmetric kernel
    (45_000, 50, 10, torch.float32, 1, "symmetric"),  # pair kernel, row tile in TMEM
]


@pytest.mark.parametrize("n,d,C,dt,sym,variant", CASES)
@pytest.mark.parametrize("noise", ["softmax", "diag"])
def test_fused_epilogue_matches_composition(n, d, C, dt, sym, variant, noise):
    rng = np.random.default_rng(n + C)
    X = rng.standard_normal((n, d))
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.5 if d < 20 else 5.0, 2.0),) * C)
    op = PriorOperator(prior, X, dtype=dt)
    kop = op.groups[0][0]
    kop.set_sym(sym)
    v = torch.from_numpy(rng.standard_normal(n * C)).to("cuda", dt)
    base = torch.from_numpy(rng.standard_normal(n * C)).to("cuda", dt)
    if noise == "softmax":
        f = torch.from_numpy(2.0 * rng.standard_normal(n * C)).to("cuda", dt)
        f[:C] = 30.0  # one saturated point
        lik = P.SoftmaxLikelihood(rng.integers(0, C, n), C)
        st = lik.noise_state(f)
    else:
        d_ = torch.from_numpy(0.1 + rng.random(n * C)).to("cuda", dt)
        st = P.likelihoods.NoiseState(lambda V, b, a, bb, o: K.diag_apply(d_, V, b, a, bb, o),
                                      None, None, fused=("diag", d_))
    kv = op.apply(v)
    assert kop.last_variant == variant
    winv = st.apply(v)
    tol = 1e-13 if dt == torch.float64 else 1e-6
    # residual form: r = rhs - K v - W^-1 v
    r = op.apply_fused(v, K.Epi(alpha=-1.0, beta=1.0, base=base, gamma=-1.0, noise=st.fused))
    assert _rel(r, base - kv - winv) < tol
    # action form: z = K s + W^-1 s with t = K s
    t = torch.empty_like(v)
    z = op.apply_fused(v, K.Epi(gamma=1.0, noise=st.fused, out2=t))
    assert torch.equal(t, kv)
    assert _rel(z, kv + winv) < tol
    # Newton form: f = K w + m with g = K w
    m = torch.from_numpy(np.tile(rng.standard_normal(C), n)).to("cuda", dt)
    g = torch.empty_like(v)
    fn = op.apply_fused(v, K.Epi(beta=1.0, base=m, out2=g))
    assert torch.equal(g, kv)
    assert _rel(fn, kv + m) < tol


def test_fused_epilogue_validation():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((500, 2))
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0),) * 3)
    op = PriorOperator(prior, X, dtype=torch.float32)
    v = torch.ones(1500, device="cuda")
    pi = torch.full((500, 3), 1.0 / 3, device="cuda")
    # a noise term needs a square operator
    rect = K.KernelOperator("rbf", 1.0, 1.0, op.X_rows[:256], op.X_rows, w_max=3)
    with pytest.raises(P.DimensionMismatch):
        rect.apply(v.view(500, 3), epi=K.Epi(gamma=1.0, noise=("softmax", pi)))
    # mixed specs cannot fuse
    mixed = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0), P.KernelSpec("rbf", 2.0, 1.0)))
    assert not PriorOperator(mixed, X, dtype=torch.float32).supports_fused
    assert op.supports_fused


def test_fit_fused_and_unfused_agree():
    """The solver's fused path (default) and the unfused composition (an
    operator wrapper without apply_fused) run the same fit.  fp64: equal to
    rounding (no recycling, a well-conditioned schedule).  fp32: K^ carries
    W^+ entries up to 1e12 next to K's O(1), so fp32 CG iterates move by
    percents under any rounding change; the fused fp32 fit must be no further
    from the fp64 fit than the unfused fp32 fit is."""
    from paper_2310_20285_b200 import configs
    c = configs.cfg2(seed=3, n=1200, n_test=10)
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 2.0),) * 3)
    ds = P.Dataset(c["X"], c["y"], "class-index", 3)
    lik = P.SoftmaxLikelihood(ds.targets, 3)
    outer = P.OuterConfig(max_newton_steps=3, delta=1e-6, inner_schedule=12, recycle=False)

    class Unfused:
        def __init__(self, inner):
            self.inner = inner

        def __call__(self, v, out=None):
            return self.inner.apply(v, out=out)

    res = {}
    for dt in (torch.float64, torch.float32):
        op = PriorOperator(prior, c["X"], dtype=dt)
        for name, o in (("fused", op), ("unfused", Unfused(op))):
            res[dt, name] = P.fit(prior, ds, lik, outer, P.InnerConfig(max_iters=1), dtype=dt,
                                  operator=o)
    (b1, t1), (b2, t2) = res[torch.float64, "fused"], res[torch.float64, "unfused"]
    assert [s.inner_iterations for s in t1.steps] == [s.inner_iterations for s in t2.steps]
    assert t1.total_kernel_matvecs == t2.total_kernel_matvecs
    assert np.linalg.norm(b1.weights - b2.weights) / np.linalg.norm(b2.weights) < 1e-9
    f64 = t1.latent.double()
    err = {k: float((res[torch.float32, k][1].latent.double() - f64).norm() / f64.norm())
           for k in ("fused", "unfused")}
    print(err)
    assert err["fused"] <= 1.5 * err["unfused"] + 1e-4, err
