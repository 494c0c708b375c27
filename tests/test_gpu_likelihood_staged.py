"""The staged likelihood kernels (round 2: 256-point shared-memory tiles,
cp.async sweeps, W+ over all column blocks from one pi tile) and the
4-elements-per-thread elementwise kernels, against the oracle's restatement
of likelihoods.py on ragged sizes (n not a multiple of the tile, a partial
last tile), every C bucket (C <= 4, <= 16, and C = 20 on the per-thread
fallback), column blocks k = 1 and 5, and leading dimensions that break the
16-byte alignment of the vector sweeps (element-wise path)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2310_20285_b200 import kernels as K  # noqa: E402
from oracle import ncgp_oracle as O  # noqa: E402

F32, F64 = torch.float32, torch.float64


def rel(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# fp32: 2e-5 as in test_gpu_solver.test_softmax_kernels (1 - pi cancels for a
# confident point: ~7e-6 relative at n = 1)
@pytest.mark.parametrize("dt,tol", [(F64, 1e-13), (F32, 2e-5)])
@pytest.mark.parametrize("n,C", [(1, 3), (300, 4), (1001, 10), (257, 16), (513, 20)])
def test_softmax_stats_staged(n, C, dt, tol):
    rng = np.random.default_rng(n + C)
    f = rng.standard_normal(n * C) * 3
    y = rng.integers(0, C, n)
    fd = torch.from_numpy(f).to("cuda", dt)
    pi, grad, yhat = K.softmax_stats(fd, torch.from_numpy(y).cuda(), n, C)
    assert rel(pi.cpu().numpy(), O.softmax_probabilities(f, C)) < tol
    assert rel(grad.cpu().numpy(), O.softmax_grad(f, y, C)) < tol
    lik = O.OracleLikelihood("softmax", y, C)
    assert rel(yhat.cpu().numpy(), O.pseudo_targets(lik, f)) < tol * 10


@pytest.mark.parametrize("dt,tol", [(F64, 1e-12), (F32, 1e-5)])
@pytest.mark.parametrize("n,C,k,pad", [(1001, 10, 1, 0), (1001, 10, 5, 0), (777, 3, 5, 1),
                                       (300, 16, 2, 3), (513, 20, 3, 0)])
def test_softmax_winv_and_w_staged(n, C, k, pad, dt, tol):
    """pad > 0: leading dimension n*C + pad (unaligned column blocks)."""
    rng = np.random.default_rng(7 * n + C)
    f = rng.standard_normal(n * C) * 2
    pi = O.softmax_probabilities(f, C)
    ld = n * C + pad
    Vb = rng.standard_normal((k, ld))
    Bb = rng.standard_normal((k, ld))
    pid = torch.from_numpy(pi).to("cuda", dt)
    Vd = torch.from_numpy(Vb).to("cuda", dt)
    Bd = torch.from_numpy(Bb).to("cuda", dt)
    V = Vd[:, :n * C]
    base = Bd[:, :n * C]
    out = K.softmax_winv(pid, n, C, V, base=base, alpha=-0.5, beta=2.0)
    w = K.softmax_w(pid, n, C, V)
    for b in range(k):
        ref = 2.0 * Bb[b, :n * C] - 0.5 * O.softmax_w_inv_matvec(f, Vb[b, :n * C], C)
        assert rel(out[b].cpu().numpy(), ref) < tol, b
        refw = O.softmax_w_matvec(f, Vb[b, :n * C], C)
        assert rel(w[b].cpu().numpy(), refw) < tol, b


@pytest.mark.parametrize("dt,tol", [(F64, 1e-13), (F32, 3e-6)])
@pytest.mark.parametrize("n", [1, 1023, 4097])
def test_elementwise_four_per_thread(n, dt, tol):
    rng = np.random.default_rng(n)
    f = rng.standard_normal(n) * 4
    y = rng.integers(0, 2, n)
    winv, w, grad, yhat = K.bernoulli_stats(torch.from_numpy(f).to("cuda", dt), torch.from_numpy(y).cuda())
    assert rel(w.cpu().numpy(), O.bernoulli_w_diag(f)) < tol
    assert rel(grad.cpu().numpy(), O.bernoulli_grad(f, y)) < tol
    if dt == F64:
        assert rel(winv.cpu().numpy(), O.bernoulli_w_inv_diag(f)) < tol
    d = rng.random(n) + 0.5
    v = rng.standard_normal((3, n))
    base = rng.standard_normal((3, n))
    out = K.diag_apply(torch.from_numpy(d).to("cuda", dt), torch.from_numpy(v).to("cuda", dt),
                       base=torch.from_numpy(base).to("cuda", dt), alpha=1.5, beta=-1.0)
    assert rel(out.cpu().numpy(), 1.5 * d * v - base) < tol
