"""Symmetric K(X, X) kernel (one P tile serves O_I += P V_J and O_J += P^T V_I)
against the CPU oracle and the plain kernel.

Tolerances (north_star): fp32 operator products within 1e-4 relative of
|K||V| per entry; checked here at 1e-5 of the entry scale (measured 1-4e-6)
and against the plain kernel at 2e-5 in norm -- 5e-5 for both with the
blocked kernel (K1-sym2), whose P_lo . Vhi split term runs in E4M3 (measured
0.7-2.3e-5 in norm, 1.8e-5 of the entry scale at worst).

Determinism (hard part 5; the reference pins tile-size
invariance at test_gp.py:106-110): the symmetric kernels accumulate in int64
fixed point, so their products are bitwise identical run to run and for any
split of the work list into parts -- asserted with ``torch.equal`` below.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2310_20285_b200.kernels import KernelOperator  # noqa: E402
from oracle import ncgp_oracle as O  # noqa: E402


class _Env:
    """Creation-time knobs (read by ncgp_kop_create)."""

    def __init__(self, **kw):
        self.kw = {k: v for k, v in kw.items() if v is not None}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kw}
        os.environ.update({k: str(v) for k, v in self.kw.items()})

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _case(n, d, w, spec, seed, cg=None, **env):
    """cg: symmetric kernel flavour the operator's work list is built for
    (1 single-CTA, 2 CTA pairs; None = the default choice)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    V = rng.standard_normal((n, w))
    with _Env(NCGP_SYM_CG=cg, **env):
        op = KernelOperator(spec[0], spec[1], spec[2], torch.from_numpy(X).float().cuda(), w_max=32)
    return X, V, op, torch.from_numpy(V).float().cuda()


# ncgp_kop_last_variant of each flavour (NCGP_SYM_CG): 1 single-CTA K1-sym1,
# 2 CTA pairs, 3 the blocked K1-sym2
CODE = {1: 2, 2: 1, 3: 4}


def _code(x):
    return x if isinstance(x, int) else x.last_variant_code


def ntol(x):
    """Norm tolerance against the plain kernel for the flavour that ran
    (an operator after its symmetric apply, or its variant code)."""
    return 5e-5 if _code(x) == 4 else 2e-5


def etol(x):
    """Entry-scale tolerance (|error| / (K |V|)) for the flavour that ran."""
    return 5e-5 if _code(x) == 4 else 1e-5


def _plain(op, V):
    with op.sym_mode(0):
        out = op.apply(V)
    assert op.last_variant == "plain"
    return out


@pytest.mark.parametrize("n,d,w,spec", [
    (300, 3, 4, ("matern32", 1.0, 1.0)),
    (1000, 2, 1, ("matern32", 1.0, 2.0)),
    (3000, 8, 32, ("matern32", 1.5, 1.0)),
    (5000, 20, 10, ("matern32", 3.0, 1.0)),
    (2561, 8, 7, ("rbf", 1.5, 1.0)),
    (4096, 8, 32, ("rbf", 1.2, 0.7)),
])
@pytest.mark.parametrize("cg", [1, 2, 3])
def test_symmetric_kernel_matches_oracle(n, d, w, spec, cg):
    X, V, op, Vd = _case(n, d, w, spec, n + d, cg)
    with op.sym_mode(1):
        got = op.apply(Vd).double().cpu().numpy()
    assert op.last_variant_code == CODE[cg]
    ref = O.kernel_matmul_rows(spec, X, X, V)
    bound = O.kernel_matmul_rows(spec, X, X, np.abs(V))
    assert np.all(np.abs(got - ref) <= etol(op) * bound), float(np.max(np.abs(got - ref) / bound))


@pytest.mark.parametrize("item", [16, 48, 128])
def test_symmetric_kernel_item_transitions(item):
    """Several work items per CTA (short items force many row-tile and V-block
    switches): the result must not depend on the item length beyond the
    flush boundaries."""
    X, V, op, Vd = _case(20000, 8, 16, ("matern32", 1.5, 1.0), 7)
    plain = _plain(op, Vd).double()
    for cg in (1, 2, 3):
        with _Env(NCGP_SYM=1, NCGP_SYM_ITEM=item, NCGP_SYM2_ITEM=item, NCGP_SYM_CG=cg):
            op2 = KernelOperator("matern32", 1.5, 1.0, op.X_rows, w_max=32)  # table built at creation
        got = op2.apply(Vd).double()
        assert op2.last_variant_code == CODE[cg]
        assert float((got - plain).norm() / plain.norm()) < ntol(op2)


def test_symmetric_kernel_only_on_full_square_launches():
    """Row-range launches (shards) and rectangular operators use the plain
    kernel, bitwise identical to the plain policy."""
    X, V, op, Vd = _case(3000, 8, 8, ("matern32", 1.5, 1.0), 3)
    plain = _plain(op, Vd)
    part = torch.empty_like(plain)
    with op.sym_mode(1):
        for r0, r1 in ((0, 1280), (1280, 3000)):
            op.apply(Vd, out=part, row_begin=r0, row_end=r1)
    rect = KernelOperator("matern32", 1.5, 1.0, op.X_rows[:2000], op.X_rows, w_max=32)
    with rect.sym_mode(1):
        rr = rect.apply(Vd)
    assert torch.equal(part, plain)
    assert torch.equal(rr, _plain(rect, Vd))


@pytest.mark.parametrize("n,w,fam,variant", [
    (3000, 8, "rbf", "plain"),             # small: the triangular list balances poorly
    (3000, 8, "matern32", "plain"),
    (70001, 32, "rbf", "symmetric"),       # single-CTA symmetric kernel (D = 8)
    (70001, 10, "rbf", "symmetric"),
    (70001, 32, "matern32", "symmetric"),
])
def test_symmetric_default_policy(n, w, fam, variant):
    """Default kernel choice (kop_tc.cu sym_enabled) and, for the symmetric
    kernel, agreement with the plain kernel and with fp64 on a row block."""
    X, V, op, Vd = _case(n, 8, w, (fam, 1.5, 1.0), 11)
    got = op.apply(Vd)
    assert op.last_variant == variant
    code = op.last_variant_code
    if variant == "plain":
        assert torch.equal(got, _plain(op, Vd))
        return
    plain = _plain(op, Vd)
    assert float((got.double() - plain.double()).norm() / plain.double().norm()) < ntol(code)
    # fp64 CUDA-core reference on the first and last row blocks (ragged tail)
    op64 = KernelOperator(fam, 1.5, 1.0, op.X_rows.double(), w_max=32, impl="simt")
    Vd64, Va64 = Vd.double(), Vd.double().abs()
    for r0, r1 in ((0, 512), (n - 300, n)):
        ref = torch.zeros((n, w), dtype=torch.float64, device=Vd.device)
        sc = torch.zeros_like(ref)
        op64.apply(Vd64, out=ref, row_begin=r0, row_end=r1)
        op64.apply(Va64, out=sc, row_begin=r0, row_end=r1)
        err = (got[r0:r1].double() - ref[r0:r1]).abs() / sc[r0:r1]
        assert float(err.max()) < etol(code)


@pytest.mark.parametrize("n,d,w,fam,cg", [
    (200_000, 8, 32, "rbf", None),        # cfg3 path (blocked kernel, WP = 32)
    (100_000, 20, 10, "matern32", None),  # cfg4 path (blocked kernel, WP = 16)
    (70_001, 8, 32, "rbf", 1),            # K1-sym1
    (70_001, 50, 10, "rbf", None),        # cfg5 path (pair kernel, row tile in TMEM)
    (70_001, 8, 32, "matern32", 2),       # pair kernel, WP = 32
])
def test_symmetric_bitwise_run_to_run(n, d, w, fam, cg):
    """The default symmetric kernels are bitwise reproducible: integer
    accumulation makes the sum independent of the CTAs' flush order."""
    X, V, op, Vd = _case(n, d, w, (fam, 2.0, 1.0), 23, cg)
    a = op.apply(Vd)
    assert op.last_variant == "symmetric"
    for _ in range(3):
        b = op.apply(Vd)
        assert torch.equal(a, b)
    # and a second operator over the same inputs
    with _Env(NCGP_SYM_CG=cg):
        op2 = KernelOperator(fam, 2.0, 1.0, op.X_rows, w_max=32)
    assert torch.equal(a, op2.apply(Vd))


def test_symmetric_work_list_order_invariant():
    """Block-major (default) and pair-major work lists give the same product
    up to the fp32 flush boundaries."""
    X, V, op, Vd = _case(40000, 8, 10, ("rbf", 1.5, 1.0), 5)
    outs = []
    for order in ("block", "pair"):
        with _Env(NCGP_SYM=1, NCGP_SYM_ORDER=order, NCGP_SYM_CG=2):
            o = KernelOperator("rbf", 1.5, 1.0, op.X_rows, w_max=32)  # table built at creation
        outs.append(o.apply(Vd).double())
        assert o.last_variant == "symmetric"
    assert float((outs[0] - outs[1]).norm() / outs[1].norm()) < 5e-6


@pytest.mark.parametrize("n,d,w,fam,env", [
    (70001, 50, 10, "matern32", {"NCGP_SYM_ATM": 0}),  # one P buffer (D = 50 outgrows two)
    (3000, 8, 8, "rbf", {"NCGP_SYM": 1, "NCGP_SYM_NPB": 1}),  # forced one buffer, small RBF
    (20000, 8, 32, "matern32", {"NCGP_SYM": 1, "NCGP_SYM_NPB": 1}),
])
def test_symmetric_kernel_single_p_buffer(n, d, w, fam, env):
    """One shared P buffer: each epilogue group waits for the other group's
    previous tile (pt_free barriers alternate by tile parity)."""
    X, V, op, Vd = _case(n, d, w, (fam, 3.0, 1.0), 13, cg=2, **env)
    got = op.apply(Vd).double()
    assert op.last_variant_code == 1
    plain = _plain(op, Vd).double()
    assert float((got - plain).norm() / plain.norm()) < ntol(1)


@pytest.mark.parametrize("n,d,w,fam,cg,parts", [
    (45000, 8, 32, "rbf", 1, (1, 2, 3, 8)),
    (45000, 8, 32, "rbf", 3, (1, 2, 3, 8)),
    (50001, 20, 10, "matern32", 3, (2, 7)),
    (70001, 8, 10, "matern32", 2, (1, 2, 5)),
    (70001, 50, 10, "matern32", None, (2, 8)),   # pair kernel, row tile in TMEM
])
def test_symmetric_split_across_parts(n, d, w, fam, cg, parts):
    """ncgp_kop_sym_partial / _finalize (the multi-GPU split of the
    triangular work list, parallel.SymmetricSplitOperator): the parts'
    int64 accumulators sum exactly, so every split gives the one-launch
    product bit for bit (1-GPU == N-GPU)."""
    X, V, op, Vd = _case(n, d, w, (fam, 2.0, 1.0), 17, cg)
    full = op.apply(Vd)
    assert op.last_variant == "symmetric"
    code = op.last_variant_code
    plain = _plain(op, Vd).double()
    assert float((full.double() - plain).norm() / plain.norm()) < ntol(code)
    m = op.sym_acc_elems(w)
    assert m >= n * w
    for P in parts:
        tot = torch.zeros(m, dtype=torch.int64, device="cuda")
        acc = torch.empty(m, dtype=torch.int64, device="cuda")
        for k in range(P):
            op.sym_partial(Vd, k, P, acc)
            tot += acc
        got = op.sym_finalize(tot, w)
        assert torch.equal(got, full), P


def test_symmetric_split_unavailable():
    """No symmetric kernel (small, rectangular or forced off): acc size 0 and
    the split entry points refuse (the caller row-shards instead)."""
    from paper_2310_20285_b200 import _native as N
    X, V, op, Vd = _case(3000, 8, 8, ("rbf", 1.5, 1.0), 3)
    assert op.sym_acc_elems(8) == 0
    with pytest.raises(N.Unsupported):
        op.sym_partial(Vd, 0, 1, torch.empty(3000 * 32, dtype=torch.int64, device="cuda"))
    rect = KernelOperator("rbf", 1.5, 1.0, op.X_rows[:2000], op.X_rows, w_max=32)
    with rect.sym_mode(1), op.sym_mode(1):
        assert rect.sym_acc_elems(8) == 0
        assert op.sym_acc_elems(8) > 0       # forced on for the square operator
        assert op.sym_acc_elems(40) == 0     # wider than w_max
        with pytest.raises(N.DimensionMismatch):  # accumulator too small (C ABI checks the size)
            op.sym_partial(Vd, 0, 1, torch.empty(100, dtype=torch.int64, device="cuda"))


def test_sharded_prior_operator_reduce_single_rank():
    """ShardedPriorOperator(gather='reduce') without a process group (one
    rank): the split path end to end through the public operator, bitwise
    equal to the one-launch product."""
    import paper_2310_20285_b200 as P
    from paper_2310_20285_b200.parallel import ShardedPriorOperator
    rng = np.random.default_rng(2)
    n, C = 45000, 10
    X = rng.standard_normal((n, 8)).astype(np.float32)
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("matern32", 2.0, 1.5),) * C)
    v = torch.from_numpy(rng.standard_normal(n * C)).float().cuda()
    red = ShardedPriorOperator(prior, X, dtype=torch.float32, gather="auto")
    assert red.gather == "reduce"
    rows = ShardedPriorOperator(prior, X, dtype=torch.float32, gather="nccl")
    one = P.PriorOperator(prior, X, dtype=torch.float32)
    a, b = red(v), rows(v)
    assert torch.equal(a, one(v))
    assert float((a.double() - b.double()).norm() / b.double().norm()) < 5e-5  # blocked kernel


@pytest.mark.parametrize("n,d,w,fam", [
    (38401, 1, 1, "rbf"),          # just above the default threshold, D = 1, w = 1
    (38529, 8, 17, "matern32"),    # ragged last tile, WP = 32 with 15 padding columns
    (70000, 24, 16, "rbf"),        # D = 24: pair kernel (sym1 lacks a 3-deep XB ring)
    (70000, 20, 32, "matern32"),   # WP = 32, D = 20: pair kernel
    (39000, 3, 5, "rbf"),
])
def test_symmetric_default_shapes_sweep(n, d, w, fam):
    """Default policy at the edges of the symmetric kernels' ranges: whichever
    flavour runs, it agrees with the plain kernel."""
    X, V, op, Vd = _case(n, d, w, (fam, 1.7, 1.3), n + w)
    got = op.apply(Vd).double()
    assert op.last_variant == "symmetric"
    code = op.last_variant_code
    with op.sym_mode(0):
        plain = op.apply(Vd).double()
        scale = op.apply(Vd.abs()).double()  # K |V|: the entry scale
    assert float((got - plain).norm() / plain.norm()) < ntol(code)
    assert float(((got - plain).abs() / scale).max()) < etol(code)


@pytest.mark.parametrize("n,d,w,fam,item", [
    (70001, 50, 10, "rbf", None),
    (70001, 50, 10, "matern32", None),
    (70001, 40, 3, "rbf", None),
    (3000, 50, 16, "rbf", 16),      # many items per cluster: the row tile is reloaded into TMEM
    (9000, 52, 7, "matern32", 16),  # D = 52: K = 160, 80 TMEM columns (D >= 56 does not fit)
])
def test_symmetric_row_tile_in_tmem(n, d, w, fam, item):
    """Pair kernel with its row tile in TMEM (large D, WP = 16): GEMM1 reads
    A from TMEM, the drain warps load it per item."""
    X, V, op, Vd = _case(n, d, w, (fam, 4.0, 1.0), n + d, cg=2, NCGP_SYM=1, NCGP_SYM_ITEM=item)
    got = op.apply(Vd).double()
    assert op.last_variant_code == 1
    code = 1
    with op.sym_mode(0):
        plain = op.apply(Vd).double()
        scale = op.apply(Vd.abs()).double()
    assert float((got - plain).norm() / plain.norm()) < ntol(code)
    assert float(((got - plain).abs() / scale).max()) < etol(code)


@pytest.mark.parametrize("spec", [("rbf", 1.5, 1.0), ("rbf", 1.5, 1e-12), ("matern32", 2.0, 3e-9)])
def test_symmetric_tiny_column_scale(spec):
    """A right-hand column of magnitude ~1e-30 next to ordinary ones, with a
    tiny outputscale: the per-column power-of-two scaling (2^-(s + e_c)) stays
    exact in fp64 and every column keeps its relative accuracy."""
    rng = np.random.default_rng(5)
    n, w = 45000, 8
    X = rng.standard_normal((n, 8))
    V = rng.standard_normal((n, w))
    V[:, 3] *= 1e-30
    V[:, 5] *= 1e30
    Xd = torch.from_numpy(X).float().cuda()
    op = KernelOperator(*spec, Xd, w_max=32)
    Vd = torch.from_numpy(V).float().cuda()
    with op.sym_mode(1):
        got = op.apply(Vd).double()
    assert op.last_variant == "symmetric"
    tol = ntol(op)
    assert bool(torch.isfinite(got).all())
    plain = _plain(op, Vd).double()
    for c in range(w):
        g, p_ = got[:, c], plain[:, c]
        assert float((g - p_).norm() / p_.norm()) < tol, c
