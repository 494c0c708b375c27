"""Row-sharded solver state on 2 CPU ranks (gloo): the host logic of
``parallel.fit_sharded`` -- operand all-gather, row-block / work-list-split
products finalised for the rank's rows, all-reduced dots / Q' z / Gram, the
redundant eigensolve, the sharded posterior -- against the one-process fit
and the oracle.

The vector and likelihood kernels are the numpy stand-ins of
``tests/fake_native.py`` behind the real ``kernels.py`` wrappers (so the
reducer hook sits where it sits on the GPU); the K1 operator is an
oracle-backed stand-in injected into :class:`ShardedStateOperator`.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

SPEC = ("rbf", 1.0, 2.0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(n, C, seed=0):
    rng = np.random.default_rng(seed)
    y = rng.integers(0, C, n)
    ang = 2 * np.pi * y / C
    X = np.stack([2 * np.cos(ang), 2 * np.sin(ang)], axis=1) + 0.8 * rng.standard_normal((n, 2))
    Xt = 1.5 * rng.standard_normal((64, 2))
    return X, y, Xt


class OracleKop:
    """CPU stand-in for kernels.KernelOperator on K(X, X): the oracle's tile
    body for row ranges, and a block-pair work list for the split."""

    B = 128

    def __init__(self, X):
        from oracle import ncgp_oracle as O
        self.O, self.X, self.n = O, X, X.shape[0]
        nb = (self.n + self.B - 1) // self.B
        self.items = [(i, j) for j in range(nb) for i in range(j + 1)]

    def _epi(self, kv, V, epi, r0, r1):
        if epi is None:
            return kv
        res = epi.alpha * kv
        if epi.base is not None:
            res = res + epi.beta * epi.base
        if epi.noise is not None and epi.gamma != 0.0:
            kind, st = epi.noise   # the rank's shard of the noise state
            Vl = V[r0:r1].double()
            if kind == "diag":
                res = res + epi.gamma * st.view(r1 - r0, -1) * Vl
            else:  # softmax pseudo-inverse P diag(1 / pi) P v per point (likelihoods.py:291-310)
                proj = Vl - Vl.mean(dim=1, keepdim=True)
                scaled = proj / st.view(r1 - r0, -1).clamp_min(1e-12)
                res = res + epi.gamma * (scaled - scaled.mean(dim=1, keepdim=True))
        if epi.out2 is not None:
            epi.out2.copy_(kv)
        return res

    def apply(self, V, out=None, row_begin=0, row_end=None, epi=None, out_row0=0, peers=None):
        r0, r1 = row_begin, self.n if row_end is None else row_end
        assert epi is None or epi.row0 == out_row0 == r0
        kv = torch.from_numpy(self.O.kernel_matmul_rows(SPEC, self.X[r0:r1], self.X,
                                                         V.double().numpy())).to(V.dtype)
        res = self._epi(kv, V, epi, r0, r1)
        if out is None:
            return res
        out[r0 - out_row0:r1 - out_row0] = res
        return out

    def sym_acc_elems(self, w):
        return self.n * w

    def sym_partial(self, V, part, nparts, acc):
        lo, hi = len(self.items) * part // nparts, len(self.items) * (part + 1) // nparts
        A = acc.view(self.n, -1)
        A.zero_()
        Vn, b = V.double().numpy(), self.B
        for i, j in self.items[lo:hi]:
            ri, rj = slice(i * b, min(self.n, (i + 1) * b)), slice(j * b, min(self.n, (j + 1) * b))
            Kij = self.O.kernel_matmul_rows(SPEC, self.X[ri], self.X[rj], np.eye(rj.stop - rj.start))
            A[ri] += torch.from_numpy(np.rint(Kij @ Vn[rj] * 2.0 ** 40)).to(torch.int64)
            if i != j:
                A[rj] += torch.from_numpy(np.rint(Kij.T @ Vn[ri] * 2.0 ** 40)).to(torch.int64)

    def sym_finalize(self, acc, w, out=None, V=None, epi=None, row_begin=0, row_end=None):
        r0, r1 = row_begin, self.n if row_end is None else row_end
        kv = acc.view(self.n, -1)[r0:r1, :w].double() * 2.0 ** -40
        res = self._epi(kv, V, epi, r0, r1)
        out.copy_(res)
        return out


class OracleInner:
    """gp.PriorOperator's interface over one OracleKop (one spec for all outputs)."""

    supports_fused = True

    def __init__(self, X, C):
        self.C, self.n_rows, self.dtype = C, X.shape[0], torch.float64
        self.groups = [(OracleKop(X), list(range(C)))]
        self.impl = "oracle"


def _fit(P, PP, comm, X, y, Xt, C, likelihood, policy, recycle, gather):
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec(*SPEC),) * C)
    if likelihood == "softmax":
        ds = P.Dataset(X, y, "class-index", C)
        lik = P.SoftmaxLikelihood(ds.targets, C)
    else:
        ds = P.Dataset(X, (y > 0).astype(int), "binary")
        lik = P.BernoulliLogisticLikelihood(ds.targets)
    oc = P.OuterConfig(max_newton_steps=3, delta=1e-12, inner_schedule=6, recycle=recycle,
                       compression_rank=8 if recycle else None)
    op = PP.ShardedStateOperator(prior, X, comm, dtype=torch.float64, gather=gather,
                                 inner=OracleInner(X, C))
    belief, trace = PP.fit_sharded(prior, ds, lik, oc, P.InnerConfig(max_iters=1), policy,
                                   comm=comm, dtype=torch.float64, operator=op)
    return op, belief, trace


def _worker(rank, world, port, n, C, likelihood, policy, recycle, gather, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import fake_native
        fake_native.install()
        import paper_2310_20285_b200 as P
        from paper_2310_20285_b200 import parallel as PP
        X, y, Xt = _problem(n, C)
        comm = PP.TorchDistComm()
        assert (comm.rank, comm.world) == (rank, world)
        op, belief, trace = _fit(P, PP, comm, X, y, Xt, C, likelihood, policy, recycle,
                                       gather)
        tag = f"w{world}r{rank}"
        np.savez(os.path.join(result_dir, tag + ".npz"),
                 weights=belief.weights, root=belief.root.columns, shard=np.array([op.r0, op.r1]),
                 iters=np.array([s.inner_iterations for s in trace.steps]),
                 norms=np.array([s.pseudo_target_norm for s in trace.steps]),
                 resid=np.array([s.residual_norm for s in trace.steps]),
                 matvecs=trace.total_kernel_matvecs, peak=trace.peak_buffer_entries,
                 latent=trace.latent.numpy(), op_matvecs=op.matvecs)
    finally:
        if world > 1:
            dist.destroy_process_group()


CASES = [
    # n, C, likelihood, policy, recycle, gather
    (600, 3, "softmax", "residual", True, "rows"),
    (600, 3, "softmax", "residual", True, "reduce"),
    (520, 1, "bernoulli", "unit", False, "rows"),
]


@pytest.mark.parametrize("n,C,likelihood,policy,recycle,gather", CASES)
def test_two_rank_sharded_fit_matches_one_process(tmp_path, n, C, likelihood, policy, recycle,
                                                  gather):
    args = (n, C, likelihood, policy, recycle, gather, str(tmp_path))
    mp.spawn(_worker, args=(1, _free_port()) + args, nprocs=1, join=True)
    mp.spawn(_worker, args=(2, _free_port()) + args, nprocs=2, join=True)
    one = np.load(tmp_path / "w1r0.npz")
    parts = [np.load(tmp_path / f"w2r{r}.npz") for r in range(2)]
    # the partition: 256-aligned contiguous row blocks covering all rows once
    assert [tuple(p["shard"]) for p in parts] == [(0, 512), (512, n)]
    assert tuple(one["shard"]) == (0, n)
    for p in parts:  # identical control flow and trace on every rank
        np.testing.assert_array_equal(p["iters"], one["iters"])
        assert int(p["matvecs"]) == int(one["matvecs"]) == int(p["op_matvecs"])
        assert int(p["peak"]) == int(one["peak"])       # reported for the global state
        np.testing.assert_allclose(p["norms"], one["norms"], rtol=1e-10)
        np.testing.assert_allclose(p["resid"], one["resid"], rtol=1e-6, atol=1e-12)
    np.testing.assert_array_equal(parts[0]["norms"], parts[1]["norms"])
    # the shards concatenate to the one-process state (fp64 partial sums in a
    # different order: rounding-level differences)
    w = np.concatenate([p["weights"] for p in parts])
    np.testing.assert_allclose(w, one["weights"], rtol=1e-7, atol=1e-9)
    f = np.concatenate([p["latent"] for p in parts])
    np.testing.assert_allclose(f, one["latent"], rtol=1e-7, atol=1e-9)
    assert parts[0]["root"].shape[1] == parts[1]["root"].shape[1] == one["root"].shape[1]
    Q = np.concatenate([p["root"] for p in parts], axis=0)
    # columns are defined up to the eigensolver's sign / rotation: compare Q Q'
    np.testing.assert_allclose(Q @ Q.T, one["root"] @ one["root"].T, rtol=1e-5, atol=1e-7)
    if likelihood == "bernoulli":
        # unit actions e_0 .. e_5 all live in rank 0's shard
        assert np.abs(parts[1]["root"]).max() == 0.0


def test_one_process_stand_in_fit_matches_the_oracle(tmp_path):
    """The stand-ins themselves: the world-1 fit through fake_native and the
    oracle-backed operator equals the oracle's fit (so the 2-rank comparison
    above is anchored to the reference's algorithm, not to itself)."""
    from oracle import ncgp_oracle as O
    n, C = 600, 3
    mp.spawn(_worker, args=(1, _free_port(), n, C, "softmax", "residual", True, "rows",
                            str(tmp_path)), nprocs=1, join=True)
    one = np.load(tmp_path / "w1r0.npz")
    X, y, _ = _problem(n, C)
    ref = O.fit([SPEC] * C, X, O.OracleLikelihood("softmax", y, C), 3, 6, recycle=True, rank=8,
                delta=1e-12, policy="residual")
    np.testing.assert_array_equal(one["iters"], [s["iterations"] for s in ref["steps"]])
    assert int(one["matvecs"]) == ref["total_matvecs"]
    np.testing.assert_allclose(one["weights"], ref["weights"], rtol=1e-6, atol=1e-9)
