"""Multi-process (world_size 2, gloo, CPU) tests of the row-sharded operator's
host logic: partition, local row-block compute, all-gather assembly.

The local compute is the CPU oracle's row-block product (test-only
injection); on the GPU the same class wraps the fused kernel-matmul.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_20285_b200.parallel import RowShardedOperator, row_partition


def test_row_partition_covers_rows_once():
    for n in (1, 127, 128, 129, 1000, 12345):
        for world in (1, 2, 3, 4, 8):
            seen = np.zeros(n, dtype=int)
            for r in range(world):
                r0, r1, per = row_partition(n, world, r)
                assert per % 256 == 0
                assert r0 % 256 == 0 or r0 == n
                seen[r0:r1] += 1
            assert (seen == 1).all(), (n, world)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, d, w, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ncgp_oracle as O
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n, d))
        V = rng.standard_normal((n, w))
        spec = ("rbf", 1.2, 1.0)

        def local_apply(Vt, out, r0, r1):
            if r1 > r0:
                blk = O.kernel_matmul_rows(spec, X[r0:r1], X, Vt.double().numpy())
                out[r0:r1] = torch.from_numpy(blk).to(out.dtype)

        op = RowShardedOperator(n, local_apply, dtype=torch.float64)
        res = op.apply(torch.from_numpy(V))
        np.save(os.path.join(result_dir, f"r{rank}.npy"), res.numpy())
        # vector operand path
        resv = op.apply(torch.from_numpy(V[:, 0].copy()))
        np.save(os.path.join(result_dir, f"v{rank}.npy"), resv.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [300, 1000])
def test_two_rank_gather_matches_single_process(tmp_path, n):
    from oracle import ncgp_oracle as O
    d, w, world = 3, 4, 2
    mp.spawn(_worker, args=(world, _free_port(), n, d, w, str(tmp_path)), nprocs=world,
             join=True)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, d))
    V = rng.standard_normal((n, w))
    ref = O.kernel_matmul_rows(("rbf", 1.2, 1.0), X, X, V)
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npy")
        # row blocks are computed independently: bitwise identical to one process
        np.testing.assert_array_equal(got, ref)
        gv = np.load(tmp_path / f"v{r}.npy")
        np.testing.assert_array_equal(gv, ref[:, 0])


class _FileSymmetricMemory:
    """CPU stand-in for TorchSymmetricMemory: each rank's gather buffer is a
    shared file mapping that every other rank maps too, so peer stores are
    real cross-process writes; the barrier is a gloo barrier."""

    def __init__(self, root):
        self.root = root

    def alloc(self, shape, dtype, device):
        rank, world = dist.get_rank(), dist.get_world_size()
        numel = int(np.prod(shape))

        def mapped(r):
            path = os.path.join(self.root, f"symm_{shape[1]}_{r}.bin")
            return torch.from_file(path, shared=True, size=numel, dtype=dtype).view(shape)

        own = mapped(rank)
        own.fill_(float("nan"))  # every row must be written by some rank
        dist.barrier()
        peers = [mapped(r) for r in range(world) if r != rank]
        return own, (lambda channel: dist.barrier()), peers


def _fused_worker(rank, world, port, n, d, w, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ncgp_oracle as O
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n, d))
        V = rng.standard_normal((n, w))
        spec = ("rbf", 1.2, 1.0)
        writes = []

        def local_apply(Vt, out, r0, r1, peers=None):
            writes.append((r0, r1, len(peers or ())))
            if r1 > r0:
                blk = torch.from_numpy(
                    O.kernel_matmul_rows(spec, X[r0:r1], X, Vt.double().numpy())).to(out.dtype)
                for dst in [out] + list(peers or ()):
                    dst[r0:r1] = blk

        op = RowShardedOperator(n, local_apply, dtype=torch.float64, gather="fused",
                                symm=_FileSymmetricMemory(result_dir))
        res = op.apply(torch.from_numpy(V))
        np.save(os.path.join(result_dir, f"f{rank}.npy"), res.numpy())
        # a second product reuses the mapped buffers (barrier before the stores)
        res2 = op.apply(torch.from_numpy(2.0 * V))
        np.save(os.path.join(result_dir, f"g{rank}.npy"), res2.numpy())
        r0, r1, _ = row_partition(n, world, rank)
        assert writes == [(r0, r1, world - 1)] * 2, writes
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [300, 1000])
def test_two_rank_fused_peer_stores_match_single_process(tmp_path, n):
    """gather='fused': each rank stores its rows into every rank's buffer; no
    collective moves data, and every rank ends with the full product."""
    from oracle import ncgp_oracle as O
    d, w, world = 3, 4, 2
    mp.spawn(_fused_worker, args=(world, _free_port(), n, d, w, str(tmp_path)), nprocs=world,
             join=True)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, d))
    V = rng.standard_normal((n, w))
    ref = O.kernel_matmul_rows(("rbf", 1.2, 1.0), X, X, V)
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"f{r}.npy"), ref)
        np.testing.assert_array_equal(np.load(tmp_path / f"g{r}.npy"),
                                      O.kernel_matmul_rows(("rbf", 1.2, 1.0), X, X, 2.0 * V))


def test_gather_mode_is_validated():
    with pytest.raises(ValueError):
        RowShardedOperator(10, lambda *a, **k: None, gather="bogus")


def _tri_items(n, b):
    """Upper-triangle block pairs (I <= J) in block-major order, with tile
    counts: the CPU stand-in for the symmetric kernel's work list."""
    nb = (n + b - 1) // b
    return [(i, j) for j in range(nb) for i in range(j + 1)]


def _sym_worker(rank, world, port, n, d, w, b, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ncgp_oracle as O
        from paper_2310_20285_b200.parallel import SymmetricSplitOperator
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n, d))
        V = rng.standard_normal((n, w))
        spec = ("rbf", 1.2, 1.0)
        items = _tri_items(n, b)
        seen = []

        def partial(Vt, part, nparts, acc):
            # slice of equal item count (the GPU slices by tile count)
            lo, hi = len(items) * part // nparts, len(items) * (part + 1) // nparts
            seen.append((part, nparts, lo, hi))
            A = acc.view(n, -1)
            A.zero_()
            Vn = Vt.double().numpy()
            for i, j in items[lo:hi]:
                ri, rj = slice(i * b, min(n, (i + 1) * b)), slice(j * b, min(n, (j + 1) * b))
                Kij = O.kernel_matmul_rows(spec, X[ri], X[rj], np.eye(rj.stop - rj.start))
                A[ri] += torch.from_numpy(Kij @ Vn[rj])
                if i != j:
                    A[rj] += torch.from_numpy(Kij.T @ Vn[ri])

        def finalize(acc, w_, out):
            res = acc.view(n, -1)[:, :w_].clone()
            if out is not None:
                out.copy_(res)
                return out
            return res

        op = SymmetricSplitOperator(n, partial, finalize, lambda w_: n * w_, dtype=torch.float64,
                                    acc_dtype=torch.float64)
        res = op.apply(torch.from_numpy(V))
        np.save(os.path.join(result_dir, f"s{rank}.npy"), res.numpy())
        resv = op.apply(torch.from_numpy(V[:, 0].copy()))
        np.save(os.path.join(result_dir, f"t{rank}.npy"), resv.numpy())
        assert [s[:2] for s in seen] == [(rank, world)] * 2, seen
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,b", [(300, 64), (1000, 128)])
def test_two_rank_symmetric_split_matches_single_process(tmp_path, n, b):
    """gather='reduce': each rank evaluates a slice of the triangular work
    list into an accumulator, a gloo all-reduce sums them, and every rank
    finalises the full product."""
    from oracle import ncgp_oracle as O
    d, w, world = 3, 4, 2
    assert len(_tri_items(n, b)) >= world
    mp.spawn(_sym_worker, args=(world, _free_port(), n, d, w, b, str(tmp_path)), nprocs=world,
             join=True)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, d))
    V = rng.standard_normal((n, w))
    ref = O.kernel_matmul_rows(("rbf", 1.2, 1.0), X, X, V)
    outs = [np.load(tmp_path / f"s{r}.npy") for r in range(world)]
    np.testing.assert_array_equal(outs[0], outs[1])  # every rank holds the same product
    np.testing.assert_allclose(outs[0], ref, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(np.load(tmp_path / "t0.npy"), ref[:, 0], rtol=1e-12, atol=1e-12)


def _epi_worker(rank, world, port, n, d, w, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import ncgp_oracle as O
        from paper_2310_20285_b200.kernels import Epi
        rng = np.random.default_rng(0)
        X = rng.standard_normal((n, d))
        V = rng.standard_normal((n, w))
        base = torch.from_numpy(rng.standard_normal((n, w)))
        dvec = torch.from_numpy(0.1 + rng.random(n * w))
        spec = ("rbf", 1.2, 1.0)
        calls = []

        def local_apply(Vt, out, r0, r1, epi=None):
            # CPU stand-in for K1 + its fused epilogue on rows [r0, r1)
            calls.append((r0, r1, epi is not None))
            if r1 <= r0:
                return
            kv = torch.from_numpy(O.kernel_matmul_rows(spec, X[r0:r1], X, Vt.double().numpy()))
            res = epi.alpha * kv + epi.beta * epi.base[r0:r1] + \
                epi.gamma * epi.noise[1].view(n, w)[r0:r1] * Vt[r0:r1]
            out[r0:r1] = res
            if epi.out2 is not None:
                epi.out2[r0:r1] = kv

        op = RowShardedOperator(n, local_apply, dtype=torch.float64)
        t = torch.empty((n, w), dtype=torch.float64)
        z = op.apply(torch.from_numpy(V),
                     epi=Epi(alpha=-1.0, beta=1.0, base=base, gamma=0.5, noise=("diag", dvec),
                             out2=t))
        np.save(os.path.join(result_dir, f"z{rank}.npy"), z.numpy())
        np.save(os.path.join(result_dir, f"t{rank}.npy"), t.numpy())
        r0, r1, _ = row_partition(n, world, rank)
        assert calls == [(r0, r1, True)], calls
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [300, 1000])
def test_two_rank_fused_epilogue_row_shards(tmp_path, n):
    """Row shards with the fused K^ epilogue (gather='nccl'): each rank runs
    the epilogue on its own rows and the all-gather moves both the epilogue
    output and the raw K V rows (out2), so every rank ends with both."""
    from oracle import ncgp_oracle as O
    d, w, world = 3, 4, 2
    mp.spawn(_epi_worker, args=(world, _free_port(), n, d, w, str(tmp_path)), nprocs=world,
             join=True)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((n, d))
    V = rng.standard_normal((n, w))
    base = rng.standard_normal((n, w))
    dvec = (0.1 + rng.random(n * w)).reshape(n, w)
    kv = O.kernel_matmul_rows(("rbf", 1.2, 1.0), X, X, V)
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"t{r}.npy"), kv)
        np.testing.assert_allclose(np.load(tmp_path / f"z{r}.npy"), -kv + base + 0.5 * dvec * V,
                                   rtol=1e-14, atol=1e-14)
