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
