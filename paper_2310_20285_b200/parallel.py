"""Row-block sharding of the kernel operator across the GPUs of one node.

SURVEY.md 8(e): output rows of K V are independent.  Each rank keeps the full
inputs X (replicated, <= 200 MB at cfg5), computes a contiguous, 256-aligned
block of output rows with the fused kernel-matmul directly into its slice of
the gather buffer, and the blocks are exchanged so every rank holds the full
product for the next solver step: either by the kernel itself, which stores
each finished row into every rank's symmetric-memory gather buffer over
NVLink (``gather="fused"``), or by an in-place NCCL all-gather after it.
With these operators (``ShardedPriorOperator``) the solver state (v, r, s, z,
d, Q, S, T) is replicated; :func:`fit_sharded` (second half of this module)
row-shards the state as well, as SURVEY.md 8(e) specifies: per-rank memory and
vector work scale as 1 / world, and the exchanges become an all-gather of each
product's operand plus all-reduces of the solver's global sums.

Because the operator plans its column splits on the *full* row count and
flushes its fp32 partial sums at fixed global column boundaries, a row is
reduced in exactly the same order on 1 or P GPUs: the sharded product is
bitwise identical to the single-GPU one.

For K(X, X) the symmetric kernel evaluates each
off-diagonal tile once; a row split would lose that.  :class:`SymmetricSplitOperator`
instead splits the triangular work list itself: every rank evaluates a slice
of equal tile count into an int64 fixed-point accumulator, an all-reduce
sums the accumulators (the exchange step: a reduction, twice the bytes of
the fp32 all-gather it replaces), and every rank writes the full product
from the sum.  Integer sums are exact and associative, so the product is
bitwise identical to the one-GPU product for any number of ranks.

The partition and gather logic takes the local compute as a callable so it
is unit-tested on CPU with the ``gloo`` backend (tests/test_parallel_gloo.py).
"""

from __future__ import annotations

import threading
from typing import Callable, Optional, Tuple

import numpy as np

import torch
import torch.distributed as dist

from .device import nvtx_range

ROW_ALIGN = 256  # the tcgen05 operator's row-tile pair (2 x 128 rows)


def row_partition(n: int, world: int, rank: int, align: int = ROW_ALIGN) -> Tuple[int, int, int]:
    """(row_begin, row_end, rows_per_rank) of ``rank``'s contiguous block.

    Blocks are multiples of ``align`` rows (the last one may be short or
    empty), so every block starts on a row-tile boundary.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    tiles = (n + align - 1) // align
    per = (tiles + world - 1) // world * align
    r0 = min(n, rank * per)
    r1 = min(n, (rank + 1) * per)
    return r0, r1, per


class TorchSymmetricMemory:
    """Peer-mapped gather buffers from ``torch.distributed._symmetric_memory``
    (CUDA, NCCL process group): one buffer per rank, every rank's mapped into
    every process over NVLink, plus a device-side cross-rank barrier."""

    def __init__(self, group=None):
        import torch.distributed._symmetric_memory as symm
        self._symm = symm
        self.group = group if group is not None else dist.group.WORLD

    def alloc(self, shape, dtype, device):
        """(own buffer, barrier(channel), [peer buffers in rank order, self excluded])."""
        buf = self._symm.empty(shape, dtype=dtype, device=device)
        hdl = self._symm.rendezvous(buf, self.group)
        rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
        peers = [hdl.get_buffer(r, shape, dtype) for r in range(world) if r != rank]
        return buf, (lambda channel: hdl.barrier(channel=channel)), peers


class RowShardedOperator:
    """y = K V with rows of K split across ranks, every rank ending with all rows.

    ``local_apply(V, out, row_begin, row_end, peers=None)`` must write rows
    [row_begin, row_end) of K V into ``out`` (an (n_rows, w) tensor) and, when
    ``peers`` is given, into each of those buffers too; in production it is
    :meth:`KernelOperator.apply` / :meth:`PriorOperator.apply`.

    Two exchange paths (``gather``):

    - ``"nccl"`` (default): the rows land in this rank's slice of a gather
      buffer and an in-place ``all_gather_into_tensor`` follows the kernel.
    - ``"fused"``: the gather buffers are symmetric memory (``symm``; by
      default :class:`TorchSymmetricMemory`), and the K1 epilogue stores each
      finished row into every rank's buffer (``ncgp_kop_apply_multi``), so
      the exchange overlaps the kernel instead of following it.  A barrier
      before the kernel (the peers are done reading the previous product) and
      one after it (every row has landed) replace the collective.
    """

    def __init__(self, n_rows: int, local_apply: Callable, group=None,
                 dtype: torch.dtype = torch.float32, device=None, gather: str = "nccl",
                 symm=None):
        if gather not in ("nccl", "fused"):
            raise ValueError(f"gather must be 'nccl' or 'fused', got {gather!r}")
        self.n_rows = n_rows
        self.local_apply = local_apply
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.r0, self.r1, self.per = row_partition(n_rows, self.world, self.rank)
        self.dtype = dtype
        self.device = device
        self.gather = gather
        self._symm_provider = symm
        self._bufs = {}
        self._symm = {}

    def _buffer(self, w: int, device):
        key = (w, str(device))
        full = self._bufs.get(key)
        if full is None:
            full = torch.empty((self.per * self.world, w), dtype=self.dtype, device=device)
            self._bufs[key] = full
        return full

    def symmetric(self, w: int, device):
        """(own gather buffer, barrier, peers' buffers) for RHS width ``w``."""
        key = (w, str(device))
        hit = self._symm.get(key)
        if hit is None:
            if self._symm_provider is None:
                self._symm_provider = TorchSymmetricMemory(self.group)
            hit = self._symm_provider.alloc((self.per * self.world, w), self.dtype, device)
            self._symm[key] = hit
        return hit

    def product(self, V2: torch.Tensor) -> torch.Tensor:
        """All n_rows rows of K V2 as a view of the internal gather buffer
        (valid until the next call)."""
        w = V2.shape[1]
        if self.gather == "fused":
            full, barrier, peers = self.symmetric(w, V2.device)
            barrier(0)   # every peer has consumed the previous product
            self.local_apply(V2, full, self.r0, self.r1, peers=peers)
            barrier(1)   # every rank's rows have landed everywhere
        elif self.world == 1:
            full = self._buffer(w, V2.device)
            self.local_apply(V2, full, 0, self.n_rows)
        else:
            # rank r's rows [r0, r1) are rows [r * per, r * per + (r1 - r0)) of
            # the gather buffer: the operator writes them in place and the
            # gather runs in place (input = this rank's slice of the output)
            full = self._buffer(w, V2.device)
            self.local_apply(V2, full, self.r0, self.r1)
            mine = full[self.rank * self.per:(self.rank + 1) * self.per]
            dist.all_gather_into_tensor(full, mine, group=self.group)
        return full[: self.n_rows]

    def _apply_epi(self, V2: torch.Tensor, out, epi) -> torch.Tensor:
        """Row shards with a fused epilogue (gather='nccl'): each rank runs the
        epilogue on its own rows -- base, noise state and V are replicated --
        and the all-gather moves the epilogue's output (and the raw K V rows
        when ``epi.out2`` is set) instead of K V."""
        from .kernels import Epi
        n, w = self.n_rows, V2.shape[1]
        if self.world == 1:
            dst = out.view(n, w) if out is not None else torch.empty(
                (n, w), dtype=self.dtype, device=V2.device)
            self.local_apply(V2, dst, 0, n, epi=epi)
            return dst
        full = self._buffer(w, V2.device)
        full2 = None
        if epi.out2 is not None:
            key = ("out2", w, str(V2.device))
            full2 = self._bufs.get(key)
            if full2 is None:
                full2 = torch.empty_like(full)
                self._bufs[key] = full2
        e = Epi(epi.alpha, epi.beta, epi.base, epi.gamma, epi.noise, full2)
        self.local_apply(V2, full, self.r0, self.r1, epi=e)
        sl = slice(self.rank * self.per, (self.rank + 1) * self.per)
        dist.all_gather_into_tensor(full, full[sl], group=self.group)
        if full2 is not None:
            dist.all_gather_into_tensor(full2, full2[sl], group=self.group)
            epi.out2.view(n, w).copy_(full2[:n])
        if out is not None:
            out.view(n, w).copy_(full[:n])
            return out.view(n, w)
        return full[:n].clone()

    def apply(self, V: torch.Tensor, out: Optional[torch.Tensor] = None, epi=None) -> torch.Tensor:
        vec = V.dim() == 1
        V2 = V.view(-1, 1) if vec else V
        w = V2.shape[1]
        if epi is not None:
            if self.gather != "nccl":
                raise ValueError("fused epilogues on row shards need gather='nccl'")
            res = self._apply_epi(V2, out, epi)
            return res.view(-1) if vec else res
        if self.world == 1 and self.gather == "nccl":
            dst = out.view(self.n_rows, w) if out is not None else torch.empty(
                (self.n_rows, w), dtype=self.dtype, device=V2.device)
            self.local_apply(V2, dst, 0, self.n_rows)
            res = dst
        else:
            res = self.product(V2)
            if out is not None:
                out.view(self.n_rows, w).copy_(res)
                res = out.view(self.n_rows, w)
            else:
                res = res.clone()
        return res.view(-1) if vec else res

    __call__ = apply


class SymmetricSplitOperator:
    """y = K(X, X) V with the symmetric kernel's triangular work list split
    across the ranks of ``group``; every rank ends with all rows.

    ``partial(V, part, nparts, acc)`` writes part ``part`` of ``nparts`` of the
    product's contributions into ``acc`` (zeroing it first), ``finalize(acc,
    w, out, V=None, epi=None)`` writes the (n_rows, w) product from the summed
    accumulators (through a fused epilogue) and ``acc_elems(w)`` sizes the
    accumulator; in production they are :meth:`KernelOperator.sym_partial` /
    ``sym_finalize`` / ``sym_acc_elems``.
    """

    def __init__(self, n_rows: int, partial: Callable, finalize: Callable, acc_elems: Callable,
                 group=None, dtype: torch.dtype = torch.float32,
                 acc_dtype: torch.dtype = torch.int64):
        self.n_rows = n_rows
        self.partial, self.finalize, self.acc_elems = partial, finalize, acc_elems
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.dtype = dtype
        self.acc_dtype = acc_dtype  # the kernel's accumulators are int64 fixed point
        self._acc = {}

    def accumulator(self, w: int, device) -> torch.Tensor:
        key = (w, str(device))
        acc = self._acc.get(key)
        if acc is None:
            acc = torch.empty(int(self.acc_elems(w)), dtype=self.acc_dtype, device=device)
            self._acc[key] = acc
        return acc

    def apply(self, V: torch.Tensor, out: Optional[torch.Tensor] = None, epi=None) -> torch.Tensor:
        vec = V.dim() == 1
        V2 = V.view(-1, 1) if vec else V
        w = V2.shape[1]
        acc = self.accumulator(w, V2.device)
        self.partial(V2, self.rank, self.world, acc)
        if self.world > 1:
            dist.all_reduce(acc, group=self.group)
        dst = None if out is None else out.view(self.n_rows, w)
        res = self.finalize(acc, w, dst, V=V2, epi=epi) if epi is not None else \
            self.finalize(acc, w, dst)
        return res.view(-1) if vec else res

    __call__ = apply


class ShardedPriorOperator:
    """Drop-in for :class:`gp.PriorOperator` in ``fit(..., operator=...)``:
    the block-diagonal prior product on CN vectors, row-sharded across the
    ranks of ``group``."""

    def __init__(self, prior, X, dtype=None, group=None, gather: str = "auto", symm=None):
        """``gather``: ``"reduce"`` splits the symmetric kernel's work list
        (:class:`SymmetricSplitOperator`), ``"nccl"`` / ``"fused"`` shard rows
        (:class:`RowShardedOperator`), ``"auto"`` takes ``"reduce"`` when the
        operator has a symmetric kernel for the C-wide product (one kernel
        spec for all outputs), else ``"nccl"``."""
        from .gp import PriorOperator
        if gather not in ("auto", "reduce", "nccl", "fused"):
            raise ValueError(f"gather must be auto, reduce, nccl or fused, got {gather!r}")
        self.inner = PriorOperator(prior, X, dtype=dtype)
        self.C = self.inner.C
        self.n_rows = self.inner.n_rows
        self.dtype = self.inner.dtype
        self.matvecs = 0
        C = self.C
        g0 = self.inner.groups[0]
        sym_ok = (len(self.inner.groups) == 1 and len(g0[1]) == C and hasattr(g0[0], "sym_acc_elems")
                  and g0[0].sym_acc_elems(C) > 0)
        if gather == "auto":
            gather = "reduce" if sym_ok else "nccl"
        if gather == "reduce" and not sym_ok:
            raise ValueError("gather='reduce' needs a symmetric kernel for this prior / width")
        self.gather = gather
        if gather == "reduce":
            kop = g0[0]
            self.sharded = SymmetricSplitOperator(self.n_rows, kop.sym_partial, kop.sym_finalize,
                                                  kop.sym_acc_elems, group=group, dtype=self.dtype)
            self._C = C
            return

        def local_apply(V, out, r0, r1, peers=None, epi=None):
            # ``out`` may be the (per * world)-row gather buffer: rows >= n_rows
            # are padding and never written
            n = self.n_rows
            if epi is not None:
                self.inner.apply_fused(V.reshape(-1), epi, out=out[:n].reshape(-1),
                                       row_begin=r0, row_end=r1)
                return
            self.inner.apply(V.reshape(-1), out=out[:n].reshape(-1), row_begin=r0, row_end=r1,
                             peers=[p[:n].reshape(-1) for p in peers] if peers else None)

        self.sharded = RowShardedOperator(self.n_rows, local_apply, group=group,
                                          dtype=self.dtype, gather=gather, symm=symm)
        self.gather = gather
        self._C = C

    @property
    def impl(self):
        return self.inner.impl

    @property
    def supports_fused(self) -> bool:
        """The fused K^ epilogue runs in every rank's finalize (work-list
        split) or on every rank's own rows before the all-gather (row shards
        with gather='nccl'); the peer-store gather keeps the unfused
        composition."""
        return self.gather in ("reduce", "nccl") and self.inner.supports_fused

    def apply(self, v: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        flat = v.dim() == 1
        V = v.reshape(self.n_rows, self._C)
        res = self.sharded.apply(V, out=None if out is None else out.view(self.n_rows, self._C))
        self.matvecs += 1
        return res.reshape(-1) if flat else res

    def apply_fused(self, v: torch.Tensor, epi, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """alpha K v + beta base + gamma W^-1 v (and K v into epi.out2) in one
        product: the epilogue runs in every rank's finalize."""
        if not self.supports_fused:
            raise ValueError("fused epilogues need gather='reduce' or 'nccl'")
        from .kernels import Epi
        flat = v.dim() == 1
        C = self._C
        V = v.reshape(self.n_rows, C)
        rows = lambda t: None if t is None else t.view(-1, C)
        e = Epi(epi.alpha, epi.beta, rows(epi.base), epi.gamma, epi.noise, rows(epi.out2))
        res = self.sharded.apply(V, out=None if out is None else out.view(self.n_rows, C), epi=e)
        self.matvecs += 1
        return res.reshape(-1) if flat else res

    __call__ = apply


# --------------------------------------------------------------------------
# Row-sharded solver state
#
# Every CN vector of the fit (v, r, s, z, d, f, y^, pi) and every column block
# (S, T, Q) is split by the same contiguous, 256-aligned partition of the N
# points.  Elementwise kernels, the W^-1 / W^+ applications, Q y and the
# rotation are then purely local, and the collectives are exactly the
# reference algorithm's global reductions:
#   * all-gather of the next K product's operand (N*C values; 40 MB at cfg5);
#   * all-reduce of the fp64 partials of the fused dots, of Q' z (<= R values)
#     and of the Gram blocks S'(T + W^+ S) (B x B, once per Newton step);
#   * for the symmetric kernels' work-list split, the all-reduce of the int64
#     accumulators (as SymmetricSplitOperator), finalised for the rank's rows.
# The small eigenproblem is solved redundantly on every rank from the same
# (all-reduced) Gram matrix, so U and Lambda agree without a broadcast.
# Per-rank memory and vector work scale as 1 / world.

class TorchDistComm:
    """Collectives of a ``torch.distributed`` group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def all_reduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return t

    def all_gather_(self, full: torch.Tensor, mine: torch.Tensor) -> torch.Tensor:
        """In place: ``mine`` is this rank's equal-sized slice of ``full``."""
        if self.world > 1:
            dist.all_gather_into_tensor(full, mine, group=self.group)
        return full


class ThreadComm:
    """The same collectives between ``world`` Python threads of one process
    sharing one device: N ranks' host logic and kernels exercised on a single
    GPU (tests, per-rank timing).  Ranks meet at a host barrier; no kernel
    waits on another rank's kernel.  Results are summed in rank order, so
    every rank gets the same bits."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.slots = [None] * world
            self.barrier = threading.Barrier(world)

    @classmethod
    def create(cls, world: int):
        shared = cls._Shared(world)
        return [cls(shared, r) for r in range(world)]

    def __init__(self, shared, rank):
        self._s, self.rank, self.world = shared, rank, shared.world

    def _exchange(self, t):
        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()
        self._s.slots[self.rank] = t
        self._s.barrier.wait()
        peers = list(self._s.slots)
        return peers

    def _done(self, t):
        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()
        self._s.barrier.wait()

    def all_reduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return t
        peers = self._exchange(t)
        total = peers[0].clone()
        for p in peers[1:]:
            total += p
        self._done(total)   # every rank has read every slot
        t.copy_(total)
        return t

    def all_gather_(self, full: torch.Tensor, mine: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return full
        peers = self._exchange(mine)
        per = mine.numel()
        parts = [p.reshape(-1).clone() for p in peers]
        self._done(parts[0])
        flat = full.view(-1)
        for r, p in enumerate(parts):
            flat[r * per:(r + 1) * per].copy_(p)
        return full


class sharded_state:
    """Context: the solver's global reductions (kernels.dots / gemv_t / gram,
    the posterior's partial products) are summed over ``comm``'s ranks, and
    the unit-vector policy indexes the global vector."""

    def __init__(self, comm, offset: int, global_dim: int):
        self.comm, self.offset, self.global_dim = comm, offset, global_dim

    def __enter__(self):
        from . import kernels as K
        self._old = (K.get_reducer(), K.get_shard())
        K.set_reducer(self.comm.all_reduce_, (self.offset, self.global_dim))
        return self

    def __exit__(self, *exc):
        from . import kernels as K
        K.set_reducer(*self._old)
        return False


class ShardedStateOperator:
    """K product on a row shard of the solver state: takes this rank's rows of
    the CN operand, returns this rank's rows of K v (or of the fused K^
    epilogue, whose base / noise state / raw-product tensors are shards too).

    The operand is all-gathered (the path's one exchange per product); then
    either the rank's row block of the plain kernel (``gather="rows"``: no
    further communication -- north_star's partition), or its slice of the
    symmetric kernel's work list, an all-reduce of the int64 accumulators
    and a finalize of its own rows (``gather="reduce"``, the default where a
    symmetric kernel exists: half the kernel evaluations).
    """

    def __init__(self, prior, X, comm, dtype=None, gather: str = "auto", inner=None):
        """``inner``: a pre-built replicated operator with :class:`gp.PriorOperator`'s
        interface (``C``, ``n_rows``, ``dtype``, ``groups`` of (kernel operator,
        output columns), ``supports_fused``); by default it is built from
        ``prior`` and the full ``X``.  The CPU tests inject a stand-in."""
        if gather not in ("auto", "reduce", "rows"):
            raise ValueError(f"gather must be auto, reduce or rows, got {gather!r}")
        self.comm = comm
        if inner is None:
            from .gp import PriorOperator
            inner = PriorOperator(prior, X, dtype=dtype)
        self.inner = inner
        self.C, self.n_rows, self.dtype = self.inner.C, self.inner.n_rows, self.inner.dtype
        self.r0, self.r1, self.per = row_partition(self.n_rows, comm.world, comm.rank)
        if self.r1 <= self.r0:
            raise ValueError(f"rank {comm.rank} of {comm.world} holds no rows of {self.n_rows}")
        g0 = self.inner.groups[0]
        sym_ok = (len(self.inner.groups) == 1 and len(g0[1]) == self.C
                  and hasattr(g0[0], "sym_acc_elems") and g0[0].sym_acc_elems(self.C) > 0)
        if gather == "auto":
            gather = "reduce" if sym_ok else "rows"
        if gather == "reduce" and not sym_ok:
            raise ValueError("gather='reduce' needs a symmetric kernel for this prior / width")
        self.gather = gather
        self.matvecs = 0
        self._full = None
        self._acc = None

    @property
    def n_local(self) -> int:
        return self.r1 - self.r0

    @property
    def impl(self):
        return self.inner.impl

    @property
    def supports_fused(self) -> bool:
        return self.inner.supports_fused

    def shard(self, full: torch.Tensor) -> torch.Tensor:
        """This rank's rows of a replicated CN vector / (n, C) matrix."""
        C = self.C
        return full.reshape(self.n_rows, C)[self.r0:self.r1].reshape(
            -1 if full.dim() == 1 else (self.n_local, C)).contiguous()

    def gather_vector(self, v_loc: torch.Tensor) -> torch.Tensor:
        """All ranks' shards of a CN vector as the full (n, C) operand (a view
        of an internal buffer, valid until the next call)."""
        C, per = self.C, self.per
        if self._full is None or self._full.device != v_loc.device:
            self._full = torch.zeros((per * self.comm.world, C), dtype=self.dtype,
                                     device=v_loc.device)
        mine = self._full[self.comm.rank * per:(self.comm.rank + 1) * per]
        mine[:self.n_local].copy_(v_loc.view(self.n_local, C))
        self.comm.all_gather_(self._full, mine)
        return self._full[:self.n_rows]

    def _row_block(self, V, O, e):
        """This rank's rows of K V by the plain kernel, straight into the shard."""
        C, r0, r1 = self.C, self.r0, self.r1
        for kop, cols in self.inner.groups:
            if len(cols) == C:
                kop.apply(V, out=O, row_begin=r0, row_end=r1, epi=e, out_row0=r0)
            else:  # mixed specs: one pass per spec group on its outputs
                idx = torch.tensor(cols, device=V.device)
                sub = kop.apply(V.index_select(1, idx).contiguous(), row_begin=r0,
                                row_end=r1, out_row0=r0)
                O[:, cols] = sub[:self.n_local]

    def _product(self, v_loc, out, epi):
        from .kernels import Epi
        C, r0, r1 = self.C, self.r0, self.r1
        flat = v_loc.dim() == 1
        if v_loc.numel() != self.n_local * C:
            raise ValueError(f"operand shard has {v_loc.numel()} entries, expected "
                             f"{self.n_local} * {C}")
        with nvtx_range("operand all-gather"):
            V = self.gather_vector(v_loc)
        if out is None:
            out = torch.empty((self.n_local, C), dtype=self.dtype, device=V.device)
        O = out.view(self.n_local, C)
        e = None
        if epi is not None:
            rows = lambda t: None if t is None else t.view(self.n_local, C)
            e = Epi(epi.alpha, epi.beta, rows(epi.base), epi.gamma, epi.noise, rows(epi.out2),
                    row0=r0)
        if self.gather == "reduce":
            kop = self.inner.groups[0][0]
            if self._acc is None:
                self._acc = torch.empty(int(kop.sym_acc_elems(C)), dtype=torch.int64,
                                        device=V.device)
            with nvtx_range("K products"):
                kop.sym_partial(V, self.comm.rank, self.comm.world, self._acc)
            with nvtx_range("accumulator all-reduce"):
                self.comm.all_reduce_(self._acc)
            with nvtx_range("K products"):
                kop.sym_finalize(self._acc, C, O, V=V, epi=e, row_begin=r0, row_end=r1)
        else:
            with nvtx_range("K products"):
                self._row_block(V, O, e)
        self.matvecs += 1
        return out.reshape(-1) if flat else out

    def apply(self, v_loc: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        return self._product(v_loc, out, None)

    def apply_fused(self, v_loc: torch.Tensor, epi, out: Optional[torch.Tensor] = None):
        if not self.supports_fused:
            raise ValueError("fused epilogues need one kernel spec for all outputs")
        return self._product(v_loc, out, epi)

    __call__ = apply


def fit_sharded(prior, dataset, likelihood, outer_config, inner_config, policy_kind="residual",
                comm=None, dtype=None, gather: str = "auto", on_step=None, on_inner=None,
                operator=None):
    """:func:`outer.fit` with the solver state row-sharded over ``comm``'s
    ranks (default: the ``torch.distributed`` world).  Every rank passes the
    full dataset and likelihood (replicated inputs);
    it returns this rank's shard of the belief -- ``belief.train_inputs`` are
    its rows of X, ``belief.weights`` / ``belief.root`` its rows of v and Q --
    and the trace (identical on every rank).  ``operator``: a pre-built
    :class:`ShardedStateOperator` (reused across fits, or a test stand-in).  Use :func:`sharded_posterior`
    to predict from the sharded belief, or :func:`gather_belief`."""
    from .gp import Dataset
    from .outer import fit
    comm = comm if comm is not None else TorchDistComm()
    op = operator if operator is not None else \
        ShardedStateOperator(prior, dataset.inputs, comm, dtype=dtype, gather=gather)
    r0, r1, C = op.r0, op.r1, op.C
    idx = np.arange(r0, r1)
    local = Dataset(inputs=dataset.inputs[r0:r1], targets=dataset.targets[r0:r1],
                    domain=dataset.domain, num_classes=dataset.num_classes)
    lik = likelihood.subset(idx)
    with sharded_state(comm, r0 * C, dataset.n_points * C):
        belief, trace = fit(prior, local, lik, outer_config, inner_config, policy_kind,
                            on_step=on_step, on_inner=on_inner, dtype=dtype, operator=op)
    trace.shard = (r0, r1)
    return belief, trace


def sharded_posterior(belief, X_test, comm=None, dtype=None):
    """(mean, marginal variance) at ``X_test`` from a row-sharded belief: every
    rank multiplies its columns of K(X*, X) with its rows of v and Q, the
    partial products are all-reduced, and the squares are taken after the
    sum.  Identical on every rank."""
    from .posterior import posterior_marginal_var, posterior_mean
    comm = comm if comm is not None else TorchDistComm()
    with sharded_state(comm, 0, 0):
        mean = posterior_mean(belief, X_test, dtype=dtype)
        var = posterior_marginal_var(belief, X_test, dtype=dtype)
    return mean, var


def gather_belief(belief, comm=None):
    """The full belief on every rank from its row shards (weights N*C and the
    root R x N*C: 10 GB at cfg5's rank 256 in fp32 -- prefer
    :func:`sharded_posterior` at scale)."""
    from .device import to_device
    from .linalg import LowRankRoot
    from .posterior import PosteriorBelief
    comm = comm if comm is not None else TorchDistComm()
    C = belief.prior.num_outputs
    X_loc = np.asarray(belief.train_inputs)
    dt = belief.dtype
    w = belief.weights_device(dt)
    counts = torch.zeros(comm.world, dtype=torch.int64, device=w.device)
    counts[comm.rank] = X_loc.shape[0]
    comm.all_reduce_(counts)
    counts = [int(c) for c in counts.tolist()]
    per = max(counts)
    dev = w.device

    def gather(block, width):  # (k, n_loc * width) row block -> (k, n * width)
        k = block.shape[0]
        full = torch.zeros((comm.world, k, per * width), dtype=block.dtype, device=dev)
        full[comm.rank, :, :block.shape[1]].copy_(block)
        comm.all_gather_(full, full[comm.rank])
        return torch.cat([full[r, :, :counts[r] * width] for r in range(comm.world)], dim=1)

    weights = gather(w.view(1, -1), C)[0]
    Xd = to_device(X_loc, torch.float64)
    X = gather(Xd.reshape(1, -1), X_loc.shape[1])[0].view(-1, X_loc.shape[1])
    R = belief.root.rank
    root = LowRankRoot(block=gather(belief.root.block(dt), C)) if R else \
        LowRankRoot.zero(weights.numel())
    return PosteriorBelief(prior=belief.prior, train_inputs=X.cpu().numpy(), weights=weights,
                           root=root, newton_step=belief.newton_step,
                           solver_iterations=belief.solver_iterations)
