"""Dry run of bench.py's N-GPU code path on ONE GPU: torch.distributed is
replaced by an in-process stand-in for rank 0 of a world of size W (the
all-gather copies this rank's block into every slot, the other collectives
are identities).  It checks the shapes, the partition and the JSON line of
the multi-rank path; it is not a timing of N GPUs.

usage: [FAKE_RANK=r] python tools/fake_dist_bench.py W [bench args...]
(rank r != 0 prints nothing: bench.py prints on rank 0 only; its kernel time
is reported on stderr with NCGP_BENCH_RANK_REPORT=1)
"""
import os
import runpy
import sys

import torch
import torch.distributed as dist

W = int(sys.argv[1])
R = int(os.environ.get("FAKE_RANK", "0"))  # which rank's share this process times
os.environ.update(WORLD_SIZE=str(W), RANK=str(R), LOCAL_RANK="0")


def _gather(out, inp, group=None, **kw):
    per = inp.shape[0]
    for r in range(W):
        if out[r * per:(r + 1) * per].data_ptr() != inp.data_ptr():
            out[r * per:(r + 1) * per].copy_(inp)


dist.init_process_group = lambda *a, **k: None
dist.destroy_process_group = lambda *a, **k: None
dist.is_initialized = lambda: True
dist.get_world_size = lambda group=None: W
dist.get_rank = lambda group=None: R
dist.barrier = lambda *a, **k: None
dist.all_reduce = lambda t, op=None, group=None: t
dist.all_gather_into_tensor = _gather

sys.argv = ["bench.py", "--gpus", str(W)] + sys.argv[2:]
runpy.run_path(os.path.join(os.path.dirname(__file__), "..", "bench.py"), run_name="__main__")
