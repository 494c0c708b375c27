"""NCGP v1 belief artifacts: the reference's persisted posterior, read and
written byte for byte (artifact.py:1-92 of the reference package).

Layout, little-endian: the magic ``NCGP``; the format version (u32, 1); six
u64 (N, D, C, rank, newton step, solver iterations); the float64 payloads
X (N, D), weights (N C,) and root columns (N C, rank), each row-major; then
a u64-length-prefixed JSON echo of the fit configuration (keys sorted).

Differences from the reference are in *how*, not *what*: payloads are
streamed to / from the file in row blocks (a cfg5 root is 1e7 x 256 fp64 =
20 GB, which the reference would first assemble in one bytes object), the
device-resident root block (rank, N C) is transposed block by block on its
way to disk, and :func:`load_belief` can hand the root straight to the
device.  The file is written to a temporary name and renamed, like the
reference, so a reader never sees a partial artifact.
"""

from __future__ import annotations

import json
import os
import struct
import tempfile
from typing import Optional, Tuple

import numpy as np

from .device import is_device, to_device
from .exceptions import ArtifactError, ConfigError
from .gp import KernelSpec, MultiOutputPrior
from .linalg import LowRankRoot
from .posterior import PosteriorBelief

MAGIC = b"NCGP"
VERSION = 1
_HEADER = struct.Struct("<4sI6Q")   # magic, version, N, D, C, rank, step, iterations
_ROW_BLOCK = 1 << 16                  # rows of the root streamed per chunk


def _kernel(d: dict) -> KernelSpec:
    try:
        return KernelSpec(d["family"], float(d["lengthscale"]), float(d["outputscale"]))
    except KeyError as e:
        raise ConfigError(f"kernel entry lacks {e}") from None


def build_prior(prior_cfg: dict, num_outputs: int) -> MultiOutputPrior:
    """Prior from the config echo (config.py:227-244 semantics): ``kernels``
    (one per output) or a shared ``kernel``; ``mean`` scalar or per output."""
    if "kernels" in prior_cfg:
        kernels = tuple(_kernel(k) for k in prior_cfg["kernels"])
        if len(kernels) != num_outputs:
            raise ConfigError(f"{len(kernels)} kernels for {num_outputs} outputs")
    elif "kernel" in prior_cfg:
        kernels = (_kernel(prior_cfg["kernel"]),) * num_outputs
    else:
        raise ConfigError("prior needs 'kernel' or 'kernels'")
    mean = prior_cfg.get("mean", 0.0)
    if isinstance(mean, (int, float)):
        mean = (float(mean),) * num_outputs
    else:
        mean = tuple(float(m) for m in mean)
        if len(mean) != num_outputs:
            raise ConfigError(f"{len(mean)} mean entries for {num_outputs} outputs")
    return MultiOutputPrior(kernels=kernels, mean=mean)


def _write_f8(fh, arr: np.ndarray) -> None:
    fh.write(np.ascontiguousarray(arr, dtype="<f8").tobytes())


def _write_root(fh, root: LowRankRoot, dim: int) -> None:
    """Root columns as a row-major (dim, rank) float64 matrix."""
    rank = root.rank
    if rank == 0:
        return
    blk = getattr(root, "_block", None)
    if blk is not None:  # device (rank, dim): transpose one row block at a time
        for i0 in range(0, dim, _ROW_BLOCK):
            i1 = min(dim, i0 + _ROW_BLOCK)
            part = blk[:, i0:i1].t().double().contiguous().cpu().numpy()
            _write_f8(fh, part)
    else:
        _write_f8(fh, root.columns)


def save_belief(path, belief: PosteriorBelief, config_echo: dict) -> None:
    """Write ``belief`` as an NCGP v1 artifact at ``path`` (atomic)."""
    X = belief.train_inputs
    X = X.detach().double().cpu().numpy() if is_device(X) else np.asarray(X, np.float64)
    n, d = X.shape
    c = belief.prior.num_outputs
    rank = belief.root.rank
    blob = json.dumps(config_echo, sort_keys=True).encode("utf-8")
    directory = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=directory, suffix=".tmp")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(_HEADER.pack(MAGIC, VERSION, n, d, c, rank, int(belief.newton_step),
                                  int(belief.solver_iterations)))
            _write_f8(fh, X)
            _write_f8(fh, belief.weights)
            _write_root(fh, belief.root, n * c)
            fh.write(struct.pack("<Q", len(blob)))
            fh.write(blob)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def load_belief(path, device: bool = False, dtype=None) -> Tuple[PosteriorBelief, dict]:
    """Read an NCGP v1 artifact; returns (belief, config echo).

    With ``device=True`` the weights and the root are placed on the GPU in
    ``dtype`` (the root as the (rank, N C) block the posterior kernels use);
    otherwise they are host float64 arrays, as in the reference.
    """
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(_HEADER.size)
        if len(head) < 4 or head[:4] != MAGIC:
            raise ArtifactError(f"{path}: not a belief artifact (bad magic)")
        if len(head) < _HEADER.size:
            raise ArtifactError(f"{path}: truncated header")
        _, version, n, d, c, rank, step, iters = _HEADER.unpack(head)
        if version != VERSION:
            raise ArtifactError(
                f"{path}: artifact format version {version} is not supported by this build "
                f"(expected {VERSION}); re-fit or upgrade the package")
        dim = n * c
        need = _HEADER.size + 8 * (n * d + dim + dim * rank) + 8
        if size < need:
            raise ArtifactError(f"{path}: truncated payload ({size} < {need} bytes)")

        def take(count):
            a = np.fromfile(fh, dtype="<f8", count=count)
            if a.size != count:
                raise ArtifactError(f"{path}: truncated payload")
            return a.astype(np.float64, copy=False)

        X = take(n * d).reshape(n, d)
        weights = take(dim)
        if device and rank:
            block = None
            for i0 in range(0, dim, _ROW_BLOCK):
                i1 = min(dim, i0 + _ROW_BLOCK)
                part = to_device(take((i1 - i0) * rank).reshape(i1 - i0, rank).T, dtype)
                if block is None:
                    block = part.new_empty((rank, dim))
                block[:, i0:i1] = part
            root = LowRankRoot(block=block)
        else:
            root = LowRankRoot(take(dim * rank).reshape(dim, rank))
        (blob_len,) = struct.unpack("<Q", fh.read(8))
        blob = fh.read(blob_len)
        if len(blob) != blob_len:
            raise ArtifactError(f"{path}: truncated configuration echo")
    echo = json.loads(blob.decode("utf-8"))
    prior = build_prior(echo.get("prior", {}), int(c))
    w = to_device(weights, dtype) if device else weights
    belief = PosteriorBelief(prior=prior, train_inputs=X, weights=w, root=root,
                             newton_step=int(step), solver_iterations=int(iters))
    return belief, echo
