"""Multi-output GP priors on the device (mirror of ncgp/gp.py).

Public names and semantics follow the reference: ``KernelSpec``
(gp.py:45-63), ``MultiOutputPrior`` (gp.py:116-141), CN layout
(gp.py:4-8, entry n*C + c), ``reorder`` (gp.py:31-42), ``kernel_eval``
(gp.py:66-75), ``prior_matvec`` (gp.py:144-172) and ``cross_covariance``
(gp.py:175-196).  The products run on the B200 through
:class:`PriorOperator`, which groups outputs by unique kernel spec (the
reference's per-tile dedup, gp.py:165-170) and issues one fused
kernel-matmul per group with all of that group's outputs as right-hand
columns.  The ``tile`` argument is accepted for signature compatibility;
the device operator's reduction order does not depend on it.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from .device import nvtx_range, to_host_tensor, is_device, resolve_dtype, to_device, to_host
from .exceptions import DimensionMismatch, InvalidInput
from .kernels import KernelOperator

DOMAIN_TAGS = ("counts", "binary", "class-index", "real")


class Ordering(enum.Enum):
    CN = "cn"  # output index fastest
    NC = "nc"  # point index fastest


def reorder(v, src: Ordering, dst: Ordering, n_points: int, n_outputs: int):
    """CN <-> NC permutation of a length N*C vector (gp.py:31-42)."""
    dev = is_device(v)
    a = v if dev else np.asarray(v)
    if a.shape[0] != n_points * n_outputs:
        raise DimensionMismatch(f"vector length {a.shape[0]} != {n_points} * {n_outputs}")
    if src == dst:
        return a.clone() if dev else a.copy()
    shape = (n_points, n_outputs) if src == Ordering.CN else (n_outputs, n_points)
    if dev:
        return a.reshape(shape).t().contiguous().reshape(-1)
    return a.reshape(shape).T.ravel().copy()


@dataclass(frozen=True)
class KernelSpec:
    """Stationary kernel (gp.py:45-63).

    rbf:      s2 * exp(-d^2 / (2 l^2))
    matern32: s2 * (1 + sqrt(3) d / l) * exp(-sqrt(3) d / l)
    """

    family: str
    lengthscale: float
    outputscale: float

    def __post_init__(self):
        if self.family not in ("rbf", "matern32"):
            raise InvalidInput(f"unknown kernel family {self.family!r}")
        for name in ("lengthscale", "outputscale"):
            val = getattr(self, name)
            if not (val > 0 and np.isfinite(val)):
                raise InvalidInput(f"{name} must be a positive finite real")


@dataclass(frozen=True)
class MultiOutputPrior:
    """Independent constant-mean GPs, one kernel per output (gp.py:116-141)."""

    kernels: Tuple[KernelSpec, ...]
    mean: Tuple[float, ...] = ()

    def __post_init__(self):
        if len(self.kernels) < 1:
            raise InvalidInput("at least one output kernel is required")
        if self.mean and len(self.mean) != len(self.kernels):
            raise DimensionMismatch("one mean constant per output is required")
        if not self.mean:
            object.__setattr__(self, "mean", (0.0,) * len(self.kernels))

    @property
    def num_outputs(self) -> int:
        return len(self.kernels)

    def mean_vector(self, n_points: int) -> np.ndarray:
        """Prior mean at n_points inputs, CN layout."""
        return np.tile(np.asarray(self.mean, dtype=np.float64), n_points)

    def marginal_prior_variance(self) -> np.ndarray:
        return np.array([k.outputscale for k in self.kernels])

    def spec_groups(self) -> List[Tuple[KernelSpec, List[int]]]:
        """Outputs grouped by identical spec, in first-appearance order."""
        groups: Dict[KernelSpec, List[int]] = {}
        for c, spec in enumerate(self.kernels):
            groups.setdefault(spec, []).append(c)
        return list(groups.items())


def _check_inputs(X):
    if isinstance(X, torch.Tensor):
        ok = bool(torch.isfinite(X).all())
    else:
        ok = bool(np.isfinite(np.asarray(X, dtype=np.float64)).all())
    if not ok:
        raise InvalidInput("kernel inputs must be finite")


class PriorOperator:
    """Device K = blockdiag_c K_c(X_rows, X_cols) acting on CN vectors.

    ``apply(v)`` takes a CN vector (n_cols*C,) or an (n_cols, C) matrix and
    returns K v in the same layout over the rows.
    """

    def __init__(self, prior: MultiOutputPrior, X_rows, X_cols=None, dtype=None,
                 impl: str = "auto"):
        self.prior = prior
        self.dtype = resolve_dtype(dtype)
        _check_inputs(X_rows)
        self.X_rows = to_device(X_rows, self.dtype)
        if X_cols is None:
            self.X_cols = self.X_rows
        else:
            _check_inputs(X_cols)
            self.X_cols = to_device(X_cols, self.dtype)
        if self.X_rows.dim() != 2 or self.X_cols.dim() != 2 or \
                self.X_rows.shape[1] != self.X_cols.shape[1]:
            raise DimensionMismatch(
                f"incompatible input shapes {tuple(self.X_rows.shape)} vs "
                f"{tuple(self.X_cols.shape)}")
        self.C = prior.num_outputs
        self.n_rows = self.X_rows.shape[0]
        self.n_cols = self.X_cols.shape[0]
        self.groups = []
        for spec, cols in prior.spec_groups():
            op = KernelOperator(spec.family, spec.lengthscale, spec.outputscale,
                                self.X_rows, None if X_cols is None else self.X_cols,
                                w_max=min(64, len(cols)), impl=impl)
            self.groups.append((op, cols))
        self.matvecs = 0

    @property
    def impl(self) -> str:
        return self.groups[0][0].impl

    @property
    def supports_fused(self) -> bool:
        """One kernel spec for all outputs and the whole CN row in one K1
        block: the Newton-step epilogues fuse into the product."""
        op, cols = self.groups[0]
        return len(self.groups) == 1 and len(cols) == self.C and self.C <= op.w_max

    def apply_fused(self, v: torch.Tensor, epi, out: Optional[torch.Tensor] = None,
                    row_begin: int = 0, row_end: Optional[int] = None) -> torch.Tensor:
        """``epi.alpha K v + epi.beta base + epi.gamma W^-1 v`` in one K1 call
        (``ncgp_kop_apply_ex``), with the raw K v into ``epi.out2`` when set.
        ``base`` / ``out2`` may be CN vectors (viewed as (n_rows, C)).  This is
        the fused K^ = K + W^-1 of SURVEY.md 2.3: the solver residual
        (solver.py:249), z = t + W^-1 s (solver.py:262,265) and the Newton
        update K v + m (outer.py:134-137)."""
        if not self.supports_fused:
            raise DimensionMismatch("fused epilogues need one kernel spec for all outputs")
        C = self.C
        if v.numel() != self.n_cols * C:
            raise DimensionMismatch(f"vector length {v.numel()} != {self.n_cols} * {C}")
        flat = v.dim() == 1
        V = v.reshape(self.n_cols, C)
        if out is None:
            out = torch.empty((self.n_rows, C), dtype=self.dtype, device=V.device)
        rows = lambda t: None if t is None else t.view(-1, C)
        from .kernels import Epi
        e = Epi(epi.alpha, epi.beta, rows(epi.base), epi.gamma, epi.noise, rows(epi.out2))
        with nvtx_range("K product (fused epilogue)"):
            self.groups[0][0].apply(V, out=out.view(self.n_rows, C), row_begin=row_begin,
                                    row_end=row_end, epi=e)
        self.matvecs += 1
        return out.reshape(-1) if flat else out

    def apply(self, v: torch.Tensor, out: Optional[torch.Tensor] = None,
              row_begin: int = 0, row_end: Optional[int] = None,
              peers: Optional[Sequence[torch.Tensor]] = None) -> torch.Tensor:
        """K v over rows [row_begin, row_end).  ``peers``: further (n_rows, C)
        buffers (other ranks' gather buffers mapped into this process) that
        receive the same rows; the K1 epilogue stores into all of them."""
        C = self.C
        flat = v.dim() == 1
        if (v.numel() != self.n_cols * C):
            raise DimensionMismatch(f"vector length {v.numel()} != {self.n_cols} * {C}")
        V = v.reshape(self.n_cols, C)
        if out is None:
            out = torch.empty((self.n_rows, C), dtype=self.dtype, device=V.device)
        O = out.view(self.n_rows, C)
        P = [p.view(self.n_rows, C) for p in peers] if peers else None
        with nvtx_range("K product"):
            self._apply_groups(V, O, C, row_begin, row_end, P)
        self.matvecs += 1
        return out.reshape(-1) if flat else out

    def _apply_groups(self, V, O, C, row_begin, row_end, peers=None):
        r1 = self.n_rows if row_end is None else row_end
        for op, cols in self.groups:
            if len(cols) == C:
                op.apply(V, out=O, row_begin=row_begin, row_end=row_end, peers=peers)
            else:
                idx = torch.tensor(cols, device=V.device)
                sub = op.apply(V.index_select(1, idx).contiguous(),
                               row_begin=row_begin, row_end=row_end)
                for dst in [O] + list(peers or ()):
                    dst[row_begin:r1, cols] = sub[row_begin:r1]

    __call__ = apply


_OP_CACHE: Dict[tuple, PriorOperator] = {}
_OP_CACHE_MAX = 4


def _snapshot(X):
    """An exact copy of the input's contents (host or device)."""
    if isinstance(X, torch.Tensor):
        return X.detach().clone()
    return np.array(X, copy=True)


def _unchanged(snap, X) -> bool:
    """Full-content equality with the snapshot taken when the operator was
    packed: any in-place edit of the input invalidates the cached operator
    (the reference keeps no state, gp.py:144-172, so it can never return a
    product of stale inputs; neither may this cache)."""
    if isinstance(X, torch.Tensor):
        return (isinstance(snap, torch.Tensor) and snap.shape == X.shape and
                snap.dtype == X.dtype and snap.device == X.device and torch.equal(snap, X))
    a = np.asarray(X)
    return isinstance(snap, np.ndarray) and snap.shape == a.shape and snap.dtype == a.dtype \
        and np.array_equal(snap, a)


def clear_operator_cache() -> None:
    """Drop every cached packed operator (and its device workspace)."""
    _OP_CACHE.clear()


def _cached_operator(prior, X, dtype) -> PriorOperator:
    """Reuse the packed operator across calls on the same, unmodified input
    array (packing K1's operands costs about one product's worth of HBM
    traffic).  The entry is validated against a full copy of the inputs on
    every call (memcmp speed on the host, an on-device compare for CUDA
    tensors), so an edit of any single element is noticed."""
    key = (prior, id(X), getattr(X, "shape", None), resolve_dtype(dtype))
    op = _OP_CACHE.get(key)
    if op is not None and op.X_host is X and _unchanged(op.X_snapshot, X):
        return op
    op = PriorOperator(prior, X, dtype=dtype)
    op.X_host = X
    op.X_snapshot = _snapshot(X)
    _OP_CACHE.pop(key, None)
    while len(_OP_CACHE) >= _OP_CACHE_MAX:
        _OP_CACHE.pop(next(iter(_OP_CACHE)))
    _OP_CACHE[key] = op
    return op


def prior_matvec(prior: MultiOutputPrior, X, v, tile: int = 256, dtype=None):
    """K v for a CN vector (gp.py:144-172), computed by the fused device
    kernel-matmul.  Returns the same kind of array it is given (numpy in,
    numpy out; CUDA tensor in, CUDA tensor out)."""
    if tile < 1:
        raise InvalidInput("tile size must be >= 1")
    n = X.shape[0]
    if v.shape[0] != n * prior.num_outputs:
        raise DimensionMismatch(f"vector length {v.shape[0]} != {n} * {prior.num_outputs}")
    dt = resolve_dtype(dtype if dtype is not None else
                       (v.dtype if isinstance(v, torch.Tensor) else None))
    op = _cached_operator(prior, X, dt)
    out = op.apply(to_device(v, dt))
    if is_device(v):
        return out
    if isinstance(v, torch.Tensor):       # host tensor in -> host tensor out
        return to_host_tensor(out)
    return to_host(out)


def kernel_eval(spec: KernelSpec, x, x2) -> float:
    """Kernel on one pair of input vectors (gp.py:66-75), on the device."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    x2 = np.atleast_1d(np.asarray(x2, dtype=np.float64))
    if not (np.isfinite(x).all() and np.isfinite(x2).all()):
        raise InvalidInput("kernel inputs must be finite")
    if x.shape != x2.shape:
        raise DimensionMismatch(f"input shapes differ: {x.shape} vs {x2.shape}")
    op = KernelOperator(spec.family, spec.lengthscale, spec.outputscale,
                        to_device(x[None, :], torch.float64), to_device(x2[None, :], torch.float64),
                        w_max=1)
    one = torch.ones((1, 1), dtype=torch.float64, device=op.X_rows.device)
    return float(op.apply(one)[0, 0].item())


def cross_covariance(prior: MultiOutputPrior, X_train, X_test, dtype=None) -> np.ndarray:
    """Dense (N_test*C) x (N_train*C) cross-covariance (gp.py:175-196).

    Materialised by applying the device operator to identity column blocks;
    intended, like the reference, for small problems only.
    """
    X_train = np.asarray(X_train, dtype=np.float64)
    X_test = np.asarray(X_test, dtype=np.float64)
    if X_train.ndim != 2 or X_test.ndim != 2 or X_train.shape[1] != X_test.shape[1]:
        raise DimensionMismatch(f"incompatible input shapes {X_test.shape} vs {X_train.shape}")
    dt = resolve_dtype(dtype)
    nt, n, C = X_test.shape[0], X_train.shape[0], prior.num_outputs
    out = np.zeros((nt * C, n * C))
    Xr, Xc = to_device(X_test, dt), to_device(X_train, dt)
    for spec, cols in prior.spec_groups():
        op = KernelOperator(spec.family, spec.lengthscale, spec.outputscale, Xr, Xc, w_max=64)
        block = np.empty((nt, n))
        for j0 in range(0, n, 64):
            j1 = min(n, j0 + 64)
            eye = torch.zeros((n, j1 - j0), dtype=dt, device=Xr.device)
            eye[torch.arange(j0, j1), torch.arange(j1 - j0)] = 1.0
            block[:, j0:j1] = to_host(op.apply(eye))
        for c in cols:
            out[c::C, c::C] = block
    return out


@dataclass(frozen=True)
class Dataset:
    """Inputs, targets and a target-domain tag (gp.py:199-241)."""

    inputs: np.ndarray
    targets: np.ndarray
    domain: str
    num_classes: int = 0

    def __post_init__(self):
        X = np.asarray(self.inputs, dtype=np.float64)
        object.__setattr__(self, "inputs", X)
        if X.ndim != 2 or X.shape[0] < 1:
            raise DimensionMismatch("inputs must be a non-empty (N, D) matrix")
        if self.domain not in DOMAIN_TAGS:
            raise InvalidInput(f"unknown domain tag {self.domain!r}")
        if self.domain == "real":
            y = np.asarray(self.targets, dtype=np.float64)
        else:
            raw = np.asarray(self.targets)
            rounded = np.round(np.asarray(raw, dtype=np.float64))
            if not np.allclose(raw, rounded):
                raise InvalidInput(f"{self.domain} targets must be integers")
            y = rounded.astype(np.int64)
        object.__setattr__(self, "targets", y)
        if y.shape != (X.shape[0],):
            raise DimensionMismatch("one target per input row is required")
        if self.domain == "counts" and (y < 0).any():
            raise InvalidInput("counts must be nonnegative")
        if self.domain == "binary" and not np.isin(y, (0, 1)).all():
            raise InvalidInput("binary labels must be in {0, 1}")
        if self.domain == "class-index":
            k = int(self.num_classes) if self.num_classes else int(y.max()) + 1
            object.__setattr__(self, "num_classes", k)
            if (y < 0).any() or (y >= k).any():
                raise InvalidInput(f"class indices must lie in [0, {k})")

    @property
    def n_points(self) -> int:
        return self.inputs.shape[0]

    @property
    def n_features(self) -> int:
        return self.inputs.shape[1]


def _fmt_value(x) -> str:
    """repr of a float (round-trip exact) or an integer (gp.py:244-247)."""
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    return repr(float(x))


def write_dataset_csv(path, dataset: Dataset) -> None:
    """CSV with header x_0..x_{D-1}, y; integer targets except for 'real'
    data (gp.py:250-260)."""
    import csv
    import io
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow([f"x_{d}" for d in range(dataset.n_features)] + ["y"])
    ints = dataset.domain != "real"
    for row, y in zip(dataset.inputs, dataset.targets):
        w.writerow([_fmt_value(x) for x in row] + [str(int(y)) if ints else _fmt_value(y)])
    with open(path, "w", newline="") as fh:
        fh.write(buf.getvalue())


def read_dataset_csv(path, domain: str, num_classes: int = 0) -> Dataset:
    """Read a dataset CSV written by :func:`write_dataset_csv` (gp.py:263-278)."""
    import csv
    with open(path, newline="") as fh:
        rows = list(csv.reader(fh))
    header, body = (rows[0] if rows else []), [r for r in rows[1:] if r]
    if not header or header[-1] != "y":
        raise InvalidInput(f"{path}: expected header ending in 'y'")
    if any(not h.startswith("x_") for h in header[:-1]):
        raise InvalidInput(f"{path}: expected feature columns named x_0..x_{{D-1}}")
    if not body:
        raise InvalidInput(f"{path}: dataset has no rows")
    data = np.array([[float(x) for x in r] for r in body])
    return Dataset(inputs=data[:, :-1], targets=data[:, -1], domain=domain,
                   num_classes=num_classes)


def write_sidecar_json(path, payload: dict) -> None:
    import json
    with open(path, "w") as fh:
        json.dump(payload, fh, indent=2, sort_keys=True)
        fh.write("\n")
