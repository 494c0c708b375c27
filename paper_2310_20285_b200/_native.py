"""ctypes binding of ``libncgp_b200.so`` (the C ABI in include/ncgp_b200.h).

The library is built in-tree by ``csrc/Makefile`` (or ``__graft_entry__.build``).
There is no fallback: if the shared object is missing or no CUDA device is
present, every compute entry point raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .exceptions import DimensionMismatch, InvalidInput, NcgpError

HERE = os.path.dirname(os.path.abspath(__file__))
# NCGP_LIB: an alternative build of the same library (timing A/B of build-time
# variants, tools/sym_ab.py); entry points it lacks stay unbound
LIB_PATH = os.environ.get("NCGP_LIB") or os.path.join(HERE, "libncgp_b200.so")

F32, F64 = 0, 1
RBF, MATERN32 = 0, 1
KOP_AUTO, KOP_TCGEN05, KOP_SIMT = 0, 1, 2


NOISE_NONE, NOISE_SOFTMAX, NOISE_DIAG = 0, 1, 2


class Epilogue(ctypes.Structure):
    """``ncgp_kop_epilogue`` (include/ncgp_b200.h)."""

    _fields_ = [("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("gamma", ctypes.c_double), ("base", ctypes.c_void_p),
                ("ldb", ctypes.c_int64), ("noise", ctypes.c_int),
                ("noise_state", ctypes.c_void_p), ("out2", ctypes.c_void_p),
                ("ld2", ctypes.c_int64)]


class NativeUnavailable(NcgpError, RuntimeError):
    """The CUDA library could not be loaded (not built, or no GPU)."""


class CudaError(NcgpError, RuntimeError):
    """A CUDA call inside the native library failed."""


class Unsupported(NcgpError, NotImplementedError):
    """The native library does not support this shape / dtype."""


_STATUS = {1: DimensionMismatch, 2: InvalidInput, 3: CudaError, 4: Unsupported}

_vp, _i64, _i32, _f64, _sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                              ctypes.c_double, ctypes.c_size_t)

# name -> (restype, argtypes)
_SIGS = {
    "ncgp_last_error": (ctypes.c_char_p, []),
    "ncgp_version": (_i32, []),
    "ncgp_device_info": (_i32, [ctypes.POINTER(_i32)] * 3),
    "ncgp_launch_count": (_i64, []),
    "ncgp_kop_workspace_bytes": (_sz, [_i32, _i32, _i64, _i64, _i32, _i32]),
    "ncgp_kop_create": (_i32, [ctypes.POINTER(_vp), _i32, _i32, _f64, _f64, _i32, _vp, _i64,
                               _vp, _i64, _i32, _i32, _vp, _sz, _vp]),
    "ncgp_kop_apply": (_i32, [_vp, _vp, _i64, _i32, _vp, _i64, _i64, _i64, _vp]),
    "ncgp_kop_apply_multi": (_i32, [_vp, _vp, _i64, _i32, ctypes.POINTER(_vp), _i32, _i64, _i64,
                                    _i64, _vp]),
    "ncgp_kop_apply_ex": (_i32, [_vp, _vp, _i64, _i32, _vp, _i64, _i64, _i64,
                                 ctypes.POINTER(Epilogue), _vp]),
    "ncgp_kop_impl": (_i32, [_vp]),
    "ncgp_kop_set_sym": (_i32, [_vp, _i32]),
    "ncgp_kop_last_variant": (_i32, [_vp]),
    "ncgp_kop_posterior_var": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp, _vp, _i64, _vp]),
    "ncgp_kop_sym_acc_elems": (_i64, [_vp, _i32]),
    "ncgp_kop_sym_partial": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _i64, _vp]),
    "ncgp_kop_sym_finalize": (_i32, [_vp, _vp, _i64, _vp, _i64, _i32, _vp, _i64,
                                     ctypes.POINTER(Epilogue), _vp]),
    "ncgp_kop_sym_finalize_rows": (_i32, [_vp, _vp, _i64, _vp, _i64, _i32, _vp, _i64,
                                          ctypes.POINTER(Epilogue), _i64, _i64, _vp]),
    "ncgp_kop_destroy": (_i32, [_vp]),
    "ncgp_softmax_stats": (_i32, [_i32, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp]),
    "ncgp_softmax_winv": (_i32, [_i32, _vp, _i64, _i32, _vp, _i64, _i32, _vp, _i64, _f64, _f64,
                                 _vp, _i64, _vp]),
    "ncgp_softmax_w": (_i32, [_i32, _vp, _i64, _i32, _vp, _i64, _i32, _vp, _i64, _vp]),
    "ncgp_bernoulli_stats": (_i32, [_i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "ncgp_poisson_stats": (_i32, [_i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]),
    "ncgp_diag_apply": (_i32, [_i32, _vp, _i64, _vp, _i64, _i32, _vp, _i64, _f64, _f64, _vp,
                               _i64, _vp]),
    "ncgp_reduce_workspace_bytes": (_sz, [_i64, _i32]),
    "ncgp_dots": (_i32, [_i32, _i64, _i32, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp, _vp,
                         _sz, _vp]),
    "ncgp_gemv_t": (_i32, [_i32, _vp, _i64, _i32, _vp, _i64, _vp, _vp, _sz, _vp]),
    "ncgp_gemv_n": (_i32, [_i32, _vp, _i64, _i32, _vp, _vp, _f64, _vp, _i64, _vp]),
    "ncgp_lincomb": (_i32, [_i32, _i64, _f64, _vp, _f64, _vp, _f64, _vp, _vp, _vp]),
    "ncgp_gram_workspace_bytes": (_sz, [_i64, _i32, _i32]),
    "ncgp_gram": (_i32, [_i32, _vp, _i64, _i32, _vp, _i64, _i32, _i64, _vp, _i64, _vp, _sz,
                         _vp]),
    "ncgp_rotate": (_i32, [_i32, _vp, _i64, _i32, _vp, _i64, _i32, _vp, _i64, _i64, _vp]),
    "ncgp_marginal_var": (_i32, [_i32, _vp, _i64, _i64, _i32, _i32, _vp, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree library once; raise loudly when it is unusable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing: build it with `make -C "
                f"paper_2310_20285_b200/csrc` or __graft_entry__.build()")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("NCGP_LIB") and not hasattr(lib, name):
                continue
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def call(name: str, *args):
    """Invoke a status-returning entry point, mapping failures to exceptions."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.ncgp_last_error().decode("utf-8", "replace")
        raise _STATUS.get(rc, NcgpError)(f"{name}: {msg}")
    return rc


def query(name: str, *args):
    return getattr(load(), name)(*args)


def launch_count() -> int:
    return int(load().ncgp_launch_count())


def ptr_array(ptrs):
    arr = (_vp * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
