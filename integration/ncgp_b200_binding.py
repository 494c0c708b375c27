# ncgp/b200.py -- optional accelerator binding (ctypes) a maintainer would add
# to the reference package; INTEGRATION.md shows this file verbatim and
# tests/test_integration_binding.py runs it against a stand-in package.
import ctypes
import os

import numpy as np
import torch

from . import outer

_lib = ctypes.CDLL(os.environ.get("NCGP_B200_LIB", "libncgp_b200.so"))
vp, i64, i32, f64, sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                         ctypes.c_double, ctypes.c_size_t)
_lib.ncgp_kop_workspace_bytes.restype = sz
_lib.ncgp_kop_workspace_bytes.argtypes = [i32, i32, i64, i64, i32, i32]
_lib.ncgp_kop_create.argtypes = [ctypes.POINTER(vp), i32, i32, f64, f64, i32, vp, i64,
                                 vp, i64, i32, i32, vp, sz, vp]
_lib.ncgp_kop_apply.argtypes = [vp, vp, i64, i32, vp, i64, i64, i64, vp]
_lib.ncgp_kop_destroy.argtypes = [vp]
_lib.ncgp_last_error.restype = ctypes.c_char_p
FAM = {"rbf": 0, "matern32": 1}
_reference_prior_matvec = outer.prior_matvec


def _check(rc):
    if rc:
        raise RuntimeError(_lib.ncgp_last_error().decode())


class DeviceKernel:
    """K(X, X) @ V on the B200 for one KernelSpec (fp32 -> tcgen05 path)."""

    def __init__(self, spec, X, w):
        self.X = torch.as_tensor(X, dtype=torch.float32, device="cuda").contiguous()
        n, d = self.X.shape
        nb = _lib.ncgp_kop_workspace_bytes(0, 0, n, n, d, w)
        self.ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        self.h = vp()
        _check(_lib.ncgp_kop_create(ctypes.byref(self.h), 0, FAM[spec.family],
                                    spec.lengthscale, spec.outputscale, 0,
                                    self.X.data_ptr(), n, self.X.data_ptr(), n, d, w,
                                    self.ws.data_ptr(), nb,
                                    torch.cuda.current_stream().cuda_stream))
        self.n = n

    def __call__(self, V):                       # V: (n, w) float32 cuda tensor
        out = torch.empty_like(V)
        _check(_lib.ncgp_kop_apply(self.h, V.data_ptr(), V.stride(0), V.shape[1],
                                   out.data_ptr(), out.stride(0), 0, self.n,
                                   torch.cuda.current_stream().cuda_stream))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            _lib.ncgp_kop_destroy(self.h)


def accelerated_prior_matvec(prior, X, v, tile=256):
    """Same contract as gp.prior_matvec (CN numpy vector in, numpy out)."""
    C = prior.num_outputs
    assert len(set(prior.kernels)) == 1, "one shared spec (group outputs otherwise)"
    op = DeviceKernel(prior.kernels[0], X, C)
    V = torch.as_tensor(np.asarray(v).reshape(-1, C), dtype=torch.float32, device="cuda")
    return op(V).double().cpu().numpy().ravel()


def enable():
    outer.prior_matvec = accelerated_prior_matvec   # fit / newton_update use this name


def disable():
    outer.prior_matvec = _reference_prior_matvec
