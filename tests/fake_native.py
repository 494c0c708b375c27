"""CPU stand-in for libncgp_b200.so's vector / likelihood entry points.

Test infrastructure only (like ``oracle/``): it lets the *host logic* above
the C ABI -- the solver, the Newton loop, the row-sharded state's collective
placement in ``kernels.py`` / ``parallel.py`` -- run on CPU tensors in
multi-process ``gloo`` tests, where no GPU exists.  ``install()`` replaces
``_native.call`` / ``_native.query`` by numpy implementations of the entry
points those paths use (same argument lists as include/ncgp_b200.h, pointers
to host memory) and makes the device helpers accept CPU tensors.  The product
never imports this module; the K1 kernel operator is not emulated here (the
tests inject an oracle-backed operator for it).
"""

import ctypes
import sys

import numpy as np
import torch

F64, F32 = 1, 0


def _arr(p, n, dtype):
    """numpy view of ``n`` elements at host address ``p``."""
    if p is None or n == 0:
        return None
    p = p.value if isinstance(p, ctypes.c_void_p) else int(p)
    ct = {np.float64: ctypes.c_double, np.float32: ctypes.c_float, np.int64: ctypes.c_int64}[dtype]
    return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ct)), shape=(int(n),))


def _block(p, ld, k, n, dt):
    """(k, n) view of a column block with row stride ld."""
    flat = _arr(p, (k - 1) * ld + n, dt)
    return np.lib.stride_tricks.as_strided(flat, shape=(k, n),
                                           strides=(ld * flat.itemsize, flat.itemsize))


def _install_native(native):
    np_dt = lambda code: np.float64 if code == native.F64 else np.float32

    def softmax_rows(f, n, C):
        z = f.reshape(n, C).astype(np.float64)
        z = z - z.max(axis=1, keepdims=True)
        e = np.exp(z)
        return e / e.sum(axis=1, keepdims=True)

    def pinv_apply(pi, V):  # (n, C), (n, C, k) -> W^+ V   (likelihoods.py:291-310)
        proj = V - V.mean(axis=1, keepdims=True)
        scaled = proj / np.maximum(pi, 1e-12)[:, :, None]
        return scaled - scaled.mean(axis=1, keepdims=True)

    def call(name, *a):
        if name == "ncgp_dots":
            code, n, npairs, xs, ys, out = a[:6]
            dt = np_dt(code)
            o = _arr(out, npairs, np.float64)
            for p in range(npairs):
                o[p] = np.dot(_arr(xs[p], n, dt).astype(np.float64),
                              _arr(ys[p], n, dt).astype(np.float64))
        elif name == "ncgp_gemv_t":
            code, Q, ldq, k, z, n, out = a[:7]
            dt = np_dt(code)
            _arr(out, k, np.float64)[:] = _block(Q, ldq, k, n, dt).astype(np.float64) @ \
                _arr(z, n, dt).astype(np.float64)
        elif name == "ncgp_gemv_n":
            code, Q, ldq, k, y, s, alpha, out, n = a[:9]
            dt = np_dt(code)
            res = np.zeros(n) if s is None else _arr(s, n, dt).astype(np.float64)
            if k:
                res = res + alpha * (_arr(y, k, np.float64) @ _block(Q, ldq, k, n, dt).astype(np.float64))
            _arr(out, n, dt)[:] = res
        elif name == "ncgp_lincomb":
            code, n, ca, x, cb, y, cc, z, out = a[:9]
            dt = np_dt(code)
            res = ca * _arr(x, n, dt).astype(np.float64)
            if y is not None:
                res = res + cb * _arr(y, n, dt)
            if z is not None:
                res = res + cc * _arr(z, n, dt)
            _arr(out, n, dt)[:] = res
        elif name == "ncgp_gram":
            code, S, lds, ka, Y, ldy, kb, n, M, ldm = a[:10]
            dt = np_dt(code)
            _block(M, ldm, ka, kb, np.float64)[:] = _block(S, lds, ka, n, dt).astype(np.float64) @ \
                _block(Y, ldy, kb, n, dt).astype(np.float64).T
        elif name == "ncgp_softmax_stats":
            code, f, labels, n, C, pi, grad, yhat = a[:8]
            dt = np_dt(code)
            fv = _arr(f, n * C, dt)
            p = softmax_rows(fv, n, C)
            _arr(pi, n * C, dt)[:] = p.reshape(-1)
            if labels is not None and (grad is not None or yhat is not None):
                onehot = np.zeros((n, C))
                onehot[np.arange(n), _arr(labels, n, np.int64)] = 1.0
                g = onehot - p
                if grad is not None:
                    _arr(grad, n * C, dt)[:] = g.reshape(-1)
                if yhat is not None:
                    _arr(yhat, n * C, dt)[:] = fv + pinv_apply(p, g[:, :, None])[:, :, 0].reshape(-1)
        elif name == "ncgp_softmax_winv":
            code, pi, n, C, V, ldv, k, base, ldb, alpha, beta, out, ldo = a[:13]
            dt = np_dt(code)
            p = _arr(pi, n * C, dt).reshape(n, C).astype(np.float64)
            Vb = _block(V, ldv, k, n * C, dt).astype(np.float64)
            res = alpha * pinv_apply(p, Vb.T.reshape(n, C, k)).reshape(n * C, k).T
            if base is not None:
                res = res + beta * _block(base, ldb, k, n * C, dt)
            _block(out, ldo, k, n * C, dt)[:] = res
        elif name == "ncgp_bernoulli_stats":
            code, f, labels, n, winv, w, grad, yhat = a[:8]
            dt = np_dt(code)
            fv = _arr(f, n, dt).astype(np.float64)
            s = np.clip(1.0 / (1.0 + np.exp(-fv)), 1e-12, 1 - 1e-12)
            wi = 1.0 / (s * (1.0 - s))
            if winv is not None:
                _arr(winv, n, dt)[:] = wi
            if w is not None:
                _arr(w, n, dt)[:] = s * (1.0 - s)
            if labels is not None:
                g = _arr(labels, n, np.int64) - 1.0 / (1.0 + np.exp(-fv))
                if grad is not None:
                    _arr(grad, n, dt)[:] = g
                if yhat is not None:
                    _arr(yhat, n, dt)[:] = fv + wi * g
        elif name == "ncgp_diag_apply":
            code, dvec, n, V, ldv, k, base, ldb, alpha, beta, out, ldo = a[:12]
            dt = np_dt(code)
            res = alpha * _arr(dvec, n, dt)[None, :] * _block(V, ldv, k, n, dt)
            if base is not None:
                res = res + beta * _block(base, ldb, k, n, dt)
            _block(out, ldo, k, n, dt)[:] = res
        elif name == "ncgp_marginal_var":
            code, A, lda, nt, C, R, s2, var = a[:8]
            dt = np_dt(code)
            Ab = _block(A, lda, nt, C * R, dt).astype(np.float64).reshape(nt, C, R)
            _arr(var, nt * C, dt)[:] = np.maximum(
                _arr(s2, C, np.float64)[None, :] - (Ab ** 2).sum(axis=2), 0.0).reshape(-1)
        else:
            raise NotImplementedError(f"fake native: {name}")
        return 0

    def query(name, *a):
        if name in ("ncgp_reduce_workspace_bytes", "ncgp_gram_workspace_bytes"):
            return 256
        raise NotImplementedError(f"fake native query: {name}")

    native.call, native.query, native.load = call, query, (lambda: None)


def install():
    """Route the package's native calls to the CPU stand-ins (this process only)."""
    import paper_2310_20285_b200  # noqa: F401
    from paper_2310_20285_b200 import _native, device

    _install_native(_native)
    cpu = torch.device("cpu")
    is_dev = lambda x: isinstance(x, torch.Tensor)

    def to_device(x, dtype=None, contiguous=True):
        dt = device.resolve_dtype(dtype)
        t = x.to(dt) if isinstance(x, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(x), dtype=np.float64 if dt == torch.float64
                                 else np.float32))
        return t.contiguous() if contiguous else t

    def labels_to_device(y):
        if isinstance(y, torch.Tensor):
            return y.to(torch.int64).contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.asarray(y), dtype=np.int64))

    class _WS:
        def get(self, key, nbytes):
            return torch.empty(max(int(nbytes), 256), dtype=torch.uint8)

    repl = {"require_cuda": lambda: cpu, "stream": lambda: None, "is_device": is_dev,
            "to_device": to_device, "labels_to_device": labels_to_device,
            "workspace": lambda: _WS()}
    for name, mod in list(sys.modules.items()):
        if name.startswith("paper_2310_20285_b200") and mod is not None:
            for k, v in repl.items():
                if hasattr(mod, k):
                    setattr(mod, k, v)
