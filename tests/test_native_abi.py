"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/ncgp_b200.h declares, and the host-side mirror of the
reference API validates inputs like the reference (no compute without GPU).
"""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

HEADER = os.path.join(ROOT, "include", "ncgp_b200.h")
LIB = os.path.join(ROOT, "paper_2310_20285_b200", "libncgp_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ncgp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        pytest.fail(f"{LIB} not built (run __graft_entry__.build())")
    from paper_2310_20285_b200 import _native
    return _native.load()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for required in ("ncgp_kop_create", "ncgp_kop_apply", "ncgp_softmax_winv",
                     "ncgp_softmax_stats", "ncgp_bernoulli_stats", "ncgp_gram", "ncgp_rotate",
                     "ncgp_gemv_t", "ncgp_gemv_n", "ncgp_dots", "ncgp_marginal_var"):
        assert required in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_signatures_cover_header(lib):
    from paper_2310_20285_b200 import _native
    assert set(declared_symbols()) <= set(_native._SIGS)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_mapping_without_gpu(lib):
    """Argument validation happens before any device work."""
    from paper_2310_20285_b200 import _native
    from paper_2310_20285_b200.exceptions import DimensionMismatch, InvalidInput
    h = _native._vp()
    with pytest.raises(InvalidInput):
        _native.call("ncgp_kop_create", _native.ctypes.byref(h), 0, 7, 1.0, 1.0, 0, 1, 4, 1,
                     4, 2, 1, None, 0, None)
    with pytest.raises(InvalidInput):
        _native.call("ncgp_kop_create", _native.ctypes.byref(h), 0, 0, -1.0, 1.0, 0, 1, 4, 1,
                     4, 2, 1, None, 0, None)
    with pytest.raises(DimensionMismatch):
        _native.call("ncgp_kop_create", _native.ctypes.byref(h), 0, 0, 1.0, 1.0, 0, 1, -4, 1,
                     4, 2, 1, None, 0, None)
    with pytest.raises(_native.Unsupported):
        _native.call("ncgp_softmax_stats", 0, 1, 1, 4, 1, 1, None, None, None)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2310_20285_b200 as P
    from paper_2310_20285_b200._native import NativeUnavailable
    prior = P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0),))
    with pytest.raises(NativeUnavailable):
        P.prior_matvec(prior, np.zeros((4, 2)), np.ones(4))


def test_host_side_validation_mirrors_reference():
    import paper_2310_20285_b200 as P
    with pytest.raises(P.InvalidInput):
        P.KernelSpec("cubic", 1.0, 1.0)
    with pytest.raises(P.InvalidInput):
        P.KernelSpec("rbf", -1.0, 1.0)
    with pytest.raises(P.DimensionMismatch):
        P.MultiOutputPrior(kernels=(P.KernelSpec("rbf", 1.0, 1.0),), mean=(0.0, 1.0))
    with pytest.raises(P.InvalidInput):
        P.OuterConfig(max_newton_steps=0)
    with pytest.raises(P.InvalidInput):
        P.InnerConfig(max_iters=-1)
    with pytest.raises(P.InvalidInput):
        P.Dataset(np.zeros((2, 1)), np.array([0, 2]), "binary")
    with pytest.raises(P.InvalidInput):
        P.SoftmaxLikelihood(np.array([0, 3]), 3)
    cfg = P.OuterConfig(max_newton_steps=3, inner_schedule=[5, 7])
    assert [cfg.budget_for(i) for i in range(4)] == [5, 7, 7, 7]


def test_reorder_and_probit_host_paths():
    import paper_2310_20285_b200 as P
    v = np.array([11.0, 12.0, 21.0, 22.0])
    np.testing.assert_array_equal(P.reorder(v, P.Ordering.CN, P.Ordering.NC, 2, 2),
                                  [11.0, 21.0, 12.0, 22.0])
    g = golden("fit_cfg1")
    np.testing.assert_allclose(P.probit_predict(g["mean"], g["var"]), g["probs"], atol=1e-15)
