"""NCGP v1 belief artifacts (reference artifact.py): byte compatibility with
a file written by the reference package itself (tests/golden/belief_v1.ncgp,
from tests/golden/make_artifact_golden.py), round trips and error handling."""

import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2310_20285_b200 as P
from paper_2310_20285_b200.artifact import VERSION, build_prior, load_belief, save_belief

REF = os.path.join(GOLDEN, "belief_v1.ncgp")


def _ref_arrays():
    with np.load(os.path.join(GOLDEN, "belief_v1_arrays.npz")) as z:
        return {k: z[k] for k in z.files}


def test_loads_reference_artifact():
    b, echo = load_belief(REF)
    a = _ref_arrays()
    np.testing.assert_array_equal(b.train_inputs, a["X"])
    np.testing.assert_array_equal(b.weights, a["weights"])
    np.testing.assert_array_equal(b.root.columns, a["Q"])
    assert (b.newton_step, b.solver_iterations) == (3, 17)
    assert b.prior.kernels == (P.KernelSpec("rbf", 1.3, 0.7), P.KernelSpec("matern32", 0.9, 2.0))
    assert b.prior.mean == (0.25, -1.0)
    assert echo["seed"] == 7


def test_writes_reference_bytes(tmp_path):
    b, echo = load_belief(REF)
    out = tmp_path / "b.ncgp"
    save_belief(out, b, echo)
    assert out.read_bytes() == open(REF, "rb").read()


def test_round_trip_shared_kernel(tmp_path):
    rng = np.random.default_rng(0)
    n, C, R = 9, 3, 0
    prior = build_prior({"kernel": {"family": "rbf", "lengthscale": 2.0, "outputscale": 1.5},
                         "mean": 0.5}, C)
    b = P.PosteriorBelief(prior, rng.standard_normal((n, 2)), rng.standard_normal(n * C),
                          P.LowRankRoot(np.zeros((n * C, R))), newton_step=1, solver_iterations=2)
    p = tmp_path / "z.ncgp"
    save_belief(p, b, {"prior": {"kernel": {"family": "rbf", "lengthscale": 2.0,
                                            "outputscale": 1.5}, "mean": 0.5}})
    b2, _ = load_belief(p)
    np.testing.assert_array_equal(b2.weights, b.weights)
    assert b2.root.rank == 0 and b2.prior == prior


def test_errors(tmp_path):
    bad = tmp_path / "bad.ncgp"
    bad.write_bytes(b"XXXX" + bytes(60))
    with pytest.raises(P.ArtifactError, match="magic"):
        load_belief(bad)
    data = bytearray(open(REF, "rb").read())
    data[4:8] = struct.pack("<I", VERSION + 1)
    bad.write_bytes(bytes(data))
    with pytest.raises(P.ArtifactError, match="version"):
        load_belief(bad)
    bad.write_bytes(open(REF, "rb").read()[:200])
    with pytest.raises(P.ArtifactError, match="truncated"):
        load_belief(bad)
    with pytest.raises(P.ConfigError):
        build_prior({"kernels": [{"family": "rbf", "lengthscale": 1.0, "outputscale": 1.0}]}, 2)
    with pytest.raises(P.ConfigError):
        build_prior({}, 2)
