"""Host-side logic that needs no GPU: CN/NC layout (property test, like the
reference's hypothesis round trip), kernel-spec and prior validation, config
dataclasses, row partitioning and the artifact prior builder."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2310_20285_b200 as P
from paper_2310_20285_b200.gp import Ordering, reorder
from paper_2310_20285_b200.parallel import row_partition


@settings(max_examples=60, deadline=None)
@given(n=st.integers(1, 40), c=st.integers(1, 7), seed=st.integers(0, 2 ** 31 - 1))
def test_reorder_round_trip(n, c, seed):
    v = np.random.default_rng(seed).standard_normal(n * c)
    nc = reorder(v, Ordering.CN, Ordering.NC, n, c)
    # NC entry c*N + i is CN entry i*C + c
    np.testing.assert_array_equal(nc.reshape(c, n).T.ravel(), v)
    np.testing.assert_array_equal(reorder(nc, Ordering.NC, Ordering.CN, n, c), v)


def test_reorder_rejects_bad_length():
    with pytest.raises(P.DimensionMismatch):
        reorder(np.zeros(5), Ordering.CN, Ordering.NC, 2, 3)


@pytest.mark.parametrize("kw", [dict(family="rbf", lengthscale=0.0, outputscale=1.0),
                                dict(family="rbf", lengthscale=1.0, outputscale=-1.0),
                                dict(family="cauchy", lengthscale=1.0, outputscale=1.0),
                                dict(family="rbf", lengthscale=float("nan"), outputscale=1.0)])
def test_kernel_spec_validation(kw):
    with pytest.raises((P.InvalidInput, ValueError)):
        P.KernelSpec(**kw)


def test_prior_spec_groups_and_mean():
    a, b = P.KernelSpec("rbf", 1.0, 1.0), P.KernelSpec("matern32", 2.0, 0.5)
    prior = P.MultiOutputPrior(kernels=(a, b, a), mean=(0.0, 1.0, 2.0))
    groups = {spec: list(cols) for spec, cols in prior.spec_groups()}
    assert groups == {a: [0, 2], b: [1]}
    np.testing.assert_array_equal(prior.mean_vector(2), [0, 1, 2, 0, 1, 2])
    with pytest.raises(P.DimensionMismatch):
        P.MultiOutputPrior(kernels=(a, b), mean=(0.0,))


def test_inner_config_validation():
    with pytest.raises(P.InvalidInput):
        P.InnerConfig(max_iters=-1)
    with pytest.raises(P.InvalidInput):
        P.InnerConfig(max_iters=1, residual="lanczos")
    assert P.InnerConfig(max_iters=1).residual == "explicit"


@settings(max_examples=80, deadline=None)
@given(n=st.integers(0, 100_000), world=st.integers(1, 8))
def test_row_partition_property(n, world):
    seen = 0
    prev_end = 0
    for r in range(world):
        r0, r1, per = row_partition(n, world, r)
        assert r0 == prev_end or r0 == n
        assert per % 256 == 0 and r0 % 256 == 0 or r0 == n
        seen += r1 - r0
        prev_end = r1
    assert seen == n
