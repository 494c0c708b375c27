"""CPU tests of the reference-compatible harness pieces that need no GPU:
config schema and builders (config.py:21-328 of the reference), the CLI's
argument / exit-code contract (cli.py:416-460), and the host metrics and
Monte-Carlo predictions (posterior.py:125-271) against outputs of the
reference itself (tests/golden/make_golden_cli.py)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2310_20285_b200 as P
from paper_2310_20285_b200 import cli
from paper_2310_20285_b200 import config as cfgmod

CLI = os.path.join(GOLDEN, "cli")


def _cfg(name):
    with open(os.path.join(CLI, name, "config.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", ["mixture_softmax", "binary_sod", "poisson_iter"])
def test_reference_configs_validate(name):
    cfg = cfgmod.validate_fit_config(_cfg(name))
    oc = cfgmod.build_outer_config(cfg)
    assert oc.max_newton_steps == cfg["outer"]["max_newton_steps"]
    prior = cfgmod.build_prior(cfg["prior"], 3)
    assert prior.num_outputs == 3


@pytest.mark.parametrize("mutate, msg", [
    (lambda c: c.update(bogus=1), "Additional properties"),
    (lambda c: c["prior"]["kernel"].update(lengthscale=-1.0), "fit config invalid"),
    (lambda c: c.update(method="sod"), "subset_size"),
    (lambda c: c["data"].update(csv="x.csv"), "exactly one"),
])
def test_invalid_configs_rejected(mutate, msg):
    cfg = _cfg("mixture_softmax")
    mutate(cfg)
    with pytest.raises(P.ConfigError, match=msg):
        cfgmod.validate_fit_config(cfg)


def test_cli_config_error_exit_code(tmp_path, capsys):
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"seed": 1}))
    assert cli.main(["fit", "--config", str(bad), "--out", str(tmp_path)]) == cli.EXIT_CONFIG
    assert "config error" in capsys.readouterr().err
    nojson = tmp_path / "nojson.json"
    nojson.write_text("{")
    assert cli.main(["generate", "--config", str(nojson), "--out", str(tmp_path)]) == \
        cli.EXIT_CONFIG


def test_metrics_header_matches_reference_file():
    with open(os.path.join(CLI, "mixture_softmax", "metrics.csv")) as fh:
        assert fh.readline().strip().split(",") == cli.METRICS_HEADER


def test_dataset_csv_round_trip(tmp_path):
    ds = P.read_dataset_csv(os.path.join(CLI, "mixture_softmax", "dataset.csv"), "class-index", 3)
    p = tmp_path / "d.csv"
    P.write_dataset_csv(p, ds)
    assert p.read_text() == open(os.path.join(CLI, "mixture_softmax", "dataset.csv")).read()


def test_host_metrics_match_reference():
    g = np.load(os.path.join(CLI, "metrics.npz"))
    assert P.metric_nll(g["probs"], g["y"]) == float(g["nll"])
    assert P.metric_ece(g["probs"], g["y"]) == float(g["ece"])
    assert P.metric_ece(g["probs"], g["y"], 7) == float(g["ece7"])
    np.testing.assert_array_equal(
        P.poisson_predictive_density(g["mean"][:, :1], g["var"][:, :1], g["counts"], 50, 14),
        g["dens"])


def test_mc_predict_matches_reference():
    """The Philox per-(point, output) streams make MC predictions equal to
    the reference's for the same moments (posterior.py:136-202).  The
    likelihood objects are host-only (no device use)."""
    g = np.load(os.path.join(CLI, "metrics.npz"))
    sm = P.mc_predict(g["mean"], g["var"], P.SoftmaxLikelihood(g["y"], 3), 50, 11)
    np.testing.assert_allclose(sm.class_probabilities, g["sm_probs"], rtol=1e-14)
    be = P.mc_predict(g["mean"][:, :1], g["var"][:, :1],
                      P.BernoulliLogisticLikelihood(g["y"] % 2), 50, 12)
    np.testing.assert_allclose(be.class_probabilities, g["be_probs"], rtol=1e-14)
    po = P.mc_predict(g["mean"][:, :1], g["var"][:, :1], P.PoissonLikelihood(g["counts"]), 50, 13)
    np.testing.assert_allclose(po.rate_median, g["po_med"], rtol=1e-14)
    np.testing.assert_allclose(po.rate_lower, g["po_lo"], rtol=1e-14)
    np.testing.assert_allclose(po.rate_upper, g["po_hi"], rtol=1e-14)
