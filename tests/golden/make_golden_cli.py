"""CLI golden outputs produced by the REAL reference ``ncgp`` command line
(cli.py) in this container: datasets from ``generate``, ``fit --clock none``
outputs (metrics.csv, summary.json, belief.ncgp) and ``predict`` CSVs, plus
the reference's metric / MC-prediction functions on fixed inputs.

    python tests/golden/make_golden_cli.py      # writes tests/golden/cli/

The GPU tests run this package's CLI on the same configs and compare.
"""

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")
REF = "/root/reference/pkg/src"

CONFIGS = {
    "mixture_softmax": {
        "seed": 3,
        "data": {"generator": {"kind": "gaussian-mixture-3d", "n_per_class": 60,
                               "num_classes": 3},
                 "test": {"draw_offset": 1}},
        "prior": {"kernel": {"family": "rbf", "lengthscale": 0.5, "outputscale": 2.0}},
        "likelihood": {"family": "softmax"},
        "method": "iterncgp", "policy": "residual",
        "outer": {"max_newton_steps": 4, "inner_schedule": [10, 15], "recycle": True,
                  "delta": 0.001},
        "metrics": {"cadence": "step"},
    },
    "binary_sod": {
        "seed": 5,
        "data": {"generator": {"kind": "gp-binary-2d", "n": 150}, "test": {"draw_offset": 2}},
        "prior": {"kernel": {"family": "matern32", "lengthscale": 1.0, "outputscale": 2.0}},
        "likelihood": {"family": "bernoulli_logistic"},
        "method": "sod", "sod": {"subset_size": 60},
        "outer": {"max_newton_steps": 8, "delta": 1e-4},
    },
    "poisson_iter": {
        "seed": 7,
        "data": {"generator": {"kind": "gp-poisson-1d", "n": 80}, "test": {"draw_offset": 1}},
        "prior": {"kernel": {"family": "rbf", "lengthscale": 0.1, "outputscale": 1.0},
                  "mean": 1.0},
        "likelihood": {"family": "poisson"},
        "method": "iterncgp", "policy": "residual",
        "outer": {"max_newton_steps": 3, "inner_schedule": 12, "recycle": False},
        "metrics": {"cadence": "iter", "every": 4, "mc_samples": 64},
    },
}


def main():
    sys.path.insert(0, REF)
    from ncgp import cli
    from ncgp.likelihoods import (BernoulliLogisticLikelihood, PoissonLikelihood,
                                  SoftmaxLikelihood)
    from ncgp.posterior import (mc_predict, metric_ece, metric_nll,
                                poisson_predictive_density)
    os.makedirs(OUT, exist_ok=True)
    for name, cfg in CONFIGS.items():
        d = os.path.join(OUT, name)
        os.makedirs(d, exist_ok=True)
        cp = os.path.join(d, "config.json")
        with open(cp, "w") as fh:
            json.dump(cfg, fh, indent=1, sort_keys=True)
        tmp = tempfile.mkdtemp()
        assert cli.main(["generate", "--config", cp, "--out", tmp]) == 0
        for f in ("dataset.csv", "test.csv"):
            shutil.copy(os.path.join(tmp, f), os.path.join(d, f))
        rc = cli.main(["fit", "--config", cp, "--out", tmp, "--clock", "none"])
        assert rc in (0, 4), rc
        for f in ("metrics.csv", "summary.json", "belief.ncgp"):
            shutil.copy(os.path.join(tmp, f), os.path.join(d, f))
        # the reference's own spread: the same fit with every K product
        # multiplied by (1 + 1e-14 xi); per metric column, the
        # largest deviation from the unperturbed metrics.csv
        import ncgp.outer as outer_mod
        orig = outer_mod.prior_matvec
        rng = np.random.default_rng(99)
        outer_mod.prior_matvec = lambda pr, X, v, tile=256: \
            orig(pr, X, v, tile=tile) * (1.0 + 1e-14 * rng.standard_normal(v.shape[0]))
        tmp2 = tempfile.mkdtemp()
        try:
            cli.main(["fit", "--config", cp, "--out", tmp2, "--clock", "none"])
        finally:
            outer_mod.prior_matvec = orig
        a = np.genfromtxt(os.path.join(tmp2, "metrics.csv"), delimiter=",", skip_header=1)
        b = np.genfromtxt(os.path.join(tmp, "metrics.csv"), delimiter=",", skip_header=1)
        spread = np.nan_to_num(np.abs(np.atleast_2d(a) - np.atleast_2d(b)).max(axis=0))
        with open(os.path.join(d, "spread.json"), "w") as fh:
            json.dump({"eps": 1e-14, "max_abs_dev_per_column": spread.tolist()}, fh, indent=1)
        shutil.rmtree(tmp2)
        assert cli.main(["predict", "--artifact", os.path.join(tmp, "belief.ncgp"),
                         "--inputs", os.path.join(tmp, "test.csv"),
                         "--out", os.path.join(d, "predictions.csv")]) == 0
        shutil.rmtree(tmp)
        print("wrote", d)
    # host metrics and MC prediction on fixed moments
    rng = np.random.default_rng(9)
    mean = rng.normal(size=(40, 3))
    var = 0.1 + rng.random((40, 3))
    y = rng.integers(0, 3, 40)
    probs = np.exp(mean) / np.exp(mean).sum(1, keepdims=True)
    counts = rng.poisson(2.0, 40)
    sm = mc_predict(mean, var, SoftmaxLikelihood(y, 3), 50, 11)
    be = mc_predict(mean[:, :1], var[:, :1], BernoulliLogisticLikelihood(y % 2), 50, 12)
    po = mc_predict(mean[:, :1], var[:, :1], PoissonLikelihood(counts), 50, 13)
    np.savez_compressed(os.path.join(OUT, "metrics.npz"), mean=mean, var=var, y=y,
                        probs=probs, counts=counts,
                        nll=metric_nll(probs, y), ece=metric_ece(probs, y),
                        ece7=metric_ece(probs, y, 7),
                        dens=poisson_predictive_density(mean[:, :1], var[:, :1], counts, 50, 14),
                        sm_probs=sm.class_probabilities, be_probs=be.class_probabilities,
                        po_med=po.rate_median, po_lo=po.rate_lower, po_hi=po.rate_upper)
    print("wrote metrics.npz")


if __name__ == "__main__":
    main()
