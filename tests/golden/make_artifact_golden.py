"""Write a small NCGP v1 belief artifact with the REAL reference package
(``ncgp.artifact.save_belief``), for the byte-compatibility test of
``paper_2310_20285_b200.artifact``.

    python tests/golden/make_artifact_golden.py [--ref /root/reference/pkg/src]
"""
import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from ncgp import KernelSpec, LowRankRoot, MultiOutputPrior
    from ncgp.artifact import save_belief
    from ncgp.posterior import PosteriorBelief
    rng = np.random.default_rng(7)
    n, d, c, rank = 13, 3, 2, 4
    prior = MultiOutputPrior(kernels=(KernelSpec("rbf", 1.3, 0.7), KernelSpec("matern32", 0.9, 2.0)),
                             mean=(0.25, -1.0))
    belief = PosteriorBelief(prior=prior, train_inputs=rng.standard_normal((n, d)),
                             weights=rng.standard_normal(n * c),
                             root=LowRankRoot(rng.standard_normal((n * c, rank))),
                             newton_step=3, solver_iterations=17)
    echo = {"prior": {"kernels": [{"family": "rbf", "lengthscale": 1.3, "outputscale": 0.7},
                                  {"family": "matern32", "lengthscale": 0.9, "outputscale": 2.0}],
                      "mean": [0.25, -1.0]},
            "likelihood": "softmax", "seed": 7}
    save_belief(os.path.join(HERE, "belief_v1.ncgp"), belief, echo)
    np.savez_compressed(os.path.join(HERE, "belief_v1_arrays.npz"), X=belief.train_inputs,
                        weights=belief.weights, Q=belief.root.columns)


if __name__ == "__main__":
    main()
