"""Generate the cfg5 Newton-trajectory fixture from the CPU oracle.

The oracle (oracle/ncgp_oracle.py) is pinned bit-exact to the reference
package on the golden vectors (tests/test_oracle_golden.py).  This script runs
its IterNCGP fit on the seeded cfg5 generator at reduced N and records, per
Newton step, the inner iteration count, the termination reason and |yhat|,
plus the accuracy of the posterior mean on the first 500 test points.

cfg5 (BASELINE.json configs[4]) drives the reference's undamped Newton
iteration into divergence from N ~ 5000 up; the fixture documents that
trajectory so the GPU fit can be checked against it step for step.

usage: python tests/golden/make_cfg5_trajectory.py N [N ...]   (N=1500: ~3 min,
       N=5000: ~55 min on one CPU core)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ncgp_oracle as O  # noqa: E402
from paper_2310_20285_b200 import configs  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg5_trajectory.json")


def run(n):
    c = configs.cfg5(n=n, n_test=2000)
    specs = [c["kernel"]] * 10
    lik = O.OracleLikelihood("softmax", c["y"], 10)
    t = time.time()
    res = O.fit(specs, c["X"], lik, max_steps=6, schedule=64, recycle=True, rank=256,
                delta=0.01, policy="residual")
    secs = time.time() - t
    mean = O.posterior_mean(specs, c["X"], res["weights"], c["X_test"][:500])
    acc = float(np.mean(mean.argmax(1) == c["y_test"][:500]))
    return {
        "n": n,
        "steps": [{"iterations": int(s["iterations"]), "termination": s["termination"],
                   "yhat_norm": float(s["yhat_norm"])} for s in res["steps"]],
        "accuracy_mean_500": acc,
        "oracle_seconds": secs,
    }


if __name__ == "__main__":
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for arg in sys.argv[1:]:
        r = run(int(arg))
        data[str(r["n"])] = r
        print(json.dumps(r), flush=True)
        json.dump(data, open(OUT, "w"), indent=1)
