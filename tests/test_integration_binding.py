"""INTEGRATION.md's ctypes binding (integration/ncgp_b200_binding.py, shown
there verbatim) installed as ``ncgp/b200.py`` into a stand-in package whose
``outer`` module resolves ``prior_matvec`` by name like the reference's
``fit`` / ``newton_update`` (outer.py:134-137, 180-181)."""

import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BINDING = os.path.join(ROOT, "integration", "ncgp_b200_binding.py")
LIB = os.path.join(ROOT, "paper_2310_20285_b200", "libncgp_b200.so")


def test_integration_md_shows_the_binding_verbatim():
    md = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    assert open(BINDING).read() in md


def _stand_in(tmp_path):
    pkg = tmp_path / "ncgp"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    # the reference's outer seam: newton_update calls the module-level name
    (pkg / "outer.py").write_text(textwrap.dedent(f"""
        import sys
        sys.path.insert(0, {ROOT!r})
        from oracle import ncgp_oracle as O

        def prior_matvec(prior, X, v, tile=256):
            return O.prior_matvec(prior.kernels, X, v, tile)

        def newton_update(prior, X, weights, mean_vec, tile=256):
            return prior_matvec(prior, X, weights, tile=tile) + mean_vec
    """))
    (pkg / "b200.py").write_text(open(BINDING).read())
    return pkg


@pytest.mark.gpu
def test_enable_routes_products_through_the_library(tmp_path):
    _stand_in(tmp_path)
    script = textwrap.dedent(f"""
        import sys
        from collections import namedtuple
        import numpy as np
        sys.path.insert(0, {str(tmp_path)!r})
        sys.path.insert(0, {ROOT!r})
        import ncgp.outer as outer
        import ncgp.b200 as b200
        from oracle import ncgp_oracle as O
        Spec = namedtuple("Spec", "family lengthscale outputscale")
        Prior = namedtuple("Prior", "kernels num_outputs")
        rng = np.random.default_rng(0)
        n, C = 3000, 3
        X = rng.standard_normal((n, 4))
        w = rng.standard_normal(n * C)
        m = np.tile([0.5, -0.2, 0.1], n)
        prior = Prior((Spec("rbf", 1.3, 2.0),) * C, C)
        ref = outer.newton_update(prior, X, w, m)
        b200.enable()
        assert outer.prior_matvec is b200.accelerated_prior_matvec
        got = outer.newton_update(prior, X, w, m)
        b200.disable()
        assert outer.prior_matvec is not b200.accelerated_prior_matvec
        kv = O.prior_matvec(prior.kernels, X, np.abs(w))
        err = np.max(np.abs(got - ref) / (kv + 1e-300))
        assert err < 1e-5, err
        print("BINDING_OK", err)
    """)
    env = dict(os.environ, NCGP_B200_LIB=LIB)
    r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, env=env,
                       timeout=600)
    assert r.returncode == 0 and "BINDING_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
