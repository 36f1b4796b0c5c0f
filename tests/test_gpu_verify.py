"""The executable-lemma checks (reference verify_suite, harness.py:387-543) on the GPU
path: same verdicts as the reference on its metal fixture (tests/golden/gen_verify.py),
and all checks passing at BASELINE scale (config 1: 48^3, 8 k-points)."""

import ast

import numpy as np
import pytest

from conftest import load_golden, product_gs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    _lib.require_device()


def test_verify_suite_matches_reference_verdicts():
    from paper_2505_02319_b200.harness import Perturbation
    from paper_2505_02319_b200.verify import verify_suite
    z = load_golden("verify_metal.npz")
    p = ast.literal_eval(str(z["params"]))
    gs = product_gs(z)
    out = verify_suite(gs, strategy=p["strategy"], tau=p["tau"], m=p["m"],
                       kerker_alpha=p["kerker_alpha"], seed=p["seed"],
                       perturbation=Perturbation(gaussian=p["gaussian"],
                                                 direction=p["direction"]))
    got = {c["name"]: c for c in out["checks"]}
    assert out["ok"]
    for name, passed, margin in zip(z["names"], z["passed"], z["margins"]):
        c = got[str(name)]
        assert c["passed"] == bool(passed), name
        assert "skipped" not in c, name
        if name in ("orbital_orthonormality", "row_norm_bounds"):
            assert c["margin"] == pytest.approx(float(margin), rel=1e-9), name
        elif name in ("error_bound_dominance", "sternheimer_error_bound", "y_coefficient_bound"):
            # ratios of CG-truncation errors: same draws, iteration counts +-1
            assert 0.5 < c["margin"] / float(margin) < 2.0, (name, c["margin"], margin)


def test_verify_suite_at_baseline_scale():
    import bench
    from paper_2505_02319_b200.verify import verify_suite
    gs, dv0, p = bench.build_workload(1)
    out = verify_suite(gs, strategy=p["strategy"], tau=p["tau"], m=p["m"], xc=p["xc"],
                       dv0=dv0, draws=4)
    assert out["ok"], out
    names = {c["name"]: c for c in out["checks"]}
    assert "skipped" in names["error_bound_dominance"]   # Gamma-point lemma
    assert "skipped" not in names["y_coefficient_bound"]
    assert names["chi0_gauge_invariance"]["passed"]
