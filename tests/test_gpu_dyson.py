"""Full Dyson-solve parity (RHS + device-resident inexact GMRES) on the GPU against
golden runs of the unmodified reference `run_response`.  Needs a B200.

Bar (BASELINE.json north_star): solution relative L2 within 1e-8, GMRES
iteration count within 1, same per-iteration Sternheimer tolerance schedule.
"""

import numpy as np
import pytest

from conftest import load_golden, product_gs, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    _lib.require_device()


@pytest.mark.parametrize("tag", ["a", "b"])
def test_device_igmres_matches_reference(tag):
    from paper_2505_02319_b200.igmres import igmres_solve
    z = load_golden("igmres.npz")
    a, b = z[f"{tag}_a"], z[f"{tag}_b"]
    rep = igmres_solve(lambda v, budget: (a @ v, 1), b, m=int(z[f"{tag}_m"]),
                       tau=float(z[f"{tag}_tau"]))
    assert rep.converged
    assert rep.iterations == int(z[f"{tag}_its"])
    np.testing.assert_allclose(rep.solution, z[f"{tag}_x"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(rep.est_res_history, z[f"{tag}_hist"], rtol=1e-8, atol=1e-13)


def test_device_igmres_adversarial_budgets():
    """Operator errors of exactly the granted budget keep ||b - Ax|| <= tau (test_igmres.py:78-90)."""
    from paper_2505_02319_b200.igmres import igmres_solve
    rng = np.random.default_rng(3)
    n, tau = 40, 1e-8
    for _ in range(5):
        a = np.eye(n) + 0.5 * rng.standard_normal((n, n)) / np.sqrt(n)
        b = rng.standard_normal(n)

        def op(v, budget):
            e = rng.standard_normal(n)
            return a @ v + e * budget / np.linalg.norm(e), 1

        rep = igmres_solve(op, b, m=8, tau=tau)
        assert np.linalg.norm(b - a @ rep.solution) <= tau


@pytest.mark.parametrize("fixture,strategy", [("dyson_metal.npz", "pbal"),
                                              ("dyson_metal.npz", "bal"),
                                              ("dyson_metal.npz", "d10"),
                                              ("dyson_metal.npz", "pagr"),
                                              ("dyson_cfg0.npz", "bal")])
def test_dyson_solve_matches_reference(fixture, strategy):
    from paper_2505_02319_b200.harness import solve_dyson
    z = load_golden(fixture)
    gs = product_gs(z)
    meta = z[f"{strategy}_meta"]
    res = solve_dyson(gs, z["dv0"], strategy=str(meta[0]), tau=float(meta[1]), m=int(meta[2]),
                      with_true_residual=True)
    assert res.converged
    assert abs(res.iterations - int(z[f"{strategy}_iterations"])) <= 1
    assert rel(res.rhs.cpu().numpy(), z[f"{strategy}_rhs"]) < 1e-8
    assert rel(res.solution.cpu().numpy(), z[f"{strategy}_solution"]) < 1e-8
    np.testing.assert_allclose(res.tolerance_schedule[0], z[f"{strategy}_rhs_tols"], rtol=1e-12)
    ops = z[f"{strategy}_op_tols"]
    for got, want in zip(res.tolerance_schedule[1:], ops):
        np.testing.assert_allclose(got, want, rtol=1e-5)
    want_nham = int(z[f"{strategy}_n_ham"])
    assert abs(res.n_ham - want_nham) <= max(2, 0.02 * want_nham)
    assert res.final_true_res <= float(meta[1]) * 1.5 + 1e-300
