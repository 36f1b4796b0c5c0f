"""CPU checks of the parity exchange: a workload directory
written by the product CLI (archive + dv0 + parameters) reads back bit-exact
through the product loader AND the numpy-only oracle loader (what bench.py's
reference arm uses, so its timed process never loads the CUDA library), and
`oracle.cli.compare` applies north_star's bar."""

import numpy as np

from conftest import load_golden, product_gs


def _kstate():
    from paper_2505_02319_b200.groundstate import GaussianWell, ModelSpec
    from paper_2505_02319_b200.pwbasis import Lattice
    from paper_2505_02319_b200.scf import run_scf_k
    z = load_golden("kpoint_supercell.npz")
    wells = tuple(GaussianWell(center=tuple(w[:3]), amplitude=float(w[3]), width=float(w[4]))
                  for w in z["unit_wells"])
    model = ModelSpec(lattice=Lattice.from_vectors(*z["unit_lattice"]),
                      e_cut=float(z["unit_e_cut"]), n_electrons=4, temperature=5e-3,
                      gaussians=wells)
    return run_scf_k(model, [[0, 0, 0], [0.5, 0, 0]], tol=1e-10, max_iter=600, damping=0.3)


def test_workload_round_trip_gamma_and_k(tmp_path):
    from oracle.archive import load_workload
    from paper_2505_02319_b200.cli import read_workload, write_workload
    params = {"strategy": "bal", "tau": 1e-8, "m": 10, "xc": "lda_x", "kgrid": (1, 1, 1)}
    for name, gs in (("gamma", product_gs(load_golden("metal.npz"))), ("k", _kstate())):
        d = tmp_path / name
        d.mkdir()
        rng = np.random.default_rng(1)
        g0 = gs.blocks[0].grids if hasattr(gs, "blocks") else gs.grids
        dv0 = rng.standard_normal(g0.n_g)
        write_workload(str(d), gs, dv0, params, {"config": -1})
        gs2, dv2, p2 = read_workload(str(d))
        og, dv3, p3 = load_workload(str(d))
        np.testing.assert_array_equal(dv2, dv0)
        np.testing.assert_array_equal(dv3, dv0)
        assert p2["strategy"] == p3["strategy"] == "bal" and p3["kgrid"] == [1, 1, 1]
        blocks = gs.blocks if hasattr(gs, "blocks") else [gs]
        b2 = gs2.blocks if hasattr(gs2, "blocks") else [gs2]
        ob = og.blocks if hasattr(og, "blocks") else [og]
        assert len(b2) == len(ob) == len(blocks)
        for a, b, c in zip(blocks, b2, ob):
            np.testing.assert_array_equal(a.phi, b.phi)
            np.testing.assert_array_equal(a.phi, c.phi)
            np.testing.assert_array_equal(a.eps, c.eps)
            np.testing.assert_array_equal(a.occ, c.occ)
            assert a.n_occ == c.n_occ and a.grids.n_b == c.grids.n_b
            np.testing.assert_array_equal(a.grids.g_int, c.grids.g_int)
        np.testing.assert_array_equal(gs.rho, og.rho)
        np.testing.assert_array_equal(gs.v_local, og.v_local)


def test_oracle_compare_applies_the_bar():
    from oracle.cli import compare
    sol = np.linspace(1.0, 2.0, 50)
    sched = np.full((3, 4), 1e-6)
    a = {"solution": sol, "iterations": 12, "n_ham": 100, "converged": True, "schedule": sched}
    b = dict(a, solution=sol * (1 + 1e-10), iterations=13)
    out = compare(a, b)
    assert out["pass"] and out["drho_rel_l2"] < 1e-9
    assert not compare(a, dict(b, iterations=14))["pass"]
    assert not compare(a, dict(b, solution=sol * (1 + 1e-6)))["pass"]
    assert not compare(a, dict(b, schedule=sched * (1 + 1e-3)))["pass"]
