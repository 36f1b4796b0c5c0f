"""Pin the CPU oracle (oracle/) against golden outputs of the unmodified reference.

CPU only.  tests/golden/*.npz come from tests/golden/gen_golden.py, which runs
/root/reference/pkg/src/pwdyson in this container.  The oracle calls the same
numpy/scipy routines in the same order, so most comparisons are at round-off.
"""

import numpy as np
import pytest

from conftest import grid_cases, load_golden, oracle_gs, rel
from oracle import basis as ob
from oracle import dyson as od
from oracle import model as om
from oracle import outer as oo
from oracle import response as orsp


@pytest.mark.parametrize("case", grid_cases())
def test_grid_tables_and_transforms(grids_golden, case):
    z = grids_golden
    b = ob.make_basis(ob.Cell(z[case + "_a"]), float(z[case + "_ecut"]))
    assert tuple(b.cube_dims) == tuple(z[case + "_dims"])
    np.testing.assert_array_equal(b.g_int, z[case + "_g_int"])
    np.testing.assert_array_equal(b.sphere_flat, z[case + "_sphere_flat"])
    np.testing.assert_allclose(b.g2_sphere, z[case + "_g2_sphere"], rtol=1e-14)
    np.testing.assert_allclose(b.g2_cube, z[case + "_g2_cube"], rtol=1e-14, atol=1e-14)
    assert rel(b.to_real_many(z[case + "_x"]), z[case + "_to_real"]) < 1e-14
    assert rel(b.to_real(z[case + "_x"][0]), z[case + "_to_real0"]) < 1e-14
    assert rel(b.to_fourier_many(z[case + "_u"]), z[case + "_to_fourier"]) < 1e-14
    h = np.stack([om.ham_apply(b, z[case + "_v"], xi) for xi in z[case + "_x"]])
    assert rel(h, z[case + "_h"]) < 1e-14
    assert rel(b.cube_fft(z[case + "_v"]), z[case + "_cube_fft"]) < 1e-14


@pytest.mark.parametrize("name", ["metal.npz", "insulator.npz"])
def test_response_pieces(name):
    z = load_golden(name)
    gs = oracle_gs(z)
    np.testing.assert_allclose(gs.fprime_occ(), z["fprime"], rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(orsp.pair_weights(gs), z["pair_weights"], rtol=1e-12, atol=1e-300)
    de, def_, df = orsp.eigen_shifts(gs, z["dv"][0])
    np.testing.assert_allclose(de, z["delta_eps"], rtol=1e-12, atol=1e-14)
    assert def_ == pytest.approx(float(z["delta_eps_f"]), rel=1e-12, abs=1e-14)
    np.testing.assert_allclose(df, z["delta_f"], rtol=1e-10, atol=1e-14)
    assert rel(orsp.project_out(gs.phi_occ, z["proj_x"]), z["proj_qx"]) < 1e-14


@pytest.mark.parametrize("name", ["metal.npz", "insulator.npz"])
@pytest.mark.parametrize("tag,tol", [("t6", 1e-6), ("t10", 1e-10)])
def test_sternheimer_matches_reference(name, tag, tol):
    z = load_golden(name)
    gs = oracle_gs(z)
    for n in range(gs.n_occ):
        r = orsp.sternheimer(gs, gs.v_local, n, z["cg_rhs"][:, n], tol)
        assert r.cg_iterations == int(z[f"cg_{tag}_its"][n])
        assert rel(r.solution, z[f"cg_{tag}_x"][:, n]) < 1e-9
        assert r.final_residual_norm <= tol


@pytest.mark.parametrize("name", ["metal.npz", "insulator.npz"])
def test_chi0_matches_reference(name):
    z = load_golden(name)
    gs = oracle_gs(z)
    n = gs.n_occ
    for tag, tol in (("t13", 1e-13), ("t8", 1e-8), ("t4", 1e-4)):
        drho, st = orsp.chi0(gs, z["dv"][0], np.full(n, tol))
        assert list(st.cg_iterations_per_band) == list(z[f"chi0_{tag}_its"])
        assert rel(drho, z[f"chi0_{tag}"]) < 1e-9
    drho, st = orsp.chi0(gs, z["dv"][1], z["chi0_mixed_tols"])
    assert rel(drho, z["chi0_mixed"]) < 1e-9
    drho, _ = orsp.chi0(gs, np.full(gs.grids.n_g, 2.4), np.full(n, 1e-13))
    assert np.linalg.norm(drho) <= 1e-10 * 2.4 * gs.model.n_electrons


@pytest.mark.parametrize("name", ["metal.npz", "insulator.npz"])
def test_kernels_dielectric_bounds(name):
    z = load_golden(name)
    gs = oracle_gs(z)
    for xc in ("none", "lda_x"):
        k = orsp.coulomb_kernel(xc, gs.grids, gs.rho, z["dv"][2])
        assert rel(k, z[f"kernel_{xc}"]) < 1e-13
        app = orsp.dielectric(gs, xc, z["dv"][2], np.full(gs.n_occ, 1e-12))
        assert app.kv_norm == pytest.approx(float(z[f"diel_{xc}_kv"]), rel=1e-13)
        assert rel(app.output, z[f"diel_{xc}"]) < 1e-10
    assert rel(orsp.kerker(0.8, gs.grids, z["dv"][2]), z["kerker_08"]) < 1e-13
    assert orsp.row_norm(gs.grids, gs.phi_occ) == pytest.approx(float(z["row_norm_abs"]), rel=1e-13)
    assert orsp.row_norm(gs.grids, gs.phi_occ, True) == pytest.approx(float(z["row_norm_re"]),
                                                                     rel=1e-13)
    assert orsp.error_bound(gs, 1.7, z["bound_tols"]) == pytest.approx(float(z["bound"]), rel=1e-12)


def test_strategies_match_reference():
    z = load_golden("strategies.npz")
    for i in range(int(z["n_cases"])):
        kind, pre, use_gap, it, cf = z[f"case{i}_spec"]
        spec = oo.Strategy(kind, pre == "True", 1e-8, 10, use_gap == "True")
        ctx = oo.Context(iteration=int(it), n_occ=6, occ=z["occ"], volume=1000.0, n_g=13824,
                         est_res_prev=3e-3, s=0.4, kv_norm=1.3, row_norm=0.6, rhs_norm=0.25,
                         eps_gap=z["gaps"], common_factor=None if cf == "None" else float(cf))
        np.testing.assert_array_equal(oo.select(spec, ctx), z[f"case{i}_tol"])


@pytest.mark.parametrize("tag", ["a", "b"])
def test_igmres_matches_reference(tag):
    z = load_golden("igmres.npz")
    a, b = z[f"{tag}_a"], z[f"{tag}_b"]
    rep = oo.igmres(lambda v, budget: (a @ v, 1), b, m=int(z[f"{tag}_m"]),
                    tau=float(z[f"{tag}_tau"]))
    assert rep.iterations == int(z[f"{tag}_its"])
    np.testing.assert_allclose(rep.solution, z[f"{tag}_x"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(rep.est_res_history, z[f"{tag}_hist"], rtol=1e-10)
    np.testing.assert_allclose([bb[2] for bb in rep.budgets], z[f"{tag}_budgets"], rtol=1e-10)


@pytest.mark.parametrize("fixture,strategy", [("dyson_metal.npz", "pbal"),
                                              ("dyson_metal.npz", "bal"),
                                              ("dyson_metal.npz", "d10"),
                                              ("dyson_metal.npz", "pagr"),
                                              ("dyson_cfg0.npz", "bal")])
def test_dyson_solve_matches_reference(fixture, strategy):
    z = load_golden(fixture)
    gs = oracle_gs(z)
    meta = z[f"{strategy}_meta"]
    spec = oo.parse(str(meta[0]), float(meta[1]), int(meta[2]))
    res = od.solve(gs, z["dv0"], spec, xc=gs.model.xc)
    assert res.converged
    assert abs(res.iterations - int(z[f"{strategy}_iterations"])) <= 1
    assert rel(res.rhs, z[f"{strategy}_rhs"]) < 1e-10
    assert rel(res.solution, z[f"{strategy}_solution"]) < 1e-8
    assert res.n_ham == int(z[f"{strategy}_n_ham"])
    np.testing.assert_allclose(res.tolerance_schedule[0], z[f"{strategy}_rhs_tols"], rtol=1e-12)
    ops = z[f"{strategy}_op_tols"]
    assert len(res.tolerance_schedule) - 1 == len(ops)
    for got, want in zip(res.tolerance_schedule[1:], ops):
        np.testing.assert_allclose(got, want, rtol=1e-6)


def test_kpoint_oracle_matches_gamma_supercell():
    """App. B: sum_k w_k chi0_k on the unit cell = reference chi0 of the supercell."""
    z = load_golden("kpoint_supercell.npz")
    cell = ob.Cell(z["unit_lattice"])
    wells = tuple(om.Well(center=tuple(w[:3]), amplitude=float(w[3]), width=float(w[4]))
                  for w in z["unit_wells"])
    model = om.Model(lattice=cell, e_cut=float(z["unit_e_cut"]), n_electrons=4,
                     temperature=5e-3, gaussians=wells)
    ks = om.scf_k(model, [[0, 0, 0], [0.5, 0, 0]], tol=1e-12, max_iter=600, damping=0.3)
    n = sum(b.n_occ for b in ks.blocks)
    drho_u, _ = orsp.chi0_k(ks, z["dv_unit"], np.full(n, 1e-13))
    nx, ny, nz = (int(d) for d in z["unit_dims"])
    cube = drho_u.reshape((nx, ny, nz), order="F")
    dup = np.concatenate([cube, cube], axis=0).ravel(order="F")
    assert rel(dup, z["drho_sup"]) < 1e-8
