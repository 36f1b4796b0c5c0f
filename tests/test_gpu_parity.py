"""Parity of the CUDA path (libpwb200 through the package API) with the golden
outputs of the unmodified reference and with the CPU oracle.  Needs a B200."""

import numpy as np
import pytest

from conftest import grid_cases, load_golden, oracle_gs, product_gs, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    _lib.require_device()


def _grids(z, case):
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids
    return build_grids(Lattice.from_vectors(*z[case + "_a"]), float(z[case + "_ecut"]))


@pytest.mark.parametrize("case", grid_cases())
def test_transforms_match_reference(grids_golden, case):
    from paper_2505_02319_b200 import ops
    z = grids_golden
    g = _grids(z, case)
    np.testing.assert_array_equal(g.g_int, z[case + "_g_int"])
    assert rel(ops.to_real_many(g, z[case + "_x"]), z[case + "_to_real"]) < 1e-13
    assert rel(ops.to_real(g, z[case + "_x"][0]), z[case + "_to_real0"]) < 1e-13
    assert rel(ops.to_fourier_many(g, z[case + "_u"]), z[case + "_to_fourier"]) < 1e-13
    assert rel(ops.ham_apply_many(g, z[case + "_v"], z[case + "_x"]), z[case + "_h"]) < 1e-13
    assert rel(ops.cube_fft(g, z[case + "_v"]), z[case + "_cube_fft"]) < 1e-13
    back = ops.cube_ifft(g, z[case + "_cube_fft"])
    assert rel(back.real, z[case + "_v"]) < 1e-13


def test_apply_hamiltonian_counts_and_validates(grids_golden):
    from paper_2505_02319_b200.groundstate import apply_hamiltonian, ham_counter
    z = grids_golden
    g = _grids(z, "toy_insulator")
    before = ham_counter.value
    out = apply_hamiltonian(g, z["toy_insulator_v"], z["toy_insulator_x"][1])
    assert ham_counter.value - before == 1
    assert rel(out, z["toy_insulator_h"][1]) < 1e-13
    with pytest.raises(ValueError):
        apply_hamiltonian(g, z["toy_insulator_v"], z["toy_insulator_x"][1][:-1])
    with pytest.raises(ValueError):
        apply_hamiltonian(g, z["toy_insulator_v"][:-1], z["toy_insulator_x"][1])


@pytest.mark.parametrize("name", ["metal.npz", "insulator.npz"])
def test_projector_kernels_rownorm(name):
    from paper_2505_02319_b200 import kernels as K
    from paper_2505_02319_b200 import response as R
    from paper_2505_02319_b200.sternheimer import project_out_occupied
    z = load_golden(name)
    gs = product_gs(z)
    assert rel(project_out_occupied(gs.phi_occ, z["proj_x"]), z["proj_qx"]) < 1e-13
    assert rel(project_out_occupied(gs.phi_occ, z["proj_x"][:, 0]), z["proj_qx"][:, 0]) < 1e-13
    for xc in ("none", "lda_x"):
        k = K.apply_kernel(K.KernelSpec(xc), gs.grids, gs.rho, z["dv"][2])
        assert rel(k, z[f"kernel_{xc}"]) < 1e-12
    assert rel(K.apply_kerker(K.KerkerSpec(0.8), gs.grids, z["dv"][2]), z["kerker_08"]) < 1e-12
    assert R.orbital_row_norm(gs.grids, gs.phi_occ) == pytest.approx(float(z["row_norm_abs"]),
                                                                     rel=1e-12)
    assert R.orbital_row_norm(gs.grids, gs.phi_occ, True) == pytest.approx(
        float(z["row_norm_re"]), rel=1e-12)
    assert R.dielectric_error_bound(gs, 1.7, z["bound_tols"]) == pytest.approx(float(z["bound"]),
                                                                               rel=1e-12)


@pytest.mark.parametrize("name", ["metal.npz", "insulator.npz"])
def test_eigen_shifts_and_occupied_response(name):
    from paper_2505_02319_b200 import response as R
    from oracle import response as orsp
    z = load_golden(name)
    gs = product_gs(z)
    de, def_, df = R.delta_eigen_occupations(gs, z["dv"][0])
    np.testing.assert_allclose(de, z["delta_eps"], rtol=1e-11, atol=1e-13)
    assert def_ == pytest.approx(float(z["delta_eps_f"]), rel=1e-11, abs=1e-13)
    np.testing.assert_allclose(df, z["delta_f"], rtol=1e-9, atol=1e-13)
    og = oracle_gs(z)
    assert rel(R.delta_phi_occupied(gs, z["dv"][0]), orsp.occupied_dphi(og, z["dv"][0])) < 1e-11
    np.testing.assert_allclose(R._occupied_pair_weights(gs), z["pair_weights"], rtol=1e-14)


@pytest.mark.parametrize("name", ["metal.npz", "insulator.npz"])
@pytest.mark.parametrize("tag,tol", [("t6", 1e-6), ("t10", 1e-10)])
def test_sternheimer_matches_reference(name, tag, tol):
    from paper_2505_02319_b200.groundstate import ham_counter
    from paper_2505_02319_b200.sternheimer import solve_sternheimer, solve_sternheimer_many
    z = load_golden(name)
    gs = product_gs(z)
    want_its = z[f"cg_{tag}_its"]
    before = ham_counter.value
    sols, res, its = solve_sternheimer_many(gs, gs.v_local, np.arange(gs.n_occ),
                                            z["cg_rhs"].T, np.full(gs.n_occ, tol))
    assert ham_counter.value - before == int(its.sum())
    for n in range(gs.n_occ):
        assert abs(int(its[n]) - int(want_its[n])) <= 1
        assert res[n] <= tol
        assert rel(sols[n], z[f"cg_{tag}_x"][:, n]) < max(1e-8, 50 * tol)
    r = solve_sternheimer(gs, gs.v_local, 0, z["cg_rhs"][:, 0], tol)
    assert r.cg_iterations == int(its[0])


def test_sternheimer_zero_rhs_and_max_iter(metal):
    from paper_2505_02319_b200.errors import NonConvergenceError
    from paper_2505_02319_b200.sternheimer import solve_sternheimer
    gs = product_gs(metal)
    r = solve_sternheimer(gs, gs.v_local, 0, np.zeros(gs.grids.n_b, complex), 1e-10)
    assert r.cg_iterations == 1 and np.linalg.norm(r.solution) == 0.0
    with pytest.raises(NonConvergenceError) as err:
        solve_sternheimer(gs, gs.v_local, 0, metal["cg_rhs"][:, 0], 1e-14, max_iter=2)
    assert err.value.residual is not None and err.value.residual > 0


@pytest.mark.parametrize("name", ["metal.npz", "insulator.npz"])
def test_chi0_matches_reference(name):
    from paper_2505_02319_b200.groundstate import ham_counter
    from paper_2505_02319_b200.response import apply_chi0
    z = load_golden(name)
    gs = product_gs(z)
    n = gs.n_occ
    for tag, tol in (("t13", 1e-13), ("t8", 1e-8), ("t4", 1e-4)):
        before = ham_counter.value
        drho, st = apply_chi0(gs, z["dv"][0], np.full(n, tol))
        assert ham_counter.value - before == st.ham_applications == sum(st.cg_iterations_per_band)
        want = list(z[f"chi0_{tag}_its"])
        assert all(abs(a - b) <= 1 for a, b in zip(st.cg_iterations_per_band, want))
        assert rel(drho, z[f"chi0_{tag}"]) < max(1e-9, 10 * tol)
    drho, _ = apply_chi0(gs, z["dv"][1], z["chi0_mixed_tols"])
    assert rel(drho, z["chi0_mixed"]) < 1e-5
    drho, _ = apply_chi0(gs, np.full(gs.grids.n_g, 2.4), np.full(n, 1e-13))
    assert np.linalg.norm(drho) <= 1e-10 * 2.4 * gs.model.n_electrons
    with pytest.raises(ValueError):
        apply_chi0(gs, z["dv"][0], np.full(n + 1, 1e-8))
    with pytest.raises(ValueError):
        apply_chi0(gs, z["dv"][0], np.zeros(n))


def test_chi0_bitwise_reproducible(metal):
    from paper_2505_02319_b200.response import apply_chi0
    gs = product_gs(metal)
    a, _ = apply_chi0(gs, metal["dv"][0], np.full(gs.n_occ, 1e-9), threads=1)
    b, _ = apply_chi0(gs, metal["dv"][0], np.full(gs.n_occ, 1e-9), threads=4)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name", ["metal.npz", "insulator.npz"])
def test_dielectric_matches_reference(name):
    from paper_2505_02319_b200.kernels import KernelSpec
    from paper_2505_02319_b200.response import apply_dielectric
    z = load_golden(name)
    gs = product_gs(z)
    for xc in ("none", "lda_x"):
        app = apply_dielectric(gs, KernelSpec(xc), z["dv"][2], np.full(gs.n_occ, 1e-12))
        assert app.kv_norm == pytest.approx(float(z[f"diel_{xc}_kv"]), rel=1e-12)
        assert rel(app.output, z[f"diel_{xc}"]) < 1e-9
    v = np.full(gs.grids.n_g, 3.3)
    app = apply_dielectric(gs, KernelSpec("none"), v, np.full(gs.n_occ, 1e-12))
    np.testing.assert_array_equal(app.output, v)
    assert app.kv_norm == 0.0 and app.ham_applications == 0


def test_kpoint_chi0_matches_gamma_supercell():
    """k-sampled chi0 on the GPU = reference Gamma supercell chi0."""
    from paper_2505_02319_b200.groundstate import GaussianWell, ModelSpec
    from paper_2505_02319_b200.pwbasis import Lattice
    from paper_2505_02319_b200.response import apply_chi0
    from paper_2505_02319_b200.scf import run_scf_k
    z = load_golden("kpoint_supercell.npz")
    wells = tuple(GaussianWell(center=tuple(w[:3]), amplitude=float(w[3]), width=float(w[4]))
                  for w in z["unit_wells"])
    model = ModelSpec(lattice=Lattice.from_vectors(*z["unit_lattice"]),
                      e_cut=float(z["unit_e_cut"]), n_electrons=4, temperature=5e-3,
                      gaussians=wells)
    ks = run_scf_k(model, [[0, 0, 0], [0.5, 0, 0]], tol=1e-12, max_iter=600, damping=0.3)
    drho, st = apply_chi0(ks, z["dv_unit"], np.full(ks.n_occ, 1e-13))
    nx, ny, nz = (int(d) for d in z["unit_dims"])
    cube = drho.reshape((nx, ny, nz), order="F")
    dup = np.concatenate([cube, cube], axis=0).ravel(order="F")
    assert rel(dup, z["drho_sup"]) < 1e-8


def test_two_phase_sharded_chi0_on_one_gpu(metal):
    """The per-rank C-ABI path (pwb_chi0_begin / pwb_chi0_finish on a band range),
    run for both halves in one process: the reduced Fermi numerator and the sum of
    the partial delta rho equal the unsharded chi0 (what NCCL does across GPUs)."""
    import ctypes

    import torch
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import device_state, ptr, shard_range
    from paper_2505_02319_b200.response import apply_chi0
    gs = product_gs(metal)
    tol = np.full(gs.n_occ, 1e-11)
    full, _ = apply_chi0(gs, metal["dv"][0], tol)
    ds = device_state(gs)
    lib = _lib.load()
    dv = torch.from_numpy(np.ascontiguousarray(metal["dv"][0])).cuda()
    ranges = [shard_range(ds.nocc, r, 2) for r in range(2)]
    fs = []
    for b0, b1 in ranges:
        f = torch.zeros(2, dtype=torch.float64, device="cuda")
        _lib.check(lib.pwb_chi0_begin(ds.handle, b0, b1, ptr(dv), ptr(f)))
        fs.append(f[0].item())
    total = torch.tensor([sum(fs), 0.0], dtype=torch.float64, device="cuda")
    parts = []
    for b0, b1 in ranges:
        f = torch.zeros(2, dtype=torch.float64, device="cuda")
        _lib.check(lib.pwb_chi0_begin(ds.handle, b0, b1, ptr(dv), ptr(f)))
        drho = torch.empty(gs.grids.n_g, dtype=torch.float64, device="cuda")
        its = np.zeros(b1 - b0, dtype=np.int32)
        tl = np.ascontiguousarray(tol[b0:b1])
        _lib.check(lib.pwb_chi0_finish(ds.handle, ptr(total), ctypes.c_void_p(tl.ctypes.data),
                                       ptr(drho), ctypes.c_void_p(its.ctypes.data)))
        parts.append(drho.cpu().numpy())
    assert abs(sum(fs)) > 0     # metallic: the Fermi-level term is exercised
    assert rel(parts[0] + parts[1], full) < 1e-12
