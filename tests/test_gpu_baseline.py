"""Parity at the BASELINE configurations (seeded synthetic inputs)
against the CPU oracle, plus size-independent properties of chi0 at full size.
Needs a B200; the ground states are generated on the GPU (lobpcg.run_scf_gpu)
and fed to both the CUDA path and the oracle."""

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    _lib.require_device()


def _workload(cfg):
    import bench
    return bench.build_workload(cfg)


@pytest.fixture(scope="module")
def cfg0():
    return _workload(0)


@pytest.fixture(scope="module")
def cfg1():
    return _workload(1)


def test_cfg0_full_dyson_solve_matches_oracle(cfg0):
    """BASELINE configs[0]: the whole inexact-GMRES solve, GPU vs oracle, same inputs."""
    import bench
    from oracle import dyson as od
    from oracle import outer as oo
    from paper_2505_02319_b200.harness import solve_dyson
    gs, dv0, p = cfg0
    assert gs.n_occ == 4 and tuple(gs.grids.cube_dims) == (24, 24, 24)
    res = solve_dyson(gs, dv0, strategy=p["strategy"], tau=p["tau"], m=p["m"], xc=p["xc"])
    ref = od.solve(bench.to_oracle(gs), dv0, oo.parse(p["strategy"], p["tau"], p["m"]),
                   xc=p["xc"])
    assert res.converged and ref.converged
    assert abs(res.iterations - ref.iterations) <= 1
    assert rel(res.solution.cpu().numpy(), ref.solution) < 1e-8
    for got, want in zip(res.tolerance_schedule, ref.tolerance_schedule):
        np.testing.assert_allclose(got, want, rtol=1e-6)
    assert abs(res.n_ham - ref.n_ham) <= max(2, 0.02 * ref.n_ham)


def test_cfg1_first_chi0_matches_oracle(cfg1):
    """BASELINE configs[1] (48^3, 8 k-points, metallic, ragged N_occ per k): the RHS chi0
    apply of the solve (iteration-0 tolerances), GPU vs oracle chi0_k."""
    import bench
    from oracle import dyson as od
    from oracle import outer as oo
    from oracle import response as orsp
    from paper_2505_02319_b200.response import apply_chi0
    gs, dv0, p = cfg1
    assert len(gs.blocks) == 8 and tuple(gs.grids.cube_dims) == (48, 48, 48)
    og = bench.to_oracle(gs)
    nrm = float(np.linalg.norm(dv0))
    tols = od.tolerance_vector(og, oo.parse(p["strategy"], p["tau"], p["m"]), 0, kv_norm=nrm,
                               rhs_norm=1.0)
    drho, st = apply_chi0(gs, dv0 / nrm, tols)
    ref, rst = orsp.chi0_k(og, dv0 / nrm, tols)
    diff = np.abs(np.array(st.cg_iterations_per_band) - np.array(rst.cg_iterations_per_band))
    assert diff.max() <= 1 and diff.sum() <= 0.05 * len(diff)
    assert rel(drho, ref) < 1e-8


def test_cfg1_chi0_properties_at_full_size(cfg1):
    """Size-independent checks: neutrality, symmetry, negative semi-definiteness,
    linearity and bitwise reproducibility of chi0 on the full (k, n) batch."""
    from paper_2505_02319_b200 import synth
    from paper_2505_02319_b200.response import apply_chi0
    gs, dv0, p = cfg1
    g = gs.grids
    rng = np.random.default_rng(11)
    u = synth.smoothed_noise(g.g2_cube, g.cube_dims, rng)
    v = synth.smoothed_noise(g.g2_cube, g.cube_dims, rng)
    tight = np.full(gs.n_occ, 1e-11)
    cu, _ = apply_chi0(gs, u, tight)
    cv, _ = apply_chi0(gs, v, tight)
    cuv, _ = apply_chi0(gs, 0.3 * u - 1.7 * v, tight)
    nrm = np.linalg.norm(cu)
    assert abs(cu.sum()) <= 1e-8 * nrm * np.sqrt(g.n_g)            # charge neutral
    assert abs(u @ cv - v @ cu) <= 1e-8 * np.linalg.norm(u) * np.linalg.norm(cv)   # symmetric
    assert u @ cu <= 1e-10 and v @ cv <= 1e-10                       # negative semi-definite
    assert rel(cuv, 0.3 * cu - 1.7 * cv) < 1e-8                      # linear
    again, _ = apply_chi0(gs, u, tight)
    np.testing.assert_array_equal(again, cu)                         # deterministic


def test_cfg3_microbench_step_matches_oracle():
    """BASELINE configs[3] (96^3, 256 random orthonormal bands): the batched H apply and
    the projected-CG first step (rhs = -Q(V psi), 5 Q) against the oracle on 6 bands."""
    from oracle import basis as ob
    from oracle import model as om
    from oracle import response as orsp
    from paper_2505_02319_b200 import ops, synth
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids
    from paper_2505_02319_b200.sternheimer import project_out_occupied
    p, _, rng = synth.model_parameters(3)
    g = build_grids(Lattice.from_vectors(*synth.cell_vectors(p["cell"])), p["e_cut"])
    assert tuple(g.cube_dims) == (96, 96, 96)
    phi = synth.random_orthonormal(rng, g.n_b, 256)
    v = synth.smoothed_uniform(g.g2_cube, g.cube_dims, rng)
    b = ob.make_basis(ob.Cell(g.lattice.a), p["e_cut"])
    rows = [0, 1, 77, 128, 200, 255]
    h = ops.ham_apply_many(g, v, phi[:, rows].T)
    href = np.stack([om.ham_apply(b, v, phi[:, j], count=False) for j in rows])
    assert rel(h, href) < 1e-13
    x = phi[:, rows] + 0.1 * (rng.standard_normal((g.n_b, len(rows)))
                              + 1j * rng.standard_normal((g.n_b, len(rows))))
    assert rel(project_out_occupied(phi, x), orsp.project_out(phi, x)) < 1e-12
