"""Optional extension (outside the parity path): Sternheimer
solves with the extra kept bands deflated (schur.py, the Schur-complement trick the
paper names, and the reference omits).  Checked for
consistency with the reference-parity solver, not for parity: both solve
Q (H - eps_n) Q x = b, so the solutions agree to the CG tolerance over the gap and
the deflated solve must not need more iterations.  Needs a B200."""

import numpy as np
import pytest

from conftest import load_golden, product_gs, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    _lib.require_device()


def _rhs(gs, seed):
    """Random right-hand sides in range(Q), one per occupied band."""
    rng = np.random.default_rng(seed)
    nb, nocc = gs.grids.n_b, gs.n_occ
    b = rng.standard_normal((nocc, nb)) + 1j * rng.standard_normal((nocc, nb))
    phi = gs.phi_occ
    return b - (b @ phi.conj()) @ phi.T


@pytest.mark.parametrize("name", ["dyson_cfg0.npz", "metal.npz"])
def test_schur_solve_agrees_with_parity_solver(name):
    from paper_2505_02319_b200.ops import ham_apply_many
    from paper_2505_02319_b200.schur import extra_band_residuals, solve_sternheimer_schur
    from paper_2505_02319_b200.sternheimer import solve_sternheimer_many
    gs = product_gs(load_golden(name))       # the reference's dense-eigh ground state
    assert gs.n_kept > gs.n_occ
    assert max(extra_band_residuals(gs)) < 1e-9
    bands = np.arange(gs.n_occ)
    rhs = _rhs(gs, 3)
    tol = np.full(gs.n_occ, 1e-10)
    x0, r0, it0 = solve_sternheimer_many(gs, None, bands, rhs, tol)
    x1, r1, it1 = solve_sternheimer_schur(gs, bands, rhs, tol)
    assert np.all(r1 <= tol)
    assert np.all(it1 <= it0) and it1.sum() < it0.sum()
    gap = gs.eps[gs.n_occ] - gs.eps[: gs.n_occ]
    for n in bands:
        assert np.linalg.norm(x1[n] - x0[n]) <= 4.0 * tol[n] / gap[n]
        # true residual of the ORIGINAL system: Q (H - eps_n) Q x - b
        phi = gs.phi_occ
        q = lambda v: v - phi @ (phi.conj().T @ v)
        hx = ham_apply_many(gs.grids, gs.v_local, q(x1[n])[None, :])[0]
        res = q(hx - gs.eps[n] * q(x1[n])) - rhs[n]
        assert np.linalg.norm(res) <= 2.0 * tol[n]


def test_schur_rejects_unconverged_extra_bands():
    from paper_2505_02319_b200.errors import ConfigurationError
    from paper_2505_02319_b200.schur import solve_sternheimer_schur
    gs = product_gs(load_golden("dyson_cfg0.npz"))
    phi = gs.phi.copy()
    phi[:, -1] += 1e-3 * np.roll(phi[:, -1], 1)       # spoil the last kept band
    import dataclasses
    bad = dataclasses.replace(gs, phi=phi)
    with pytest.raises(ConfigurationError):
        solve_sternheimer_schur(bad, [0], _rhs(gs, 1)[:1], [1e-8])


def test_gpu_scf_converges_kept_bands_for_schur():
    from paper_2505_02319_b200 import synth
    from paper_2505_02319_b200.groundstate import GaussianWell, ModelSpec
    from paper_2505_02319_b200.lobpcg import run_scf_gpu
    from paper_2505_02319_b200.pwbasis import Lattice
    from paper_2505_02319_b200.schur import extra_band_residuals, solve_sternheimer_schur
    from paper_2505_02319_b200.sternheimer import solve_sternheimer_many
    spec = synth.build_model(0, Lattice, GaussianWell, ModelSpec)
    gs = run_scf_gpu(spec["model"], tol=1e-9, eig_tol=1e-10, converge_kept=True)
    assert max(extra_band_residuals(gs)) < 1e-8
    bands = np.arange(gs.n_occ)
    rhs = _rhs(gs, 5)
    tol = np.full(gs.n_occ, 1e-9)
    x0, _, it0 = solve_sternheimer_many(gs, None, bands, rhs, tol)
    x1, _, it1 = solve_sternheimer_schur(gs, bands, rhs, tol)
    assert it1.sum() < it0.sum()
    assert rel(x1, x0) < 1e-6
