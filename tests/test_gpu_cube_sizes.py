"""chi0 parity on the larger BASELINE cubes (64^3 = configs[4], 96^3 = configs[3]),
where the H-apply pencil and the fused delta-rho accumulation run their two-pass
plans (64 = 16 x 4, 96 = 8 x 12), against the CPU oracle.  Small electron counts
keep the oracle's CPU solves to seconds; metallic smearing exercises the
Fermi-level term."""

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    _lib.require_device()


@pytest.mark.parametrize("e_cut,dims", [(12.0, 64), (26.0, 96)], ids=["64", "96"])
def test_chi0_on_large_cube_matches_oracle(e_cut, dims):
    import bench
    from oracle import response as orsp
    from paper_2505_02319_b200 import synth
    from paper_2505_02319_b200.groundstate import GaussianWell, ModelSpec
    from paper_2505_02319_b200.lobpcg import run_scf_gpu
    from paper_2505_02319_b200.pwbasis import Lattice
    from paper_2505_02319_b200.response import apply_chi0
    wells = (GaussianWell(center=(0.3, 0.4, 0.5), amplitude=-4.0, width=1.2),
             GaussianWell(center=(0.7, 0.6, 0.45), amplitude=-3.5, width=1.0))
    model = ModelSpec(lattice=Lattice.cubic(20.0), e_cut=e_cut, n_electrons=4,
                      temperature=2e-3, smearing="fermi_dirac", xc="lda_x", gaussians=wells)
    gs = run_scf_gpu(model, tol=1e-8, eig_tol=1e-7, n_states=16)
    assert tuple(gs.grids.cube_dims) == (dims,) * 3
    rng = np.random.default_rng(3)
    dv = synth.smoothed_noise(gs.grids.g2_cube, gs.grids.cube_dims, rng)
    dv /= np.linalg.norm(dv)
    tol = np.full(gs.n_occ, 1e-10)
    drho, st = apply_chi0(gs, dv, tol)
    ref, rst = orsp.chi0(bench.to_oracle(gs), dv, tol)
    diff = np.abs(np.array(st.cg_iterations_per_band) - np.array(rst.cg_iterations_per_band))
    assert diff.max() <= 1
    assert rel(drho, ref) < 1e-8
