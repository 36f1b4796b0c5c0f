"""The reference-side ctypes binding (integration/pwdyson_b200.py, numpy + ctypes
only) against the reference's golden outputs: what a pwdyson maintainer gets
after adding it as pwdyson/_b200.py."""

import importlib.util
import os

import numpy as np
import pytest

from conftest import ROOT, load_golden, oracle_gs, product_gs, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def binding():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    _lib.require_device()
    path = os.path.join(ROOT, "integration", "pwdyson_b200.py")
    spec = importlib.util.spec_from_file_location("pwdyson_b200", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("name", ["metal.npz", "insulator.npz"])
def test_binding_chi0_matches_reference_goldens(binding, name):
    z = load_golden(name)
    gs = product_gs(z)          # only the reference GroundState attributes are read
    n = gs.n_occ
    for tag, tol in (("t13", 1e-13), ("t8", 1e-8)):
        before = binding.ham_counter.value
        drho, st = binding.apply_chi0(gs, z["dv"][0], np.full(n, tol))
        want = list(z[f"chi0_{tag}_its"])
        assert all(abs(a - b) <= 1 for a, b in zip(st.cg_iterations_per_band, want))
        assert binding.ham_counter.value - before == st.ham_applications
        assert rel(drho, z[f"chi0_{tag}"]) < max(1e-9, 10 * tol)
    with pytest.raises(ValueError):
        binding.apply_chi0(gs, z["dv"][0], np.zeros(n))


def test_binding_hamiltonian_and_projector(binding, metal):
    from oracle import model as om
    from oracle import response as orsp
    gs = product_gs(metal)
    og = oracle_gs(metal)
    rng = np.random.default_rng(5)
    psi = rng.standard_normal(gs.grids.n_b) + 1j * rng.standard_normal(gs.grids.n_b)
    got = binding.apply_hamiltonian(gs.grids, gs.v_local, psi)
    want = om.ham_apply(og.grids, og.v_local, psi, count=False)
    assert rel(got, want) < 1e-13
    x = metal["proj_x"]
    assert rel(binding.project_out_occupied(gs.phi_occ, x), metal["proj_qx"]) < 1e-13
    assert rel(binding.project_out_occupied(gs.phi_occ, x[:, 0]),
               orsp.project_out(gs.phi_occ, x[:, 0])) < 1e-13
