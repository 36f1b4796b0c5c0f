"""install() rebinds the reference's chi0-path names (CPU: no operator is called).

Needs the reference source tree (present in the build container only); skipped
elsewhere.
"""

import importlib
import os
import sys

import pytest

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture()
def pwdyson():
    if not os.path.isdir(os.path.join(REF_SRC, "pwdyson")):
        pytest.skip("reference source tree not present")
    sys.path.insert(0, REF_SRC)
    try:
        mod = importlib.import_module("pwdyson")
        importlib.import_module("pwdyson.harness")
        yield mod
    finally:
        sys.path.remove(REF_SRC)


def test_install_rebinds_every_import_site(pwdyson):
    from paper_2505_02319_b200 import dropin as inst
    from paper_2505_02319_b200 import response, sternheimer
    import pwdyson.harness as h
    import pwdyson.response as r
    orig = r.apply_chi0
    names = inst.install(pwdyson)
    try:
        assert "harness.apply_chi0" in names and "response.solve_sternheimer" in names
        assert h.apply_chi0 is response.apply_chi0
        assert h.solve_sternheimer is sternheimer.solve_sternheimer
        assert r.apply_chi0 is response.apply_chi0
        assert r.project_out_occupied is sternheimer.project_out_occupied
        # the counter the reference's harness reads is the one our operators increment
        assert response.ham_counter is pwdyson.groundstate.ham_counter
        assert inst.install(pwdyson) == names          # idempotent
    finally:
        inst.uninstall(pwdyson)
    assert r.apply_chi0 is orig
    assert response.ham_counter is not pwdyson.groundstate.ham_counter


def test_reference_objects_have_the_duck_typed_fields(pwdyson):
    """DeviceGrid / DeviceState read only these attributes of the reference objects."""
    import numpy as np
    from pwdyson.pwbasis import Lattice, build_grids
    g = build_grids(Lattice.from_vectors([6.0, 0, 0], [0, 6.0, 0], [0, 0, 6.0]), 3.0)
    for attr in ("g_int", "g2_sphere", "g2_cube", "cube_dims", "n_b", "n_g"):
        assert hasattr(g, attr)
    assert g.lattice.volume > 0
    from pwdyson.groundstate import GroundState
    for attr in ("phi_occ", "eps_occ", "occ_occ", "fprime_occ"):
        assert hasattr(GroundState, attr)
