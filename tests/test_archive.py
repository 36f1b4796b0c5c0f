"""Ground-state archives: the reference's format for Gamma
(archive.py:1-15, 55-120) read and written bit-exactly in both directions, and
the k-point extension round trip with the reference's error behaviour."""

import json
import os
import sys

import numpy as np
import pytest

from conftest import load_golden, product_gs

REF = "/root/reference/pkg/src"


def _kstate():
    from paper_2505_02319_b200.groundstate import GaussianWell, GroundState, KGroundState, ModelSpec
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids
    model = ModelSpec(lattice=Lattice.cubic(4.0), e_cut=3.0, n_electrons=4, temperature=5e-3,
                      gaussians=(GaussianWell(center=(0.3, 0.4, 0.5), amplitude=-3.0, width=0.8),))
    rng = np.random.default_rng(5)
    kf = np.array([[0, 0, 0], [0.5, 0, 0]], dtype=float)
    g0 = build_grids(model.lattice, model.e_cut, kf[0])
    rho, v = rng.standard_normal(g0.n_g), rng.standard_normal(g0.n_g)
    blocks = []
    for k in kf:
        g = build_grids(model.lattice, model.e_cut, tuple(k))
        phi = rng.standard_normal((g.n_b, 4)) + 1j * rng.standard_normal((g.n_b, 4))
        blocks.append(GroundState(model=model, grids=g, phi=phi, eps=np.sort(rng.random(4)),
                                  occ=np.array([2.0, 2.0, 1e-3, 0.0]), fermi_level=0.3,
                                  rho=rho, n_occ=3, v_local=v, scf_residual=1e-11))
    return KGroundState(model=model, blocks=blocks, weights=np.array([0.5, 0.5]), kfracs=kf,
                        fermi_level=0.3, rho=rho, v_local=v, scf_residual=1e-11)


def _same_block(a, b):
    np.testing.assert_array_equal(a.phi, b.phi)
    np.testing.assert_array_equal(a.eps, b.eps)
    np.testing.assert_array_equal(a.occ, b.occ)
    np.testing.assert_array_equal(a.rho, b.rho)
    np.testing.assert_array_equal(a.v_local, b.v_local)
    assert a.n_occ == b.n_occ and a.fermi_level == b.fermi_level
    np.testing.assert_array_equal(a.grids.g_int, b.grids.g_int)


def test_gamma_round_trip_bit_exact(tmp_path):
    from paper_2505_02319_b200.archive import load_ground_state, save_ground_state
    gs = product_gs(load_golden("metal.npz"))
    save_ground_state(str(tmp_path / "a"), gs)
    _same_block(gs, load_ground_state(str(tmp_path / "a")))
    assert json.load(open(tmp_path / "a" / "meta.json"))["format_version"] == 1


def test_kpoint_round_trip_and_errors(tmp_path):
    from paper_2505_02319_b200.archive import load_ground_state, save_ground_state
    from paper_2505_02319_b200.errors import ArchiveError
    ks = _kstate()
    p = str(tmp_path / "k")
    save_ground_state(p, ks)
    back = load_ground_state(p)
    assert len(back.blocks) == 2
    np.testing.assert_array_equal(back.weights, ks.weights)
    np.testing.assert_array_equal(back.kfracs, ks.kfracs)
    for a, b in zip(ks.blocks, back.blocks):
        _same_block(a, b)
    # truncated blob, missing blob, wrong version: ArchiveError like the reference
    with open(os.path.join(p, "phi_re_k1.bin"), "r+b") as fh:
        fh.truncate(64)
    with pytest.raises(ArchiveError):
        load_ground_state(p)
    os.remove(os.path.join(p, "phi_re_k1.bin"))
    with pytest.raises(ArchiveError):
        load_ground_state(p)
    meta = json.load(open(os.path.join(p, "meta.json")))
    meta["format_version"] = 7
    json.dump(meta, open(os.path.join(p, "meta.json"), "w"))
    with pytest.raises(ArchiveError):
        load_ground_state(p)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present (GPU box)")
def test_interoperates_with_reference_archives(tmp_path):
    sys.path.insert(0, REF)
    from pwdyson.archive import load_ground_state as ref_load, save_ground_state as ref_save
    from paper_2505_02319_b200.archive import load_ground_state, save_ground_state
    gs = product_gs(load_golden("metal.npz"))
    save_ground_state(str(tmp_path / "ours"), gs)
    _same_block(gs, ref_load(str(tmp_path / "ours")))          # reference reads ours
    ref_save(str(tmp_path / "theirs"), ref_load(str(tmp_path / "ours")))
    _same_block(gs, load_ground_state(str(tmp_path / "theirs")))   # we read the reference's
