"""The projector Q X = X - Phi (Phi^H X) (sternheimer.py:28-30) at the shapes the
benchmark runs: configs[4]'s 64^3 sphere with 68 orbitals per k block (wide-tile
kernels, projw.cu) and configs[3]'s 256 orbitals (16-row kernels, proj.cu),
against a float64 PyTorch (cuBLAS) reference of the same two products, for row
counts from one row (the CG tail) to several wide tiles."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    _lib.require_device()


def _state(alat, ecut, nocc, seed=0):
    import bench
    from paper_2505_02319_b200 import synth
    from paper_2505_02319_b200.device import device_state
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids
    g = build_grids(Lattice.cubic(alat), ecut)
    rng = np.random.default_rng(seed)
    phi = synth.random_orthonormal(rng, g.n_b, nocc)
    v = synth.smoothed_uniform(g.g2_cube, g.cube_dims, rng)
    ms = bench._MicroState(g, phi, np.linspace(-1.0, 0.5, nocc), v)
    return ms, device_state(ms), rng


@pytest.mark.parametrize("alat,ecut,nocc", [(20.0, 12.0, 68), (15.0, 10.0, 33), (12.0, 8.0, 20)])
def test_projector_matches_cublas(alat, ecut, nocc):
    import torch
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import ptr
    ms, ds, rng = _state(alat, ecut, nocc)
    dg = ds.grid
    lib = _lib.load()
    P = dg.pack(list(ms.phi_occ.T))                       # (nocc, nbp), zero padded
    # tile heights through every (m fragments, n fragments) pair a warp can own: the
    # wide kernels dispatch their inner loops on those counts (coef_chunk<CM, CN>)
    for ncol in (1, 7, 16, 24, 33, 40, 48, 56, 68, 72, 73, 150, 300):
        x = rng.standard_normal((ncol, dg.nb[0])) + 1j * rng.standard_normal((ncol, dg.nb[0]))
        X = dg.pack(list(x))
        want = X - (X @ P.conj().T) @ P
        _lib.check(lib.pwb_project_out(ds.handle, 0, ncol, ptr(X)))
        err = float(torch.linalg.norm(X - want) / torch.linalg.norm(want))
        assert err < 1e-13, (ncol, err)
        assert float(torch.abs(X[:, dg.nb[0]:]).max()) == 0.0 if dg.nbp > dg.nb[0] else True
        # idempotent: projecting again changes nothing beyond round-off
        Y = X.clone()
        _lib.check(lib.pwb_project_out(ds.handle, 0, ncol, ptr(Y)))
        assert float(torch.linalg.norm(Y - X) / torch.linalg.norm(X)) < 1e-13


def test_projector_is_deterministic():
    import torch
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import ptr
    ms, ds, rng = _state(20.0, 12.0, 68, seed=3)
    dg = ds.grid
    lib = _lib.load()
    x = rng.standard_normal((140, dg.nb[0])) + 1j * rng.standard_normal((140, dg.nb[0]))
    outs = []
    for _ in range(3):
        X = dg.pack(list(x))
        _lib.check(lib.pwb_project_out(ds.handle, 0, 140, ptr(X)))
        outs.append(X)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
