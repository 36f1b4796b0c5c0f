"""Projector cost in the mid-width regime of a configs[4] solve: a 32-k-point state of
random orthonormal orbitals (68 per k on the 64^3 spheres, no SCF), one projected-CG
iteration (pwb_sternheimer, tol unreachable-high) on `rows` rows per k, with the
library's live per-group timing (CUDA events): projector ms per call and the
HBM rate of the Phi stream it implies (2 passes over Phi_k per Q per live k).

    python tools/qmid.py [--rows 1 2 4 8 16 32 66] [--nk 32]
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class _Block:
    def __init__(self, g, phi, eps, v):
        self.grids, self.phi_occ, self.eps_occ, self.v_local = g, phi, eps, v
        self.n_occ = phi.shape[1]
        self.occ_occ = np.full(self.n_occ, 2.0)
        self.rho = np.zeros_like(v)

    def fprime_occ(self):
        return np.zeros(self.n_occ)


class _KState:
    def __init__(self, blocks, v):
        self.blocks = blocks
        self.weights = np.full(len(blocks), 1.0 / len(blocks))
        self.v_local = v
        self.rho = np.zeros_like(v)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, nargs="*", default=[1, 2, 4, 8, 16, 32, 66])
    ap.add_argument("--nk", type=int, default=32)
    ap.add_argument("--nocc", type=int, default=68)
    a = ap.parse_args()
    import torch

    from paper_2505_02319_b200 import _lib, synth
    from paper_2505_02319_b200.device import device_state, ptr
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids, monkhorst_pack
    lat = Lattice.cubic(20.0)
    kfr = monkhorst_pack((4, 4, 2))[: a.nk]
    rng = np.random.default_rng(0)
    g0 = build_grids(lat, 12.0)
    v = synth.smoothed_uniform(g0.g2_cube, g0.cube_dims, rng)
    blocks = []
    for k in kfr:
        g = build_grids(lat, 12.0, k)
        blocks.append(_Block(g, synth.random_orthonormal(rng, g.n_b, a.nocc),
                             np.linspace(-1.0, 0.2, a.nocc), v))
    ks = _KState(blocks, v)
    ds = device_state(ks)
    lib = _lib.load()
    nbp = ds.grid.nbp
    print(f"{a.nk} k blocks x {a.nocc} orbitals, nbp {nbp}; Phi {a.nk * a.nocc * nbp * 16 / 1e6:.0f} MB")
    for rk in a.rows:
        rk = min(rk, a.nocc)
        bands = np.concatenate([ds.offsets[k] + np.arange(rk) for k in range(a.nk)]).astype(np.int32)
        n = len(bands)
        rhs = torch.randn(n, nbp, dtype=torch.complex128, device="cuda")
        for k in range(a.nk):
            rhs[k * rk:(k + 1) * rk, blocks[k].grids.n_b:] = 0
        x = torch.zeros_like(rhs)
        tol = np.full(n, 1e300)
        its = np.zeros(n, dtype=np.int32)
        res = np.zeros(n)

        def step():
            _lib.check(lib.pwb_sternheimer(ds.handle, n, ctypes.c_void_p(bands.ctypes.data),
                                           ptr(rhs), ctypes.c_void_p(tol.ctypes.data), 0, ptr(x),
                                           ctypes.c_void_p(its.ctypes.data),
                                           ctypes.c_void_p(res.ctypes.data)))
        step()
        _lib.profile(True)
        for _ in range(3):
            step()
        prof = _lib.profile_read()
        _lib.profile(False)
        ms, cnt, _ = prof["projector"]
        per = ms / max(cnt, 1)
        phi_bytes = 2.0 * a.nk * a.nocc * nbp * 16   # coef + apply stream Phi_k once each
        print(f"rows/k {rk:3d} ({n:5d} rows): projector {per * 1e3:8.1f} us per Q "
              f"(Phi stream {phi_bytes / (per * 1e-3) / 1e9:6.0f} GB/s), "
              f"H {prof['ham_apply'][0] / max(prof['ham_apply'][1], 1) * 1e3:8.1f} us")


if __name__ == "__main__":
    main()
