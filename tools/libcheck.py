"""Library cross-check: the hand-written kernels beside cuFFT and
cuBLAS on the same shapes, timed with CUDA events (inputs larger than L2).

  * H apply (pwb_ham_apply: sphere -> cube inverse FFT, x V(r), forward FFT ->
    sphere, kinetic) vs the library pipeline torch/cuFFT would run for the
    same operator: scatter into the cube, batched Z2Z ifftn, multiply, fftn,
    gather (the minimum a library version needs; no pruning).
  * projector Q X on configs[4]'s shape (68 orbitals per k, 64^3 sphere) vs
    the cuBLAS ZGEMM pair X - (X Phi^H) Phi.

    python tools/libcheck.py [--bands 256] [--reps 5] > profiles/r02_libcheck.txt
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(torch, fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bands", type=int, default=256)
    ap.add_argument("--rows", type=int, default=2119)
    ap.add_argument("--nocc", type=int, default=68)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    import bench
    from paper_2505_02319_b200 import _lib, synth
    from paper_2505_02319_b200.device import device_state, ptr
    from paper_2505_02319_b200.ops import ham_apply_dev
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids
    for alat, ecut in ((15.0, 10.0), (20.0, 12.0), (20.0, 26.0)):
        g = build_grids(Lattice.cubic(alat), ecut)
        rng = np.random.default_rng(0)
        v = synth.smoothed_uniform(g.g2_cube, g.cube_dims, rng)
        phi = synth.random_orthonormal(rng, g.n_b, a.nocc)
        ds = device_state(bench._MicroState(g, phi, np.zeros(a.nocc), v))
        dg = ds.grid
        nb = a.bands if g.n_g < 500000 else 64
        x = torch.randn(nb, dg.nbp, dtype=torch.complex128, device="cuda")
        x[:, g.n_b:] = 0
        vt = torch.from_numpy(v).cuda()
        ms_h = timed(torch, lambda: ham_apply_dev(dg, x, vt), a.reps)
        # library pipeline of the same operator
        nx, ny, nz = g.cube_dims
        flat = torch.from_numpy(np.asarray(g.sphere_flat, dtype=np.int64)).cuda()
        kin = torch.from_numpy(0.5 * g.g2_sphere).cuda()
        vc = vt.reshape(nz, ny, nx)
        cube = torch.zeros(nb, g.n_g, dtype=torch.complex128, device="cuda")

        def lib_h():
            cube.zero_()
            cube[:, flat] = x[:, : g.n_b]
            u = torch.fft.ifftn(cube.view(nb, nz, ny, nx), dim=(1, 2, 3)) * vc
            w = torch.fft.fftn(u, dim=(1, 2, 3)).reshape(nb, g.n_g)
            return w[:, flat] / g.n_g + kin * x[:, : g.n_b]
        ms_lib = timed(torch, lib_h, a.reps)
        print(f"H apply {nx}x{ny}x{nz} n_b {g.n_b}, {nb} bands: pwb {ms_h / nb * 1e3:.2f} us/band,"
              f" cuFFT pipeline {ms_lib / nb * 1e3:.2f} us/band (x{ms_lib / ms_h:.2f})")
        del cube
        if g.n_g != 64 ** 3:
            continue
        rows = a.rows
        X = torch.randn(rows, dg.nbp, dtype=torch.complex128, device="cuda")
        X[:, g.n_b:] = 0
        P = dg.pack(list(phi.T))
        lib = _lib.load()
        Y = X.clone()
        ms_q = timed(torch, lambda: _lib.check(lib.pwb_project_out(ds.handle, 0, rows, ptr(Y))), a.reps)

        def zgemm():
            return X - (X @ P.conj().T) @ P
        ms_z = timed(torch, zgemm, a.reps)
        fl = 16.0 * g.n_b * a.nocc * rows
        print(f"projector {rows} rows x {a.nocc} orbitals (n_b {g.n_b}): pwb {ms_q:.3f} ms "
              f"({fl / ms_q / 1e9:.1f} TFLOP/s), cuBLAS ZGEMM pair {ms_z:.3f} ms "
              f"({fl / ms_z / 1e9:.1f} TFLOP/s)")


if __name__ == "__main__":
    main()
