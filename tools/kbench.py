"""Kernel microbenchmark (BASELINE configs[3] style): one batched H apply and one
projector application on B random orthonormal bands, timed with CUDA events.

    python tools/kbench.py --ecut 10 --alat 15 --bands 256 --nocc 32 [--reps 20]

Used for ncu captures of the hot kernels without the SCF setup.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--alat", type=float, default=15.0)
    p.add_argument("--ecut", type=float, default=10.0)
    p.add_argument("--bands", type=int, default=256)
    p.add_argument("--nocc", type=int, default=32)
    p.add_argument("--reps", type=int, default=20)
    p.add_argument("--what", default="hq")
    a = p.parse_args()
    import torch
    from paper_2505_02319_b200 import synth
    from paper_2505_02319_b200.device import device_grid, ptr
    from paper_2505_02319_b200.ops import ham_apply_dev
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids
    from paper_2505_02319_b200 import _lib
    g = build_grids(Lattice.cubic(a.alat), a.ecut)
    dg = device_grid(g)
    rng = np.random.default_rng(0)
    v = synth.smoothed_uniform(g.g2_cube, g.cube_dims, rng)
    x = rng.standard_normal((a.bands, g.n_b)) + 1j * rng.standard_normal((a.bands, g.n_b))
    X = dg.pack(list(x))
    vt = torch.from_numpy(v).cuda()
    phi = synth.random_orthonormal(rng, g.n_b, a.nocc)
    phi_rows = torch.from_numpy(np.ascontiguousarray(phi.T)).cuda()
    lib = _lib.load()
    print(f"grid {g.cube_dims} n_b {g.n_b} nbp {dg.nbp} nxa {dg.nxa} nya {dg.nya} tile {dg.tile}")
    res = {}
    if "h" in a.what:
        for _ in range(3):
            ham_apply_dev(dg, X, vt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.reps):
            ham_apply_dev(dg, X, vt)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        bh = 64.0 * g.n_g + 32.0 * g.n_b
        res["H"] = ms
        print(f"H apply: {ms:.3f} ms per batch of {a.bands} -> {ms / a.bands * 1e3:.2f} us/band, "
              f"{a.bands / ms * 1e3:.0f} band-applies/s, B_H model {bh * a.bands / ms / 1e6:.0f} GB/s")
    if a.what == "qsweep":   # projector launches at CG-tail sizes (time them under ncu)
        nbp = dg.nbp
        phi = synth.random_orthonormal(rng, nbp, a.nocc)
        P = torch.from_numpy(np.ascontiguousarray(phi.T)).cuda()
        for ncol in (1, 4, 8, 16, 32, 64, 128, 256):
            Xs = torch.randn(ncol, nbp, dtype=torch.complex128, device="cuda")
            for _ in range(a.reps):
                lib.pwb_project_generic(nbp, a.nocc, ptr(P), ncol, ptr(Xs))
            torch.cuda.synchronize()
            print("ncol", ncol, "done")
        return
    if "q" in a.what:
        Y = X.clone()
        for _ in range(3):
            _lib.check(lib.pwb_project_generic(dg.nbp, a.nocc, ptr(torch.nn.functional.pad(
                phi_rows, (0, dg.nbp - g.n_b))), a.bands, ptr(Y)))
        pr = torch.nn.functional.pad(phi_rows, (0, dg.nbp - g.n_b)).contiguous()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.reps):
            lib.pwb_project_generic(dg.nbp, a.nocc, ptr(pr), a.bands, ptr(Y))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        fl = 16.0 * g.n_b * a.nocc * a.bands
        print(f"Q apply: {ms:.3f} ms per batch -> {fl / ms / 1e9:.2f} TFLOP/s (FP64)")
        # cuBLAS reference for the same two GEMMs (plumbing measurement of the FP64 peak)
        P = pr
        e0.record()
        for _ in range(a.reps):
            C = torch.matmul(P.conj(), X.T)
            X2 = X - torch.matmul(C.T, P)
        e1.record()
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1) / a.reps
        print(f"cuBLAS ZGEMM pair: {ms2:.3f} ms -> {fl / ms2 / 1e9:.2f} TFLOP/s")
        n = 8192
        A = torch.randn(n, n, dtype=torch.float64, device="cuda")
        torch.matmul(A, A)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            torch.matmul(A, A)
        e1.record()
        torch.cuda.synchronize()
        ms3 = e0.elapsed_time(e1) / 3
        print(f"cuBLAS DGEMM {n}^3: {2 * n ** 3 / ms3 / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
