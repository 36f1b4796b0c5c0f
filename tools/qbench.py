"""Projector microbenchmark at config-1 shapes: Q X = X - Phi (Phi^H X) through
pwb_project_out (cached plan: exactly k_proj_coef + k_proj_apply per call) for
N_occ orbitals of a 48^3 sphere (n_b 5041) and a sweep of row counts.

    python tools/qbench.py [--nocc 33] [--reps 50]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--nocc", type=int, default=33)
    p.add_argument("--reps", type=int, default=50)
    p.add_argument("--alat", type=float, default=15.0)
    p.add_argument("--ecut", type=float, default=10.0)
    p.add_argument("--rows", default="1,4,16,32,64,128,261,522")
    a = p.parse_args()
    import torch
    import bench
    from paper_2505_02319_b200 import _lib, synth
    from paper_2505_02319_b200.device import device_state, ptr
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids
    g = build_grids(Lattice.cubic(a.alat), a.ecut)
    rng = np.random.default_rng(0)
    phi = synth.random_orthonormal(rng, g.n_b, a.nocc)
    ms = bench._MicroState(g, phi, np.zeros(a.nocc), np.zeros(g.n_g))
    ds = device_state(ms)
    lib = _lib.load()
    dg = ds.grid
    f_row = 16.0 * g.n_b * a.nocc
    for n in [int(v) for v in a.rows.split(",")]:
        X = torch.randn(n, dg.nbp, dtype=torch.complex128, device="cuda")
        X[:, g.n_b:] = 0
        for _ in range(3):
            _lib.check(lib.pwb_project_out(ds.handle, 0, n, ptr(X)))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.reps):
            lib.pwb_project_out(ds.handle, 0, n, ptr(X))
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / a.reps
        # check: Q X orthogonal to Phi
        P = torch.from_numpy(np.ascontiguousarray(phi.T)).cuda()
        c = torch.matmul(P.conj(), X[:, : g.n_b].T).abs().max().item()
        print(f"rows {n:4d}: {t * 1e3:7.1f} us  {f_row * n / (t * 1e-3) / 1e12:6.2f} TFLOP/s  "
              f"|Phi^H QX| {c:.1e}", flush=True)


if __name__ == "__main__":
    main()
