"""configs[4]-shaped kernel driver for ncu captures (no SCF): a 64^3 sphere (cubic 20
bohr, E_cut 12, n_b 15 895), a state of `--nocc` random orthonormal orbitals, one
batched H apply of `--bands` rows and one projector Q X of `--rows` rows (the full
width of a configs[4] Sternheimer batch is 2 090-2 119 rows), each `--reps`
times, timed with CUDA events.

    python tools/kbench4.py [--what hq] [--rows 2119] [--bands 2119] [--nocc 68]
    ncu --set full -k regex:"k_projw|k_proj_" -s 2 -c 2 -o out python tools/kbench4.py --what q
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="hq")
    ap.add_argument("--rows", type=int, default=2119)
    ap.add_argument("--bands", type=int, default=2119)
    ap.add_argument("--nocc", type=int, default=68)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--alat", type=float, default=20.0)
    ap.add_argument("--ecut", type=float, default=12.0)
    a = ap.parse_args()
    import torch

    import bench
    from paper_2505_02319_b200 import _lib, synth
    from paper_2505_02319_b200.device import device_state, ptr
    from paper_2505_02319_b200.ops import ham_apply_dev
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids
    g = build_grids(Lattice.cubic(a.alat), a.ecut)
    rng = np.random.default_rng(0)
    v = synth.smoothed_uniform(g.g2_cube, g.cube_dims, rng)
    phi = synth.random_orthonormal(rng, g.n_b, a.nocc)
    ds = device_state(bench._MicroState(g, phi, np.zeros(a.nocc), v))
    dg = ds.grid
    lib = _lib.load()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    if "h" in a.what:
        x = torch.randn(a.bands, dg.nbp, dtype=torch.complex128, device="cuda")
        x[:, g.n_b:] = 0
        vt = torch.from_numpy(v).cuda()
        ms = timed(lambda: ham_apply_dev(dg, x, vt))
        bh = 64.0 * g.n_g + 32.0 * g.n_b
        print(f"H apply {g.cube_dims} x {a.bands}: {ms:.3f} ms, {ms / a.bands * 1e3:.2f} us/band, "
              f"B_H model {bh * a.bands / ms / 1e6:.0f} GB/s")
        del x
    if "q" in a.what:
        X = torch.randn(a.rows, dg.nbp, dtype=torch.complex128, device="cuda")
        X[:, g.n_b:] = 0
        ms = timed(lambda: _lib.check(lib.pwb_project_out(ds.handle, 0, a.rows, ptr(X))))
        fl = 16.0 * g.n_b * a.nocc * a.rows
        print(f"projector {a.rows} rows x {a.nocc} orbitals: {ms:.3f} ms, "
              f"{fl / ms / 1e9:.2f} TFLOP/s (algorithmic, 16 n_b n_occ per row)")


if __name__ == "__main__":
    main()
