"""Calibrate BASELINE config ground states on the GPU (setup): run the GPU SCF for a
config with given temperature/seed and report N_occ per k, gaps and timing."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--temperature", type=float, default=None)
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--tol", type=float, default=1e-9)
    p.add_argument("--scan", type=int, default=0, help="scan seeds 0..N-1 at loose tol")
    p.add_argument("--verbose", action="store_true")
    p.add_argument("--max-iter", type=int, default=200)
    p.add_argument("--n-electrons", type=int, nargs="*", default=None,
                   help="run the SCF for each of these electron counts (config 2 calibration)")
    args = p.parse_args()
    if args.scan:
        return scan(args)
    from paper_2505_02319_b200 import synth
    from paper_2505_02319_b200.groundstate import GaussianWell, ModelSpec
    from paper_2505_02319_b200.lobpcg import run_scf_gpu
    from paper_2505_02319_b200.pwbasis import Lattice
    from dataclasses import replace
    spec = synth.build_model(args.config, Lattice, GaussianWell, ModelSpec, seed=args.seed)
    model = spec["model"]
    if args.temperature is not None:
        model = replace(model, temperature=args.temperature)
    if args.n_electrons:
        from paper_2505_02319_b200.groundstate import fermi_and_occupations, smearing_function
        for nel in args.n_electrons:
            m = replace(model, n_electrons=nel)
            t0 = time.perf_counter()
            try:
                gs = run_scf_gpu(m, kgrid=spec["params"]["kgrid"], tol=args.tol,
                                 verbose=args.verbose, max_iter=args.max_iter,
                                 n_states=nel // 2 + max(6, nel // 4) + 20)
            except Exception as err:  # noqa: BLE001
                print(f"n_el {nel}: {err}", flush=True)
                continue
            e = np.asarray(gs.eps_all).reshape(-1)
            # N_occ implied by this spectrum for neighbouring electron counts
            occf, _ = smearing_function(m.smearing)
            implied = {}
            for n2 in range(max(2, nel - 24), nel + 25, 4):
                mu, _ = fermi_and_occupations(e, n2, m.temperature, m.smearing)
                f = occf((e - mu) / m.temperature)
                implied[n2] = int(np.max(np.nonzero(f > m.occupation_threshold)[0])) + 1
            print(f"n_el {nel}: n_occ {gs.n_occ} (scf {time.perf_counter() - t0:.0f} s, "
                  f"mu {gs.fermi_level:.5f}); same spectrum implies {implied}", flush=True)
        return
    t0 = time.perf_counter()
    gs = run_scf_gpu(model, kgrid=spec["params"]["kgrid"], tol=args.tol, verbose=True)
    dt = time.perf_counter() - t0
    blocks = gs.blocks if hasattr(gs, "blocks") else [gs]
    print(f"scf {dt:.1f} s, mu {gs.fermi_level:.6f}")
    for i, b in enumerate(blocks):
        n = b.n_occ
        print(f"k{i} n_b {b.grids.n_b} n_occ {n} eps[n-1] {b.eps[n-1]:.5f} eps[n] {b.eps[n]:.5f}"
              f" f[n-1] {b.occ[n-1]:.3e} f[n] {b.occ[n]:.3e}")


def scan(args):
    from dataclasses import replace
    from paper_2505_02319_b200 import synth
    from paper_2505_02319_b200.groundstate import GaussianWell, ModelSpec
    from paper_2505_02319_b200.lobpcg import run_scf_gpu
    from paper_2505_02319_b200.pwbasis import Lattice
    for seed in range(args.scan):
        spec = synth.build_model(args.config, Lattice, GaussianWell, ModelSpec, seed=seed)
        model = replace(spec["model"], temperature=1e-3)
        nel = model.n_electrons // 2
        try:
            gs = run_scf_gpu(model, kgrid=spec["params"]["kgrid"], tol=1e-6, eig_tol=1e-7)
        except Exception as err:  # noqa: BLE001
            print(f"seed {seed}: {err}")
            continue
        e = gs.eps_all
        gap = float(e[:, nel].min() - e[:, nel - 1].max())
        print(f"seed {seed}: indirect gap at band {nel}: {gap:+.5f} Ha  "
              f"(vbm {e[:, nel-1].max():.5f}, cbm {e[:, nel].min():.5f})", flush=True)


if __name__ == "__main__":
    main()
