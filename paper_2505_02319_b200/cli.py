"""Parity-exchange CLI: the on-disk handshake between GPU
runs and the CPU oracle.

    python -m paper_2505_02319_b200.cli ground-state --config C --out DIR
        GPU ground state of BASELINE configs[C] (lobpcg.run_scf_gpu, seeded
        App. A inputs) written as an archive (archive.py: the reference's
        format for Gamma, format 2 for k-points) + dv0.bin (the seeded
        perturbation) + workload.json (strategy, tau, m, xc, ...).
    python -m paper_2505_02319_b200.cli solve --workload DIR --out FILE.npz
        the inexact-GMRES Dyson solve of that workload on the GPU
        (harness.solve_dyson): solution, rhs, iterations, N_Ham, tolerance
        schedule.

The oracle side reads the same directory (`python -m oracle.cli solve`,
numpy only) and `python -m oracle.cli compare` applies north_star's bar.
bench.py's reference arm uses `ground-state` as its setup step, so the timed
CPU process never loads the CUDA library.
"""

import argparse
import json
import os
import sys
import time

import numpy as np


def make_workload(cfg):
    """(gs, dv0, params) for BASELINE configs[cfg] (seeded): the ground
    state from the GPU SCF, then dV0 drawn from the same generator after the wells."""
    from . import synth
    from .groundstate import GaussianWell, ModelSpec
    from .lobpcg import run_scf_gpu
    from .pwbasis import Lattice
    if cfg not in (0, 1, 2, 4):
        raise SystemExit(f"config {cfg} is not a Dyson-solve workload")
    spec = synth.build_model(cfg, Lattice, GaussianWell, ModelSpec)
    p = spec["params"]
    gs = run_scf_gpu(spec["model"], kgrid=p["kgrid"], tol=1e-9, n_states=p.get("n_states"))
    g = gs.grids
    dv0 = synth.smoothed_noise(g.g2_cube, g.cube_dims, spec["rng"])
    return gs, dv0, p


def write_workload(path, gs, dv0, params, extra=None):
    from .archive import save_ground_state
    save_ground_state(path, gs)
    np.asarray(dv0, dtype="<f8").tofile(os.path.join(path, "dv0.bin"))
    keep = {k: (list(v) if isinstance(v, tuple) else v) for k, v in params.items()}
    keep.update(extra or {})
    with open(os.path.join(path, "workload.json"), "w") as fh:
        json.dump(keep, fh, indent=1)


def read_workload(path):
    from .archive import load_ground_state
    with open(os.path.join(path, "workload.json")) as fh:
        params = json.load(fh)
    gs = load_ground_state(path)
    dv0 = np.fromfile(os.path.join(path, "dv0.bin"), dtype="<f8")
    if dv0.shape != (gs.grids.n_g,):
        raise ValueError("dv0.bin does not match the archive's grid")
    return gs, dv0, params


def _ground_state(args):
    t0 = time.perf_counter()
    gs, dv0, params = make_workload(args.config)
    scf_s = time.perf_counter() - t0
    os.makedirs(args.out, exist_ok=True)
    write_workload(args.out, gs, dv0, params, {"config": args.config, "scf_s": scf_s})
    print(json.dumps({"config": args.config, "out": args.out, "scf_s": round(scf_s, 2)}))


def _solve(args):
    from .harness import solve_dyson
    gs, dv0, p = read_workload(args.workload)
    res = solve_dyson(gs, dv0, strategy=p["strategy"], tau=p["tau"], m=p["m"], xc=p["xc"])
    sched = np.zeros((len(res.tolerance_schedule), max(len(t) for t in res.tolerance_schedule)))
    for i, t in enumerate(res.tolerance_schedule):
        sched[i, : len(t)] = t
    np.savez(args.out, solution=res.solution.cpu().numpy(), rhs=res.rhs.cpu().numpy(),
             iterations=res.iterations, n_ham=res.n_ham, converged=res.converged,
             schedule=sched, impl="gpu")
    print(json.dumps({"iterations": res.iterations, "n_ham": res.n_ham,
                      "converged": res.converged, "out": args.out}))


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2505_02319_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("ground-state")
    g.add_argument("--config", type=int, required=True)
    g.add_argument("--out", required=True)
    s = sub.add_parser("solve")
    s.add_argument("--workload", required=True)
    s.add_argument("--out", required=True)
    args = ap.parse_args(argv)
    {"ground-state": _ground_state, "solve": _solve}[args.cmd](args)


if __name__ == "__main__":
    sys.exit(main())
