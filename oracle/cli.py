"""Oracle side of the parity exchange -- TEST INFRASTRUCTURE ONLY.

    python -m oracle.cli solve --workload DIR --out FILE.npz [--threads N]
        the oracle's Dyson solve (oracle.dyson.solve, harness.py:215-292) of a
        workload directory written by `paper_2505_02319_b200.cli ground-state`
        (read with oracle.archive: numpy only).
    python -m oracle.cli compare GPU.npz ORACLE.npz
        north_star's bar: GMRES iterations within 1, delta rho within 1e-8
        relative L2, the same Sternheimer tolerance schedule (rtol 1e-6);
        exit status 0 when it holds.
"""

import argparse
import json
import sys

import numpy as np


def _solve(args):
    from threadpoolctl import threadpool_limits

    from . import dyson, outer, response
    from .archive import load_workload
    st, dv0, p = load_workload(args.workload)
    response.BAND_THREADS = max(1, args.threads)
    with threadpool_limits(limits=1):
        res = dyson.solve(st, dv0, outer.parse(p["strategy"], p["tau"], p["m"]), xc=p["xc"])
    sched = np.zeros((len(res.tolerance_schedule), max(len(t) for t in res.tolerance_schedule)))
    for i, t in enumerate(res.tolerance_schedule):
        sched[i, : len(t)] = t
    np.savez(args.out, solution=res.solution, rhs=res.rhs, iterations=res.iterations,
             n_ham=res.n_ham, converged=res.converged, schedule=sched, impl="oracle")
    print(json.dumps({"iterations": res.iterations, "n_ham": res.n_ham,
                      "converged": bool(res.converged), "out": args.out}))


def compare(a, b):
    """dict of the parity measures between two solve outputs and a pass flag."""
    its = abs(int(a["iterations"]) - int(b["iterations"]))
    ref = np.asarray(b["solution"])
    err = float(np.linalg.norm(np.asarray(a["solution"]) - ref) / np.linalg.norm(ref))
    n = min(a["schedule"].shape[0], b["schedule"].shape[0])
    sa, sb = a["schedule"][:n], b["schedule"][:n]
    mask = sb != 0
    sched = float(np.max(np.abs(sa[mask] - sb[mask]) / np.abs(sb[mask]))) if mask.any() else 0.0
    ok = its <= 1 and err <= 1e-8 and sched <= 1e-6 and bool(a["converged"]) and \
        bool(b["converged"])
    return {"iterations": [int(a["iterations"]), int(b["iterations"])], "drho_rel_l2": err,
            "schedule_max_rel": sched, "n_ham": [int(a["n_ham"]), int(b["n_ham"])], "pass": ok}


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m oracle.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve")
    s.add_argument("--workload", required=True)
    s.add_argument("--out", required=True)
    s.add_argument("--threads", type=int, default=1)
    c = sub.add_parser("compare")
    c.add_argument("gpu")
    c.add_argument("oracle")
    args = ap.parse_args(argv)
    if args.cmd == "solve":
        _solve(args)
        return 0
    out = compare(np.load(args.gpu), np.load(args.oracle))
    print(json.dumps(out))
    return 0 if out["pass"] else 1


if __name__ == "__main__":
    sys.exit(main())
