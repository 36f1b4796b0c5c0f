"""Per-rank work of the (k, n)-sharded Dyson solve, measured on ONE GPU.

Only one GPU is available to this build, so the 1/2/4/8-rank scaling of
DESIGN.md section 6 cannot be timed over NCCL.  What CAN be measured is the
time each rank would spend on its own shard: a rank's chi0 work (RHS,
Sternheimer CG, accumulation of its rows) depends on no other rank until the
single all-reduce, so running shard r of N ALONE on the GPU times exactly what
rank r would run.  This tool

  1. runs one full solve of the config and records every chi0 call's input
     (dv, per-row tolerances);
  2. replays every recorded call on the full row range (the 1-rank time) and
     on each rank's band range for N in --worlds (pwb_chi0_begin / finish on
     [b0, b1): the same kernels the sharded path launches), timed with CUDA
     events;
  3. prints, per N: sum over calls of the slowest rank's time, the replicated
     remainder of the solve (GMRES, K v, host scalars: solve - sum of full
     chi0 times), the measured cost of an all-reduce-sized device copy as a
     stand-in floor, and the projected solve time and speed-up.

It is a projection from measured single-GPU pieces, not an NCCL measurement:
no rank waits on another here, and the all-reduce itself (2 MB over NVLink,
one per chi0) is not timed.

    python tools/shard_projection.py [--config 4] [--worlds 2 4 8] [--out FILE.json]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--worlds", type=int, nargs="*", default=[2, 4, 8])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch

    import bench
    from paper_2505_02319_b200.device import DeviceState, device_state, shard_range
    from paper_2505_02319_b200.harness import solve_dyson
    gs, dv0, p = bench.build_workload(a.config)
    ds = device_state(gs)
    dv0_t = torch.from_numpy(np.ascontiguousarray(dv0)).cuda()

    def solve():
        return solve_dyson(gs, dv0_t, strategy=p["strategy"], tau=p["tau"], m=p["m"], xc=p["xc"])

    solve()   # warm-up (graphs, plans)
    calls = []
    begin0, finish0 = DeviceState.chi0_begin, DeviceState.chi0_finish

    def rec_begin(self, dv_t):
        calls.append([dv_t.clone(), None])
        return begin0(self, dv_t)

    def rec_finish(self, tol):
        calls[-1][1] = np.array(tol, dtype=float, copy=True)
        return finish0(self, tol)

    DeviceState.chi0_begin, DeviceState.chi0_finish = rec_begin, rec_finish
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    res = solve()
    e1.record()
    torch.cuda.synchronize()
    solve_ms = e0.elapsed_time(e1)
    DeviceState.chi0_begin, DeviceState.chi0_finish = begin0, finish0

    def timed_call(dv_t, tol, rng):
        ds.shard = rng
        torch.cuda.synchronize()
        e0.record()
        ds.chi0_begin(dv_t)
        _, its = ds.chi0_finish(tol)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), int(np.sum(its))

    full = (0, ds.nband)
    for dv_t, tol in calls[:2]:
        timed_call(dv_t, tol, full)
    t_full = [timed_call(dv_t, tol, full) for dv_t, tol in calls]
    chi0_ms = sum(t for t, _ in t_full)
    rest_ms = solve_ms - chi0_ms
    # an all-reduce-sized buffer copied on the device: a floor for the collective's
    # local passes, NOT its NVLink time
    pk = torch.empty(2 * ds.grid.n_g + 2 + 2 * ds.nband, dtype=torch.float64, device="cuda")
    pk2 = torch.empty_like(pk)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        pk2.copy_(pk)
    e1.record()
    torch.cuda.synchronize()
    copy_ms = e0.elapsed_time(e1) / 20
    out = {"config": a.config, "solve_ms": solve_ms, "chi0_calls": len(calls),
           "chi0_ms_full_rows": chi0_ms, "replicated_ms": rest_ms,
           "n_ham": int(res.n_ham), "gmres_iterations": int(res.iterations),
           "packet_copy_ms": copy_ms, "worlds": {}}
    print(f"config {a.config}: solve {solve_ms:.1f} ms, {len(calls)} chi0 calls "
          f"{chi0_ms:.1f} ms (replay), replicated remainder {rest_ms:.1f} ms")
    for world in a.worlds:
        per_rank = np.zeros((len(calls), world))
        its_rank = np.zeros((len(calls), world))
        for r in range(world):
            rng = shard_range(ds.nocc, r, world)
            timed_call(calls[0][0], calls[0][1], rng)   # plans / graph of this range
            for c, (dv_t, tol) in enumerate(calls):
                per_rank[c, r], its_rank[c, r] = timed_call(dv_t, tol, rng)
        slowest = per_rank.max(axis=1).sum()
        rank_tot = per_rank.sum(axis=0)
        proj = slowest + rest_ms + len(calls) * copy_ms
        out["worlds"][str(world)] = {
            "rows_per_rank": [int(np.diff(shard_range(ds.nocc, r, world))[0]) for r in range(world)],
            "rank_chi0_ms": [float(x) for x in rank_tot],
            "rank_ham_applies": [int(x) for x in its_rank.sum(axis=0)],
            "sum_of_slowest_rank_per_call_ms": float(slowest),
            "projected_solve_ms": float(proj),
            "projected_speedup": float(solve_ms / proj),
            "chi0_only_speedup": float(chi0_ms / slowest),
        }
        print(f"  N={world}: per-rank chi0 totals {np.round(rank_tot, 1).tolist()} ms; "
              f"sum of per-call slowest {slowest:.1f} ms; projected solve {proj:.1f} ms "
              f"-> x{solve_ms / proj:.2f} (chi0 alone x{chi0_ms / slowest:.2f})")
    ds.shard = full
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
