"""Host-side gaps in a config-1 Dyson solve: wall time of the solve vs device time
inside the chi0 applies (CUDA events around each apply_chi0_dev) -- what the
GMRES / tolerance / launch bookkeeping on the host costs between device work.

    python tools/host_gaps.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2505_02319_b200 import harness, response
    from paper_2505_02319_b200.harness import solve_dyson
    gs, dv0, p = bench.build_workload(1)
    dv0_t = torch.from_numpy(dv0).cuda()
    kw = dict(strategy=p["strategy"], tau=p["tau"], m=p["m"], xc=p["xc"])
    for _ in range(2):
        solve_dyson(gs, dv0_t, **kw)
    rec = []
    orig = response.apply_chi0_dev

    def timed(gs_, dv_t, tols):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        t0 = time.perf_counter()
        e0.record()
        out = orig(gs_, dv_t, tols)
        e1.record()
        rec.append((e0, e1, time.perf_counter() - t0))
        return out
    response.apply_chi0_dev = timed
    harness.apply_chi0_dev = timed
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    res = solve_dyson(gs, dv0_t, sync_timing=False, **kw)
    e1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) * 1e3
    dev = e0.elapsed_time(e1)
    chi0_dev = sum(a.elapsed_time(b) for a, b, _ in rec)
    chi0_wall = sum(w for _, _, w in rec) * 1e3
    print(f"solve: wall {wall:.1f} ms, device span {dev:.1f} ms, {len(rec)} chi0 applies: "
          f"device {chi0_dev:.1f} ms, host wall inside them {chi0_wall:.1f} ms; outside chi0 "
          f"{dev - chi0_dev:.1f} ms of device span (GMRES, kernels, host gaps)")


if __name__ == "__main__":
    main()
