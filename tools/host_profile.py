"""cProfile of one config-1 Dyson solve (after warm-up): where the host time
outside the CUDA kernels goes (GMRES bookkeeping, tolerance vectors, launches).

    python tools/host_profile.py
"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2505_02319_b200.harness import solve_dyson
    gs, dv0, p = bench.build_workload(1)
    dv0_t = torch.from_numpy(dv0).cuda()
    kw = dict(strategy=p["strategy"], tau=p["tau"], m=p["m"], xc=p["xc"])
    for _ in range(2):
        solve_dyson(gs, dv0_t, **kw)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    solve_dyson(gs, dv0_t, sync_timing=True, **kw)
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
