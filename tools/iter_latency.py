"""Per-iteration latency of the batched projected CG vs live rows (config-1 state):
pwb_sternheimer on the first n rows with tol = 1e300 (init + exactly one iteration)
and with max_iter-bounded runs; CUDA-event timed, graph mode.

    python tools/iter_latency.py
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import bench
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import device_state, ptr
    gs, dv0, params = bench.build_workload(1)
    ds = device_state(gs)
    lib = _lib.load()
    dg = ds.grid
    rng = np.random.default_rng(0)
    only = os.environ.get("ITER_ROWS")
    for n in ((int(only),) if only else (1, 4, 16, 64, 128, 261)):
        bands = np.arange(n, dtype=np.int32)
        rhs = dg.rows(n)
        rhs.real.copy_(torch.from_numpy(rng.standard_normal((n, dg.nbp))))
        _lib.check(lib.pwb_project_out(ds.handle, 0, n, ptr(rhs)))   # k = 0 only is fine for timing
        x = torch.zeros_like(rhs)
        its = np.zeros(n, dtype=np.int32)
        res = np.zeros(n)
        out = {}
        for label, tolv, mi in (("1 it", 1e300, 0), ("10 its", 0.0, 10)):
            tol = np.full(n, tolv)

            def call():
                return lib.pwb_sternheimer(ds.handle, n, ctypes.c_void_p(bands.ctypes.data),
                                           ptr(rhs), ctypes.c_void_p(tol.ctypes.data), mi, ptr(x),
                                           ctypes.c_void_p(its.ctypes.data),
                                           ctypes.c_void_p(res.ctypes.data))
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(5):
                call()
            e1.record()
            torch.cuda.synchronize()
            out[label] = e0.elapsed_time(e1) / 5
        per_it = (out["10 its"] - out["1 it"]) / 9
        print(f"rows {n:4d}: init+1 it {out['1 it'] * 1e3:8.1f} us, 10 its {out['10 its'] * 1e3:8.1f} us"
              f" -> {per_it * 1e3:7.1f} us per iteration")
    if only:
        return
    # the solve's situation: a 261-row batch of which only `live` rows keep iterating
    n = 261
    bands = np.arange(n, dtype=np.int32)
    rhs = dg.rows(n)
    rhs.real.copy_(torch.from_numpy(rng.standard_normal((n, dg.nbp))))
    x = torch.zeros_like(rhs)
    its = np.zeros(n, dtype=np.int32)
    res = np.zeros(n)
    for live in (1, 4, 16, 64):
        out = {}
        for label, mi in (("2 its", 2), ("10 its", 10)):
            tol = np.full(n, 1e300)
            tol[:live] = 0.0

            def call():
                return lib.pwb_sternheimer(ds.handle, n, ctypes.c_void_p(bands.ctypes.data),
                                           ptr(rhs), ctypes.c_void_p(tol.ctypes.data), mi, ptr(x),
                                           ctypes.c_void_p(its.ctypes.data),
                                           ctypes.c_void_p(res.ctypes.data))
            for _ in range(2):
                call()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(5):
                call()
            e1.record()
            torch.cuda.synchronize()
            out[label] = e0.elapsed_time(e1) / 5
        per_it = (out["10 its"] - out["2 its"]) / 8
        print(f"batch 261, live {live:3d}: {per_it * 1e3:7.1f} us per iteration")


if __name__ == "__main__":
    main()
