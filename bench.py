#!/usr/bin/env python
"""Benchmark: one inexact-GMRES delta_rho (Dyson) solve per step on the B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Metric (BASELINE.json): H*psi band-applies/s = N_Ham of the solve (RHS build
+ GMRES; one count per Sternheimer CG iteration of one (k, n) pair, exactly
the reference's ham_counter accounting) / device time of the solve; the
wall time per solve is `ms_per_step`.  `value` is measured with dV0 already
in HBM; `e2e` is the same solve through the public API with a host dV0 and
the host solution copied back inside the timed region.  Multi-GPU: one
process per GPU (torchrun), the (k, n) pairs are sharded, delta_rho is
NCCL-all-reduced once per chi0 apply, GMRES is replicated; time = max over
ranks; scaling "strong" (fixed total work).

`--impl reference` times the CPU oracle (numpy restatement of the
reference, oracle/) on the host cores with the same config and metric.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H*psi band-applies/s per inexact-GMRES delta_rho solve"
UNIT = "band-applies/s"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK = 6650.0
# DRAM bytes per band-apply of the H-apply kernels from the committed ncu --set full
# capture (profiles/r01_ncu_happly_summary.txt), for roofline.traffic
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=1)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget", type=float, default=15.0)
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------------------
# workload construction (setup, not timed)

def build_workload(cfg):
    """(gs, dv0 numpy, params) for a BASELINE config, seeded.

    The ground state is generated on the GPU (LOBPCG + k-point SCF, setup, not
    timed); dV0 is drawn from the same generator after the wells.
    """
    from paper_2505_02319_b200 import synth
    from paper_2505_02319_b200.groundstate import GaussianWell, ModelSpec
    from paper_2505_02319_b200.lobpcg import run_scf_gpu
    from paper_2505_02319_b200.pwbasis import Lattice
    if cfg not in (0, 1, 2, 4):
        raise SystemExit(f"config {cfg} is not a Dyson-solve workload")
    spec = synth.build_model(cfg, Lattice, GaussianWell, ModelSpec)
    gs = run_scf_gpu(spec["model"], kgrid=spec["params"]["kgrid"], tol=1e-9)
    g = gs.grids
    dv0 = synth.smoothed_noise(g.g2_cube, g.cube_dims, spec["rng"])
    return gs, dv0, spec["params"]


def workload_desc(cfg, gs, params):
    from paper_2505_02319_b200.device import state_blocks
    blocks, _ = state_blocks(gs)
    g = blocks[0].grids
    return {
        "workload": f"BASELINE configs[{cfg}]: full inexact-GMRES Dyson solve (RHS + GMRES)",
        "cube": list(g.cube_dims), "n_b": int(g.n_b), "n_k": len(blocks),
        "n_occ_per_k": [int(b.n_occ) for b in blocks],
        "strategy": params["strategy"], "tau": params["tau"], "m": params["m"],
        "xc": params["xc"], "temperature": params["temperature"],
        "perturbation": "seeded white noise, Gaussian-smoothed (sigma 1 bohr), seed 0",
        "l2": "flushed (256 MiB write) between timed steps",
    }


# ----------------------------------------------------------------------------------------
# clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() in ("active", "0x1", "1"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------------------

def peaks():
    try:
        with open(PEAKS_FILE) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


def roofline_from_profile(prof, gs):
    """Dominant kernel group of the solve and its achieved HBM bandwidth.

    The H apply's algorithmic bytes per band-apply are SURVEY.md 8(d)'s
    3-pass full-cube model B_H = 64 N_g + 32 N_b; the pruned-plane traffic
    of this implementation is reported beside it.
    """
    from paper_2505_02319_b200.device import state_blocks
    blocks, _ = state_blocks(gs)
    g = blocks[0].grids
    n_g, n_b = g.n_g, int(np.mean([b.grids.n_b for b in blocks]))
    peak, how = peaks()
    shares = {k: v[0] for k, v in prof.items()}
    total = sum(shares.values())
    ms, count, units = prof["ham_apply"]
    b_h = 64.0 * n_g + 32.0 * n_b
    avg_ms = ms / max(count, 1)
    bands = units / max(count, 1)
    bytes_per_launch = b_h * bands
    achieved = bytes_per_launch / (avg_ms * 1e-3) / 1e9 if avg_ms > 0 else 0.0
    traffic, traffic_src = None, None
    try:
        with open(TRAFFIC_FILE) as fh:
            t = json.load(fh)["ham_apply"]
        if n_g == 48 ** 3:   # the capture is of this grid
            traffic = t["dram_bytes_per_band_apply"] * bands
            traffic_src = t["capture"]
    except (OSError, KeyError, ValueError):
        pass
    return {
        "kernel": "ham_apply (plane_inv + pencil V(r) + plane_fwd, one batched H psi)",
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
        "peak_source": how,
        "algorithmic_bytes_per_band_apply": b_h,
        "avg_launch_ms": avg_ms, "bands_per_launch": units / max(count, 1),
        "share_of_kernel_time": {k: (v / total if total > 0 else 0.0) for k, v in shares.items()},
        "kernel_ms": shares,
    }


def oracle_sample(gs, dv0, params, budget_s):
    """Bounded CPU sample of the workload: the oracle's RHS + Sternheimer solves of
    the first (k, n) pairs at the solve's iteration-0 tolerances, band-applies/s."""
    from oracle import dyson as od
    from oracle import model as om
    from oracle import outer as oo
    from oracle import response as orsp
    og = to_oracle(gs)
    spec = oo.parse(params["strategy"], params["tau"], params["m"])
    nrm = float(np.linalg.norm(dv0))
    tols = od.tolerance_vector(og, spec, 0, kv_norm=nrm, rhs_norm=1.0)
    blk = og.blocks[0] if hasattr(og, "blocks") else og
    t0 = time.perf_counter()
    start = om.ham_counter.value
    b = blk.grids
    done = 0
    dv = dv0 / nrm
    for n in range(blk.n_occ):
        pr = b.to_real(blk.phi[:, n])
        rhs = -orsp.project_out(blk.phi_occ, b.to_fourier(dv * pr))
        orsp.sternheimer(blk, blk.v_local, n, rhs, tols[n])
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    nh = om.ham_counter.value - start
    return nh / dt, f"{done} (k=0, n) Sternheimer solves with RHS FFTs at the iteration-0 " \
                    f"tolerances ({nh} band-applies in {dt:.1f} s), oracle/ numpy port, 1 thread"


def cpu_baseline(gs, dv0, params, budget_s):
    """Oracle (numpy port of the reference) on the host, bounded sample."""
    from oracle import dyson as od
    from oracle import model as om
    from oracle import outer as oo
    if hasattr(gs, "blocks") or gs.grids.n_g > 100000:
        v, sample = oracle_sample(gs, dv0, params, budget_s)
        return {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample}
    og = to_oracle(gs)
    spec = oo.parse(params["strategy"], params["tau"], params["m"])
    t0 = time.perf_counter()
    n_ham, solves = 0, 0
    while True:
        start = om.ham_counter.value
        res = od.solve(og, dv0, spec, xc=params["xc"])
        n_ham += om.ham_counter.value - start
        solves += 1
        if time.perf_counter() - t0 > budget_s or solves >= 20:
            break
    dt = time.perf_counter() - t0
    return {"value": n_ham / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{solves} full Dyson solve(s) of the same workload, oracle/ numpy port "
                      f"(scipy.fft + OpenBLAS, 1 thread); {dt / solves * 1e3:.1f} ms per solve",
            "ms_per_solve": dt / solves * 1e3, "gmres_iterations": res.iterations}


def to_oracle(gs):
    from oracle import basis as ob
    from oracle import model as om
    m = gs.model
    cell = ob.Cell(m.lattice.a)
    model = om.Model(lattice=cell, e_cut=m.e_cut, n_electrons=m.n_electrons,
                     temperature=m.temperature, smearing=m.smearing, xc=m.xc,
                     gaussians=tuple(om.Well(g.center, g.amplitude, g.width)
                                     for g in m.gaussians))
    if hasattr(gs, "blocks"):
        blocks = [om.State(model=model, grids=ob.make_basis(cell, m.e_cut, b.grids.kfrac),
                           phi=b.phi, eps=b.eps, occ=b.occ, fermi_level=b.fermi_level,
                           rho=b.rho, n_occ=b.n_occ, v_local=b.v_local) for b in gs.blocks]
        return om.KState(model=model, blocks=blocks, weights=gs.weights, kfracs=gs.kfracs,
                         fermi_level=gs.fermi_level, rho=gs.rho, v_local=gs.v_local)
    return om.State(model=model, grids=ob.make_basis(cell, m.e_cut), phi=gs.phi, eps=gs.eps,
                    occ=gs.occ, fermi_level=gs.fermi_level, rho=gs.rho, n_occ=gs.n_occ,
                    v_local=gs.v_local)


# ----------------------------------------------------------------------------------------

def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing
    gs, dv0, params = build_workload(args.config)
    if hasattr(gs, "blocks") or gs.grids.n_g > 100000:
        vals = []
        t_all = time.perf_counter()
        for _ in range(args.warmup + args.steps):
            v, sample = oracle_sample(gs, dv0, params, 20.0)
            vals.append(v)
        value = float(np.mean(vals[args.warmup:]))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": (time.perf_counter() - t_all) / (args.warmup + args.steps) * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64/c128", "data": "synthetic",
                "config": workload_desc(args.config, gs, params),
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                                 "sample": "per step: " + sample +
                                 f" (host has {multiprocessing.cpu_count()} cores)"},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return
    from oracle import dyson as od
    from oracle import model as om
    from oracle import outer as oo
    og = to_oracle(gs)
    spec = oo.parse(params["strategy"], params["tau"], params["m"])
    for _ in range(args.warmup):
        od.solve(og, dv0, spec, xc=params["xc"])
    t0 = time.perf_counter()
    n_ham = 0
    for _ in range(args.steps):
        start = om.ham_counter.value
        od.solve(og, dv0, spec, xc=params["xc"])
        n_ham += om.ham_counter.value - start
    dt = time.perf_counter() - t0
    value = n_ham / dt
    cores = 1
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64/c128", "data": "synthetic",
            "config": workload_desc(args.config, gs, params),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{args.steps} full Dyson solves, oracle/ numpy port "
                                       f"(host has {multiprocessing.cpu_count()} cores)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    world, rank, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import device_state
    from paper_2505_02319_b200.harness import solve_dyson

    gs, dv0, params = build_workload(args.config)
    ds = device_state(gs)
    if world > 1:
        ds.set_sharding(rank, world, group)
    dev = torch.device("cuda", local)
    dv0_t = torch.from_numpy(dv0).to(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MiB > L2
    kw = dict(strategy=params["strategy"], tau=params["tau"], m=params["m"], xc=params["xc"])

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        solve_dyson(gs, dv0_t, **kw)

    # ---- timed region: device-resident inputs ----------------------------------------
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count()
    total_ms, n_ham, iters, step_ms = 0.0, 0, [], []
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = solve_dyson(gs, dv0_t, sync_timing=False, **kw)
        e1.record()
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        total_ms += step_ms[-1]
        n_ham += res.n_ham
        iters.append(res.iterations)
    barrier()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    # live per-kernel-group timing (CUDA events on the launching stream) over one more
    # identical solve; kept out of the timed loop so event records do not perturb it
    _lib.profile(True)
    flush.zero_()
    torch.cuda.synchronize()
    solve_dyson(gs, dv0_t, sync_timing=False, **kw)
    prof = _lib.profile_read()
    hist = _lib.profile_hist()
    _lib.profile(False)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = n_ham / (total_ms * 1e-3)

    # ---- e2e: public API with host buffers ------------------------------------------
    pinned = torch.from_numpy(dv0).pin_memory()
    e2e_ms, e2e_ham = 0.0, 0
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    for _ in range(e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        host_in = pinned.to(dev, non_blocking=True)
        r = solve_dyson(gs, host_in, sync_timing=False, **kw)
        sol = r.solution.cpu()
        e1.record()
        torch.cuda.synchronize()
        e2e_ms += e0.elapsed_time(e1)
        e2e_ham += r.n_ham
        del sol
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": e2e_ham / (e2e_ms * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": int(dv0.nbytes), "d2h_bytes_per_step": int(dv0.nbytes),
           "ms_per_step": e2e_ms / e2e_steps}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64/c128", "data": "synthetic",
            "config": dict(workload_desc(args.config, gs, params), parallelism=f"kn-shard{world}"),
            "n_ham_per_solve": n_ham / args.steps, "gmres_iterations": iters,
            "step_ms": [round(t, 3) for t in step_ms],
            "gpu_launches": int(launches), "clocks": clk, "e2e": e2e,
            "roofline": roofline_from_profile(prof, gs),
            "kernel_ms_by_live_rows": {
                cat: {f">={1 << b}": [round(ms, 2), n] for b, ms, n in rows}
                for cat, rows in hist.items() if cat in ("ham_apply", "projector", "cg_vector")}}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(gs, dv0, params, args.cpu_budget)
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
