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
import gc
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
# DRAM bytes per unit (band-apply / projected row) of the hot kernel groups from the
# committed ncu --set full captures, keyed by cube, for roofline.traffic
TRAFFIC_FILES = [os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")]


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=4)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget", type=float, default=15.0)
    return p.parse_args()


def dist_env():
    """(world, rank, local device).  PWB_SHARE_GPU=1 (control-flow check of the
    sharded path on a one-GPU box, never a measurement) maps every rank to the
    visible devices round-robin."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PWB_SHARE_GPU"):
        import torch
        local %= max(1, torch.cuda.device_count())
    return world, rank, local


# ----------------------------------------------------------------------------------------
# workload construction (setup, not timed)

def build_workload(cfg):
    """(gs, dv0 numpy, params) for a BASELINE config, seeded: the ground
    state from the GPU SCF (setup, not timed), dV0 drawn from the same generator
    after the wells (paper_2505_02319_b200.cli.make_workload)."""
    from paper_2505_02319_b200.cli import make_workload, read_workload
    wl = os.environ.get("PWB_WORKLOAD")   # development: reuse a `cli ground-state` directory
    if wl and os.path.exists(os.path.join(wl, "workload.json")):
        gs, dv0, params = read_workload(wl)
        if params.get("config") != cfg:
            raise SystemExit(f"PWB_WORKLOAD holds config {params.get('config')}, not {cfg}")
        params["kgrid"] = tuple(params["kgrid"])
        return gs, dv0, params
    return make_workload(cfg)


def workload_desc(cfg, gs, params):
    blocks = list(gs.blocks) if hasattr(gs, "blocks") else [gs]
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


def _traffic(cube, group):
    """Per-unit DRAM bytes of a kernel group from a committed ncu --set full capture
    (profiles/*_ncu_traffic.json, keyed by cube), or (None, None)."""
    key = "x".join(str(int(d)) for d in cube)
    for path in TRAFFIC_FILES:
        try:
            with open(path) as fh:
                t = json.load(fh)
        except (OSError, ValueError):
            continue
        ent = t.get(key, {}).get(group)
        if ent:
            return ent["dram_bytes_per_unit"], ent["capture"]
    return None, None


def _shares(prof):
    shares = {k: v[0] for k, v in prof.items()}
    total = sum(shares.values())
    return shares, {k: (v / total if total > 0 else 0.0) for k, v in shares.items()}


def roofline_from_profile(prof, gs):
    """HBM roofline of the H apply over the profiled solve.

    Algorithmic bytes per band-apply: SURVEY.md 8(d)'s 3-pass full-cube model
    B_H = 64 N_g + 32 N_b.  This implementation prunes the zero x planes, so
    its DRAM traffic is below B_H; `traffic` (ncu dram bytes of the same
    kernels per launch) and `frac_dram` (that traffic / launch time / peak)
    report the fraction on the bytes actually moved.
    """
    from paper_2505_02319_b200.device import state_blocks
    blocks, _ = state_blocks(gs)
    g = blocks[0].grids
    n_g, n_b = g.n_g, int(np.mean([b.grids.n_b for b in blocks]))
    peak, how = peaks()
    shares, frac = _shares(prof)
    ms, count, units = prof["ham_apply"]
    b_h = 64.0 * n_g + 32.0 * n_b
    avg_ms = ms / max(count, 1)
    bands = units / max(count, 1)
    achieved = b_h * bands / (avg_ms * 1e-3) / 1e9 if avg_ms > 0 else 0.0
    per, src = _traffic(g.cube_dims, "ham_apply")
    traffic = per * bands if per else None
    out = {
        "kernel": "ham_apply (plane_inv + pencil V(r) + plane_fwd, one batched H psi)",
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "traffic": traffic, "traffic_source": src,
        "peak_source": how,
        "algorithmic_bytes_per_band_apply": b_h,
        "avg_launch_ms": avg_ms, "bands_per_launch": bands,
        "share_of_kernel_time": frac, "kernel_ms": shares,
    }
    if traffic:
        out["achieved_dram"] = traffic / (avg_ms * 1e-3) / 1e9
        out["frac_dram"] = out["achieved_dram"] / peak
    return out


def projector_roofline(prof, gs, peak_fp64):
    """FP64 roofline of the projector GEMM group over the profiled solve.

    F_Q = 16 N_b N_occ flop per row per Q application (two complex
    GEMMs, 8 flop per complex MAC); rows = the live rows of every projector call
    (x and r count twice), N_occ the row-weighted mean over k blocks."""
    from paper_2505_02319_b200.device import state_blocks
    blocks, _ = state_blocks(gs)
    nocc = np.array([b.n_occ for b in blocks], dtype=float)
    nb = np.array([b.grids.n_b for b in blocks], dtype=float)
    f_row = 16.0 * float(np.sum(nocc * nb * nocc) / np.sum(nocc))
    ms, count, units = prof["projector"]
    achieved = f_row * units / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
    shares, frac = _shares(prof)
    per, src = _traffic(blocks[0].grids.cube_dims, "projector")
    rows = units / max(count, 1)
    wide = float(nocc.max()) <= 72   # projw.cu serves N_occ,k <= 72, proj.cu the rest
    pair = "k_projw_coef + k_projw_apply" if wide else "k_proj_coef + k_proj_apply"
    return {"kernel": f"projector Q X ({pair}), all CG calls of one solve",
            "bound": "tensor", "achieved": achieved, "peak": peak_fp64, "unit": "TFLOP/s (FP64)",
            "frac": achieved / peak_fp64, "traffic": per * rows if per else None,
            "traffic_source": src,
            "peak_source": "measured live: cuBLAS DGEMM 8192^3 best of 5 (MEASURED_PEAKS.json "
                           "has no FP64 entry)",
            "algorithmic_flop_per_row": f_row, "rows": int(units), "launch_pairs": int(count),
            "avg_rows_per_call": rows, "avg_launch_ms": ms / max(count, 1),
            "share_of_kernel_time": frac, "kernel_ms": shares}


def dominant_roofline(ham, proj):
    """The roofline object of the kernel group with the larger share of the solve."""
    sh = ham["share_of_kernel_time"]
    return dict(proj) if sh.get("projector", 0) >= sh.get("ham_apply", 0) else dict(ham)


def oracle_tolerances(og, dv0, params):
    """Iteration-0 Sternheimer tolerances of the solve (setup for oracle_sample: ~25 s
    of host time at configs[4], so the reference arm computes it once, not per step)."""
    from oracle import dyson as od
    from oracle import outer as oo
    spec = oo.parse(params["strategy"], params["tau"], params["m"])
    return od.tolerance_vector(og, spec, 0, kv_norm=float(np.linalg.norm(dv0)), rhs_norm=1.0)


def oracle_sample(og, dv0, params, budget_s, threads=1, tols=None):
    """Bounded CPU sample of the workload: the oracle's RHS + Sternheimer solves of
    the first (k, n) pairs at the solve's iteration-0 tolerances, band-applies/s.

    BLAS is pinned to one thread; `threads` > 1 runs the bands on a thread pool,
    the reference's own band parallelism (response.py:144-148, scipy.fft and
    OpenBLAS release the GIL)."""
    from concurrent.futures import ThreadPoolExecutor

    from threadpoolctl import threadpool_limits

    from oracle import dyson as od
    from oracle import model as om
    from oracle import outer as oo
    from oracle import response as orsp
    nrm = float(np.linalg.norm(dv0))
    if tols is None:
        tols = oracle_tolerances(og, dv0, params)
    blocks = og.blocks if hasattr(og, "blocks") else [og]
    pairs, off = [], 0
    for blk in blocks:                      # (k, n) pairs in the solve's order
        pairs += [(blk, n, off + n) for n in range(blk.n_occ)]
        off += blk.n_occ
    dv = dv0 / nrm

    def one(pair):
        blk, n, i = pair
        b = blk.grids
        pr = b.to_real(blk.phi[:, n])
        rhs = -orsp.project_out(blk.phi_occ, b.to_fourier(dv * pr))
        orsp.sternheimer(blk, blk.v_local, n, rhs, tols[i])

    done = 0
    with threadpool_limits(limits=1), ThreadPoolExecutor(max_workers=threads) as pool:
        t0 = time.perf_counter()
        start = om.ham_counter.value
        while done < len(pairs):
            batch = pairs[done:done + threads]
            list(pool.map(one, batch))
            done += len(batch)
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
        nh = om.ham_counter.value - start
    how = "1 thread" if threads == 1 else f"{threads}-thread band pool"
    return nh / dt, f"first {done} of {len(pairs)} (k, n) Sternheimer solves of the RHS chi0 " \
                    f"apply, with their RHS FFTs, at the iteration-0 tolerances ({nh} " \
                    f"band-applies in {dt:.1f} s), oracle/ numpy port, {how}, BLAS 1 thread"


def cpu_baseline(gs, dv0, params, budget_s):
    """Oracle (numpy port of the reference) on the host, bounded sample."""
    from oracle import dyson as od
    from oracle import model as om
    from oracle import outer as oo
    if hasattr(gs, "blocks") or gs.grids.n_g > 100000:
        v, sample = oracle_sample(to_oracle(gs), dv0, params, budget_s)
        return {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": sample}
    og = to_oracle(gs)
    spec = oo.parse(params["strategy"], params["tau"], params["m"])
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=1):
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
# BASELINE configs[3]: kernel microbench (one batched H apply + one projected-CG iteration)

def fp64_peak(dev):
    """Measured FP64 tensor throughput of this GPU: cuBLAS DGEMM 8192^3, best of 5 (TFLOP/s)."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, a)
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


class _MicroState:
    """GroundState-shaped holder for configs[3]'s random orthonormal bands."""

    def __init__(self, grids, phi, eps, v_local):
        self.grids, self.phi_occ, self.eps_occ, self.v_local = grids, phi, eps, v_local
        self.n_occ = phi.shape[1]
        self.occ_occ = np.full(self.n_occ, 2.0)
        self.rho = np.zeros_like(v_local)

    def fprime_occ(self):
        return np.zeros(self.n_occ)


def micro_setup(dev):
    """configs[3] inputs on `dev`: 96^3 grid, 256 random orthonormal bands (= Phi), V ~
    U(-1,1) smoothed, eps_n = Re <psi_n, H psi_n> (GPU H), rhs_n = -Q (V psi_n) as device
    rows, and the device state the Sternheimer step runs on."""
    import torch

    from paper_2505_02319_b200 import _lib, ops, synth
    from paper_2505_02319_b200.device import device_state, ptr
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids
    p, _, rng = synth.model_parameters(3)
    g = build_grids(Lattice.from_vectors(*synth.cell_vectors(p["cell"])), p["e_cut"])
    nb = p["n_bands"]
    phi = synth.random_orthonormal(rng, g.n_b, nb)
    v = synth.smoothed_uniform(g.g2_cube, g.cube_dims, rng)
    eps = np.zeros(nb)
    ds = device_state(_MicroState(g, phi, eps, v))
    dg = ds.grid
    vt = torch.from_numpy(v).to(dev)
    psi = dg.pack(list(phi.T))
    hpsi = ops.ham_apply_dev(dg, psi, vt)
    eps[:] = torch.sum(psi.conj() * hpsi, dim=1).real.cpu().numpy()
    ms = _MicroState(g, phi, eps, v)          # eps known now: the state the CG uses
    ds = device_state(ms)
    lib = _lib.load()
    # rhs_n = -Q (V psi_n): V psi in the sphere basis, then the projector
    rhs = -ops.to_fourier_many_dev(dg, ops.to_real_many_dev(dg, psi) * vt[None, :])
    _lib.check(lib.pwb_project_out(ds.handle, 0, nb, ptr(rhs)), "project_out")
    return dict(p=p, g=g, phi=phi, v=v, vt=vt, eps=eps, ms=ms, ds=ds, dg=dg, psi=psi, rhs=rhs,
                nb=nb)


def micro_step(m, x, rhs=None, tol_value=1e300):
    """One pwb_sternheimer call on the 256 rows of configs[3] (init Q + one iteration =
    1 batched H apply + 5 Q when tol_value is unreachable-high): returns (its, res)."""
    import ctypes

    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import ptr
    nb = m["nb"]
    bands = m.setdefault("bands", np.arange(nb, dtype=np.int32))
    tol = np.full(nb, tol_value)
    its = np.zeros(nb, dtype=np.int32)
    res = np.zeros(nb)
    _lib.check(_lib.load().pwb_sternheimer(
        m["ds"].handle, nb, ctypes.c_void_p(bands.ctypes.data),
        ptr(m["rhs"] if rhs is None else rhs), ctypes.c_void_p(tol.ctypes.data), 0, ptr(x),
        ctypes.c_void_p(its.ctypes.data), ctypes.c_void_p(res.ctypes.data)), "sternheimer")
    return its, res


def run_microbench(args):
    """configs[3]: 96^3 cube, 256 random orthonormal bands (Phi = the bands), V ~ U(-1,1)
    smoothed; eps_n = Re <psi_n, H psi_n>; step = one batched projected-CG iteration of
    the 256 Sternheimer rows rhs_n = -Q(V psi_n) through the C-ABI (pwb_sternheimer:
    init projection + one iteration = 1 batched H apply + 5 Q, the reference op
    sequence, sternheimer.py:59-91).  Separately timed: the batched H apply alone
    (HBM roofline) and one Q on the 256 rows (FP64 roofline)."""
    import torch

    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import ptr
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    m = micro_setup(dev)
    g, nb, ds, dg, psi, vt, rhs, p = (m[k] for k in ("g", "nb", "ds", "dg", "psi", "vt", "rhs",
                                                      "p"))
    lib = _lib.load()
    x = torch.zeros_like(rhs)
    its = np.zeros(nb, dtype=np.int32)

    def step():
        its[:] = micro_step(m, x)[0]

    def timed(fn, reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        step()
    assert np.all(its == 1)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count()
    step_ms = []
    gc.collect()
    gc.disable()   # no cyclic-GC pause inside the timed steps
    for _ in range(args.steps):
        flush.zero_()
        step_ms.append(timed(step, 1))
    launches = _lib.launch_count() - launches0
    gc.enable()
    clk = clocks.stop()
    ms_step = float(np.mean(step_ms))
    # the two kernel groups alone (inputs larger than L2: 256 rows x 50 685 x 16 B = 207 MB)
    out = dg.rows(nb)
    h_ms = timed(lambda: lib.pwb_ham_apply(dg.handle, nb, None, ptr(psi), ptr(vt), None,
                                           ptr(out)), 5)
    y = rhs.clone()
    q_ms = timed(lambda: lib.pwb_project_out(ds.handle, 0, nb, ptr(y)), 5)
    # e2e: host rhs in, host solution out, through the host-buffer C-ABI path
    pinned_in = rhs.cpu().pin_memory()
    pinned_out = torch.empty_like(pinned_in, device="cpu").pin_memory()
    rhs_dev = torch.empty_like(rhs)

    def e2e_step():
        rhs_dev.copy_(pinned_in, non_blocking=True)
        micro_step(m, x, rhs_dev)
        pinned_out.copy_(x, non_blocking=True)
    e2e_ms = timed(e2e_step, max(1, args.steps))
    peak_hbm, how = peaks()
    peak_fp64 = fp64_peak(dev)
    b_h = 64.0 * g.n_g + 32.0 * g.n_b
    f_q = 16.0 * g.n_b * nb * nb
    line = {"metric": "H*psi band-applies/s (batched H apply + projected-CG iteration)",
            "value": nb / (ms_step * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64/c128", "data": "synthetic",
            "config": {"workload": "BASELINE configs[3]: one batched H apply + projected-CG "
                                   "iteration (init Q + 1 iteration, 5 Q) on 256 bands",
                       "cube": list(g.cube_dims), "n_b": int(g.n_b), "bands": nb,
                       "n_occ": nb, "cell": "cubic 20 bohr", "e_cut": p["e_cut"],
                       "l2": "flushed (256 MiB write) between timed steps; operands 207 MB"},
            "step_ms": [round(t, 3) for t in step_ms], "gpu_launches": int(launches),
            "clocks": clk,
            "e2e": {"value": nb / (e2e_ms * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": int(rhs.numel() * 16),
                    "d2h_bytes_per_step": int(x.numel() * 16), "ms_per_step": e2e_ms},
            "roofline": {"kernel": "ham_apply (batched, 256 bands)", "bound": "hbm",
                         "achieved": b_h * nb / (h_ms * 1e-3) / 1e9, "peak": peak_hbm,
                         "unit": "GB/s", "frac": b_h * nb / (h_ms * 1e-3) / 1e9 / peak_hbm,
                         "traffic": None, "peak_source": how, "avg_launch_ms": h_ms,
                         "algorithmic_bytes_per_band_apply": b_h},
            "roofline_projector": {"kernel": "projector Q X (coef + apply GEMMs, 256 x 256 "
                                             "orbitals)", "bound": "tensor",
                                   "achieved": f_q / (q_ms * 1e-3) / 1e12, "peak": peak_fp64,
                                   "unit": "TFLOP/s (FP64)",
                                   "frac": f_q / (q_ms * 1e-3) / 1e12 / peak_fp64,
                                   "traffic": None,
                                   "peak_source": "measured live: cuBLAS DGEMM 8192^3 best of 5",
                                   "avg_launch_ms": q_ms,
                                   "algorithmic_flop_per_launch": f_q}}
    print(json.dumps(line))


def reference_setup(cfg):
    """Setup of the reference arm, outside the timed process: a child process runs
    the GPU ground-state generator and writes the workload directory (archive +
    dV0 + parameters, paper_2505_02319_b200.cli ground-state); this process only
    reads it back with numpy (oracle.archive) and never loads the CUDA library."""
    import tempfile
    out = os.environ.get("PWB_REF_WORKLOAD") or tempfile.mkdtemp(prefix=f"pwb_ref_cfg{cfg}_")
    cmd = [sys.executable, "-m", "paper_2505_02319_b200.cli", "ground-state", "--config",
           str(cfg), "--out", out]
    t0 = time.perf_counter()
    if not os.path.exists(os.path.join(out, "workload.json")):
        subprocess.run(cmd, check=True, cwd=ROOT, stdout=subprocess.DEVNULL)
    setup_s = time.perf_counter() - t0
    from oracle.archive import load_workload
    og, dv0, params = load_workload(out)
    return og, dv0, params, {"ground_state": "GPU SCF in a child process (" + " ".join(
        ["python"] + cmd[1:]) + "), archive format 2 read back by oracle.archive (numpy)",
        "setup_s": round(setup_s, 1), "workload_dir": out}


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing
    og, dv0, params, setup = reference_setup(args.config)
    ncores = len(os.sched_getaffinity(0))
    common = {"metric": METRIC, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
              "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
              "scaling": "strong", "vs_baseline": None, "dtype": "f64/c128", "data": "synthetic",
              "config": dict(workload_desc(args.config, og, params),
                             parallelism=f"kn-shard{args.gpus}"),
              "reference": setup}
    if hasattr(og, "blocks") or og.grids.n_g > 100000:
        vals = []
        tols0 = oracle_tolerances(og, dv0, params)
        t_all = time.perf_counter()
        for _ in range(args.warmup + args.steps):
            v, sample = oracle_sample(og, dv0, params, 10.0, threads=ncores, tols=tols0)
            vals.append(v)
        value = float(np.mean(vals[args.warmup:]))
        line = dict(common, value=value,
                    ms_per_step=(time.perf_counter() - t_all) / (args.warmup + args.steps) * 1e3,
                    cpu_baseline={"value": value, "unit": UNIT, "cores": ncores, "kind": "port",
                                  "sample": "per step: " + sample +
                                  f" (host has {multiprocessing.cpu_count()} cores)"},
                    e2e={"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                         "d2h_bytes_per_step": 0})
        print(json.dumps(line))
        return
    from threadpoolctl import threadpool_limits

    from oracle import dyson as od
    from oracle import model as om
    from oracle import outer as oo
    from oracle import response as orsp
    spec = oo.parse(params["strategy"], params["tau"], params["m"])
    orsp.BAND_THREADS = cores = ncores
    with threadpool_limits(limits=1):
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
    line = dict(common, value=value, ms_per_step=dt / args.steps * 1e3,
                cpu_baseline={"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                              "sample": f"{args.steps} full Dyson solves, oracle/ numpy port, "
                                        f"{ncores}-thread band pool, BLAS 1 thread "
                                        f"(host has {multiprocessing.cpu_count()} cores)"},
                e2e={"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                     "d2h_bytes_per_step": 0})
    print(json.dumps(line))


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 3:
        return run_microbench(args)
    world, rank, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("PWB_DIST_BACKEND", "nccl")   # gloo: the shared-GPU check
        dist.init_process_group(backend, **({"device_id": torch.device("cuda", local)}
                                            if backend == "nccl" else {}))
        group = dist.group.WORLD
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import device_state
    from paper_2505_02319_b200.harness import solve_dyson

    t_setup = time.perf_counter()
    gs, dv0, params = build_workload(args.config)
    ds = device_state(gs)
    setup_s = time.perf_counter() - t_setup
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
    region = os.environ.get("PWB_PROFILE_REGION") == "1"   # ncu --profile-from-start off
    # a full cyclic-GC pass of this process (torch + scipy heaps) stalls the host
    # launch stream for ~0.1 s at random points: collect now, none while timing
    gc.collect()
    gc.disable()
    barrier()
    if region:
        torch.cuda.cudart().cudaProfilerStart()
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
    if region:
        torch.cuda.cudart().cudaProfilerStop()
    launches = _lib.launch_count() - launches0
    gc.enable()
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
    e2e_ms, e2e_ham, e2e_list = 0.0, 0, []
    e2e_steps = max(1, min(args.steps, 3))
    gc.collect()
    gc.disable()
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
        e2e_list.append(e0.elapsed_time(e1))
        e2e_ms += e2e_list[-1]
        e2e_ham += r.n_ham
        del sol
    gc.enable()
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": e2e_ham / (e2e_ms * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": int(dv0.nbytes), "d2h_bytes_per_step": int(dv0.nbytes),
           "ms_per_step": e2e_ms / e2e_steps, "step_ms": [round(t, 3) for t in e2e_list]}

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
            "setup_s": round(setup_s, 1),
            "step_ms": [round(t, 3) for t in step_ms],
            "gpu_launches": int(launches), "clocks": clk, "e2e": e2e,
            "roofline": None,
            "roofline_ham": roofline_from_profile(prof, gs),
            "roofline_projector": projector_roofline(prof, gs, fp64_peak(dev)),
            "kernel_ms_by_live_rows": {
                cat: {f">={1 << b}": [round(ms, 2), n] for b, ms, n in rows}
                for cat, rows in hist.items() if cat in ("ham_apply", "projector", "cg_vector")}}
    line["roofline"] = dominant_roofline(line["roofline_ham"], line["roofline_projector"])
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(gs, dv0, params, args.cpu_budget)
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
