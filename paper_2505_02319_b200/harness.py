"""The Dyson solve driver: RHS build + device-resident inexact GMRES.

Mirrors the reference harness.py for the hot path: `build_perturbation`'s
right-hand side chi0 dV0 = |dV0| chi0(dV0/|dV0|) with iteration-0 budget
tau/3 (harness.py:143-204), the budgeted operator closure that turns each
granted budget into per-band tolerances (common_factor = budget,
harness.py:240-259), Kerker preconditioning (:250, :272), N_Ham accounting
(counter delta including the RHS, :231, :281), `true_residual` at
tau_CG = 1e-16 (:207-212) and eta (:291-292).  dV0 can be passed
explicitly (the BASELINE's smoothed white noise) or built from the
configured Gaussian displacement like the reference.

Everything N_g-sized stays on the GPU: dV0, b, the Krylov basis, K v, the
Kerker filter and every chi0 application; only scalars cross to the host.
"""

import time
from dataclasses import dataclass, field

import numpy as np

from .device import device_state, state_blocks, torch_mod
from .errors import NonConvergenceError
from .groundstate import ham_counter
from .igmres import igmres_solve
from .kernels import KernelSpec, KerkerSpec, apply_kerker_dev
from .ops import axpby_dev, div_dev
from .response import _norm, apply_chi0_dev, apply_dielectric_dev, orbital_row_norm
from .strategies import StrategySpec, parse_strategy, tolerances_k

TIGHT_CG_TOL = 1e-16


@dataclass(frozen=True)
class Perturbation:
    """Gaussian-displacement perturbation (reference config.py:23-27)."""
    gaussian: int = 0
    direction: tuple = (1.0, 0.0, 0.0)
    analytic: bool = True


@dataclass
class DysonResult:
    solution: object
    rhs: object
    converged: bool
    iterations: int
    n_ham: int
    n_ham_rhs: int
    final_est_res: float
    est_res_history: list
    tolerance_schedule: list = field(default_factory=list)
    cg_iterations: list = field(default_factory=list)
    budgets: list = field(default_factory=list)
    restarts: list = field(default_factory=list)
    wall_s: float = 0.0
    final_true_res: float = np.nan
    eta: float = np.nan
    y_final: object = None          # last cycle's least-squares coefficients (igmres.py:154)
    cycle_est_res: list = field(default_factory=list)
    sigma_final: float = np.nan


def row_norms(gs):
    """Real-part orbital row norm per k block (harness.py:137)."""
    blocks, _ = state_blocks(gs)
    return [orbital_row_norm(b.grids, b.phi_occ, real_part=True) for b in blocks]


def build_rhs(gs, dv0_t, spec, rows=None):
    """(b tensor, N_Ham spent, tolerances used) -- harness.py:180-204 with dV0 given."""
    torch = torch_mod()
    blocks, _ = state_blocks(gs)
    ds = device_state(gs)
    nrm = _norm(ds.grid, dv0_t)
    if nrm == 0.0:
        return torch.zeros_like(dv0_t), 0, None
    if rows is None:
        rows = row_norms(gs) if spec.kind == "grt" else [np.nan] * len(blocks)
    h = ds.grid.handle
    unit = div_dev(h, dv0_t, nrm)
    if spec.kind == "d10n":
        prov = tolerances_k(blocks, StrategySpec("d10", spec.preconditioned, spec.tau, spec.m),
                            0, rows, kv_norm=nrm, rhs_norm=1.0)
        d0, st0 = apply_chi0_dev(gs, unit, prov)
        rn = _norm(ds.grid, d0) * nrm
        tols = tolerances_k(blocks, spec, 0, rows, kv_norm=nrm, rhs_norm=rn)
        if np.all(tols >= prov):
            return axpby_dev(h, nrm, d0), st0.ham_applications, prov
        d0, st = apply_chi0_dev(gs, unit, tols)
        return axpby_dev(h, nrm, d0), st0.ham_applications + st.ham_applications, tols
    tols = tolerances_k(blocks, spec, 0, rows, kv_norm=nrm, rhs_norm=1.0)
    d0, st = apply_chi0_dev(gs, unit, tols)
    return axpby_dev(h, nrm, d0), st.ham_applications, tols


def true_residual(gs, kernel, x_t, b_t):
    """||b - E x|| with every tau_CG = 1e-16 (harness.py:207-212)."""
    blocks, _ = state_blocks(gs)
    n = sum(b.n_occ for b in blocks)
    out, _, _ = apply_dielectric_dev(gs, kernel, x_t, np.full(n, TIGHT_CG_TOL))
    dg = device_state(gs).grid
    return _norm(dg, axpby_dev(dg.handle, 1.0, b_t, -1.0, out))


def solve_dyson(gs, dv0, strategy="bal", tau=1e-8, m=10, xc=None, kerker_alpha=0.8,
                use_gap=False, with_true_residual=False, sync_timing=True):
    """Solve (I - chi0 K) drho = chi0 dV0 (run_response, harness.py:215-292).

    dv0: numpy array or float64 CUDA tensor (x-fastest grid values).  Returns a
    DysonResult whose solution / rhs are device tensors.  N_Ham excludes the
    optional final true residual, as in the reference.
    """
    torch = torch_mod()
    spec = strategy if isinstance(strategy, StrategySpec) else parse_strategy(
        strategy, tau=tau, m=m, use_gap=use_gap)
    blocks, _ = state_blocks(gs)
    ds = device_state(gs)
    dg = ds.grid
    xc = gs.model.xc if xc is None else xc
    kernel = KernelSpec(xc=xc)
    kerker = KerkerSpec(alpha=kerker_alpha) if spec.preconditioned else None
    dv0_t = (dv0.to(dtype=torch.float64).contiguous() if hasattr(dv0, "data_ptr") else
             torch.from_numpy(np.ascontiguousarray(dv0, dtype=float)).to(ds.device))
    rows = row_norms(gs) if spec.kind == "grt" else [np.nan] * len(blocks)
    if sync_timing:
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    start = ham_counter.value
    b_t, n_rhs, rhs_tols = build_rhs(gs, dv0_t, spec, rows)
    b_norm = _norm(dg, b_t)
    sched = [] if rhs_tols is None else [np.asarray(rhs_tols)]
    cgits = []

    def op(v, budget):
        def tolerances(kv):
            return tolerances_k(blocks, spec, 1, rows, kv_norm=kv, rhs_norm=b_norm,
                                common=budget)
        out, kv, stats = apply_dielectric_dev(gs, kernel, v, tolerances)
        cost = 0
        if stats is not None:
            sched.append(np.asarray(stats.tolerances_used))
            cgits.append(list(stats.cg_iterations_per_band))
            cost = stats.ham_applications
        if kerker is not None:
            out = apply_kerker_dev(kerker, dg, out)
        return out, cost

    bs = apply_kerker_dev(kerker, dg, b_t) if kerker is not None else b_t
    try:
        rep = igmres_solve(op, bs, x0=None, m=spec.m, tau=spec.tau, s_init=1.0,
                           grid_handle=dg.handle)
        ok = True
    except NonConvergenceError as err:
        rep = err.report
        ok = False
    if sync_timing:
        torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    n_ham = ham_counter.value - start
    res = DysonResult(solution=rep.solution, rhs=b_t, converged=ok, iterations=rep.iterations,
                      n_ham=n_ham, n_ham_rhs=n_rhs, final_est_res=rep.final_est_res,
                      est_res_history=list(rep.est_res_history), tolerance_schedule=sched,
                      cg_iterations=cgits, budgets=list(rep.budgets),
                      restarts=list(rep.restarts), wall_s=wall, y_final=rep.y_final,
                      cycle_est_res=list(rep.cycle_est_res), sigma_final=rep.sigma_final)
    if with_true_residual:
        res.final_true_res = true_residual(gs, kernel, rep.solution, b_t)
        if n_ham > 0 and res.final_true_res > 0 and b_norm > 0:
            res.eta = -np.log10(res.final_true_res / b_norm) / n_ham
    return res


def perturbation_from_config(gs, pert):
    """dV0 of the reference's Gaussian-displacement perturbation (harness.py:153-178)."""
    from .groundstate import external_potential_derivative
    return external_potential_derivative(gs.model, gs.grids, pert.gaussian, pert.direction)
