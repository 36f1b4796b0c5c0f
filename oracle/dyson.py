"""Oracle: the Dyson solve driver (RHS build + inexact GMRES), run_response style.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates harness.py:131-141 (_base_context), :143-204 (build_perturbation,
with the perturbation dV0 passed in explicitly so the BASELINE's smoothed
white noise can be used), :207-212 (true_residual) and :215-292 (the
budgeted operator closure, Kerker preconditioning, N_Ham accounting, eta).
For k-sampled states the tolerance prefactors are evaluated per k block
with that block's N_occ,k (with w_k N_MP = 1 this is
the paper's bal_k / grt_k).
"""

from dataclasses import dataclass, field

import numpy as np

from .model import OracleNonConvergence, ham_counter
from .outer import Context, Strategy, igmres, select
from .response import chi0, chi0_k, dielectric, kerker, row_norm

TIGHT_CG_TOL = 1e-16


def _blocks(gs):
    return list(gs.blocks) if hasattr(gs, "blocks") else [gs]


def tolerance_vector(gs, spec, iteration, kv_norm=np.nan, rhs_norm=np.nan, common=None,
                     row_cache=None):
    """Concatenated per-(k, n) tolerances (strategies.py:98 per block)."""
    out = []
    for i, blk in enumerate(_blocks(gs)):
        b = blk.grids
        if row_cache is not None and i in row_cache:
            rn = row_cache[i]
        else:
            rn = row_norm(b, blk.phi_occ, real_part=True)
            if row_cache is not None:
                row_cache[i] = rn
        ctx = Context(iteration=iteration, n_occ=blk.n_occ, occ=blk.occ_occ,
                      volume=b.lattice.volume, n_g=b.n_g, row_norm=rn, rhs_norm=rhs_norm,
                      eps_gap=(blk.eps_gap_ref - blk.eps_occ) if spec.use_gap else None,
                      kv_norm=kv_norm, common_factor=common)
        out.append(select(spec, ctx))
    return np.concatenate(out)


def apply_chi0_any(gs, dv, tols):
    if hasattr(gs, "blocks"):
        return chi0_k(gs, dv, tols)
    return chi0(gs, dv, tols)


def rhs(gs, dv0, spec):
    """chi0 dV0 = |dV0| chi0(dV0/|dV0|) with iteration-0 budget (harness.py:180-204)."""
    nrm = float(np.linalg.norm(dv0))
    if nrm == 0.0:
        return np.zeros_like(dv0), 0, None
    if spec.kind == "d10n":
        prov = tolerance_vector(gs, Strategy("d10", spec.preconditioned, spec.tau, spec.m),
                                0, kv_norm=nrm, rhs_norm=1.0)
        d0, st0 = apply_chi0_any(gs, dv0 / nrm, prov)
        rn = float(np.linalg.norm(d0)) * nrm
        t = tolerance_vector(gs, spec, 0, kv_norm=nrm, rhs_norm=rn)
        if np.all(t >= prov):
            return nrm * d0, st0.ham_applications, prov
        d0, st = apply_chi0_any(gs, dv0 / nrm, t)
        return nrm * d0, st0.ham_applications + st.ham_applications, t
    t = tolerance_vector(gs, spec, 0, kv_norm=nrm, rhs_norm=1.0)
    d0, st = apply_chi0_any(gs, dv0 / nrm, t)
    return nrm * d0, st.ham_applications, t


@dataclass
class DysonResult:
    solution: np.ndarray
    rhs: np.ndarray
    converged: bool
    iterations: int
    n_ham: int
    n_ham_rhs: int
    final_est_res: float
    est_res_history: list
    tolerance_schedule: list = field(default_factory=list)   # per op call: tol vector
    cg_iterations: list = field(default_factory=list)        # per op call: per band
    budgets: list = field(default_factory=list)


def solve(gs, dv0, spec, xc="none", kerker_alpha=0.8):
    """run_response equivalent (harness.py:215-292) without the file outputs."""
    start = ham_counter.value
    b, n_rhs, rhs_tols = rhs(gs, dv0, spec)
    bn = float(np.linalg.norm(b))
    alpha = kerker_alpha if spec.preconditioned else None
    basis = gs.grids
    rows = {}
    sched, cgits = [], []
    if rhs_tols is not None:
        sched.append(np.asarray(rhs_tols))

    def op(v, budget):
        def tols(kv):
            return tolerance_vector(gs, spec, 1, kv_norm=kv, rhs_norm=bn, common=budget,
                                    row_cache=rows)
        app = dielectric(gs, xc, v, tols)
        sched.append(np.asarray(app.tolerances_used))
        cgits.append(list(app.cg_iterations_per_band))
        out = kerker(alpha, basis, app.output) if alpha is not None else app.output
        return out, app.ham_applications

    bs = kerker(alpha, basis, b) if alpha is not None else b
    try:
        rep = igmres(op, bs, None, m=spec.m, tau=spec.tau, s_init=1.0)
        ok = True
    except OracleNonConvergence as err:
        rep = err.report
        ok = False
    return DysonResult(rep.solution, b, ok, rep.iterations, ham_counter.value - start, n_rhs,
                       rep.final_est_res, list(rep.est_res_history), sched, cgits,
                       list(rep.budgets))


def true_residual(gs, xc, x, b):
    """||b - E x|| at tau_CG = 1e-16 (harness.py:207-212)."""
    n = sum(blk.n_occ for blk in _blocks(gs))
    app = dielectric(gs, xc, np.asarray(x, dtype=float), np.full(n, TIGHT_CG_TOL))
    return float(np.linalg.norm(b - app.output))
