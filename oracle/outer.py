"""Oracle: Sternheimer tolerance strategies and the restarted inexact GMRES.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates
  * Strategy / parse / Context / select  <- strategies.py:21-129
  * Gmres state, Arnoldi MGS + reorth   <- igmres.py:56-114
  * givens_update                       <- igmres.py:117-144
  * sigma_min                           <- igmres.py:147-151
  * igmres                              <- igmres.py:173-306
"""

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

from .basis import OracleConfigError
from .model import OracleNonConvergence

TOL_FLOOR = 1e-16
BUDGET_FLOOR_REL = 1e-16
ADAPTIVE = ("grt", "bal", "agr")
STATIC = ("d10", "d100", "d10n")


@dataclass(frozen=True)
class Strategy:
    kind: str
    preconditioned: bool
    tau: float
    m: int
    use_gap: bool = False

    def __post_init__(self):
        if self.kind not in ADAPTIVE + STATIC:
            raise OracleConfigError(f"unknown strategy kind {self.kind!r}")

    @property
    def adaptive(self):
        return self.kind in ADAPTIVE

    @property
    def name(self):
        return ("p" if self.preconditioned else "") + self.kind


def parse(name, tau, m, use_gap=False):
    key = name.strip().lower()
    pre = key.startswith("p")
    return Strategy(key[1:] if pre else key, pre, tau, m, use_gap)


@dataclass
class Context:
    iteration: int
    n_occ: int
    occ: np.ndarray
    volume: float
    n_g: int
    est_res_prev: float = np.nan
    s: float = np.nan
    kv_norm: float = np.nan
    row_norm: float = np.nan
    rhs_norm: float = np.nan
    eps_gap: np.ndarray = None
    common_factor: float = None


def _pos(v, what):
    if v is None or not np.all(np.isfinite(v)) or not np.all(np.asarray(v) > 0):
        raise OracleConfigError(f"need positive finite {what}, got {v}")
    return v


def shared_factor(spec, ctx):
    """(s/3m) tau/||r_{i-1}||, or tau/3 at iteration 0 (strategies.py:88-95)."""
    if ctx.common_factor is not None:
        return float(_pos(ctx.common_factor, "common_factor"))
    if ctx.iteration == 0:
        return spec.tau / 3.0
    _pos(ctx.s, "s")
    _pos(ctx.est_res_prev, "est_res_prev")
    return (ctx.s / (3.0 * spec.m)) * spec.tau / ctx.est_res_prev


def select(spec, ctx):
    """Per-band tolerances, floored at 1e-16 (strategies.py:98-129)."""
    occ = np.asarray(_pos(ctx.occ, "occupations"), dtype=float)
    if len(occ) != ctx.n_occ:
        raise OracleConfigError("occupation vector length disagrees with n_occ")
    if spec.adaptive:
        c = shared_factor(spec, ctx)
        if spec.kind == "agr":
            pre = np.ones(ctx.n_occ)
        else:
            band = np.sqrt(ctx.volume) / (2.0 * occ * np.sqrt(ctx.n_g * ctx.n_occ))
            if spec.kind == "grt":
                pre = band / (_pos(ctx.kv_norm, "kv_norm") * _pos(ctx.row_norm, "row_norm"))
            else:
                pre = band * np.sqrt(ctx.volume) / np.sqrt(ctx.n_occ)
            if spec.use_gap:
                pre = pre * np.asarray(_pos(ctx.eps_gap, "eps_gap"), dtype=float)
        tol = pre * c
    elif spec.kind == "d10":
        tol = np.full(ctx.n_occ, spec.tau / 10.0)
    elif spec.kind == "d100":
        tol = np.full(ctx.n_occ, spec.tau / 100.0)
    else:
        tol = np.full(ctx.n_occ, spec.tau / (10.0 * _pos(ctx.rhs_norm, "rhs_norm")))
    return np.maximum(tol, TOL_FLOOR)


# -- inexact GMRES --------------------------------------------------------------

class Arnoldi:
    """Basis + Hessenberg + Givens (igmres.py:56-114)."""

    def __init__(self, m):
        self.m = m
        self.v = []
        self.h = np.zeros((m + 1, m))
        self.r = np.zeros((m + 1, m))
        self.cs = np.zeros(m)
        self.sn = np.zeros(m)
        self.g = np.zeros(m + 1)
        self.size = 0
        self.beta = 0.0
        self.history = []

    def start(self, r0):
        self.beta = float(np.linalg.norm(r0))
        self.v = [r0 / self.beta]
        self.g[:] = 0.0
        self.g[0] = self.beta
        self.size = 0
        self.history = [self.beta]

    def hess(self):
        return self.h[: self.size + 1, : self.size].copy()

    def orthogonalise(self, w):
        i = self.size
        col = np.zeros(i + 2)
        for j in range(i + 1):
            c = float(np.dot(self.v[j], w))
            w = w - c * self.v[j]
            col[j] = c
        for j in range(i + 1):
            c = float(np.dot(self.v[j], w))
            w = w - c * self.v[j]
            col[j] += c
        col[i + 1] = float(np.linalg.norm(w))
        self.v.append(w / col[i + 1] if col[i + 1] > 0 else np.zeros_like(w))
        return col

    def coefficients(self):
        i = self.size
        return scipy.linalg.solve_triangular(self.r[:i, :i], self.g[:i])

    def combine(self, x0, y):
        x = x0.copy()
        for j, c in enumerate(y):
            x = x + c * self.v[j]
        return x


def givens_update(st, col):
    """Fold a Hessenberg column into the QR; return ||r~_i|| (igmres.py:117-144)."""
    i = st.size
    col = np.array(col, dtype=float)
    st.h[: i + 2, i] = col[: i + 2]
    for j in range(i):
        t = st.cs[j] * col[j] + st.sn[j] * col[j + 1]
        col[j + 1] = -st.sn[j] * col[j] + st.cs[j] * col[j + 1]
        col[j] = t
    d = np.hypot(col[i], col[i + 1])
    if d == 0.0:
        st.cs[i], st.sn[i] = 1.0, 0.0
    else:
        st.cs[i], st.sn[i] = col[i] / d, col[i + 1] / d
    col[i], col[i + 1] = d, 0.0
    st.r[: i + 2, i] = col[: i + 2]
    st.g[i + 1] = -st.sn[i] * st.g[i]
    st.g[i] = st.cs[i] * st.g[i]
    st.size = i + 1
    est = abs(float(st.g[i + 1]))
    st.history.append(est)
    return est


def sigma_min(h):
    if h.size == 0:
        raise OracleConfigError("empty Hessenberg matrix")
    return float(scipy.linalg.svdvals(h)[-1])


@dataclass
class GmresReport:
    solution: np.ndarray
    converged: bool
    iterations: int
    total_cost: int
    est_res_history: list
    budgets: list
    restarts: list
    s_final: float
    sigma_final: float
    final_est_res: float = np.inf
    cycle_est_res: list = field(default_factory=list)


def igmres(op, b, x0=None, m=10, tau=1e-9, s_init=1.0, max_total_iterations=None, monitor=None):
    """Algorithm 1 (igmres.py:173-306). budgets: list of (iter, cycle, budget, cost)."""
    if tau <= 0 or m < 1 or s_init <= 0:
        raise OracleConfigError("need tau > 0, m >= 1, s_init > 0")
    b = np.asarray(b, dtype=float)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=float, copy=True)
    cap = 100 * m if max_total_iterations is None else max_total_iterations
    nb = float(np.linalg.norm(b))
    floor = BUDGET_FLOOR_REL * nb
    s = float(s_init)
    budgets, restarts, hist, cyc = [], [], [], []
    cost_sum = 0
    its = 0
    cycle = 0

    def report(sol, ok, sigma=np.nan, est=np.inf):
        return GmresReport(sol, ok, its, cost_sum, hist, budgets, restarts, s, sigma, est, cyc)

    if nb == 0.0 and not np.any(x):
        return report(x, True, est=0.0)
    st = Arnoldi(m)
    while True:
        cycle += 1
        if np.any(x):
            b0 = max(tau / 3.0, floor)
            w0, c0 = op(x, b0)
            cost_sum += c0
            budgets.append((0, cycle, b0, c0))
            r0 = b - w0
        else:
            r0 = b.copy()
        if np.linalg.norm(r0) == 0.0:
            return report(x, True, est=0.0)
        st.start(r0)
        hist.append(st.beta)
        est = st.beta
        exhausted = True
        for _ in range(m):
            budget = max((s / (3.0 * m)) * tau / est, floor)
            w, c = op(st.v[st.size], budget)
            cost_sum += c
            its += 1
            budgets.append((its, cycle, budget, c))
            est = givens_update(st, st.orthogonalise(w))
            hist.append(est)
            if monitor is not None:
                monitor({"iteration": its, "cycle": cycle, "est_res": est, "budget": budget,
                         "cost": c, "s": s,
                         "get_x": lambda: st.combine(x, st.coefficients())})
            if est <= tau / 3.0:
                sig = sigma_min(st.hess())
                xn = st.combine(x, st.coefficients())
                if s <= sig:
                    cyc.append(list(st.history))
                    return report(xn, True, sig, est)
                restarts.append(("s-violation", cycle, s, sig))
                s = sig
                x = xn
                exhausted = False
                break
            if its >= cap:
                xn = st.combine(x, st.coefficients())
                raise OracleNonConvergence("inexact GMRES iteration cap", residual=est,
                                           report=report(xn, False, sigma_min(st.hess()), est))
        if exhausted:
            sig = sigma_min(st.hess())
            x = st.combine(x, st.coefficients())
            restarts.append(("cycle-full", cycle, s, sig))
            s = sig
        cyc.append(list(st.history))
