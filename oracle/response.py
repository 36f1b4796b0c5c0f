"""Oracle: projector, Sternheimer PCG, chi0, dielectric operator, kernels.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates
  * project_out / sternheimer      <- sternheimer.py:28-98
  * eigen_shifts                   <- response.py:45-71
  * pair_weights / occupied_dphi   <- response.py:74-107
  * chi0                           <- response.py:110-161
  * dielectric                     <- response.py:164-187
  * row_norm / error_bound         <- response.py:190-221
  * coulomb_kernel / kerker        <- kernels.py:40-79
k-point extension (`chi0_k`): chi0 = sum_k w_k chi0_k with
a global delta eps_F; each k block is processed with the Gamma code on its
k-shifted basis.
"""

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from .model import OracleNonConvergence, ham_apply, ham_counter

PRECOND_FLOOR = 0.1            # sternheimer.py:19
DEGENERACY_RTOL = 1e-8         # response.py:25
IMAG_RTOL = 1e-10              # response.py:26
LDA_FLOOR = 1e-10              # kernels.py:16
BAND_THREADS = 1               # Sternheimer band pool width (response.py:144-148)


def project_out(phi, x):
    """Q x = x - Phi (Phi^H x) (sternheimer.py:28-30)."""
    return x - phi @ (phi.conj().T @ x)


@dataclass
class CgResult:
    solution: np.ndarray
    final_residual_norm: float
    cg_iterations: int


def sternheimer(gs, v_local, n, rhs, tol, max_iter=None):
    """Projected PCG on Q(H - eps_n)Q (sternheimer.py:33-98)."""
    basis = gs.grids
    phi = gs.phi_occ
    e_n = float(gs.eps[n])
    limit = 10 * basis.n_b if max_iter is None else max_iter
    minv = 1.0 / (0.5 * basis.g2_sphere + max(e_n, PRECOND_FLOOR))

    x = np.zeros(basis.n_b, dtype=np.complex128)
    r = np.array(rhs, dtype=np.complex128, copy=True)
    z = project_out(phi, minv * r)
    p = z.copy()
    rz = np.vdot(r, z).real
    its = 0
    while True:
        p = project_out(phi, p)
        ap = project_out(phi, ham_apply(basis, v_local, p) - e_n * p)
        its += 1
        pap = np.vdot(p, ap).real
        alpha = rz / pap if pap > 0 else 0.0
        x += alpha * p
        r -= alpha * ap
        x = project_out(phi, x)
        r = project_out(phi, r)
        res = float(np.linalg.norm(r))
        if res <= tol:
            break
        if its >= limit:
            raise OracleNonConvergence(
                f"Sternheimer CG for band {n} stalled at {res:.3e} (target {tol:.3e})", residual=res)
        z = project_out(phi, minv * r)
        rz_new = np.vdot(r, z).real
        beta = rz_new / rz if rz != 0 else 0.0
        rz = rz_new
        p = z + beta * p
    return CgResult(x, res, its)


def eigen_shifts(gs, dv):
    """delta eps_n, delta eps_F, delta f_n (response.py:45-71)."""
    b = gs.grids
    pr = b.to_real_many(gs.phi_occ.T)
    dvpsi = b.to_fourier_many(dv[None, :] * pr)
    raw = np.einsum("bn,nb->n", gs.phi_occ.conj(), dvpsi)
    scale = max(np.max(np.abs(raw), initial=0.0), float(np.linalg.norm(dv)) * b.w)
    if scale > 0 and np.max(np.abs(raw.imag)) > IMAG_RTOL * scale:
        raise FloatingPointError("first-order eigenvalue shifts have an imaginary part")
    de = raw.real
    fp = gs.fprime_occ()
    s = fp.sum()
    de_f = float(fp @ de / s) if abs(s) > 1e-14 * gs.n_occ else 0.0
    return de, de_f, fp * (de - de_f)


def pair_weights(gs):
    """W[m, n] with f_n W[m,n] + f_m W[n,m] = divided difference (response.py:74-98)."""
    f, e, fp = gs.occ_occ, gs.eps_occ, gs.fprime_occ()
    de = e[None, :] - e[:, None]
    df = f[None, :] - f[:, None]
    degen = np.abs(de) <= DEGENERACY_RTOL * np.maximum(1.0, np.abs(e[None, :]))
    ratio = np.where(degen, fp[None, :], df / np.where(degen, 1.0, de))
    w = ratio * f[None, :] / (f[None, :] ** 2 + f[:, None] ** 2)
    np.fill_diagonal(w, 0.0)
    return w


def occupied_dphi(gs, dv):
    """delta phi^P = Phi (W o M) (response.py:101-107)."""
    b = gs.grids
    pr = b.to_real_many(gs.phi_occ.T)
    dvpsi = b.to_fourier_many(dv[None, :] * pr).T
    return gs.phi_occ @ (pair_weights(gs) * (gs.phi_occ.conj().T @ dvpsi))


@dataclass
class Chi0Stats:
    cg_iterations_per_band: list = field(default_factory=list)
    tolerances_used: list = field(default_factory=list)
    ham_applications: int = 0


def _check_tols(tols, n):
    tols = np.asarray(tols, dtype=float)
    if tols.shape != (n,):
        raise ValueError(f"need one tolerance per occupied band ({n}), got shape {tols.shape}")
    if np.any(tols <= 0):
        raise ValueError("Sternheimer tolerances must be positive")
    return tols


def _chi0_block(gs, dv, tols, de_f=None, weight=1.0):
    """One k block of apply_chi0 (response.py:127-154); returns pieces."""
    b = gs.grids
    pr = b.to_real_many(gs.phi_occ.T)
    dvpsi = b.to_fourier_many(dv[None, :] * pr)
    m = gs.phi_occ.conj().T @ dvpsi.T
    de = np.diag(m).real
    fp = gs.fprime_occ()
    dphi_p = gs.phi_occ @ (pair_weights(gs) * m)
    def one(n):
        rhs = -project_out(gs.phi_occ, dvpsi[n])
        return sternheimer(gs, gs.v_local, n, rhs, tols[n])

    if BAND_THREADS > 1:   # the reference's band pool (response.py:144-148); same results
        with ThreadPoolExecutor(max_workers=BAND_THREADS) as pool:
            results = list(pool.map(one, range(gs.n_occ)))
    else:
        results = [one(n) for n in range(gs.n_occ)]
    return dict(pr=pr, de=de, fp=fp, dphi_p=dphi_p, results=results, weight=weight)


def _accumulate(gs, blk, df):
    b = gs.grids
    dphi = blk["dphi_p"] + np.stack([r.solution for r in blk["results"]], axis=1)
    dr = b.to_real_many(dphi.T)
    pr = blk["pr"]
    c = (2.0 * gs.occ_occ[:, None]) * (pr.conj() * dr).real
    c += df[:, None] * np.abs(pr) ** 2
    return c.sum(axis=0)


def chi0(gs, dv, tolerances, threads=1):
    """apply_chi0 (response.py:110-161). Gamma-point ground state."""
    tols = _check_tols(tolerances, gs.n_occ)
    blk = _chi0_block(gs, dv, tols)
    fp, de = blk["fp"], blk["de"]
    s = fp.sum()
    de_f = float(fp @ de / s) if abs(s) > 1e-14 * gs.n_occ else 0.0
    drho = _accumulate(gs, blk, fp * (de - de_f))
    its = [r.cg_iterations for r in blk["results"]]
    return drho, Chi0Stats(its, list(tols), int(sum(its)))


def chi0_k(ks, dv, tolerances):
    """k-sampled chi0: sum_k w_k chi0_k with a global Fermi shift (App. B).

    `tolerances` is a list (one array per k block) or a flat array over
    (k, n) pairs in block order.
    """
    nocc = [blk.n_occ for blk in ks.blocks]
    if not isinstance(tolerances, (list, tuple)):
        flat = np.asarray(tolerances, dtype=float)
        if flat.shape != (sum(nocc),):
            raise ValueError("need one tolerance per (k, n) pair")
        tolerances = np.split(flat, np.cumsum(nocc)[:-1])
    pieces = []
    for gs, t, w in zip(ks.blocks, tolerances, ks.weights):
        pieces.append(_chi0_block(gs, dv, _check_tols(t, gs.n_occ), weight=w))
    num = sum(w * float(p["fp"] @ p["de"]) for p, w in zip(pieces, ks.weights))
    den = sum(w * float(p["fp"].sum()) for p, w in zip(pieces, ks.weights))
    thresh = 1e-14 * sum(w * n for w, n in zip(ks.weights, nocc))
    de_f = num / den if abs(den) > thresh else 0.0
    drho = np.zeros(ks.grids.n_g)
    its = []
    for gs, p, w in zip(ks.blocks, pieces, ks.weights):
        drho += w * _accumulate(gs, p, p["fp"] * (p["de"] - de_f))
        its += [r.cg_iterations for r in p["results"]]
    flat_t = np.concatenate([np.asarray(t, float) for t in tolerances])
    return drho, Chi0Stats(its, list(flat_t), int(sum(its)))


# -- kernels (kernels.py) ----------------------------------------------------------

def coulomb_kernel(xc, basis, rho_ref, v):
    """K v: Hartree 4pi/|G|^2 (+ LDA-x pointwise) (kernels.py:40-57)."""
    vf = basis.cube_fft(v)
    with np.errstate(divide="ignore", invalid="ignore"):
        vf *= 4 * np.pi / basis.g2_cube
    vf[basis.g2_cube == 0] = 0.0
    out = basis.cube_ifft(vf).real
    if xc == "lda_x":
        rho = np.clip(rho_ref, LDA_FLOOR, None)
        out = out - (1.0 / 3.0) * (3.0 / np.pi) ** (1.0 / 3.0) * rho ** (-2.0 / 3.0) * v
    return out


def kerker(alpha, basis, v):
    """T v = F^-1 D F v, D = |G|^2/(|G|^2+alpha^2), D(0)=1 (kernels.py:60-70)."""
    if alpha is None:
        return np.array(v, dtype=float, copy=True)
    if alpha == 0.0:
        return np.array(v, dtype=float, copy=True)
    d = basis.g2_cube / (basis.g2_cube + alpha ** 2)
    d[basis.g2_cube == 0] = 1.0
    return basis.cube_ifft(basis.cube_fft(v) * d).real


@dataclass
class Dielectric:
    output: np.ndarray
    kv_norm: float
    cg_iterations_per_band: list
    tolerances_used: list
    ham_applications: int


def dielectric(gs, xc, v, tolerances, threads=1):
    """E v = v - |Kv| chi0(Kv/|Kv|) (response.py:164-187). gs: State or KState."""
    u = coulomb_kernel(xc, gs.grids, gs.rho, np.asarray(v, dtype=float))
    kv = float(np.linalg.norm(u))
    if kv == 0.0:
        return Dielectric(np.array(v, dtype=float, copy=True), 0.0, [], [], 0)
    t = tolerances(kv) if callable(tolerances) else tolerances
    if hasattr(gs, "blocks"):
        drho, st = chi0_k(gs, u / kv, t)
    else:
        drho, st = chi0(gs, u / kv, t)
    return Dielectric(v - kv * drho, kv, st.cg_iterations_per_band, st.tolerances_used,
                      st.ham_applications)


def row_norm(basis, phi, real_part=False):
    """max_r ||F^-1 Phi (r, :)||_2 (response.py:190-199)."""
    pr = basis.to_real_many(phi.T)
    mat = pr.real if real_part else pr
    return float(np.sqrt(np.max(np.sum(np.abs(mat) ** 2, axis=0))))


def error_bound(gs, kv_norm, tolerances):
    """Lemma bound on ||(E - E~) v|| (response.py:202-214)."""
    t = np.asarray(tolerances, dtype=float)
    worst = float(np.max(gs.occ_occ * t / (gs.eps_gap_ref - gs.eps_occ)))
    if "abs" not in gs._row_norm_cache:
        gs._row_norm_cache["abs"] = row_norm(gs.grids, gs.phi_occ)
    row = gs._row_norm_cache["abs"]
    b = gs.grids
    return 2.0 * kv_norm * row * np.sqrt(b.n_g * gs.n_occ / b.lattice.volume) * worst


__all__ = [
    "project_out", "sternheimer", "eigen_shifts", "pair_weights", "occupied_dphi",
    "chi0", "chi0_k", "coulomb_kernel", "kerker", "dielectric", "row_norm", "error_bound",
    "ham_counter",
]
