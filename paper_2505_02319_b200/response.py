"""chi0 and the dielectric operator E = I - chi0 K on the GPU.

Drop-in for the reference response.py: `apply_chi0` (response.py:110-161),
`apply_dielectric` (:164-187), `delta_eigen_occupations` (:45-71),
`delta_phi_occupied` (:101-107), `_occupied_pair_weights` (:74-98),
`orbital_row_norm` (:190-199), `dielectric_error_bound` (:202-214) -- same
arguments, results, validation errors and H-application accounting
(ham_counter += sum of CG iterations).  `gs` may be a Gamma GroundState
(this package's or the reference's) or a KGroundState; for k-sampled states
the tolerance vector has one entry per (k, n) pair in block order and the
Fermi-level shift is global over k.

The whole (k, n) batch goes to the device in one call (pwb_chi0): RHS FFTs,
Phi^H dV psi, delta eps / delta eps_F / delta f, the occupied pair term, all
Sternheimer solves as one masked batched PCG, and the fused
inverse-FFT + drho accumulation.  `threads` is accepted and ignored: the
result is bitwise reproducible regardless.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .device import device_grid, device_state, ptr, state_blocks, torch_mod
from .groundstate import ham_counter
from .kernels import KernelSpec, apply_kernel_dev
from .ops import axpby_dev, div_dev

DEGENERACY_RTOL = 1e-8
IMAG_EIGENSHIFT_RTOL = 1e-10


@dataclass
class Chi0Stats:
    cg_iterations_per_band: list = field(default_factory=list)
    tolerances_used: list = field(default_factory=list)
    ham_applications: int = 0


@dataclass
class DielectricApplication:
    output: np.ndarray
    kv_norm: float
    cg_iterations_per_band: list
    tolerances_used: list
    ham_applications: int


def _n_pairs(gs):
    blocks, _ = state_blocks(gs)
    return int(sum(b.n_occ for b in blocks))


def _validate(gs, tolerances):
    n = _n_pairs(gs)
    tols = np.asarray(tolerances, dtype=float)
    if tols.shape != (n,):
        raise ValueError(f"need one tolerance per occupied band ({n}), got shape {tols.shape}")
    if np.any(tols <= 0):
        raise ValueError("Sternheimer tolerances must be positive")
    return tols


def _to_dev(ds, v):
    torch = torch_mod()
    if hasattr(v, "data_ptr"):
        return v.to(device=ds.device, dtype=torch.float64).contiguous()
    v = np.ascontiguousarray(v, dtype=float)
    if v.shape != (ds.grid.n_g,):
        raise ValueError(f"expected grid vector of length {ds.grid.n_g}, got {v.shape}")
    return torch.from_numpy(v).to(ds.device)


def _stats(its, tols):
    """Chi0Stats of one apply; adds the H applications to ham_counter (groundstate.py:48)."""
    its = [int(i) for i in its]
    total = int(sum(its))
    ham_counter.add(total)
    return Chi0Stats(cg_iterations_per_band=its, tolerances_used=list(tols),
                     ham_applications=total)


def apply_chi0_dev(gs, dv_t, tolerances):
    """Device-resident chi0: (drho tensor, Chi0Stats); dv_t a float64 device tensor."""
    tols = _validate(gs, tolerances)
    ds = device_state(gs)
    drho, its = ds.chi0(_to_dev(ds, dv_t), tols)
    return drho, _stats(its, tols)


def apply_chi0(gs, dv, tolerances, threads=1):
    """Density response chi0 dv with per-band Sternheimer tolerances (response.py:110-161)."""
    tols = _validate(gs, tolerances)
    drho, stats = apply_chi0_dev(gs, dv, tols)
    return drho.cpu().numpy(), stats


def _diag_and_dphi(gs, dv, want_dphi):
    torch = torch_mod()
    ds = device_state(gs)
    dvt = _to_dev(ds, dv)
    diag = np.zeros(2 * ds.nband)
    dphi = ds.grid.rows(ds.nband) if want_dphi else None
    _lib.check(_lib.load().pwb_chi0_parts(ds.handle, ptr(dvt), ctypes.c_void_p(diag.ctypes.data),
                                          ptr(dphi)), "chi0_parts")
    return ds, diag[0::2] + 1j * diag[1::2], dphi


def delta_eigen_occupations(gs, dv):
    """delta eps_n, delta eps_F, delta f_n (response.py:45-71), Gamma or k-sampled."""
    ds, raw, _ = _diag_and_dphi(gs, dv, False)
    g0 = ds.blocks[0].grids
    scale = max(np.max(np.abs(raw), initial=0.0), float(np.linalg.norm(dv)) * g0.w)
    if scale > 0 and np.max(np.abs(raw.imag)) > IMAG_EIGENSHIFT_RTOL * scale:
        raise FloatingPointError(
            f"first-order eigenvalue shifts have imaginary part "
            f"{np.max(np.abs(raw.imag)):.2e} relative to {scale:.2e}")
    de = raw.real
    wb = ds.weights[ds.band_k]
    if abs(ds.fp_den) > ds.fp_thresh:
        def_ = float(np.sum(wb * ds.fprime * de) / ds.fp_den)
    else:
        def_ = 0.0
    return de, def_, ds.fprime * (de - def_)


def _occupied_pair_weights(gs):
    """W[m, n]: f_n W[m,n] + f_m W[n,m] = (f_n - f_m)/(eps_n - eps_m) (response.py:74-98)."""
    f, e, fp = gs.occ_occ, gs.eps_occ, gs.fprime_occ()
    de = e[None, :] - e[:, None]
    df = f[None, :] - f[:, None]
    degen = np.abs(de) <= DEGENERACY_RTOL * np.maximum(1.0, np.abs(e[None, :]))
    ratio = np.where(degen, fp[None, :], df / np.where(degen, 1.0, de))
    w = ratio * f[None, :] / (f[None, :] ** 2 + f[:, None] ** 2)
    np.fill_diagonal(w, 0.0)
    return w


def delta_phi_occupied(gs, dv):
    """Occupied-subspace orbital response (n_b, n_occ) (response.py:101-107), Gamma state."""
    ds, _, dphi = _diag_and_dphi(gs, dv, True)
    return np.stack(ds.grid.unpack(dphi, ds.band_k), axis=1)


def apply_dielectric_dev(gs, kernel, v_t, tolerances):
    """Device E v: returns (output tensor, kv_norm, Chi0Stats or None)."""
    torch = torch_mod()
    ds = device_state(gs)
    v_t = _to_dev(ds, v_t)
    u = apply_kernel_dev(kernel, ds.grid, ds.rho_t, v_t)
    kv = _norm(ds.grid, u)
    if kv == 0.0:
        return v_t.clone(), 0.0, None
    h = ds.grid.handle
    if callable(tolerances):
        # the tolerance vector depends on |Kv| only: build chi0's right-hand side on
        # the GPU while the host evaluates the strategy (strategies.py, numpy)
        ds.chi0_begin(div_dev(h, u, kv))
        tols = _validate(gs, tolerances(kv))
        drho, its = ds.chi0_finish(tols)
        stats = _stats(its, tols)
    else:
        drho, stats = apply_chi0_dev(gs, div_dev(h, u, kv), tolerances)
    return axpby_dev(h, 1.0, v_t, -kv, drho), kv, stats


def _norm(dg, x):
    """||x||_2 via the library's deterministic reduction."""
    torch = torch_mod()
    out = torch.zeros(1, dtype=torch.float64, device=x.device)
    _lib.check(_lib.load().pwb_vec_dot(dg.handle, x.numel(), ptr(x), ptr(x), ptr(out)), "dot")
    return float(np.sqrt(out.item()))


def apply_dielectric(gs, kernel, v, tolerances, threads=1):
    """E v = v - |Kv| chi0(Kv/|Kv|); identity when Kv = 0 (response.py:164-187)."""
    v = np.asarray(v, dtype=float)
    out, kv, stats = apply_dielectric_dev(gs, kernel, v, tolerances)
    if stats is None:
        return DielectricApplication(output=np.array(v, dtype=float, copy=True), kv_norm=0.0,
                                     cg_iterations_per_band=[], tolerances_used=[],
                                     ham_applications=0)
    return DielectricApplication(output=out.cpu().numpy(), kv_norm=kv,
                                 cg_iterations_per_band=stats.cg_iterations_per_band,
                                 tolerances_used=stats.tolerances_used,
                                 ham_applications=stats.ham_applications)


def orbital_row_norm(grids, phi, real_part=False):
    """max_r ||to_real(Phi)(r, :)||_2 (response.py:190-199), computed on the GPU."""
    dg = device_grid(grids)
    phi = np.asarray(phi)
    rows = dg.pack(list(np.ascontiguousarray(phi.T)))
    out = ctypes.c_double(0.0)
    _lib.check(_lib.load().pwb_row_norm_rows(dg.handle, rows.shape[0], None, ptr(rows),
                                             1 if real_part else 0, ctypes.byref(out)),
               "row_norm")
    return float(out.value)


def _cached_row_norm(gs, real_part=False):
    key = "re" if real_part else "abs"
    cache = gs._row_norm_cache
    if key not in cache:
        cache[key] = orbital_row_norm(gs.grids, gs.phi_occ, real_part)
    return cache[key]


def dielectric_error_bound(gs, kv_norm, tolerances):
    """Lemma bound on ||(E - E~) v|| (response.py:202-214)."""
    tolerances = np.asarray(tolerances, dtype=float)
    gaps = gs.eps_gap_ref - gs.eps_occ
    worst = float(np.max(gs.occ_occ * tolerances / gaps))
    row = _cached_row_norm(gs)
    g = gs.grids
    return 2.0 * kv_norm * row * np.sqrt(g.n_g * gs.n_occ / g.lattice.volume) * worst
