"""Projected Sternheimer PCG on the GPU (drop-in for the reference sternheimer.py).

`project_out_occupied` (sternheimer.py:28-30) and `solve_sternheimer`
(sternheimer.py:33-98) with the same signatures, results and exceptions.
The arithmetic runs in libpwb200: complex-FP64 projector GEMMs and the
batched masked PCG (one CG row per right-hand side; `solve_sternheimer_many`
solves many bands at once, which is how apply_chi0 uses it).
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import device_state, ptr, torch_mod
from .errors import NonConvergenceError
from .groundstate import ham_counter

PRECONDITIONER_SHIFT_FLOOR = 0.1


@dataclass
class SternheimerResult:
    solution: np.ndarray
    final_residual_norm: float
    cg_iterations: int


def project_out_occupied(phi, psi):
    """Q psi = psi - Phi (Phi^H psi) for psi of shape (n_b,) or (n_b, k), on the GPU."""
    torch = torch_mod()
    phi = np.asarray(phi)
    psi = np.asarray(psi)
    vec = psi.ndim == 1
    cols = psi[:, None] if vec else psi
    nb, nocc = phi.shape
    if cols.shape[0] != nb:
        raise ValueError(f"psi has {cols.shape[0]} rows, phi has {nb}")
    dev = torch.device("cuda", torch.cuda.current_device())
    phi_rows = torch.from_numpy(np.ascontiguousarray(phi.T, dtype=np.complex128)).to(dev)
    x = torch.from_numpy(np.ascontiguousarray(cols.T, dtype=np.complex128)).to(dev)
    _lib.check(_lib.load().pwb_project_generic(nb, nocc, ptr(phi_rows), x.shape[0], ptr(x)),
               "project_out_occupied")
    out = x.cpu().numpy().T
    return out[:, 0].copy() if vec else np.ascontiguousarray(out)


def _state_for(gs, v_local):
    ds = device_state(gs)
    if v_local is not None and v_local is not gs.v_local and not np.array_equal(v_local,
                                                                                 gs.v_local):
        raise ValueError("solve_sternheimer on the GPU uses the ground state's own v_local "
                         "(the reference always passes gs.v_local, response.py:142)")
    return ds


def solve_sternheimer_many(gs, v_local, bands, rhs_rows, tols, max_iter=None):
    """Batched solve_sternheimer: rows of rhs (host (m, n_b)) for global bands `bands`.

    Returns (solutions (m, n_b), residuals, iterations).  Raises
    NonConvergenceError (with the first failing residual) like the reference.
    """
    torch = torch_mod()
    ds = _state_for(gs, v_local)
    bands = np.asarray(bands, dtype=np.int32)
    order = np.argsort(ds.band_k[bands], kind="stable")   # the batch runs k-grouped
    if np.any(order != np.arange(len(bands))):
        rhs_rows = np.asarray(rhs_rows)
        sol, res, its = solve_sternheimer_many(gs, v_local, bands[order], rhs_rows[order],
                                               np.asarray(tols, dtype=float)[order], max_iter)
        inv = np.argsort(order)
        return sol[inv], res[inv], its[inv]
    bands = np.ascontiguousarray(bands)
    tols = np.ascontiguousarray(tols, dtype=float)
    m = len(bands)
    rhs = ds.grid.pack(list(rhs_rows), ds.band_k[bands])
    x = torch.zeros_like(rhs)
    its = np.zeros(m, dtype=np.int32)
    res = np.zeros(m, dtype=float)
    status = _lib.load().pwb_sternheimer(
        ds.handle, m, ctypes.c_void_p(bands.ctypes.data), ptr(rhs),
        ctypes.c_void_p(tols.ctypes.data), int(max_iter or 0), ptr(x),
        ctypes.c_void_p(its.ctypes.data), ctypes.c_void_p(res.ctypes.data))
    done = its[its > 0]
    if status == _lib.PWB_ERR_NONCONV:
        bad = int(np.argmax(its < 0))
        # every row iterated until max_iter or convergence; count what was spent
        # (a failed row ran its full budget: max_iter, else 10 n_b of its k block,
        # sternheimer.py:60-61)
        failed_k = ds.band_k[bands[its < 0]]
        limits = (np.full(len(failed_k), int(max_iter)) if max_iter else
                  10 * np.asarray(ds.grid.nb, dtype=np.int64)[failed_k])
        spent = int(done.sum()) + int(np.sum(limits))
        ham_counter.add(spent)
        raise NonConvergenceError(
            f"Sternheimer CG for band {int(bands[bad])} stalled at {res[bad]:.3e} "
            f"(target {tols[bad]:.3e})", residual=float(res[bad]))
    _lib.check(status, "solve_sternheimer")
    ham_counter.add(int(its.sum()))
    sols = ds.grid.unpack(x, ds.band_k[bands])
    return np.stack(sols), res, its


def solve_sternheimer(gs, v_local, n, rhs, tol, max_iter=None):
    """CG on A_n = Q (H - eps_n) Q with kinetic preconditioning (sternheimer.py:33-98)."""
    rhs = np.asarray(rhs, dtype=np.complex128)
    if rhs.shape != (gs.grids.n_b,):
        raise ValueError(f"expected sphere vector of length {gs.grids.n_b}, got {rhs.shape}")
    sol, res, its = solve_sternheimer_many(gs, v_local, [n], rhs[None, :], [tol], max_iter)
    return SternheimerResult(solution=sol[0], final_residual_norm=float(res[0]),
                             cg_iterations=int(its[0]))
