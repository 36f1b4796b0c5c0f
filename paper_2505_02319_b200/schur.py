"""Sternheimer solves with the extra computed bands deflated (optional extension).

The paper solves its Sternheimer equations with the Schur-complement trick of
Cances et al.; the reference package omits it
(SPEC.md:275), so this module is OUTSIDE the parity path:
nothing in `apply_chi0` / `solve_dyson` calls it, and its results agree with
`solve_sternheimer` only to the CG tolerance, not iteration by iteration.

A ground state keeps N_ex extra eigenpairs above the occupied ones
(groundstate.py:373-377: max(3, 10% of N_occ) of them).  With those CONVERGED,
H is block diagonal on span(Phi_ex) + R, R the complement of all kept bands,
and the solution of Q (H - eps_n) Q x = b, b in range(Q), splits exactly:

    x = Phi_ex (Lambda_ex - eps_n)^-1 Phi_ex^H b  +  x_R,
    Q_all (H - eps_n) Q_all x_R = Q_all b,        Q_all = 1 - Phi_kept Phi_kept^H.

The CG then runs on R, where the smallest eigenvalue of the operator is
eps_{N_kept+1} - eps_n instead of eps_{N_occ+1} - eps_n: fewer iterations for the
same residual (the explicit part carries no residual, so the stopping test
||r|| <= tol is the reference's).  For extra bands that are only approximately
converged the full Schur complement of Cances et al. adds a coupling term; here
the residual of every extra band is checked against `resid_tol` and a
ConfigurationError is raised instead (lobpcg.run_scf_gpu(converge_kept=True)
converges them).

The CG is the same batched device PCG (`pwb_sternheimer`) on a second device
state whose projector block holds all kept bands; Q_all b is formed on the device
(`pwb_project_out`).
"""

import ctypes
from dataclasses import replace

import numpy as np

from . import _lib
from .device import device_state, ptr, state_blocks, torch_mod
from .errors import ConfigurationError
from .sternheimer import solve_sternheimer_many


def extended_state(gs):
    """The same ground state with every kept band in the projector block (cached)."""
    ext = getattr(gs, "_pwb_schur_state", None)
    if ext is not None:
        return ext
    if hasattr(gs, "blocks"):
        ext = replace(gs, blocks=[replace(b, n_occ=b.n_kept) for b in gs.blocks])
    else:
        ext = replace(gs, n_occ=gs.n_kept)
    try:
        object.__setattr__(gs, "_pwb_schur_state", ext)
    except (AttributeError, TypeError):
        pass
    return ext


def extra_band_residuals(gs):
    """max_m ||H phi_m - eps_m phi_m|| over the extra bands of each k block (device H)."""
    from .ops import ham_apply_many
    out = []
    for blk in state_blocks(gs)[0]:
        ex = np.ascontiguousarray(blk.phi[:, blk.n_occ:].T)
        if ex.shape[0] == 0:
            out.append(0.0)
            continue
        h = ham_apply_many(blk.grids, gs.v_local, ex)
        r = h - blk.eps[blk.n_occ:, None] * ex
        out.append(float(np.linalg.norm(r, axis=1).max()))
    return out


def solve_sternheimer_schur(gs, bands, rhs_rows, tols, max_iter=None, resid_tol=1e-8):
    """Batched Sternheimer solves with the extra bands deflated.

    bands: global occupied-band indices ((k, n) pairs in block order, as in
    `solve_sternheimer_many`); rhs_rows (m, n_b) in range(Q); tols absolute l2
    tolerances.  Returns (solutions (m, n_b), residual norms, CG iterations).
    """
    torch = torch_mod()
    blocks, _ = state_blocks(gs)
    if any(b.n_kept <= b.n_occ for b in blocks):
        raise ConfigurationError("the ground state keeps no extra bands to deflate")
    worst = max(extra_band_residuals(gs))
    if worst > resid_tol:
        raise ConfigurationError(
            f"extra bands are not converged (max residual {worst:.2e} > {resid_tol:.1e}); "
            "run the SCF with converge_kept=True")
    ds = device_state(gs)
    ext = extended_state(gs)
    dx = device_state(ext)
    lib = _lib.load()
    bands = np.asarray(bands, dtype=np.int64)
    ks = ds.band_k[bands]
    order = np.argsort(ks, kind="stable")
    inv = np.argsort(order)
    bands, ks = bands[order], ks[order]
    rhs_rows = np.asarray(rhs_rows, dtype=np.complex128)[order]
    tols = np.asarray(tols, dtype=float)[order]
    local = bands - ds.offsets[ks]                 # band index inside its k block
    ext_bands = (dx.offsets[ks] + local).astype(np.int32)
    # Q_all b on the device, one call per k block present
    rhs = dx.grid.pack(list(rhs_rows), ks)
    for k in np.unique(ks):
        sel = np.nonzero(ks == k)[0]
        rows = rhs[sel[0]: sel[-1] + 1]            # contiguous: the batch is k-grouped
        _lib.check(lib.pwb_project_out(dx.handle, int(k), len(sel), ptr(rows)), "project_out")
    rhs_r = np.stack(dx.grid.unpack(rhs, ks))
    x_r, res, its = solve_sternheimer_many(ext, None, ext_bands, rhs_r, tols, max_iter)
    # explicit part on the converged extra bands
    sols = np.empty_like(x_r)
    for i, (k, n) in enumerate(zip(ks, local)):
        blk = blocks[k]
        ex = blk.phi[:, blk.n_occ:]
        coef = (ex.conj().T @ rhs_rows[i]) / (blk.eps[blk.n_occ:] - blk.eps[n])
        sols[i] = x_r[i] + ex @ coef
    torch.cuda.synchronize()
    return sols[inv], res[inv], its[inv]
