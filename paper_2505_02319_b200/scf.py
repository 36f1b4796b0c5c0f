"""Ground-state generation (setup for the hot path).

The chi0 hot path consumes a converged ground state (Phi, eps, f, V_local,
rho); producing it is a prerequisite, not part of the path.  This module
provides the damped Kerker-mixed SCF of the reference (groundstate.py:
333-394) with dense diagonalisation, plus its k-sampled extension (density
sum_k w_k sum_n f_nk |psi_nk|^2 and a global Fermi level).  Dense `eigh` is
O(n_b^3) and is only used for the small configs (n_b <= ~3000); the large
configs use `lobpcg.py` on the GPU H apply.
"""

import numpy as np
import scipy.linalg

from .errors import ConfigurationError, NonConvergenceError
from .groundstate import (GroundState, KGroundState, external_potential,
                          fermi_and_occupations)
from .pwbasis import build_grids, monkhorst_pack


def _fft(grids, v):
    return np.fft.fftn(grids.cube_view(np.asarray(v, dtype=np.complex128))).ravel(order="F")


def _ifft(grids, c):
    return np.fft.ifftn(grids.cube_view(c)).ravel(order="F")


def dense_hamiltonian(grids, v_local):
    """H_{GG'} = |G+k|^2/2 delta + V^(G - G') (groundstate.py:222-234)."""
    vhat = _fft(grids, v_local) / grids.n_g
    nx, ny, nz = grids.cube_dims
    d = grids.g_int[:, None, :] - grids.g_int[None, :, :]
    idx = (d[..., 0] % nx) + nx * ((d[..., 1] % ny) + ny * (d[..., 2] % nz))
    h = vhat[idx]
    h[np.arange(grids.n_b), np.arange(grids.n_b)] += 0.5 * grids.g2_sphere
    return h


def diagonalize_dense(grids, v_local, n_states):
    if n_states > grids.n_b:
        raise ConfigurationError(f"n_states={n_states} exceeds basis size {grids.n_b}")
    return scipy.linalg.eigh(dense_hamiltonian(grids, v_local), subset_by_index=[0, n_states - 1])


def _to_real_host(grids, phi):
    k = phi.shape[1]
    buf = np.zeros((k, grids.n_g), dtype=np.complex128)
    buf[:, grids.sphere_flat] = phi.T
    cube = buf.reshape((k, *grids.cube_dims), order="F")
    vals = np.fft.ifftn(cube, axes=(1, 2, 3)).reshape(k, grids.n_g, order="F")
    return vals * (grids.n_g / np.sqrt(grids.lattice.volume))


def density(grids, phi, occ):
    psi = _to_real_host(grids, phi)
    return np.einsum("n,nr->r", np.asarray(occ, dtype=float), np.abs(psi) ** 2)


def hartree(grids, rho):
    rf = _fft(grids, rho)
    with np.errstate(divide="ignore", invalid="ignore"):
        vf = 4 * np.pi * rf / grids.g2_cube
    vf[grids.g2_cube == 0] = 0.0
    return _ifft(grids, vf).real


def lda_x(rho):
    return -((3.0 / np.pi) ** (1.0 / 3.0)) * np.cbrt(np.clip(rho, 0.0, None))


def local_potential(model, grids, v_ext, rho):
    v = v_ext + hartree(grids, rho)
    if model.xc == "lda_x":
        v = v + lda_x(rho)
    return v


def kerker_mix(grids, v, alpha):
    d = grids.g2_cube / (grids.g2_cube + alpha ** 2)
    d[grids.g2_cube == 0] = 1.0
    return _ifft(grids, _fft(grids, v) * d).real


def run_scf(model, tol, max_iter=200, *, mixing="kerker", kerker_alpha=0.8, damping=0.8,
            grids=None, verbose=False):
    """Damped fixed-point SCF (groundstate.py:333-394), dense diagonalisation."""
    if not tol > 0:
        raise ConfigurationError("scf tolerance must be positive")
    if mixing not in ("kerker", "identity"):
        raise ConfigurationError(f"unknown mixing {mixing!r}")
    grids = grids if grids is not None else build_grids(model.lattice, model.e_cut)
    v_ext = external_potential(model, grids)
    rho = np.full(grids.n_g, model.n_electrons / model.lattice.volume)
    n_states = min(grids.n_b, model.n_electrons // 2 + max(6, model.n_electrons // 4))
    weight = np.sqrt(model.lattice.volume / grids.n_g)
    res = np.inf
    for it in range(max_iter):
        v_loc = local_potential(model, grids, v_ext, rho)
        eps, phi = diagonalize_dense(grids, v_loc, n_states)
        mu, occ = fermi_and_occupations(eps, model.n_electrons, model.temperature, model.smearing)
        n_occ = int(np.max(np.nonzero(occ > model.occupation_threshold)[0])) + 1
        n_extra = max(3, int(np.ceil(0.1 * n_occ)))
        if n_occ + n_extra > n_states:
            if n_occ + n_extra > grids.n_b:
                raise NonConvergenceError(f"basis too small: need {n_occ + n_extra} states")
            n_states = min(grids.n_b, n_occ + n_extra + 4)
            continue
        rho_new = density(grids, phi, occ)
        resid = rho_new - rho
        res = float(np.linalg.norm(resid) * weight)
        if verbose:
            print(f"scf iter {it:3d}  residual {res:.3e}  fermi {mu:+.6f}")
        if res <= tol:
            keep = n_occ + n_extra
            return GroundState(model=model, grids=grids, phi=np.ascontiguousarray(phi[:, :keep]),
                               eps=eps[:keep].copy(), occ=occ[:keep].copy(), fermi_level=mu,
                               rho=rho_new, n_occ=n_occ, v_local=v_loc, scf_residual=res)
        step = kerker_mix(grids, resid, kerker_alpha) if mixing == "kerker" else resid
        rho = rho + damping * step
    raise NonConvergenceError(f"SCF did not reach {tol:.1e} in {max_iter} iterations",
                              residual=res)


def run_scf_k(model, kgrid, tol, max_iter=200, kerker_alpha=0.8, damping=0.8, n_states=None,
              verbose=False, eigensolver=None):
    """k-sampled SCF with a global Fermi level; returns a KGroundState.

    `eigensolver(grids, v_loc, n_states, guess)` -> (eps, phi) may replace the
    dense diagonalisation (e.g. lobpcg.gpu_lowest_states for large n_b).
    """
    kfr = monkhorst_pack(kgrid) if np.ndim(kgrid) == 1 else np.asarray(kgrid, dtype=float)
    nk = len(kfr)
    wk = np.full(nk, 1.0 / nk)
    grids = [build_grids(model.lattice, model.e_cut, k) for k in kfr]
    g0 = grids[0]
    v_ext = external_potential(model, g0)
    rho = np.full(g0.n_g, model.n_electrons / model.lattice.volume)
    if n_states is None:
        n_states = model.n_electrons // 2 + max(6, model.n_electrons // 4)
    weight = np.sqrt(model.lattice.volume / g0.n_g)
    res = np.inf
    guesses = [None] * nk
    for it in range(max_iter):
        v_loc = local_potential(model, g0, v_ext, rho)
        spectra = []
        for i, g in enumerate(grids):
            if eigensolver is None:
                spectra.append(diagonalize_dense(g, v_loc, n_states))
            else:
                spectra.append(eigensolver(g, v_loc, n_states, guesses[i]))
                guesses[i] = spectra[-1][1]
        all_eps = np.concatenate([e for e, _ in spectra])
        mu, _ = fermi_and_occupations(all_eps, model.n_electrons, model.temperature,
                                      model.smearing, np.repeat(wk, n_states))
        occf, _ = _smear(model)
        rho_new = np.zeros(g0.n_g)
        parts = []
        grow = False
        for g, (eps, phi), w in zip(grids, spectra, wk):
            occ = occf((eps - mu) / model.temperature)
            n_occ = int(np.max(np.nonzero(occ > model.occupation_threshold)[0])) + 1
            n_extra = max(3, int(np.ceil(0.1 * n_occ)))
            grow |= n_occ + n_extra > n_states
            rho_new += w * density(g, phi, occ)
            parts.append((g, eps, phi, occ, n_occ, n_extra))
        if grow:
            n_states += 8
            guesses = [None] * nk
            continue
        resid = rho_new - rho
        res = float(np.linalg.norm(resid) * weight)
        if verbose:
            print(f"k-scf iter {it:3d}  residual {res:.3e}  fermi {mu:+.6f}")
        if res <= tol:
            blocks = []
            for g, eps, phi, occ, n_occ, n_extra in parts:
                keep = n_occ + n_extra
                blocks.append(GroundState(model=model, grids=g,
                                          phi=np.ascontiguousarray(phi[:, :keep]),
                                          eps=eps[:keep].copy(), occ=occ[:keep].copy(),
                                          fermi_level=mu, rho=rho_new, n_occ=n_occ,
                                          v_local=v_loc, scf_residual=res))
            return KGroundState(model=model, blocks=blocks, weights=wk, kfracs=kfr,
                                fermi_level=mu, rho=rho_new, v_local=v_loc, scf_residual=res)
        rho = rho + damping * kerker_mix(g0, resid, kerker_alpha)
    raise NonConvergenceError(f"k-SCF did not reach {tol:.1e} in {max_iter} iterations",
                              residual=res)


def _smear(model):
    from .groundstate import smearing_function
    return smearing_function(model.smearing)
