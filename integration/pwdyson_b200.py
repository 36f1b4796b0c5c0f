"""Reference-side binding of libpwb200 -- the file a pwdyson maintainer would add
as `pwdyson/_b200.py` (numpy + ctypes only: no torch, no import of the
B200 package).

It binds the C-ABI declared in include/pwb200.h and re-exposes the
reference's operator signatures on top of it:

    apply_hamiltonian(grids, v_local, psi)                groundstate.py:211-219
    project_out_occupied(phi, psi)                        sternheimer.py:28-30
    apply_chi0(gs, dv, tolerances, threads=1)             response.py:110-161

so `pwdyson.response.apply_chi0 = _b200.apply_chi0` (plus the harness import
site) moves the hot path onto the GPU.  Inside pwdyson
the relative imports below resolve to the reference's own Chi0Stats,
ham_counter and exceptions; standalone (tests) it uses local stand-ins.

Library path: $PWB200_LIB, else ../paper_2505_02319_b200/libpwb200.so
relative to this file.
"""

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

try:                                   # inside pwdyson
    from .errors import ConfigurationError, NonConvergenceError, PwdysonError
    from .groundstate import ham_counter
    from .response import Chi0Stats
except ImportError:                    # standalone
    class PwdysonError(Exception):
        pass

    class ConfigurationError(PwdysonError):
        pass

    class NonConvergenceError(PwdysonError):
        def __init__(self, message, residual=None, report=None):
            super().__init__(message)
            self.residual = residual
            self.report = report

    class _Counter:
        value = 0

        def add(self, n=1):
            self.value += n

    ham_counter = _Counter()

    @dataclass
    class Chi0Stats:
        cg_iterations_per_band: list = field(default_factory=list)
        tolerances_used: list = field(default_factory=list)
        ham_applications: int = 0


_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_SIG = {
    "pwb_last_error": (ctypes.c_char_p, []),
    "pwb_grid_create": (_I, [_I, _I, _I, _D, _I, _P, _P, _P, _P, ctypes.POINTER(_P)]),
    "pwb_grid_destroy": (_I, [_P]),
    "pwb_grid_info": (_I, [_P, _P]),
    "pwb_ham_apply_host": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "pwb_state_create": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.POINTER(_P)]),
    "pwb_state_destroy": (_I, [_P]),
    "pwb_project_host": (_I, [_I, _I, _P, _I, _P]),
    "pwb_chi0_host": (_I, [_P, _P, _P, _P, _P]),
}
_lib = None


def lib():
    global _lib
    if _lib is None:
        path = os.environ.get("PWB200_LIB") or os.path.join(
            os.path.dirname(os.path.abspath(__file__)), "..", "paper_2505_02319_b200",
            "libpwb200.so")
        cdll = ctypes.CDLL(path)
        for name, (res, args) in _SIG.items():
            getattr(cdll, name).restype = res
            getattr(cdll, name).argtypes = args
        _lib = cdll
    return _lib


def _check(status, what):
    """Status codes -> the reference's exceptions (include/pwb200.h:35-43)."""
    if status == 0:
        return
    msg = f"{what}: {lib().pwb_last_error().decode(errors='replace')}"
    if status == 1:
        raise ValueError(msg)
    if status == 2:
        raise ConfigurationError(msg)
    if status == 3:
        raise NonConvergenceError(msg)
    raise PwdysonError(msg)


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


class _Grid:
    """pwb_grid for one (Gamma) FourierGrids, cached on the grids object."""

    def __init__(self, grids):
        nx, ny, nz = (int(d) for d in grids.cube_dims)
        self.n_b = int(grids.n_b)
        nb = np.array([self.n_b], dtype=np.int32)
        gint = np.ascontiguousarray(grids.g_int, dtype=np.int32)
        g2s = np.ascontiguousarray(grids.g2_sphere, dtype=np.float64)
        g2c = np.ascontiguousarray(grids.g2_cube, dtype=np.float64)
        h = ctypes.c_void_p()
        _check(lib().pwb_grid_create(nx, ny, nz, float(grids.lattice.volume), 1, _p(nb),
                                     _p(gint), _p(g2s), _p(g2c), ctypes.byref(h)),
               "pwb_grid_create")
        self.handle = h
        info = np.zeros(8, dtype=np.int32)
        _check(lib().pwb_grid_info(h, _p(info)), "pwb_grid_info")
        self.nbp = int(info[4])

    def __del__(self):
        if getattr(self, "handle", None) is not None and _lib is not None:
            _lib.pwb_grid_destroy(self.handle)


def _grid(grids):
    g = getattr(grids, "_b200_grid", None)
    if g is None:
        g = _Grid(grids)
        grids._b200_grid = g
    return g


def apply_hamiltonian(grids, v_local, psi):
    """H psi = |G|^2/2 psi + to_fourier(v_local * to_real(psi)) (groundstate.py:211-219)."""
    g = _grid(grids)
    rows = np.zeros((1, g.nbp), dtype=np.complex128)
    rows[0, : g.n_b] = psi
    out = np.empty_like(rows)
    v = np.ascontiguousarray(v_local, dtype=np.float64)
    _check(lib().pwb_ham_apply_host(g.handle, 1, None, _p(rows), _p(v), None, _p(out)),
           "pwb_ham_apply_host")
    ham_counter.add(1)
    return out[0, : g.n_b].copy()


def project_out_occupied(phi, psi):
    """psi - Phi (Phi^H psi) (sternheimer.py:28-30) on the FP64 tensor cores."""
    phi = np.ascontiguousarray(phi, dtype=np.complex128)
    psi = np.asarray(psi, dtype=np.complex128)
    vec = psi.ndim == 1
    x = np.ascontiguousarray((psi[:, None] if vec else psi).T)     # rows = columns of psi
    phit = np.ascontiguousarray(phi.T)
    n_b, n_occ = phi.shape
    _check(lib().pwb_project_host(n_b, n_occ, _p(phit), x.shape[0], _p(x)), "pwb_project_host")
    return x[0] if vec else x.T


class _State:
    """pwb_state for a reference GroundState (Gamma), cached on it."""

    def __init__(self, gs):
        g = _grid(gs.grids)
        self.grid = g
        n = int(gs.n_occ)
        phi = np.ascontiguousarray(gs.phi_occ.T, dtype=np.complex128)
        eps = np.ascontiguousarray(gs.eps_occ, dtype=np.float64)
        occ = np.ascontiguousarray(gs.occ_occ, dtype=np.float64)
        fpr = np.ascontiguousarray(gs.fprime_occ(), dtype=np.float64)
        v = np.ascontiguousarray(gs.v_local, dtype=np.float64)
        rho = np.ascontiguousarray(gs.rho, dtype=np.float64)
        nocc = np.array([n], dtype=np.int32)
        w = np.ones(1)
        h = ctypes.c_void_p()
        _check(lib().pwb_state_create(g.handle, _p(nocc), _p(w), _p(phi), _p(eps), _p(occ),
                                      _p(fpr), _p(v), _p(rho), ctypes.byref(h)),
               "pwb_state_create")
        self.handle = h
        self.n_occ = n

    def __del__(self):
        if getattr(self, "handle", None) is not None and _lib is not None:
            _lib.pwb_state_destroy(self.handle)


def apply_chi0(gs, dv, tolerances, threads=1):
    """(delta_rho, Chi0Stats) for a Gamma GroundState (response.py:110-161).

    `threads` is accepted for signature compatibility; the (k, n) solves run
    as one batched PCG on the GPU.
    """
    tolerances = np.asarray(tolerances, dtype=float)
    if tolerances.shape != (gs.n_occ,):
        raise ValueError(f"need one tolerance per occupied band ({gs.n_occ}), "
                         f"got shape {tolerances.shape}")
    if np.any(tolerances <= 0):
        raise ValueError("Sternheimer tolerances must be positive")
    st = gs.__dict__.get("_b200_state")
    if st is None:
        st = _State(gs)
        gs.__dict__["_b200_state"] = st
    dv = np.ascontiguousarray(dv, dtype=np.float64)
    tol = np.ascontiguousarray(tolerances)
    drho = np.empty(int(gs.grids.n_g))
    its = np.zeros(gs.n_occ, dtype=np.int32)
    _check(lib().pwb_chi0_host(st.handle, _p(dv), _p(tol), _p(drho), _p(its)), "pwb_chi0_host")
    total = int(its.sum())
    ham_counter.add(total)
    return drho, Chi0Stats(cg_iterations_per_band=[int(i) for i in its],
                           tolerances_used=list(tolerances), ham_applications=total)
