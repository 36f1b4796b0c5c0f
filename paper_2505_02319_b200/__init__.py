"""B200-native (sm_100a) chi0 / Sternheimer hot path for the pwdyson Dyson solver.

Drop-in for the operator API of the reference package `pwdyson`
(arXiv 2505.02319): `apply_hamiltonian`, `project_out_occupied`,
`solve_sternheimer`, `apply_chi0`, `apply_dielectric`, `apply_kernel`,
`apply_kerker`, `igmres_solve`, `run_response`.  All hot arithmetic runs in
hand-written CUDA kernels (libpwb200.so, C-ABI in include/pwb200.h); the
Python modules hold host-side setup and the scalar logic of the outer
solver.  There is no CPU fallback: the operators raise if the CUDA library
or a GPU is missing.

The CUDA library is loaded lazily (first operator call), so setup-only
modules (`synth`, `pwbasis`) import without a GPU.
"""

__version__ = "0.1.0"

from .errors import (ArchiveError, ConfigurationError, InvariantViolationError,  # noqa: F401
                     NonConvergenceError, PwdysonError)


def install(package="pwdyson"):
    """Route the reference package's chi0 path through libpwb200 (see dropin.py)."""
    from .dropin import install as _install
    return _install(package)


def uninstall(package="pwdyson"):
    from .dropin import uninstall as _uninstall
    return _uninstall(package)
