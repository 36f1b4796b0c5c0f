"""Drop-in installation into the reference package `pwdyson`.

`install()` rebinds the reference's chi0-path operators to this package's
B200 implementations, in the defining modules AND in the modules that
imported them by name at load time (`from .response import apply_chi0` in
harness.py:30-36, `from .sternheimer import ...` in response.py:23, ...),
so `pwdyson.harness.run_response` and the reference CLI run on the GPU
unchanged.  The H-application counter stays the reference's own object
(groundstate.py:50), which this package's operators then increment.

The reference's GroundState / FourierGrids objects are accepted as they are
(duck-typed: `grids.g_int`, `g2_sphere`, `g2_cube`, `cube_dims`,
`lattice.volume`; `gs.phi`, `eps`, `occ`, `n_occ`, `v_local`, `rho`,
`fprime_occ()`), so ground states loaded from the reference's archives work.

There is no CPU fallback: after install() the patched operators raise
DeviceError on a machine without a B200.
"""

import importlib

from . import groundstate as _gs
from . import harness as _harness
from . import kernels as _kernels
from . import response as _response
from . import sternheimer as _stern

# reference module -> {name: replacement}; citations are the reference definitions
PATCHES = {
    "groundstate": {
        "apply_hamiltonian": _gs.apply_hamiltonian,             # groundstate.py:211
    },
    "sternheimer": {
        "project_out_occupied": _stern.project_out_occupied,     # sternheimer.py:28
        "solve_sternheimer": _stern.solve_sternheimer,           # sternheimer.py:33
        "apply_hamiltonian": _gs.apply_hamiltonian,              # imported at sternheimer.py:16
    },
    "kernels": {
        "apply_kernel": _kernels.apply_kernel,                   # kernels.py:40
        "apply_kerker": _kernels.apply_kerker,                   # kernels.py:60
    },
    "response": {
        "delta_eigen_occupations": _response.delta_eigen_occupations,   # response.py:45
        "delta_phi_occupied": _response.delta_phi_occupied,             # response.py:101
        "apply_chi0": _response.apply_chi0,                             # response.py:110
        "apply_dielectric": _response.apply_dielectric,                 # response.py:164
        "orbital_row_norm": _response.orbital_row_norm,                 # response.py:190
        "dielectric_error_bound": _response.dielectric_error_bound,     # response.py:202
        "apply_kernel": _kernels.apply_kernel,                          # imported at :22
        "project_out_occupied": _stern.project_out_occupied,            # imported at :23
        "solve_sternheimer": _stern.solve_sternheimer,                  # imported at :23
    },
    "harness": {                                                        # imports at :20-37
        "apply_chi0": _response.apply_chi0,
        "apply_dielectric": _response.apply_dielectric,
        "dielectric_error_bound": _response.dielectric_error_bound,
        "orbital_row_norm": _response.orbital_row_norm,
        "project_out_occupied": _stern.project_out_occupied,
        "solve_sternheimer": _stern.solve_sternheimer,
        "apply_kerker": _kernels.apply_kerker,
    },
}

# this package's modules that hold a module-level reference to the counter
_COUNTER_USERS = (_gs, _harness, _response, _stern)

_saved = {}


def install(package="pwdyson"):
    """Route `package`'s chi0 path through libpwb200.  Returns the patched names.

    `package` is the importable name (or the module object) of the reference.
    Idempotent; `uninstall()` restores the originals.
    """
    root = importlib.import_module(package) if isinstance(package, str) else package
    name = root.__name__
    patched = []
    for sub, names in PATCHES.items():
        mod = importlib.import_module(f"{name}.{sub}")
        for attr, repl in names.items():
            if not hasattr(mod, attr):
                raise AttributeError(f"{name}.{sub} has no {attr}: not the expected pwdyson")
            key = (name, sub, attr)
            if key not in _saved:
                _saved[key] = getattr(mod, attr)
            setattr(mod, attr, repl)
            patched.append(f"{sub}.{attr}")
    counter = importlib.import_module(f"{name}.groundstate").ham_counter
    key = ("__counter__",)
    if key not in _saved:
        _saved[key] = _gs.ham_counter
    for m in _COUNTER_USERS:
        m.ham_counter = counter
    return patched


def uninstall(package="pwdyson"):
    """Restore everything install() replaced."""
    root = importlib.import_module(package) if isinstance(package, str) else package
    name = root.__name__
    for key, orig in list(_saved.items()):
        if key == ("__counter__",):
            for m in _COUNTER_USERS:
                m.ham_counter = orig
            del _saved[key]
        elif key[0] == name:
            setattr(importlib.import_module(f"{name}.{key[1]}"), key[2], orig)
            del _saved[key]
