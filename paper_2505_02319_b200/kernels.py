"""Hartree (+ LDA exchange) kernel and the Kerker preconditioner on the GPU.

Drop-in for the reference kernels.py: `KernelSpec` (:18), `KerkerSpec` (:29),
`apply_kernel` (:40-57), `apply_kerker` (:60-70), `kerker_fourier_diagonal`
(:73-79).  Both operators are one full-cube FFT round trip with the Fourier
diagonal fused into the plane pass (and the pointwise LDA-x term fused into
the final pencil pass).
"""

from dataclasses import dataclass

import numpy as np

from .device import device_grid, torch_mod
from .errors import ConfigurationError
from .ops import kernel_apply_dev, kerker_apply_dev

LDA_X_DENSITY_FLOOR = 1e-10


@dataclass(frozen=True)
class KernelSpec:
    xc: str = "none"

    def __post_init__(self):
        if self.xc not in ("none", "lda_x"):
            raise ConfigurationError(f"unknown xc kernel {self.xc!r}")


@dataclass(frozen=True)
class KerkerSpec:
    alpha: float = 0.8

    def __post_init__(self):
        if not self.alpha >= 0:
            raise ConfigurationError(f"kerker alpha must be >= 0, got {self.alpha}")


def apply_kernel_dev(spec, dg, rho_t, v_t):
    return kernel_apply_dev(dg, spec.xc == "lda_x", rho_t, v_t)


def apply_kerker_dev(spec, dg, v_t):
    if spec.alpha == 0.0:
        return v_t.clone()
    return kerker_apply_dev(dg, spec.alpha, v_t)


def _dev(dg, v):
    torch = torch_mod()
    v = np.ascontiguousarray(v, dtype=float)
    if v.shape != (dg.n_g,):
        raise ValueError(f"expected grid vector of length {dg.n_g}, got {v.shape}")
    return torch.from_numpy(v).to(dg.device)


def apply_kernel(spec, grids, rho_ref, v):
    """K v = K_Hartree v (+ K_x v) (kernels.py:40-57)."""
    dg = device_grid(grids)
    return apply_kernel_dev(spec, dg, _dev(dg, rho_ref), _dev(dg, v)).cpu().numpy()


def apply_kerker(spec, grids, v):
    """T v = W^-1 D W v, D = |G|^2/(|G|^2+alpha^2), D(0) = 1 (kernels.py:60-70)."""
    if spec.alpha == 0.0:
        return np.array(v, dtype=float, copy=True)
    dg = device_grid(grids)
    return apply_kerker_dev(spec, dg, _dev(dg, v)).cpu().numpy()


def kerker_fourier_diagonal(spec, grids):
    """Fourier diagonal of T with the unit G = 0 entry (kernels.py:73-79); host table."""
    if spec.alpha == 0.0:
        return np.ones(grids.n_g)
    d = grids.g2_cube / (grids.g2_cube + spec.alpha ** 2)
    d[grids.g2_cube == 0] = 1.0
    return d
