"""Toy-solid model, ground-state containers and the GPU Hamiltonian apply.

Public surface mirrors the reference's groundstate.py: `ham_counter`
(groundstate.py:22-48), `GaussianWell` / `ModelSpec` (:51-85),
`smearing_function` (:90-108), `fermi_and_occupations` (:111-149),
`external_potential[_derivative]` (:172-206), `apply_hamiltonian`
(:211-219), `GroundState` (:280-326) and `run_scf` (:333-394, in scf.py).

`apply_hamiltonian` is the hot operator and runs on the B200 through
libpwb200 (fused pruned FFT + V(r) + kinetic).  The model helpers and the
ground-state generation are setup code that produce the inputs of the hot
path (out of the hot-path scope).
"""

import threading
from dataclasses import dataclass, field

import numpy as np
from scipy.special import erfc, expit

from .errors import ConfigurationError, NonConvergenceError
from .pwbasis import FourierGrids, Lattice


class HamiltonianCounter:
    """Thread-safe count of Hamiltonian applications (groundstate.py:22-45)."""

    def __init__(self):
        self._lock = threading.Lock()
        self._count = 0

    def add(self, n=1):
        with self._lock:
            self._count += int(n)

    def reset(self):
        with self._lock:
            self._count = 0

    @property
    def value(self):
        with self._lock:
            return self._count


ham_counter = HamiltonianCounter()


@dataclass(frozen=True)
class GaussianWell:
    center: tuple
    amplitude: float
    width: float

    def __post_init__(self):
        if not self.width > 0:
            raise ConfigurationError(f"gaussian width must be positive, got {self.width}")


@dataclass(frozen=True)
class ModelSpec:
    lattice: Lattice
    e_cut: float
    n_electrons: int
    temperature: float
    smearing: str = "fermi_dirac"
    occupation_threshold: float = 1e-8
    xc: str = "none"
    gaussians: tuple = ()

    def __post_init__(self):
        if self.n_electrons <= 0 or self.n_electrons % 2 != 0:
            raise ConfigurationError("n_electrons must be an even positive integer")
        if not self.temperature > 0:
            raise ConfigurationError("temperature must be positive")
        if self.smearing not in ("fermi_dirac", "gaussian"):
            raise ConfigurationError(f"unknown smearing {self.smearing!r}")
        if self.xc not in ("none", "lda_x"):
            raise ConfigurationError(f"unknown xc {self.xc!r}")
        if not 0 < self.occupation_threshold < 2:
            raise ConfigurationError("occupation_threshold must lie in (0, 2)")


def smearing_function(kind):
    """(f, f') on [0, 2) for Fermi-Dirac or Gaussian smearing (groundstate.py:90-108)."""
    if kind == "fermi_dirac":
        def occ(x):
            return 2.0 * expit(-np.asarray(x, dtype=float))

        def docc(x):
            s = expit(-np.asarray(x, dtype=float))
            return -2.0 * s * (1.0 - s)
    elif kind == "gaussian":
        def occ(x):
            return erfc(np.asarray(x, dtype=float))

        def docc(x):
            x = np.asarray(x, dtype=float)
            return -2.0 / np.sqrt(np.pi) * np.exp(-np.clip(x * x, 0, 700))
    else:
        raise ConfigurationError(f"unknown smearing {kind!r}")
    return occ, docc


def fermi_and_occupations(eps, n_electrons, temperature, smearing="fermi_dirac", weights=None):
    """Fermi level by bisection (groundstate.py:111-149); `weights` = k weights per state."""
    eps = np.asarray(eps, dtype=float)
    occ, _ = smearing_function(smearing)
    w = np.ones_like(eps) if weights is None else np.asarray(weights, dtype=float)
    target = float(n_electrons)
    if 2 * float(np.sum(w)) <= n_electrons:
        raise NonConvergenceError(
            f"{len(eps)} states cannot hold {n_electrons} electrons; retain more states")

    def count(mu):
        return float(np.sum(w * occ((eps - mu) / temperature)))

    lo = float(eps.min()) - temperature
    hi = float(eps.max()) + temperature
    while count(lo) >= target:
        lo -= 10 * temperature + abs(lo) * 0.1 + 1.0
    while count(hi) < target:
        hi += 10 * temperature + abs(hi) * 0.1 + 1.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if mid <= lo or mid >= hi:
            break
        if count(mid) < target:
            lo = mid
        else:
            hi = mid
    mu = min((lo, hi), key=lambda m: abs(count(m) - target))
    return mu, occ((eps - mu) / temperature)


def _shifts(lattice, r_cut):
    spacing = 2 * np.pi / np.linalg.norm(lattice.b, axis=1)
    lim = np.ceil(r_cut / spacing).astype(int)
    mesh = np.meshgrid(*[np.arange(-m, m + 1) for m in lim], indexing="ij")
    return np.stack([c.ravel() for c in mesh], axis=1) @ lattice.a


def _cutoff(model):
    widths = [g.width for g in model.gaussians] or [0.0]
    return 3.0 * max(widths) + float(np.sum(np.linalg.norm(model.lattice.a, axis=1)))


def external_potential(model, grids):
    """Lattice-summed Gaussian wells on the cube (groundstate.py:172-184)."""
    v = np.zeros(grids.n_g)
    if not model.gaussians:
        return v
    a = np.asarray(model.lattice.a, dtype=float)
    if not np.any(a - np.diag(np.diag(a))):
        return _external_potential_orthogonal(model, grids)
    pts = grids.real_space_points()
    shifts = _shifts(model.lattice, _cutoff(model))
    for g in model.gaussians:
        c = np.asarray(g.center, dtype=float) @ model.lattice.a
        for s in shifts:
            d = pts - (c + s)
            v += g.amplitude * np.exp(-np.einsum("ij,ij->i", d, d) / (2 * g.width ** 2))
    return v


def _external_potential_orthogonal(model, grids):
    """The same lattice sum for an orthogonal cell: the shift set is a product mesh
    (_shifts) and the Gaussian factorises over the axes, so each well is an outer
    product of three 1-D image sums.  The point-by-point loop above costs
    wells x images x N_g (40 x 3645 x 327 680 at configs[2]: ten minutes of host
    time); this is wells x (images + N) per axis.  Same value up to summation order."""
    a = np.diag(np.asarray(model.lattice.a, dtype=float))
    spacing = 2 * np.pi / np.linalg.norm(model.lattice.b, axis=1)
    lim = np.ceil(_cutoff(model) / spacing).astype(int)
    v = np.zeros(tuple(grids.cube_dims))
    for g in model.gaussians:
        c = np.asarray(g.center, dtype=float) * a
        f = []
        for ax in range(3):
            x = np.arange(grids.cube_dims[ax]) / grids.cube_dims[ax] * a[ax]
            s = np.arange(-lim[ax], lim[ax] + 1) * a[ax]
            d = x[:, None] - (c[ax] + s[None, :])
            f.append(np.exp(-d * d / (2 * g.width ** 2)).sum(axis=1))
        v += g.amplitude * f[0][:, None, None] * f[1][None, :, None] * f[2][None, None, :]
    return np.ascontiguousarray(v.ravel(order="F"))


def external_potential_derivative(model, grids, index, direction):
    """Centre derivative of one well's lattice sum along a unit direction (:187-206)."""
    if not 0 <= index < len(model.gaussians):
        raise ConfigurationError(f"gaussian index {index} out of range")
    direction = np.asarray(direction, dtype=float)
    nrm = np.linalg.norm(direction)
    if nrm == 0 or not np.all(np.isfinite(direction)):
        raise ConfigurationError("perturbation direction must be a nonzero vector")
    direction = direction / nrm
    g = model.gaussians[index]
    pts = grids.real_space_points()
    c = np.asarray(g.center, dtype=float) @ model.lattice.a
    dv = np.zeros(grids.n_g)
    for s in _shifts(model.lattice, _cutoff(model)):
        d = pts - (c + s)
        gauss = np.exp(-np.einsum("ij,ij->i", d, d) / (2 * g.width ** 2))
        dv += g.amplitude * gauss * (d @ direction) / g.width ** 2
    return dv


def apply_hamiltonian(grids, v_local, psi):
    """H psi = |G|^2/2 psi + to_fourier(v_local to_real(psi)) on the GPU; +1 count.

    Drop-in for groundstate.py:211-219 (same argument checks and counting).
    """
    psi = np.asarray(psi)
    v_local = np.asarray(v_local)
    if psi.shape != (grids.n_b,):
        raise ValueError(f"expected sphere vector of length {grids.n_b}, got {psi.shape}")
    if v_local.shape != (grids.n_g,):
        raise ValueError(f"expected grid potential of length {grids.n_g}, got {v_local.shape}")
    from .ops import ham_apply_many
    out = ham_apply_many(grids, v_local, psi[None, :])[0]
    ham_counter.add(1)
    return out


def apply_hamiltonian_many(grids, v_local, psi_rows):
    """Batched H over rows of (k, n_b); counts k applications."""
    from .ops import ham_apply_many
    out = ham_apply_many(grids, v_local, psi_rows)
    ham_counter.add(len(out))
    return out


@dataclass
class GroundState:
    """Converged Gamma-point ground state (groundstate.py:280-326)."""

    model: ModelSpec
    grids: FourierGrids
    phi: np.ndarray
    eps: np.ndarray
    occ: np.ndarray
    fermi_level: float
    rho: np.ndarray
    n_occ: int
    v_local: np.ndarray
    scf_residual: float = 0.0
    _row_norm_cache: dict = field(default_factory=dict, repr=False)

    @property
    def n_kept(self):
        return self.phi.shape[1]

    @property
    def phi_occ(self):
        return self.phi[:, : self.n_occ]

    @property
    def occ_occ(self):
        return self.occ[: self.n_occ]

    @property
    def eps_occ(self):
        return self.eps[: self.n_occ]

    @property
    def eps_gap_ref(self):
        return float(self.eps[self.n_occ])

    def fprime_occ(self):
        _, fp = smearing_function(self.model.smearing)
        x = (self.eps_occ - self.fermi_level) / self.model.temperature
        return fp(x) / self.model.temperature


@dataclass
class KGroundState:
    """k-sampled ground state: one GroundState-like block per k.

    All blocks share `v_local`, `rho` and the Fermi level; `weights` are the
    k weights w_k (sum 1) and `kfracs` the fractional k-vectors.
    """

    model: ModelSpec
    blocks: list
    weights: np.ndarray
    kfracs: np.ndarray
    fermi_level: float
    rho: np.ndarray
    v_local: np.ndarray
    scf_residual: float = 0.0

    @property
    def grids(self):
        return self.blocks[0].grids

    @property
    def n_occ(self):
        return int(sum(b.n_occ for b in self.blocks))


def run_scf(*args, **kwargs):
    """Ground-state generation (setup; see scf.py)."""
    from .scf import run_scf as _run
    return _run(*args, **kwargs)
