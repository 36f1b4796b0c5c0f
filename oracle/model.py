"""Oracle: toy solid, smearing, Hamiltonian apply, dense diagonalisation, SCF.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates pkg/src/pwdyson/groundstate.py:
  * Counter                  <- groundstate.py:22-48
  * Well / Model             <- groundstate.py:51-85
  * smearing                 <- groundstate.py:90-108
  * fermi_level              <- groundstate.py:111-149
  * v_external (+derivative) <- groundstate.py:154-206
  * ham_apply                <- groundstate.py:211-219
  * dense_h / lowest_states  <- groundstate.py:222-243
  * density / hartree / lda  <- groundstate.py:248-275
  * State (GroundState)      <- groundstate.py:280-326
  * scf                      <- groundstate.py:329-394
k-point extension: `KState` holds one State-like block per
k with a common V_local and a global Fermi level; `scf_k` restates the SCF
with a k-weighted density.
"""

import threading
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
from scipy.special import erfc, expit

from .basis import OracleConfigError, make_basis


class OracleNonConvergence(RuntimeError):
    """Mirror of pwdyson.errors.NonConvergenceError."""

    def __init__(self, message, residual=None, report=None):
        super().__init__(message)
        self.residual = residual
        self.report = report


class Counter:
    """Locked H-application counter (groundstate.py:22-48)."""

    def __init__(self):
        self._lock = threading.Lock()
        self._n = 0

    def add(self, n=1):
        with self._lock:
            self._n += n

    @property
    def value(self):
        with self._lock:
            return self._n


ham_counter = Counter()


@dataclass(frozen=True)
class Well:
    center: tuple
    amplitude: float
    width: float


@dataclass(frozen=True)
class Model:
    lattice: object
    e_cut: float
    n_electrons: int
    temperature: float
    smearing: str = "fermi_dirac"
    occupation_threshold: float = 1e-8
    xc: str = "none"
    gaussians: tuple = ()


def smearing(kind):
    """(f, f') pair on [0, 2) (groundstate.py:90-108)."""
    if kind == "fermi_dirac":
        return (lambda x: 2.0 * expit(-np.asarray(x, dtype=float)),
                lambda x: _fd_prime(np.asarray(x, dtype=float)))
    if kind == "gaussian":
        return (lambda x: erfc(np.asarray(x, dtype=float)),
                lambda x: -2.0 / np.sqrt(np.pi) * np.exp(-np.clip(np.asarray(x, float) ** 2, 0, 700)))
    raise OracleConfigError(f"unknown smearing {kind!r}")


def _fd_prime(x):
    s = expit(-x)
    return -2.0 * s * (1.0 - s)


def fermi_level(eps, n_el, temp, kind="fermi_dirac", weights=None):
    """Bisection for sum_n w_n f((eps_n - mu)/T) = N (groundstate.py:111-149).

    `weights` (k-point weights per state) is the k-extension; None is the
    reference's unit weight.
    """
    eps = np.asarray(eps, dtype=float)
    f, _ = smearing(kind)
    w = np.ones_like(eps) if weights is None else np.asarray(weights, dtype=float)
    target = float(n_el)
    if 2 * np.sum(w) <= n_el:
        raise OracleNonConvergence("retained states cannot hold the electrons")

    def filled(mu):
        return float(np.sum(w * f((eps - mu) / temp)))

    lo, hi = float(eps.min()) - temp, float(eps.max()) + temp
    while filled(lo) >= target:
        lo -= 10 * temp + abs(lo) * 0.1 + 1.0
    while filled(hi) < target:
        hi += 10 * temp + abs(hi) * 0.1 + 1.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if mid <= lo or mid >= hi:
            break
        if filled(mid) < target:
            lo = mid
        else:
            hi = mid
    mu = min((lo, hi), key=lambda m: abs(filled(m) - target))
    return mu, f((eps - mu) / temp)


def _images(cell, rcut):
    spacing = 2 * np.pi / np.linalg.norm(cell.b, axis=1)
    lim = np.ceil(rcut / spacing).astype(int)
    mesh = np.meshgrid(*[np.arange(-m, m + 1) for m in lim], indexing="ij")
    return np.stack([c.ravel() for c in mesh], axis=1) @ cell.a


def _rcut(model):
    widths = [g.width for g in model.gaussians] or [0.0]
    return 3.0 * max(widths) + float(np.sum(np.linalg.norm(model.lattice.a, axis=1)))


def v_external(model, basis):
    """Lattice-summed Gaussians on the cube (groundstate.py:172-184)."""
    v = np.zeros(basis.n_g)
    if not model.gaussians:
        return v
    pts = basis.points()
    shifts = _images(model.lattice, _rcut(model))
    for g in model.gaussians:
        c = np.asarray(g.center, dtype=float) @ model.lattice.a
        for s in shifts:
            d = pts - (c + s)
            v += g.amplitude * np.exp(-np.einsum("ij,ij->i", d, d) / (2 * g.width ** 2))
    return v


def ham_apply(basis, v_local, psi, count=True):
    """H psi = |G+k|^2/2 psi + F(V F^-1 psi), +1 count (groundstate.py:211-219)."""
    if psi.shape != (basis.n_b,):
        raise ValueError(f"expected sphere vector of length {basis.n_b}, got {psi.shape}")
    if v_local.shape != (basis.n_g,):
        raise ValueError(f"expected grid potential of length {basis.n_g}, got {v_local.shape}")
    out = 0.5 * basis.g2_sphere * psi + basis.to_fourier(v_local * basis.to_real(psi))
    if count:
        ham_counter.add(1)
    return out


def dense_h(basis, v_local):
    """Explicit Hamiltonian matrix (groundstate.py:222-234)."""
    vhat = basis.cube_fft(v_local) / basis.n_g
    nx, ny, nz = basis.cube_dims
    d = basis.g_int[:, None, :] - basis.g_int[None, :, :]
    idx = (d[..., 0] % nx) + nx * ((d[..., 1] % ny) + ny * (d[..., 2] % nz))
    h = vhat[idx]
    h[np.arange(basis.n_b), np.arange(basis.n_b)] += 0.5 * basis.g2_sphere
    return h


def lowest_states(basis, v_local, n):
    """Lowest n eigenpairs (groundstate.py:237-243)."""
    if n > basis.n_b:
        raise OracleConfigError(f"n_states={n} exceeds basis size {basis.n_b}")
    return scipy.linalg.eigh(dense_h(basis, v_local), subset_by_index=[0, n - 1])


def density(basis, phi, occ):
    """rho = sum_n f_n |F^-1 phi_n|^2 (groundstate.py:248-252)."""
    pr = basis.to_real_many(phi.T)
    return np.einsum("n,nr->r", np.asarray(occ, dtype=float), np.abs(pr) ** 2)


def hartree(basis, rho):
    """Zero-mean Poisson solution (groundstate.py:255-262)."""
    rf = basis.cube_fft(rho)
    with np.errstate(divide="ignore", invalid="ignore"):
        vf = 4 * np.pi * rf / basis.g2_cube
    vf[basis.g2_cube == 0] = 0.0
    return basis.cube_ifft(vf).real


def lda_x(rho):
    """Slater exchange potential (groundstate.py:265-267)."""
    return -((3.0 / np.pi) ** (1.0 / 3.0)) * np.cbrt(np.clip(rho, 0.0, None))


def v_total(model, basis, v_ext, rho):
    v = v_ext + hartree(basis, rho)
    if model.xc == "lda_x":
        v = v + lda_x(rho)
    return v


@dataclass
class State:
    """Converged ground state (groundstate.py:280-326)."""

    model: object
    grids: object
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
        _, fp = smearing(self.model.smearing)
        return fp((self.eps_occ - self.fermi_level) / self.model.temperature) / self.model.temperature


def _kerker(basis, v, alpha):
    damp = basis.g2_cube / (basis.g2_cube + alpha ** 2)
    damp[basis.g2_cube == 0] = 1.0
    return basis.cube_ifft(basis.cube_fft(v) * damp).real


def scf(model, tol, max_iter=200, mixing="kerker", kerker_alpha=0.8, damping=0.8, grids=None):
    """Damped Kerker/identity-mixed SCF (groundstate.py:333-394)."""
    if not tol > 0:
        raise OracleConfigError("scf tolerance must be positive")
    basis = grids if grids is not None else make_basis(model.lattice, model.e_cut)
    v_ext = v_external(model, basis)
    rho = np.full(basis.n_g, model.n_electrons / model.lattice.volume)
    n_states = min(basis.n_b, model.n_electrons // 2 + max(6, model.n_electrons // 4))
    weight = np.sqrt(model.lattice.volume / basis.n_g)
    res = np.inf
    for _ in range(max_iter):
        v_loc = v_total(model, basis, v_ext, rho)
        eps, phi = lowest_states(basis, v_loc, n_states)
        mu, occ = fermi_level(eps, model.n_electrons, model.temperature, model.smearing)
        n_occ = int(np.max(np.nonzero(occ > model.occupation_threshold)[0])) + 1
        n_extra = max(3, int(np.ceil(0.1 * n_occ)))
        if n_occ + n_extra > n_states:
            if n_occ + n_extra > basis.n_b:
                raise OracleNonConvergence("basis too small")
            n_states = min(basis.n_b, n_occ + n_extra + 4)
            continue
        rho_new = density(basis, phi, occ)
        resid = rho_new - rho
        res = np.linalg.norm(resid) * weight
        if res <= tol:
            keep = n_occ + n_extra
            return State(model=model, grids=basis, phi=np.ascontiguousarray(phi[:, :keep]),
                         eps=eps[:keep].copy(), occ=occ[:keep].copy(), fermi_level=mu,
                         rho=rho_new, n_occ=n_occ, v_local=v_loc, scf_residual=res)
        step = _kerker(basis, resid, kerker_alpha) if mixing == "kerker" else resid
        rho = rho + damping * step
    raise OracleNonConvergence(f"SCF did not reach {tol:.1e}", residual=res)


# -- k-point extension (no reference counterpart) -------------------

@dataclass
class KState:
    """Ground state sampled on k-points sharing V_local and the Fermi level.

    `blocks[i]` is a State-like object for k-point i (its own grids with the
    k-shifted sphere, phi, eps, occ, n_occ); `weights[i]` = w_k (sum 1).
    """

    model: object
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


def scf_k(model, kfracs, tol, max_iter=200, kerker_alpha=0.8, damping=0.8, n_states=None):
    """k-sampled restatement of scf(): density sum_k w_k sum_n f_nk |psi_nk|^2."""
    kfracs = np.asarray(kfracs, dtype=float)
    nk = len(kfracs)
    wk = np.full(nk, 1.0 / nk)
    bases = [make_basis(model.lattice, model.e_cut, k) for k in kfracs]
    b0 = bases[0]
    v_ext = v_external(model, b0)
    rho = np.full(b0.n_g, model.n_electrons / model.lattice.volume)
    if n_states is None:
        n_states = model.n_electrons // 2 + max(6, model.n_electrons // 4)
    weight = np.sqrt(model.lattice.volume / b0.n_g)
    res = np.inf
    for _ in range(max_iter):
        v_loc = v_total(model, b0, v_ext, rho)
        spectra = [lowest_states(b, v_loc, n_states) for b in bases]
        all_eps = np.concatenate([e for e, _ in spectra])
        all_w = np.repeat(wk, n_states)
        mu, _ = fermi_level(all_eps, model.n_electrons, model.temperature, model.smearing, all_w)
        f, _ = smearing(model.smearing)
        blocks = []
        rho_new = np.zeros(b0.n_g)
        grow = False
        for b, (eps, phi), w in zip(bases, spectra, wk):
            occ = f((eps - mu) / model.temperature)
            n_occ = int(np.max(np.nonzero(occ > model.occupation_threshold)[0])) + 1
            n_extra = max(3, int(np.ceil(0.1 * n_occ)))
            if n_occ + n_extra > n_states:
                grow = True
            rho_new += w * density(b, phi, occ)
            blocks.append((b, eps, phi, occ, n_occ, n_extra))
        if grow:
            n_states += 8
            continue
        resid = rho_new - rho
        res = np.linalg.norm(resid) * weight
        if res <= tol:
            out = []
            for b, eps, phi, occ, n_occ, n_extra in blocks:
                keep = n_occ + n_extra
                out.append(State(model=model, grids=b, phi=np.ascontiguousarray(phi[:, :keep]),
                                 eps=eps[:keep].copy(), occ=occ[:keep].copy(), fermi_level=mu,
                                 rho=rho_new, n_occ=n_occ, v_local=v_loc, scf_residual=res))
            return KState(model=model, blocks=out, weights=wk, kfracs=kfracs, fermi_level=mu,
                          rho=rho_new, v_local=v_loc, scf_residual=res)
        rho = rho + damping * _kerker(b0, resid, kerker_alpha)
    raise OracleNonConvergence(f"k-SCF did not reach {tol:.1e}", residual=res)
