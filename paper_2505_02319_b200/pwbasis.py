"""Plane-wave sphere / FFT-cube geometry (host-side setup, no hot arithmetic).

Mirrors the public surface of the reference's pwbasis.py (Lattice
pwbasis.py:32-64, FourierGrids pwbasis.py:95-224, build_grids :227-236) so
user code and tests read the same, and adds the k-point sphere
|G + k| <= sqrt(2 E_cut).  The index tables built here
(lexicographic sphere order, wrapped x-fastest cube indices, |G|^2 on the
cube) define the layout contract with the CUDA library; the transforms
themselves (`to_real`, `to_fourier`, `cube_fft`, ...) run on the GPU through
libpwb200 and return numpy arrays.
"""

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError

TWO_PI = 2.0 * np.pi


@dataclass(frozen=True)
class Lattice:
    """Cell with lattice vectors as rows of `a`; b_i . a_j = 2 pi delta_ij."""

    a: np.ndarray
    b: np.ndarray
    volume: float

    @classmethod
    def from_vectors(cls, a1, a2, a3):
        a = np.array([a1, a2, a3], dtype=float)
        if not np.all(np.isfinite(a)):
            raise ConfigurationError("lattice vectors must be finite")
        det = float(np.linalg.det(a))
        if abs(det) < 1e-14:
            raise ConfigurationError("lattice vectors are linearly dependent")
        return cls(a=a, b=TWO_PI * np.linalg.inv(a).T, volume=abs(det))

    @classmethod
    def cubic(cls, alat):
        return cls.from_vectors([alat, 0, 0], [0, alat, 0], [0, 0, alat])

    @classmethod
    def orthorhombic(cls, ax, ay, az):
        return cls.from_vectors([ax, 0, 0], [0, ay, 0], [0, 0, az])

    def duality_defect(self):
        return float(np.max(np.abs(self.b @ self.a.T / TWO_PI - np.eye(3))))


def fft_size(n):
    """Smallest even 2,3,5-smooth integer >= max(2, n)."""
    n = max(2, int(n))
    while True:
        if n % 2 == 0:
            r = n
            for p in (2, 3, 5):
                while r % p == 0:
                    r //= p
            if r == 1:
                return n
        n += 1


def _candidates(a, radius):
    lim = np.floor(radius * np.linalg.norm(a, axis=1) / TWO_PI).astype(int)
    axes = np.meshgrid(*[np.arange(-m, m + 1) for m in lim], indexing="ij")
    return np.stack([ax.ravel() for ax in axes], axis=1)


class FourierGrids:
    """Sphere of orbital coefficients and the density cube for one k-point.

    Attributes follow the reference (pwbasis.py:101-112): lattice, e_cut,
    g_int, g_cart, g2_sphere, cube_dims, n_b, n_g, w, g2_cube, sphere_flat,
    plus `kfrac` (fractional k; zero for Gamma).
    """

    def __init__(self, lattice, e_cut, kfrac=(0.0, 0.0, 0.0)):
        if not np.isfinite(e_cut) or e_cut <= 0:
            raise ConfigurationError(f"e_cut must be positive, got {e_cut}")
        self.lattice = lattice
        self.e_cut = float(e_cut)
        self.kfrac = np.asarray(kfrac, dtype=float).copy()
        kc = self.kfrac @ lattice.b
        radius = np.sqrt(2.0 * e_cut)

        extra = np.linalg.norm(kc) if np.any(self.kfrac != 0) else 0.0
        ints = _candidates(lattice.a, radius + extra)
        vec = ints @ lattice.b + kc
        ints = ints[np.einsum("ij,ij->i", vec, vec) <= radius * radius * (1 + 1e-14)]
        ints = ints[np.lexsort((ints[:, 2], ints[:, 1], ints[:, 0]))]
        self.g_int = np.ascontiguousarray(ints)
        self.g_cart = self.g_int @ lattice.b + kc
        self.g2_sphere = np.einsum("ij,ij->i", self.g_cart, self.g_cart)
        self.n_b = len(self.g_int)

        box = _candidates(lattice.a, np.sqrt(3.0) * 2.0 * radius)
        inside = np.max(np.abs(box @ lattice.b), axis=1) <= 2.0 * radius * (1 + 1e-14)
        reach = np.max(np.abs(box[inside]), axis=0)
        self.cube_dims = tuple(fft_size(2 * int(r) + 2) for r in reach)
        self.n_g = int(np.prod(self.cube_dims))
        self.w = np.sqrt(lattice.volume) / np.sqrt(self.n_g)

        dims = np.array(self.cube_dims)
        wrapped = self.g_int % dims
        self.sphere_flat = np.ascontiguousarray(
            wrapped[:, 0] + dims[0] * (wrapped[:, 1] + dims[1] * wrapped[:, 2]))
        if len(np.unique(self.sphere_flat)) != self.n_b:
            raise ConfigurationError("cube grid cannot hold the sphere without aliasing")

        freq = [np.fft.fftfreq(n, 1.0 / n).astype(int) for n in self.cube_dims]
        fx, fy, fz = np.meshgrid(*freq, indexing="ij")
        cube = np.stack([fx.ravel(order="F"), fy.ravel(order="F"), fz.ravel(order="F")], axis=1)
        cc = cube @ lattice.b
        self.g2_cube = np.einsum("ij,ij->i", cc, cc)

    # -- layout helpers (pwbasis.py:166-180) -----------------------------------
    def cube_view(self, flat):
        return flat.reshape(self.cube_dims, order="F")

    def flat_view(self, cube):
        return cube.ravel(order="F")

    def real_space_points(self):
        fr = [np.arange(n) / n for n in self.cube_dims]
        fx, fy, fz = np.meshgrid(*fr, indexing="ij")
        st = np.stack([fx.ravel(order="F"), fy.ravel(order="F"), fz.ravel(order="F")], axis=1)
        return st @ self.lattice.a

    # -- transforms: GPU (libpwb200) ---------------------------------------------
    def to_real(self, coeffs):
        from . import ops
        return ops.to_real(self, coeffs)

    def to_fourier(self, values):
        from . import ops
        return ops.to_fourier(self, values)

    def to_real_many(self, coeffs):
        from . import ops
        return ops.to_real_many(self, coeffs)

    def to_fourier_many(self, values):
        from . import ops
        return ops.to_fourier_many(self, values)

    def cube_fft(self, values):
        from . import ops
        return ops.cube_fft(self, values)

    def cube_ifft(self, coeffs):
        from . import ops
        return ops.cube_ifft(self, coeffs)


def build_grids(lattice, e_cut, kfrac=(0.0, 0.0, 0.0)):
    """Sphere/cube grids for one cutoff (pwbasis.py:227-236), optionally k-shifted."""
    if lattice.duality_defect() > 1e-12:
        raise ConfigurationError("lattice reciprocal vectors violate b_i . a_j = 2 pi delta_ij")
    return FourierGrids(lattice, e_cut, kfrac)


def monkhorst_pack(shape):
    """Gamma-centred Monkhorst-Pack fractions in [-1/2, 1/2), k-point order n1 slowest."""
    out = []
    for i in range(shape[0]):
        for j in range(shape[1]):
            for m in range(shape[2]):
                f = np.array([i / shape[0], j / shape[1], m / shape[2]])
                out.append(f - np.floor(f + 0.5))
    return np.array(out)
