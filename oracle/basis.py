"""Oracle: lattice, plane-wave sphere, FFT cube and the normalised transforms.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates pkg/src/pwdyson/pwbasis.py of the reference:
  * Lattice                 <- pwbasis.py:32-64
  * 5-smooth even dims      <- pwbasis.py:67-80
  * integer search box      <- pwbasis.py:83-92
  * Basis (FourierGrids)    <- pwbasis.py:95-162
  * to_real / to_fourier    <- pwbasis.py:184-214
  * cube_fft / cube_ifft    <- pwbasis.py:218-224
The k-point extension (sphere |G+k| <= sqrt(2 Ecut)) is
new: the reference is Gamma-only.  With k = 0 it reduces to the
reference construction exactly.
"""

import numpy as np
import scipy.fft

TWO_PI = 2.0 * np.pi


class OracleConfigError(ValueError):
    """Mirror of pwdyson.errors.ConfigurationError for oracle-side checks."""


class Cell:
    """Real-space cell; rows of `a` are lattice vectors (pwbasis.py:32-52)."""

    def __init__(self, a):
        a = np.array(a, dtype=float)
        if not np.all(np.isfinite(a)):
            raise OracleConfigError("lattice vectors must be finite")
        det = np.linalg.det(a)
        if abs(det) < 1e-14:
            raise OracleConfigError("lattice vectors are linearly dependent")
        self.a = a
        self.b = TWO_PI * np.linalg.inv(a).T
        self.volume = abs(det)

    @staticmethod
    def cubic(alat):
        return Cell(np.diag([alat, alat, alat]))

    @staticmethod
    def box(ax, ay, az):
        return Cell(np.diag([ax, ay, az]))


def smooth_even(n):
    """Smallest even 2,3,5-smooth integer >= max(2, n) (pwbasis.py:67-80)."""
    n = max(2, int(n))
    while True:
        if n % 2 == 0:
            m = n
            for p in (2, 3, 5):
                while m % p == 0:
                    m //= p
            if m == 1:
                return n
        n += 1


def search_box(a, radius):
    """Integer triples possibly inside a ball of `radius` (pwbasis.py:83-92)."""
    lim = np.floor(radius * np.linalg.norm(a, axis=1) / TWO_PI).astype(int)
    axes = [np.arange(-m, m + 1) for m in lim]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([c.ravel() for c in mesh], axis=1)


class Basis:
    """Sphere of orbital coefficients plus the density cube.

    Restates FourierGrids.__init__ (pwbasis.py:114-162).  `kfrac` (fractional
    reciprocal coordinates) shifts the sphere to |G+k| <= sqrt(2 Ecut); the
    cube is always the Gamma cube so all k share one real-space grid.
    """

    def __init__(self, cell, e_cut, kfrac=(0.0, 0.0, 0.0)):
        if not np.isfinite(e_cut) or e_cut <= 0:
            raise OracleConfigError(f"e_cut must be positive, got {e_cut}")
        self.lattice = cell
        self.e_cut = float(e_cut)
        self.kfrac = np.asarray(kfrac, dtype=float)
        kcart = self.kfrac @ cell.b
        rs = np.sqrt(2.0 * e_cut)

        # sphere: lexicographic on (i1, i2, i3)  [pwbasis.py:123-132]
        pad = 1 if np.any(self.kfrac != 0) else 0
        cand = search_box(cell.a, rs + pad * np.linalg.norm(kcart))
        shifted = cand @ cell.b + kcart
        keep = np.einsum("ij,ij->i", shifted, shifted) <= rs * rs * (1 + 1e-14)
        gi = cand[keep]
        gi = gi[np.lexsort((gi[:, 2], gi[:, 1], gi[:, 0]))]
        self.g_int = np.ascontiguousarray(gi)
        self.g_cart = self.g_int @ cell.b + kcart
        self.g2_sphere = np.einsum("ij,ij->i", self.g_cart, self.g_cart)
        self.n_b = len(self.g_int)

        # cube: even 5-smooth box holding |G|_inf <= 2 sqrt(2 Ecut) [:134-142]
        rc = 2.0 * rs
        cand = search_box(cell.a, np.sqrt(3.0) * rc)
        inside = np.max(np.abs(cand @ cell.b), axis=1) <= rc * (1 + 1e-14)
        extent = np.max(np.abs(cand[inside]), axis=0)
        self.cube_dims = tuple(smooth_even(2 * int(e) + 2) for e in extent)
        self.n_g = int(np.prod(self.cube_dims))
        self.w = np.sqrt(cell.volume) / np.sqrt(self.n_g)

        nx, ny, nz = self.cube_dims
        wrap = self.g_int % np.array(self.cube_dims)
        self.sphere_flat = np.ascontiguousarray(wrap[:, 0] + nx * (wrap[:, 1] + ny * wrap[:, 2]))
        if len(np.unique(self.sphere_flat)) != self.n_b:
            raise OracleConfigError("cube grid cannot hold the sphere without aliasing")

        # |G|^2 on the cube, x fastest [:152-159]
        f = [np.fft.fftfreq(n, 1.0 / n).astype(int) for n in self.cube_dims]
        fx, fy, fz = np.meshgrid(*f, indexing="ij")
        ci = np.stack([fx.ravel(order="F"), fy.ravel(order="F"), fz.ravel(order="F")], axis=1)
        cc = ci @ cell.b
        self.g2_cube = np.einsum("ij,ij->i", cc, cc)
        self._up = self.n_g / np.sqrt(cell.volume)      # to_real scale
        self._down = np.sqrt(cell.volume) / self.n_g    # to_fourier scale

    # layout helpers (pwbasis.py:166-180)
    def cube(self, flat):
        return flat.reshape(self.cube_dims, order="F")

    def flat(self, cube):
        return cube.ravel(order="F")

    def points(self):
        fr = [np.arange(n) / n for n in self.cube_dims]
        fx, fy, fz = np.meshgrid(*fr, indexing="ij")
        st = np.stack([fx.ravel(order="F"), fy.ravel(order="F"), fz.ravel(order="F")], axis=1)
        return st @ self.lattice.a

    # transforms (pwbasis.py:184-224)
    def to_real(self, c):
        if c.shape != (self.n_b,):
            raise ValueError(f"expected sphere vector of length {self.n_b}, got {c.shape}")
        buf = np.zeros(self.n_g, dtype=np.complex128)
        buf[self.sphere_flat] = c
        return self.flat(scipy.fft.ifftn(self.cube(buf))) * self._up

    def to_fourier(self, u):
        if u.shape != (self.n_g,):
            raise ValueError(f"expected grid vector of length {self.n_g}, got {u.shape}")
        spec = scipy.fft.fftn(self.cube(u.astype(np.complex128)))
        return self.flat(spec)[self.sphere_flat] * self._down

    def to_real_many(self, c):
        k = c.shape[0]
        buf = np.zeros((k, self.n_g), dtype=np.complex128)
        buf[:, self.sphere_flat] = c
        out = scipy.fft.ifftn(buf.reshape((k, *self.cube_dims), order="F"), axes=(1, 2, 3))
        return out.reshape(k, self.n_g, order="F") * self._up

    def to_fourier_many(self, u):
        k = u.shape[0]
        spec = scipy.fft.fftn(u.astype(np.complex128).reshape((k, *self.cube_dims), order="F"),
                              axes=(1, 2, 3))
        return spec.reshape(k, self.n_g, order="F")[:, self.sphere_flat] * self._down

    def cube_fft(self, u):
        return self.flat(scipy.fft.fftn(self.cube(u.astype(np.complex128))))

    def cube_ifft(self, c):
        return self.flat(scipy.fft.ifftn(self.cube(c)))


def make_basis(cell, e_cut, kfrac=(0.0, 0.0, 0.0)):
    """build_grids (pwbasis.py:227-236) with the duality check."""
    defect = float(np.max(np.abs(cell.b @ cell.a.T / TWO_PI - np.eye(3))))
    if defect > 1e-12:
        raise OracleConfigError("reciprocal vectors violate b.a = 2 pi")
    return Basis(cell, e_cut, kfrac)


def monkhorst_pack(shape):
    """Gamma-centred MP grid as fractional k-vectors in [-1/2, 1/2)."""
    n1, n2, n3 = shape
    ks = []
    for i in range(n1):
        for j in range(n2):
            for l in range(n3):
                f = np.array([i / n1, j / n2, l / n3])
                f = f - np.floor(f + 0.5)
                ks.append(f)
    return np.array(ks)
