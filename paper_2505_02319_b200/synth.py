"""Seeded synthetic inputs for the BASELINE configs.

Pure numpy setup code (no hot-path arithmetic).  The benchmark configs of
BASELINE.json describe models by distribution, not by data; this module
fixes the draw order so the oracle, the GPU path and the reference (via
tests/golden/gen_golden.py) all see the same inputs:

  * rng = numpy.random.default_rng(seed), seed 0 unless stated;
  * per well: centre (3 fractional uniforms), depth U(1, 3) -> amplitude =
    -depth, width U(0.5, 1.0);
  * then dV0: one standard normal per grid point (x-fastest), filtered in
    Fourier space by exp(-|G|^2 sigma^2 / 2) with sigma = 1 bohr, real part.

The model-building helpers take the classes to instantiate as arguments so
the same draws can build reference objects (golden generation) or this
package's objects.
"""

import numpy as np

SIGMA_SMOOTH = 1.0


def draw_wells(rng, count):
    """[(center, amplitude, width)] with the App. A draw order."""
    out = []
    for _ in range(count):
        center = tuple(float(c) for c in rng.uniform(0.0, 1.0, 3))
        depth = float(rng.uniform(1.0, 3.0))
        width = float(rng.uniform(0.5, 1.0))
        out.append((center, -depth, width))
    return out


def smoothed_noise(g2_cube, cube_dims, rng, sigma=SIGMA_SMOOTH):
    """White noise on the cube filtered by exp(-|G|^2 sigma^2/2) (real part)."""
    n_g = int(np.prod(cube_dims))
    raw = rng.standard_normal(n_g)
    cube = raw.reshape(cube_dims, order="F")
    spec = np.fft.fftn(cube) * np.exp(-0.5 * sigma * sigma * g2_cube.reshape(cube_dims, order="F"))
    return np.ascontiguousarray(np.fft.ifftn(spec).real.ravel(order="F"))


def smoothed_uniform(g2_cube, cube_dims, rng, lo=-1.0, hi=1.0, sigma=SIGMA_SMOOTH):
    """U(lo, hi) per grid point, smoothed with the same filter (config 3's V_loc)."""
    n_g = int(np.prod(cube_dims))
    raw = rng.uniform(lo, hi, n_g)
    cube = raw.reshape(cube_dims, order="F")
    spec = np.fft.fftn(cube) * np.exp(-0.5 * sigma * sigma * g2_cube.reshape(cube_dims, order="F"))
    return np.ascontiguousarray(np.fft.ifftn(spec).real.ravel(order="F"))


# name -> parameters (choices recorded in DESIGN.md)
CONFIGS = {
    0: dict(cell=("cubic", 10.0), e_cut=6.0, n_electrons=8, n_wells=4, temperature=2e-4,
            smearing="fermi_dirac", xc="lda_x", kgrid=(1, 1, 1), tau=1e-8, strategy="bal", m=10,
            seed=0),
    1: dict(cell=("cubic", 15.0), e_cut=10.0, n_electrons=64, n_wells=16, temperature=2e-4,
            smearing="fermi_dirac", xc="lda_x", kgrid=(2, 2, 2), tau=1e-9, strategy="bal", m=10,
            seed=0),
    2: dict(cell=("box", 7.6, 7.6, 76.0), e_cut=20.0, n_electrons=120, n_wells=40,
            temperature=1e-2, smearing="fermi_dirac", xc="lda_x", kgrid=(1, 1, 1), tau=1e-8,
            strategy="pbal", m=10, seed=0, n_states=128),   # 90 states reach the block edge
    3: dict(cell=("cubic", 20.0), e_cut=26.0, n_bands=256, kgrid=(1, 1, 1), seed=0),
    4: dict(cell=("cubic", 20.0), e_cut=12.0, n_electrons=128, n_wells=32, temperature=2e-4,
            smearing="fermi_dirac", xc="lda_x", kgrid=(4, 4, 2), tau=1e-8, strategy="bal", m=10,
            seed=0),
}


def cell_vectors(cell):
    if cell[0] == "cubic":
        a = cell[1]
        return [[a, 0, 0], [0, a, 0], [0, 0, a]]
    return [[cell[1], 0, 0], [0, cell[2], 0], [0, 0, cell[3]]]


def fcc_slab_wells(rng, a=7.6, layers=10, disp=0.05, depth=2.0, width=0.8):
    """Config 2: fcc sites of an a-cube stacked `layers` times along z, N(0, disp) shifts."""
    base = [(0, 0, 0), (0.5, 0.5, 0), (0.5, 0, 0.5), (0, 0.5, 0.5)]
    out = []
    lz = a * layers
    for layer in range(layers):
        for (fx, fy, fz) in base:
            d = rng.normal(0.0, disp, 3)
            cart = np.array([fx * a, fy * a, (fz + layer) * a]) + d
            frac = (cart[0] / a, cart[1] / a, cart[2] / lz)
            out.append((tuple(float(f) for f in frac), -depth, width))
    return out


def model_parameters(config_id, seed=None):
    """(params dict, wells, rng) with the rng positioned after the well draws."""
    p = dict(CONFIGS[config_id])
    rng = np.random.default_rng(p["seed"] if seed is None else seed)
    if config_id == 2:
        wells = fcc_slab_wells(rng)
    elif config_id == 3:
        wells = []
    else:
        wells = draw_wells(rng, p["n_wells"])
    return p, wells, rng


def config0_model(Lattice, GaussianWell, ModelSpec, seed=None):
    """Config 0 model built from the given classes; returns dict(model, rng)."""
    return build_model(0, Lattice, GaussianWell, ModelSpec, seed)


def build_model(config_id, Lattice, GaussianWell, ModelSpec, seed=None):
    p, wells, rng = model_parameters(config_id, seed)
    lat = Lattice.from_vectors(*cell_vectors(p["cell"]))
    model = ModelSpec(lattice=lat, e_cut=p["e_cut"], n_electrons=p["n_electrons"],
                      temperature=p["temperature"], smearing=p["smearing"], xc=p["xc"],
                      gaussians=tuple(GaussianWell(center=c, amplitude=a, width=w)
                                      for c, a, w in wells))
    return dict(model=model, rng=rng, params=p)


def random_orthonormal(rng, n_b, n_bands):
    """Config 3: complex normal columns (real then imaginary draws), QR-orthonormalised."""
    re = rng.standard_normal((n_b, n_bands))
    im = rng.standard_normal((n_b, n_bands))
    q, _ = np.linalg.qr(re + 1j * im)
    return np.ascontiguousarray(q)
