"""Transform / H-apply parity at the BASELINE grid sizes and the reference's toy
grids (compile-time FFT codelets and the runtime engine) against the CPU oracle."""

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

# (name, lattice vectors, e_cut, k fraction)
CASES = [
    ("cfg1_48", np.diag([15.0] * 3), 10.0, (0, 0, 0)),
    ("cfg1_48_k", np.diag([15.0] * 3), 10.0, (0.5, 0.5, 0.0)),
    ("cfg4_64", np.diag([20.0] * 3), 12.0, (0.25, 0, 0.5)),
    ("cfg2_32x320", np.diag([7.6, 7.6, 76.0]), 20.0, (0, 0, 0)),
    ("cfg3_96", np.diag([20.0] * 3), 26.0, (0, 0, 0)),
    ("toy_metal_216x6", np.diag([87.5, 2.6, 2.6]), 6.5, (0, 0, 0)),
    ("odd_10_12", np.diag([4.0, 5.0, 6.0]), 4.0, (0, 0, 0)),
]


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    _lib.require_device()


@pytest.mark.parametrize("name,a,ecut,k", CASES, ids=[c[0] for c in CASES])
def test_h_and_transforms_vs_oracle(name, a, ecut, k):
    from oracle import basis as ob
    from oracle import model as om
    from paper_2505_02319_b200 import ops
    from paper_2505_02319_b200.pwbasis import Lattice, build_grids
    g = build_grids(Lattice.from_vectors(*a), ecut, k)
    b = ob.make_basis(ob.Cell(a), ecut, k)
    np.testing.assert_array_equal(g.g_int, b.g_int)
    assert tuple(g.cube_dims) == tuple(b.cube_dims)
    rng = np.random.default_rng(7)
    nb = 3
    x = rng.standard_normal((nb, g.n_b)) + 1j * rng.standard_normal((nb, g.n_b))
    v = rng.standard_normal(g.n_g)
    h = ops.ham_apply_many(g, v, x)
    href = np.stack([om.ham_apply(b, v, xi, count=False) for xi in x])
    assert rel(h, href) < 1e-13
    r = ops.to_real_many(g, x[:2])
    assert rel(r, b.to_real_many(x[:2])) < 1e-13
    u = r[0] * v
    assert rel(ops.to_fourier(g, u), b.to_fourier(u)) < 1e-13
    assert rel(ops.cube_fft(g, v), b.cube_fft(v)) < 1e-13
