"""Numpy-facing wrappers of the libpwb200 sphere/cube operators.

Each function is the GPU implementation of one reference call site and
returns numpy arrays (host in, host out), so it can replace the reference
function one-for-one.  Device-resident variants (`*_dev`) take and return
torch tensors for use inside the device-resident solvers.
"""

import numpy as np

from . import _lib
from .device import device_grid, ptr, torch_mod


def _dg(grids):
    return device_grid(grids)


def _rows_from(dg, coeffs):
    coeffs = np.asarray(coeffs)
    if coeffs.ndim != 2 or coeffs.shape[1] != dg.nb[0]:
        raise ValueError(f"expected (k, {dg.nb[0]}) sphere rows, got {coeffs.shape}")
    return dg.pack(coeffs.astype(np.complex128))


def to_real_many_dev(dg, rows, band_k=None):
    """pwb_to_real on device rows -> (n, n_g) complex device tensor."""
    torch = torch_mod()
    n = rows.shape[0]
    out = torch.empty((n, dg.n_g), dtype=torch.complex128, device=dg.device)
    _lib.check(_lib.load().pwb_to_real(dg.handle, n, ptr(band_k), ptr(rows), ptr(out)), "to_real")
    return out


def to_fourier_many_dev(dg, values, band_k=None):
    torch = torch_mod()
    n = values.shape[0]
    out = dg.rows(n)
    _lib.check(_lib.load().pwb_to_fourier(dg.handle, n, ptr(band_k), ptr(values), ptr(out)),
               "to_fourier")
    return out


def to_real_many(grids, coeffs):
    """to_real_many (pwbasis.py:200-207) on the GPU."""
    dg = _dg(grids)
    out = to_real_many_dev(dg, _rows_from(dg, coeffs))
    return out.cpu().numpy()


def to_real(grids, coeffs):
    """to_real (pwbasis.py:184-191) on the GPU."""
    coeffs = np.asarray(coeffs)
    if coeffs.shape != (grids.n_b,):
        raise ValueError(f"expected sphere vector of length {grids.n_b}, got {coeffs.shape}")
    return to_real_many(grids, coeffs[None, :])[0]


def to_fourier_many(grids, values):
    """to_fourier_many (pwbasis.py:209-214) on the GPU."""
    torch = torch_mod()
    dg = _dg(grids)
    values = np.asarray(values)
    if values.ndim != 2 or values.shape[1] != dg.n_g:
        raise ValueError(f"expected (k, {dg.n_g}) grid rows, got {values.shape}")
    vt = torch.from_numpy(np.ascontiguousarray(values, dtype=np.complex128)).to(dg.device)
    out = to_fourier_many_dev(dg, vt)
    return np.stack(dg.unpack(out))


def to_fourier(grids, values):
    """to_fourier (pwbasis.py:193-198) on the GPU."""
    values = np.asarray(values)
    if values.shape != (grids.n_g,):
        raise ValueError(f"expected grid vector of length {grids.n_g}, got {values.shape}")
    return to_fourier_many(grids, values[None, :])[0]


def cube_fft_dev(dg, vt, inverse=False):
    torch = torch_mod()
    vt = vt.to(torch.complex128)
    out = torch.empty_like(vt)
    n = 1 if vt.dim() == 1 else vt.shape[0]
    _lib.check(_lib.load().pwb_cube_fft(dg.handle, n, ptr(vt), ptr(out), 1 if inverse else 0),
               "cube_fft")
    return out


def cube_fft(grids, values):
    """cube_fft (pwbasis.py:218-220): unnormalised forward DFT of a grid vector."""
    torch = torch_mod()
    dg = _dg(grids)
    vt = torch.from_numpy(np.ascontiguousarray(values, dtype=np.complex128)).to(dg.device)
    return cube_fft_dev(dg, vt).cpu().numpy()


def cube_ifft(grids, coeffs):
    """cube_ifft (pwbasis.py:222-224): 1/N-normalised inverse DFT."""
    torch = torch_mod()
    dg = _dg(grids)
    vt = torch.from_numpy(np.ascontiguousarray(coeffs, dtype=np.complex128)).to(dg.device)
    return cube_fft_dev(dg, vt, inverse=True).cpu().numpy()


def ham_apply_dev(dg, rows, vloc_t, shift_t=None, band_k=None):
    """(|G+k|^2/2 - shift) psi + F(V F^-1 psi) for device rows."""
    n = rows.shape[0]
    out = dg.rows(n)
    _lib.check(_lib.load().pwb_ham_apply(dg.handle, n, ptr(band_k), ptr(rows), ptr(vloc_t),
                                         ptr(shift_t), ptr(out)), "ham_apply")
    return out


def ham_apply_many(grids, v_local, psi_rows):
    """Batched apply_hamiltonian over rows of a (k, n_b) array (no counting)."""
    torch = torch_mod()
    dg = _dg(grids)
    v_local = np.asarray(v_local, dtype=float)
    if v_local.shape != (dg.n_g,):
        raise ValueError(f"expected grid potential of length {dg.n_g}, got {v_local.shape}")
    vt = torch.from_numpy(np.ascontiguousarray(v_local)).to(dg.device)
    out = ham_apply_dev(dg, _rows_from(dg, psi_rows), vt)
    return np.stack(dg.unpack(out))


def kernel_apply_dev(dg, lda, rho_t, v_t):
    torch = torch_mod()
    out = torch.empty_like(v_t)
    _lib.check(_lib.load().pwb_kernel_apply(dg.handle, 1 if lda else 0, ptr(rho_t), ptr(v_t),
                                            ptr(out)), "kernel_apply")
    return out


def kerker_apply_dev(dg, alpha, v_t):
    torch = torch_mod()
    out = torch.empty_like(v_t)
    _lib.check(_lib.load().pwb_kerker_apply(dg.handle, float(alpha), ptr(v_t), ptr(out)),
               "kerker_apply")
    return out


def axpby_dev(handle, a, x_t, b=0.0, y_t=None, out=None):
    """a x + b y (numpy's rounding: no FMA contraction) on float64 device vectors."""
    torch = torch_mod()
    out = torch.empty_like(x_t) if out is None else out
    _lib.check(_lib.load().pwb_vec_axpby(handle, x_t.numel(), float(a), ptr(x_t), float(b),
                                         ptr(y_t), ptr(out)), "vec_axpby")
    return out


def div_dev(handle, x_t, d, out=None):
    """x / d on a float64 device vector."""
    torch = torch_mod()
    out = torch.empty_like(x_t) if out is None else out
    _lib.check(_lib.load().pwb_vec_div(handle, x_t.numel(), ptr(x_t), float(d), ptr(out)),
               "vec_div")
    return out
