"""ctypes binding of libpwb200.so (C-ABI in include/pwb200.h).

The library is loaded on first use.  There is no fallback: if the shared
object is missing, or no CUDA device is visible when an operator runs, a
DeviceError is raised.  Status codes are mapped onto the reference's
exception types (errors.py).
"""

import ctypes
import os
import threading

from .errors import ConfigurationError, DeviceError, NonConvergenceError, PwdysonError

HERE = os.path.dirname(os.path.abspath(__file__))
# PWB200_VARIANT selects a performance-experiment build (build.py --variant); default = product
LIB_PATH = os.path.join(HERE, f"libpwb200_{os.environ['PWB200_VARIANT']}.so"
                        if os.environ.get("PWB200_VARIANT") else "libpwb200.so")

PWB_OK, PWB_ERR_VALUE, PWB_ERR_CONFIG, PWB_ERR_NONCONV = 0, 1, 2, 3
PWB_ERR_CUDA, PWB_ERR_UNSUPPORTED, PWB_ERR_NOMEM = 4, 5, 6

_c_int_p = ctypes.POINTER(ctypes.c_int)
_c_dbl_p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p

# name -> (restype, argtypes); every entry point of include/pwb200.h
SIGNATURES = {
    "pwb_last_error": (ctypes.c_char_p, []),
    "pwb_version": (ctypes.c_int, []),
    "pwb_launch_count": (ctypes.c_ulonglong, []),
    "pwb_device_count": (ctypes.c_int, [_c_int_p]),
    "pwb_grid_set_stream": (ctypes.c_int, [_vp, _vp]),
    "pwb_grid_create": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.c_int, _vp, _vp, _vp, _vp,
                                       ctypes.POINTER(_vp)]),
    "pwb_grid_destroy": (ctypes.c_int, [_vp]),
    "pwb_grid_info": (ctypes.c_int, [_vp, _vp]),
    "pwb_to_real": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    "pwb_to_fourier": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    "pwb_ham_apply": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp]),
    "pwb_ham_apply_host": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp]),
    "pwb_cube_fft": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, ctypes.c_int]),
    "pwb_kernel_apply": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    "pwb_kerker_apply": (ctypes.c_int, [_vp, ctypes.c_double, _vp, _vp]),
    "pwb_state_create": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                        ctypes.POINTER(_vp)]),
    "pwb_state_destroy": (ctypes.c_int, [_vp]),
    "pwb_state_nbands": (ctypes.c_int, [_vp, _c_int_p]),
    "pwb_project_out": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp]),
    "pwb_sternheimer": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp, ctypes.c_int, _vp, _vp,
                                       _vp]),
    "pwb_chi0": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pwb_chi0_host": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pwb_chi0_begin": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp]),
    "pwb_chi0_finish": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "pwb_row_norm": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _c_dbl_p]),
    "pwb_row_norm_rows": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, ctypes.c_int, _c_dbl_p]),
    "pwb_chi0_parts": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "pwb_project_generic": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp]),
    "pwb_project_host": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp]),
    "pwb_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "pwb_profile_reset": (ctypes.c_int, []),
    "pwb_profile_read": (ctypes.c_int, [_vp, _vp, _vp]),
    "pwb_profile_hist": (ctypes.c_int, [_vp, _vp]),
    "pwb_vec_dot": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    "pwb_vec_axpy": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_double, _vp, _vp]),
    "pwb_vec_axpby": (ctypes.c_int, [_vp, ctypes.c_longlong, ctypes.c_double, _vp,
                                     ctypes.c_double, _vp, _vp]),
    "pwb_vec_div": (ctypes.c_int, [_vp, ctypes.c_longlong, _vp, ctypes.c_double, _vp]),
    "pwb_arnoldi_mgs": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]),
    "pwb_vec_combine": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp]),
    "pwb_chi0_packet_size": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_longlong)]),
    "pwb_chi0_finish_local": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "pwb_chi0_reduce_apply": (ctypes.c_int, [_vp, _vp, _vp, _vp, _c_dbl_p]),
    "pwb_chi0_finish_sharded": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _c_dbl_p]),
    "pwb_comm_unique_id": (ctypes.c_int, [_vp]),
    "pwb_comm_init": (ctypes.c_int, [_vp, _vp, ctypes.c_int, ctypes.c_int]),
    "pwb_comm_destroy": (ctypes.c_int, [_vp]),
    "pwb_allreduce": (ctypes.c_int, [_vp, _vp, ctypes.c_longlong]),
    "pwb_last_residual": (ctypes.c_double, []),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the CDLL with every signature declared."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2505_02319_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error():
    return load().pwb_last_error().decode(errors="replace")


def check(status, what=""):
    """Map a PWB status code onto the reference exception types."""
    if status == PWB_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if status == PWB_ERR_VALUE:
        raise ValueError(msg)
    if status == PWB_ERR_CONFIG:
        raise ConfigurationError(msg)
    if status == PWB_ERR_NONCONV:
        res = float(load().pwb_last_residual())
        raise NonConvergenceError(msg, residual=None if res != res else res)
    if status in (PWB_ERR_CUDA, PWB_ERR_NOMEM):
        raise DeviceError(msg)
    raise PwdysonError(msg)


def device_count():
    n = ctypes.c_int(0)
    load().pwb_device_count(ctypes.byref(n))
    return n.value


def launch_count():
    return int(load().pwb_launch_count())


PROFILE_CATEGORIES = ("ham_apply", "projector", "cg_vector", "chi0_rhs", "drho_accumulate")


def profile(on=True):
    load().pwb_profile_enable(1 if on else 0)
    load().pwb_profile_reset()


def profile_read():
    """{category: (ms, launches-groups, units)} accumulated since profile()."""
    import numpy as np
    ms = np.zeros(8)
    cnt = np.zeros(8, dtype=np.int64)
    units = np.zeros(8, dtype=np.int64)
    load().pwb_profile_read(ctypes.c_void_p(ms.ctypes.data), ctypes.c_void_p(cnt.ctypes.data),
                            ctypes.c_void_p(units.ctypes.data))
    return {name: (float(ms[i]), int(cnt[i]), int(units[i]))
            for i, name in enumerate(PROFILE_CATEGORIES)}


def profile_hist():
    """{category: [(bucket, ms, launch groups)]}: time split by log2(live rows)."""
    import numpy as np
    ms = np.zeros(8 * 16)
    cnt = np.zeros(8 * 16, dtype=np.int64)
    load().pwb_profile_hist(ctypes.c_void_p(ms.ctypes.data), ctypes.c_void_p(cnt.ctypes.data))
    return {name: [(b, float(ms[i * 16 + b]), int(cnt[i * 16 + b])) for b in range(16)
                   if cnt[i * 16 + b]]
            for i, name in enumerate(PROFILE_CATEGORIES)}


def require_device():
    if device_count() < 1:
        raise DeviceError("no CUDA device visible: the B200 path has no CPU fallback")
