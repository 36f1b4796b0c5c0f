"""CPU checks of the drop-in boundary: the C-ABI library builds, loads and exports
every symbol declared in include/pwb200.h; the Python binding declares each
one; the product package never imports the oracle."""

import ast
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "pwb200.h")
PKG = os.path.join(ROOT, "paper_2505_02319_b200")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pwb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_core_entry_points():
    syms = declared_symbols()
    for name in ("pwb_grid_create", "pwb_ham_apply", "pwb_to_real", "pwb_to_fourier",
                 "pwb_state_create", "pwb_project_out", "pwb_sternheimer", "pwb_chi0",
                 "pwb_chi0_host", "pwb_chi0_begin", "pwb_chi0_finish", "pwb_kernel_apply",
                 "pwb_kerker_apply", "pwb_arnoldi_mgs"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"


def test_no_gpu_is_a_loud_error():
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.errors import DeviceError
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(DeviceError):
        _lib.require_device()


def test_status_codes_map_to_reference_exceptions():
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.errors import (ConfigurationError, DeviceError,
                                              NonConvergenceError)
    with pytest.raises(ValueError):
        _lib.check(_lib.PWB_ERR_VALUE)
    with pytest.raises(ConfigurationError):
        _lib.check(_lib.PWB_ERR_CONFIG)
    with pytest.raises(NonConvergenceError):
        _lib.check(_lib.PWB_ERR_NONCONV)
    with pytest.raises(DeviceError):
        _lib.check(_lib.PWB_ERR_CUDA)


def test_product_never_imports_the_oracle():
    for root, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith(".py"):
                continue
            tree = ast.parse(open(os.path.join(root, f)).read())
            for node in ast.walk(tree):
                if isinstance(node, ast.Import):
                    assert not any(a.name.split(".")[0] == "oracle" for a in node.names), f
                if isinstance(node, ast.ImportFrom) and node.module:
                    assert node.module.split(".")[0] != "oracle", f
