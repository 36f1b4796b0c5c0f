"""bench.py's JSON contract pieces that do not need a GPU: argument defaults, the
roofline objects built from a (synthetic) live profile, the rank environment."""

import sys

import pytest

from conftest import load_golden, product_gs


def test_defaults_are_one_gpu_config4(monkeypatch):
    """The default workload is BASELINE configs[4], the config the metric's 1/2/4/8-GPU
    series is quoted on (it fits one B200)."""
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert (a.gpus, a.config, a.impl) == (1, 4, "ours")
    assert a.warmup >= 3 and a.steps >= 1


def test_roofline_objects_from_profile():
    import bench
    gs = product_gs(load_golden("metal.npz"))
    # category -> (ms, launch groups, units): units = band rows per group
    prof = {"ham_apply": (10.0, 100, 1000), "projector": (20.0, 400, 4000),
            "cg_vector": (3.0, 300, 3000), "chi0_rhs": (1.0, 10, 100),
            "drho_accumulate": (1.0, 10, 100)}
    r = bench.roofline_from_profile(prof, gs)
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    b_h = 64.0 * gs.grids.n_g + 32.0 * gs.grids.n_b
    assert r["achieved"] == pytest.approx(b_h * 10 / 0.1e-3 / 1e9)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    q = bench.projector_roofline(prof, gs, 35.0)
    assert q["bound"] == "tensor" and q["peak"] == 35.0
    f_row = 16.0 * gs.grids.n_b * gs.n_occ
    assert q["achieved"] == pytest.approx(f_row * 4000 / 20e-3 / 1e12)
    # the line's `roofline` is the group with the larger share (the projector here)
    d = bench.dominant_roofline(r, q)
    assert d["bound"] == "tensor" and d["frac"] == q["frac"]
    flip = {"projector": 0.1, "ham_apply": 0.5}
    assert bench.dominant_roofline(dict(r, share_of_kernel_time=flip), q)["bound"] == "hbm"


def test_traffic_lookup_by_cube():
    import bench
    per, src = bench._traffic((64, 64, 64), "ham_apply")
    if per is not None:
        assert per > 0 and "ncu" in src
    assert bench._traffic((7, 7, 7), "ham_apply") == (None, None)


def test_rank_environment(monkeypatch):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setenv("RANK", "2")
    monkeypatch.setenv("LOCAL_RANK", "2")
    monkeypatch.delenv("PWB_SHARE_GPU", raising=False)
    assert bench.dist_env() == (4, 2, 2)
