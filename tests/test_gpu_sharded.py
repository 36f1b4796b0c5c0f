"""The sharded chi0 protocol on the GPU (pwb200.h: pwb_chi0_finish_local ->
one all-reduce of the packet -> pwb_chi0_reduce_apply), checked against the
unsharded pwb_chi0 of the same state.  Only one GPU is available, so the two
shards run one after the other in one process and their packets are summed
on the device (what the all-reduce does across GPUs); the library's own NCCL
path runs with a one-rank communicator."""

import ctypes

import numpy as np
import pytest

from conftest import load_golden, product_gs, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2505_02319_b200 import _lib, build
    build.build()
    _lib.require_device()


def _np(a):
    return ctypes.c_void_p(a.ctypes.data)


def _kstate():
    from paper_2505_02319_b200.groundstate import GaussianWell, ModelSpec
    from paper_2505_02319_b200.pwbasis import Lattice
    from paper_2505_02319_b200.scf import run_scf_k
    z = load_golden("kpoint_supercell.npz")
    wells = tuple(GaussianWell(center=tuple(w[:3]), amplitude=float(w[3]), width=float(w[4]))
                  for w in z["unit_wells"])
    model = ModelSpec(lattice=Lattice.from_vectors(*z["unit_lattice"]),
                      e_cut=float(z["unit_e_cut"]), n_electrons=4, temperature=5e-3,
                      gaussians=wells)
    ks = run_scf_k(model, [[0, 0, 0], [0.5, 0, 0]], tol=1e-12, max_iter=600, damping=0.3)
    return ks, z["dv_unit"]


def _states():
    metal = load_golden("metal.npz")
    ins = load_golden("insulator.npz")
    ks, dvk = _kstate()
    return [("metal", product_gs(metal), metal["dv"][0]),
            ("insulator", product_gs(ins), ins["dv"][0]),
            ("kpoints", ks, dvk)]


@pytest.mark.parametrize("case", [0, 1, 2])
def test_packet_protocol_equals_unsharded(case):
    import torch
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import device_state, packet_layout, ptr, shard_range
    from paper_2505_02319_b200.response import apply_chi0
    name, gs, dv_h = _states()[case]
    ds = device_state(gs)
    tol = np.full(ds.nband, 1e-11)
    full, st = apply_chi0(gs, dv_h, tol)
    lib = _lib.load()
    n = ctypes.c_longlong(0)
    _lib.check(lib.pwb_chi0_packet_size(ds.handle, ctypes.byref(n)))
    metal = abs(ds.fp_den) > ds.fp_thresh
    lay = packet_layout(ds.grid.n_g, ds.nband, metal)
    assert n.value == lay["size"]
    assert metal == (name != "insulator")
    dv = torch.from_numpy(np.ascontiguousarray(dv_h)).cuda()
    total = torch.zeros(n.value, dtype=torch.float64, device="cuda")
    for world in (2, 3):
        total.zero_()
        for r in range(world):
            b0, b1 = shard_range(ds.nocc, r, world)
            f = torch.zeros(2, dtype=torch.float64, device="cuda")
            _lib.check(lib.pwb_chi0_begin(ds.handle, b0, b1, ptr(dv), ptr(f)))
            pk = torch.empty(n.value, dtype=torch.float64, device="cuda")
            tl = np.ascontiguousarray(tol[b0:b1]) if b1 > b0 else np.zeros(1)
            _lib.check(lib.pwb_chi0_finish_local(ds.handle, ptr(f), _np(tl), ptr(pk)))
            total += pk                      # the all-reduce across ranks
        drho = torch.empty(ds.grid.n_g, dtype=torch.float64, device="cuda")
        its = np.zeros(ds.nband, dtype=np.int32)
        res = ctypes.c_double(0.0)
        _lib.check(lib.pwb_chi0_reduce_apply(ds.handle, ptr(total), ptr(drho), _np(its),
                                             ctypes.byref(res)))
        assert rel(drho.cpu().numpy(), full) < 1e-12, (name, world)
        np.testing.assert_array_equal(its, st.cg_iterations_per_band)
        assert total[lay["nfail"]].item() == 0.0


def test_nccl_one_rank_communicator():
    """The library's NCCL path end to end (unique id, communicator, ncclAllReduce on
    the state's stream, fold) with one rank: equal to the unsharded chi0."""
    import torch
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import device_state, ptr
    from paper_2505_02319_b200.response import apply_chi0
    z = load_golden("metal.npz")
    gs = product_gs(z)
    ds = device_state(gs)
    tol = np.full(ds.nband, 1e-11)
    full, st = apply_chi0(gs, z["dv"][0], tol)
    lib = _lib.load()
    uid = ctypes.create_string_buffer(128)
    _lib.check(lib.pwb_comm_unique_id(uid))
    _lib.check(lib.pwb_comm_init(ds.handle, uid, 0, 1))
    try:
        n = ctypes.c_longlong(0)
        _lib.check(lib.pwb_chi0_packet_size(ds.handle, ctypes.byref(n)))
        dv = torch.from_numpy(np.ascontiguousarray(z["dv"][0])).cuda()
        f = torch.zeros(2, dtype=torch.float64, device="cuda")
        pk = torch.empty(n.value, dtype=torch.float64, device="cuda")
        drho = torch.empty(gs.grids.n_g, dtype=torch.float64, device="cuda")
        its = np.zeros(ds.nband, dtype=np.int32)
        res = ctypes.c_double(0.0)
        _lib.check(lib.pwb_chi0_begin(ds.handle, 0, ds.nband, ptr(dv), ptr(f)))
        _lib.check(lib.pwb_chi0_finish_sharded(ds.handle, ptr(f), _np(tol), ptr(pk), ptr(drho),
                                               _np(its), ctypes.byref(res)))
        assert rel(drho.cpu().numpy(), full) < 1e-12
        np.testing.assert_array_equal(its, st.cg_iterations_per_band)
    finally:
        _lib.check(lib.pwb_comm_destroy(ds.handle))


def test_failure_reaches_every_rank_with_residual():
    """A row that cannot converge on one shard fails the reduced chi0 (every rank
    raises NonConvergenceError, carrying the failed row's residual)."""
    import torch
    from paper_2505_02319_b200 import _lib
    from paper_2505_02319_b200.device import device_state, ptr, shard_range
    from paper_2505_02319_b200.errors import NonConvergenceError
    z = load_golden("insulator.npz")
    gs = product_gs(z)
    ds = device_state(gs)
    tol = np.full(ds.nband, 1e-10)
    tol[-1] = -1.0              # unreachable (C-ABI level): runs to max_iter = 10 n_b
    lib = _lib.load()
    n = ctypes.c_longlong(0)
    _lib.check(lib.pwb_chi0_packet_size(ds.handle, ctypes.byref(n)))
    dv = torch.from_numpy(np.ascontiguousarray(z["dv"][0])).cuda()
    total = torch.zeros(n.value, dtype=torch.float64, device="cuda")
    for r in range(2):
        b0, b1 = shard_range(ds.nocc, r, 2)
        f = torch.zeros(2, dtype=torch.float64, device="cuda")
        _lib.check(lib.pwb_chi0_begin(ds.handle, b0, b1, ptr(dv), ptr(f)))
        pk = torch.empty(n.value, dtype=torch.float64, device="cuda")
        tl = np.ascontiguousarray(tol[b0:b1])
        _lib.check(lib.pwb_chi0_finish_local(ds.handle, ptr(f), _np(tl), ptr(pk)))
        total += pk
    drho = torch.empty(gs.grids.n_g, dtype=torch.float64, device="cuda")
    its = np.zeros(ds.nband, dtype=np.int32)
    res = ctypes.c_double(0.0)
    status = lib.pwb_chi0_reduce_apply(ds.handle, ptr(total), ptr(drho), _np(its),
                                       ctypes.byref(res))
    with pytest.raises(NonConvergenceError) as err:
        _lib.check(status, "chi0")
    assert err.value.residual is not None and err.value.residual >= 0.0
    assert res.value == err.value.residual
    assert its[-1] == -1 and np.all(its[:-1] > 0)
