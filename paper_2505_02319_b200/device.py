"""Device-resident grids and ground states (handles onto libpwb200 objects).

`DeviceGrid` wraps a `pwb_grid` (sphere/cube tables + FFT plans for one or
more k-points sharing a cube); `DeviceState` wraps a `pwb_state` (occupied
orbitals, eigenvalues, occupations, V_local and rho in HBM).  Both are built
once and cached on the host objects they mirror (attribute
`_pwb_device_grid` / `_pwb_device_state`), the way the reference caches
row norms on its GroundState (groundstate.py:299).

PyTorch is used only to own device buffers and for torch.distributed
(NCCL) when the (k, n) batch is sharded over ranks.
"""

import ctypes

import numpy as np

from . import _lib
from .errors import DeviceError


def torch_mod():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device visible: the B200 path has no CPU fallback")
    return torch


def ptr(t):
    """Device pointer of a torch tensor (or None)."""
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _np_ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


class DeviceGrid:
    """pwb_grid for a list of FourierGrids sharing one cube (one per k-point)."""

    def __init__(self, grids_list):
        torch = torch_mod()
        lib = _lib.load()
        _lib.require_device()
        grids_list = list(grids_list)
        g0 = grids_list[0]
        for g in grids_list[1:]:
            if tuple(g.cube_dims) != tuple(g0.cube_dims):
                raise ValueError("k-point grids must share one FFT cube")
        self.grids = grids_list
        self.cube_dims = tuple(int(d) for d in g0.cube_dims)
        self.n_g = int(np.prod(self.cube_dims))
        self.volume = float(g0.lattice.volume)
        self.nk = len(grids_list)
        self.nb = [int(g.n_b) for g in grids_list]
        nb = np.array(self.nb, dtype=np.int32)
        gint = np.ascontiguousarray(np.concatenate([g.g_int for g in grids_list]).astype(np.int32))
        g2s = np.ascontiguousarray(np.concatenate([g.g2_sphere for g in grids_list]), dtype=float)
        g2c = np.ascontiguousarray(g0.g2_cube, dtype=float)
        handle = ctypes.c_void_p()
        nx, ny, nz = self.cube_dims
        _lib.check(lib.pwb_grid_create(nx, ny, nz, self.volume, self.nk, _np_ptr(nb),
                                       _np_ptr(gint), _np_ptr(g2s), _np_ptr(g2c),
                                       ctypes.byref(handle)), "pwb_grid_create")
        self.handle = handle
        self._lib = lib
        _lib.check(lib.pwb_grid_set_stream(handle, ctypes.c_void_p(
            torch.cuda.current_stream().cuda_stream)))
        info = np.zeros(8, dtype=np.int32)
        _lib.check(lib.pwb_grid_info(handle, _np_ptr(info)))
        self.nbp = int(info[4])
        self.nxa = int(info[5])
        self.nya = int(info[6])
        self.tile = int(info[7])
        self.device = torch.device("cuda", torch.cuda.current_device())

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.pwb_grid_destroy(h)
            except Exception:
                pass
            self.handle = None

    # -- packing of sphere rows -------------------------------------------------
    def rows(self, n):
        torch = torch_mod()
        return torch.zeros((n, self.nbp), dtype=torch.complex128, device=self.device)

    def pack(self, vectors, ks=None):
        """Host sphere vectors (list / 2-D array, row b for k ks[b]) -> padded device rows."""
        torch = torch_mod()
        vecs = list(vectors)
        n = len(vecs)
        host = np.zeros((n, self.nbp), dtype=np.complex128)
        for i, v in enumerate(vecs):
            k = 0 if ks is None else int(ks[i])
            v = np.asarray(v)
            if v.shape != (self.nb[k],):
                raise ValueError(f"expected sphere vector of length {self.nb[k]}, got {v.shape}")
            host[i, : self.nb[k]] = v
        return torch.from_numpy(host).to(self.device)

    def unpack(self, rows, ks=None):
        """Device rows -> list of host sphere vectors (trimmed to n_b of each k)."""
        host = rows.cpu().numpy()
        out = []
        for i in range(host.shape[0]):
            k = 0 if ks is None else int(ks[i])
            out.append(host[i, : self.nb[k]].copy())
        return out

    def band_k_tensor(self, ks):
        torch = torch_mod()
        return torch.tensor(np.asarray(ks, dtype=np.int32), dtype=torch.int32, device=self.device)


def device_grid(grids_list):
    """Cached DeviceGrid for one FourierGrids (Gamma) or a tuple of k-grids."""
    if not isinstance(grids_list, (list, tuple)):
        grids_list = [grids_list]
    owner = grids_list[0]
    key = tuple(id(g) for g in grids_list)
    cache = getattr(owner, "_pwb_device_grid", None)
    if cache is not None and cache[0] == key:
        return cache[1]
    dg = DeviceGrid(grids_list)
    try:
        owner._pwb_device_grid = (key, dg)
    except AttributeError:
        pass
    return dg


def state_blocks(gs):
    """(blocks, weights): the k blocks of a ground state (Gamma -> one block, w=1)."""
    if hasattr(gs, "blocks"):
        return list(gs.blocks), np.asarray(gs.weights, dtype=float)
    return [gs], np.ones(1)


class DeviceState:
    """pwb_state for a (possibly k-sampled) ground state."""

    def __init__(self, gs):
        torch = torch_mod()
        lib = _lib.load()
        blocks, weights = state_blocks(gs)
        self.gs = gs
        self.blocks = blocks
        self.weights = weights
        self.grid = device_grid([b.grids for b in blocks])
        self.nocc = [int(b.n_occ) for b in blocks]
        self.nband = int(sum(self.nocc))
        self.band_k = np.repeat(np.arange(len(blocks)), self.nocc).astype(np.int32)
        self.offsets = np.concatenate([[0], np.cumsum(self.nocc)]).astype(int)
        phi = np.ascontiguousarray(np.concatenate(
            [np.ascontiguousarray(b.phi_occ.T).ravel() for b in blocks]), dtype=np.complex128)
        eps = np.ascontiguousarray(np.concatenate([b.eps_occ for b in blocks]), dtype=float)
        occ = np.ascontiguousarray(np.concatenate([b.occ_occ for b in blocks]), dtype=float)
        fpr = np.ascontiguousarray(np.concatenate([b.fprime_occ() for b in blocks]), dtype=float)
        self.eps, self.occ, self.fprime = eps, occ, fpr
        wb = weights[self.band_k]
        self.fp_den = float(np.sum(wb * fpr))          # sum_k w_k sum_n f'_nk
        self.fp_thresh = 1e-14 * float(np.sum(wb))     # response.py:135 with k weights
        nocc = np.array(self.nocc, dtype=np.int32)
        w = np.ascontiguousarray(weights, dtype=float)
        vloc = np.ascontiguousarray(gs.v_local, dtype=float)
        rho = np.ascontiguousarray(gs.rho, dtype=float)
        handle = ctypes.c_void_p()
        _lib.check(lib.pwb_state_create(self.grid.handle, _np_ptr(nocc), _np_ptr(w), _np_ptr(phi),
                                        _np_ptr(eps), _np_ptr(occ), _np_ptr(fpr), _np_ptr(vloc),
                                        _np_ptr(rho), ctypes.byref(handle)), "pwb_state_create")
        self.handle = handle
        self._lib = lib
        self.device = self.grid.device
        self.rho_t = torch.from_numpy(rho).to(self.device)
        self.vloc_t = torch.from_numpy(vloc).to(self.device)
        self._fsum = torch.zeros(2, dtype=torch.float64, device=self.device)
        self.shard = (0, self.nband)
        self.comm = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.pwb_state_destroy(h)
            except Exception:
                pass
            self.handle = None

    # -- sharding over ranks ---------------------------------------------------------
    def set_sharding(self, rank, world, group=None, transport=None):
        """Own the contiguous band range of `rank` (k blocks stay whole when N_k >= world).

        transport "nccl" (default; env PWB_DIST_BACKEND): the library's own NCCL
        communicator, whose unique id rank 0 creates and `group` broadcasts once;
        anything else (the gloo shared-GPU control-flow check) sums the packet with
        torch.distributed instead.  Either way a chi0 apply costs ONE all-reduce.
        """
        import os
        torch = torch_mod()
        self.shard = shard_range(self.nocc, rank, world)
        self.comm = None
        if world <= 1:
            return
        import torch.distributed as dist
        transport = transport or os.environ.get("PWB_DIST_BACKEND", "nccl")
        if transport == "nccl":
            uid = ctypes.create_string_buffer(128)
            if rank == 0:
                _lib.check(self._lib.pwb_comm_unique_id(uid), "pwb_comm_unique_id")
            obj = [uid.raw if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = ctypes.create_string_buffer(obj[0], 128)
            _lib.check(self._lib.pwb_comm_init(self.handle, uid, rank, world), "pwb_comm_init")
        n = ctypes.c_longlong(0)
        _lib.check(self._lib.pwb_chi0_packet_size(self.handle, ctypes.byref(n)))
        self.layout = packet_layout(self.grid.n_g, self.nband, abs(self.fp_den) > self.fp_thresh)
        assert n.value == self.layout["size"], "packet layout out of sync with the library"
        self._packet = torch.empty(n.value, dtype=torch.float64, device=self.device)
        self.comm = (rank, world, group, transport)

    def chi0(self, dv_t, tol):
        """drho (device tensor) and per-(k, n) iteration counts of the local shard.

        With sharding active the result is already all-reduced over ranks, and
        the returned iteration counts cover the whole (k, n) list.
        """
        self.chi0_begin(dv_t)
        return self.chi0_finish(tol)

    def chi0_begin(self, dv_t):
        """Launch the right-hand side of chi0 dv (asynchronous: the host is free to
        compute the tolerance vector while the GPU builds the RHS)."""
        b0, b1 = self.shard
        self._dv_pending = dv_t   # keep the input alive until finish
        _lib.check(self._lib.pwb_chi0_begin(self.handle, b0, b1, ptr(dv_t), ptr(self._fsum)),
                   "chi0_begin")

    def chi0_finish(self, tol):
        """Sternheimer solves + delta rho accumulation of the pending chi0.

        Sharded: the rank's solves and accumulation (delta eps_F = 0), ONE
        all-reduce of the packet [drho | C(r) | sum w f' delta eps | failures |
        iterations], then drho -= delta eps_F C(r) on the device (pwb200.h)."""
        torch = torch_mod()
        tol = np.ascontiguousarray(tol, dtype=float)
        drho = torch.empty(self.grid.n_g, dtype=torch.float64, device=self.device)
        b0, b1 = self.shard
        tl = np.ascontiguousarray(tol[b0:b1]) if b1 > b0 else np.zeros(1)
        hold = self._dv_pending   # noqa: F841 -- dv stays alive until the calls below return
        self._dv_pending = None
        if self.comm is None:
            its = np.zeros(max(b1 - b0, 1), dtype=np.int32)
            status = self._lib.pwb_chi0_finish(self.handle, ptr(self._fsum), _np_ptr(tl),
                                               ptr(drho), _np_ptr(its))
            _lib.check(status, "chi0_finish")
            return drho, its[: b1 - b0]
        _, _, group, transport = self.comm
        its = np.zeros(self.nband, dtype=np.int32)
        resid = ctypes.c_double(np.nan)
        if transport == "nccl":
            status = self._lib.pwb_chi0_finish_sharded(
                self.handle, ptr(self._fsum), _np_ptr(tl), ptr(self._packet), ptr(drho),
                _np_ptr(its), ctypes.byref(resid))
        else:
            import torch.distributed as dist
            _lib.check(self._lib.pwb_chi0_finish_local(self.handle, ptr(self._fsum), _np_ptr(tl),
                                                       ptr(self._packet)), "chi0_finish_local")
            dist.all_reduce(self._packet, group=group)
            status = self._lib.pwb_chi0_reduce_apply(self.handle, ptr(self._packet), ptr(drho),
                                                     _np_ptr(its), ctypes.byref(resid))
        _lib.check(status, "chi0_finish")
        return drho, its


def packet_layout(n_g, nband, metal):
    """Offsets (in doubles) of the per-chi0 all-reduce packet (pwb200.h,
    pwb_chi0_finish_local): slices drho / fermi (C(r), metals only) / iters /
    resid, scalar offsets fsum / nfail, and the total size."""
    base = n_g * (2 if metal else 1)
    return {"drho": slice(0, n_g), "fermi": slice(n_g, 2 * n_g) if metal else None,
            "fsum": base, "nfail": base + 1, "iters": slice(base + 2, base + 2 + nband),
            "resid": slice(base + 2 + nband, base + 2 + 2 * nband),
            "size": base + 2 + 2 * nband}


def shard_range(nocc, rank, world):
    """Contiguous [b0, b1) of the (k, n) list for `rank`, balanced by band count."""
    total = int(sum(nocc))
    if world <= 1:
        return 0, total
    bounds = [round(total * r / world) for r in range(world + 1)]
    return bounds[rank], bounds[rank + 1]


def device_state(gs):
    """Cached DeviceState of a ground state (the reference's or this package's)."""
    cache = getattr(gs, "_pwb_device_state", None)
    if cache is not None:
        return cache
    ds = DeviceState(gs)
    try:
        object.__setattr__(gs, "_pwb_device_state", ds)
    except (AttributeError, TypeError):
        pass
    return ds
