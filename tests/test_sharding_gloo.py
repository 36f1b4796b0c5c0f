"""Multi-rank decomposition of chi0 on CPU (gloo, world size 2).

The B200 path shards the (k, n) Sternheimer solves over ranks
(`DeviceState.set_sharding` -> `shard_range`); each rank accumulates its
bands with delta eps_F = 0 into ONE packet laid out by
`device.packet_layout` ([drho | C(r) = sum w f' |psi|^2 | sum w f' d eps |
failed rows | iterations | failed residuals]), the packets are summed by ONE
all-reduce per chi0 apply, and the global Fermi shift is folded in
afterwards (drho -= d eps_F C(r), the device kernel k_fermi_apply).  This
test runs exactly that protocol with the CPU oracle's per-band pieces on two
gloo ranks and checks it against the unsharded oracle chi0 (the same sum in
a different order), and that a failure on one rank reaches every rank.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_golden


def _k_state():
    from oracle import basis as ob
    from oracle import model as om
    z = load_golden("kpoint_supercell.npz")
    wells = tuple(om.Well(center=tuple(w[:3]), amplitude=float(w[3]), width=float(w[4]))
                  for w in z["unit_wells"])
    model = om.Model(lattice=ob.Cell(z["unit_lattice"]), e_cut=float(z["unit_e_cut"]),
                     n_electrons=4, temperature=5e-3, gaussians=wells)
    return om.scf_k(model, [[0, 0, 0], [0.5, 0, 0]], tol=1e-11, max_iter=600, damping=0.3), z


def _pieces(ks, dv, tols, bands):
    """Per-(k, n) RHS, d eps, Sternheimer solution and accumulation pieces (response.py:127-154)."""
    from oracle import response as orsp
    out = {}
    offs = np.cumsum([0] + [b.n_occ for b in ks.blocks])
    for gb in bands:
        k = int(np.searchsorted(offs, gb, side="right") - 1)
        n = gb - offs[k]
        blk = ks.blocks[k]
        b = blk.grids
        pr = b.to_real_many(blk.phi_occ.T)
        dvpsi = b.to_fourier_many(dv[None, :] * pr)
        m = blk.phi_occ.conj().T @ dvpsi.T
        dphi_p = blk.phi_occ @ (orsp.pair_weights(blk) * m)
        rhs = -orsp.project_out(blk.phi_occ, dvpsi[n])
        sol = orsp.sternheimer(blk, blk.v_local, n, rhs, tols[gb]).solution
        out[gb] = dict(k=k, n=n, de=float(m[n, n].real), fp=float(blk.fprime_occ()[n]),
                       f=float(blk.occ_occ[n]), psi_r=pr[n],
                       dphi_r=b.to_real(dphi_p[:, n] + sol))
    return out


def fold_packet(packet, layout, fp_den):
    """k_fermi_apply's arithmetic: sum of partials - (sum w f' d eps / sum w f') C(r)."""
    drho = packet[layout["drho"]]
    if layout["fermi"] is None:
        return drho
    return drho - (packet[layout["fsum"]] / fp_den) * packet[layout["fermi"]]


def _worker(rank, world, port, result_file):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_02319_b200.device import packet_layout, shard_range
    ks, z = _k_state()
    nocc = [b.n_occ for b in ks.blocks]
    b0, b1 = shard_range(nocc, rank, world)
    dv = z["dv_unit"]
    ntot = sum(nocc)
    tols = np.full(ntot, 1e-12)
    pieces = _pieces(ks, dv, tols, range(b0, b1))
    w = ks.weights
    den = sum(w[k] * float(blk.fprime_occ().sum()) for k, blk in enumerate(ks.blocks))
    thresh = 1e-14 * sum(wk * n for wk, n in zip(w, nocc))
    metal = abs(den) > thresh
    assert metal   # the fixture exercises the Fermi-level fold
    lay = packet_layout(ks.grids.n_g, ntot, metal)
    pk = np.zeros(lay["size"])
    for gb, p in pieces.items():   # this rank's rows, delta eps_F = 0
        wk = w[p["k"]]
        pk[lay["drho"]] += wk * (2.0 * p["f"] * (p["psi_r"].conj() * p["dphi_r"]).real
                                 + p["fp"] * p["de"] * np.abs(p["psi_r"]) ** 2)
        pk[lay["fermi"]] += wk * p["fp"] * np.abs(p["psi_r"]) ** 2
        pk[lay["fsum"]] += wk * p["fp"] * p["de"]
        pk[lay["iters"]][gb] = 1.0
    if rank == 1:   # a failed row on one rank only
        pk[lay["nfail"]] = 1.0
        pk[lay["resid"]][b0] = 3.5e-3
    t = torch.from_numpy(pk)
    dist.all_reduce(t)                      # the ONE all-reduce per chi0 apply
    red = t.numpy()
    # every rank sees every row's count and the other rank's failure
    assert np.all(red[lay["iters"]] == 1.0)
    assert red[lay["nfail"]] == 1.0 and red[lay["resid"]][b0 if rank == 1 else b1] == 3.5e-3
    if rank == 0:
        np.save(result_file, fold_packet(red, lay, den))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_shard_ranges_cover_all_pairs():
    from paper_2505_02319_b200.device import shard_range
    nocc = [31, 31, 32, 34, 31, 35, 33, 34]
    for world in (1, 2, 3, 4, 8):
        ranges = [shard_range(nocc, r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == sum(nocc)
        for (a0, a1), (b0, _) in zip(ranges, ranges[1:]):
            assert a1 == b0 and a0 <= a1
        sizes = [b - a for a, b in ranges]
        assert max(sizes) - min(sizes) <= 1


@pytest.mark.timeout(600)
def test_two_rank_chi0_equals_unsharded(tmp_path):
    from oracle import response as orsp
    result = str(tmp_path / "drho.npy")
    mp.spawn(_worker, args=(2, _free_port(), result), nprocs=2, join=True)
    ks, z = _k_state()
    ref, _ = orsp.chi0_k(ks, z["dv_unit"], np.full(sum(b.n_occ for b in ks.blocks), 1e-12))
    got = np.load(result)
    assert np.linalg.norm(got - ref) <= 1e-11 * np.linalg.norm(ref)
