"""Oracle: ground-state archive reader (numpy only) -- TEST INFRASTRUCTURE ONLY.

Restates the reference's load_ground_state (archive.py:83-120: meta.json,
format version, endianness tag, column-major phi_re/phi_im float64 blobs,
rho / v_local x-fastest, grid rebuild check) and reads the k-point extension
(format 2: a `kpoints` list in meta.json, per-k blobs phi_re_k<i>.bin /
phi_im_k<i>.bin) that paper_2505_02319_b200.archive writes.  It builds
oracle State / KState objects, so the reference arm of bench.py and the
parity-exchange CLI (oracle.cli) read a GPU-generated ground state without
importing the product package or loading its CUDA library.

A workload directory (`paper_2505_02319_b200.cli ground-state`) adds
`workload.json` (solve parameters) and `dv0.bin` (the perturbation).
"""

import json
import os

import numpy as np

from .basis import Cell, make_basis
from .model import KState, Model, State, Well


class OracleArchiveError(RuntimeError):
    """Mirror of pwdyson.errors.ArchiveError (errors.py:29)."""


def _blob(path, count):
    if not os.path.exists(path):
        raise OracleArchiveError(f"missing blob {os.path.basename(path)}")
    data = np.fromfile(path, dtype="<f8")
    if len(data) != count:
        raise OracleArchiveError(f"{os.path.basename(path)}: expected {count} values, "
                                 f"found {len(data)}")
    return data


def _model(d):
    """config.py:51-71 (model_from_dict)."""
    return Model(lattice=Cell(np.asarray(d["lattice"], dtype=float)), e_cut=float(d["e_cut"]),
                 n_electrons=int(d["n_electrons"]), temperature=float(d["temperature"]),
                 smearing=d.get("smearing", "fermi_dirac"),
                 occupation_threshold=float(d.get("occupation_threshold", 1e-8)),
                 xc=d.get("xc", "none"),
                 gaussians=tuple(Well(tuple(g["center"]), float(g["amplitude"]),
                                      float(g["width"])) for g in d.get("gaussians", [])))


def load_state(path):
    """archive.py:83-120 (+ format 2): oracle State (Gamma) or KState."""
    meta_path = os.path.join(path, "meta.json")
    if not os.path.exists(meta_path):
        raise OracleArchiveError(f"no meta.json under {path}")
    with open(meta_path) as fh:
        meta = json.load(fh)
    version = meta.get("format_version")
    if version not in (1, 2):
        raise OracleArchiveError(f"archive format version {version}")
    if meta.get("endianness") != "little":
        raise OracleArchiveError(f"unsupported endianness tag {meta.get('endianness')!r}")
    model = _model(meta["model"])
    n_g = int(np.prod(meta["cube_dims"]))
    rho = _blob(os.path.join(path, "rho.bin"), n_g)
    v_local = _blob(os.path.join(path, "v_local.bin"), n_g)
    fermi = float(meta["fermi_level"])
    res = float(meta.get("scf_residual", 0.0))

    def block(kfrac, m, suffix):
        basis = make_basis(model.lattice, model.e_cut, tuple(kfrac))
        n_b, n_kept = int(m["n_b"]), int(m["n_kept"])
        if basis.n_b != n_b or list(basis.cube_dims) != list(meta["cube_dims"]):
            raise OracleArchiveError("grid rebuild disagrees with the archive")
        re = _blob(os.path.join(path, f"phi_re{suffix}.bin"), n_b * n_kept)
        im = _blob(os.path.join(path, f"phi_im{suffix}.bin"), n_b * n_kept)
        phi = (re + 1j * im).reshape((n_b, n_kept), order="F")
        return State(model=model, grids=basis, phi=phi, eps=np.asarray(m["eps"], dtype=float),
                     occ=np.asarray(m["occ"], dtype=float), fermi_level=fermi, rho=rho,
                     n_occ=int(m["n_occ"]), v_local=v_local, scf_residual=res)

    if version == 1:
        return block((0.0, 0.0, 0.0), meta, "")
    kp = meta["kpoints"]
    blocks = [block(m["kfrac"], m, f"_k{i}") for i, m in enumerate(kp)]
    return KState(model=model, blocks=blocks,
                  weights=np.array([m["weight"] for m in kp], dtype=float),
                  kfracs=np.array([m["kfrac"] for m in kp], dtype=float),
                  fermi_level=fermi, rho=rho, v_local=v_local, scf_residual=res)


def load_workload(path):
    """(state, dv0, params) of a workload directory."""
    with open(os.path.join(path, "workload.json")) as fh:
        params = json.load(fh)
    state = load_state(path)
    grids = state.blocks[0].grids if hasattr(state, "blocks") else state.grids
    dv0 = _blob(os.path.join(path, "dv0.bin"), int(grids.n_g))
    return state, dv0, params
