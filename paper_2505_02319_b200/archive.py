"""Ground-state archives: the reference's format plus a k-point extension.

Gamma ground states are written in exactly the reference's layout
(archive.py:1-15, 55-120 of pwdyson): `meta.json` + raw little-endian float64
blobs `phi_re.bin` / `phi_im.bin` (column-major n_b x n_kept), `rho.bin`,
`v_local.bin` (x fastest), format version 1 -- so the reference's
`load_ground_state` reads what this module writes and vice versa.

k-sampled ground states (`KGroundState`) use the same
conventions with format version 2: `meta.json` gains a `kpoints` list (one
entry per k block: fractional k, weight, n_b, n_occ, n_kept, eps, occ) and the
orbital blobs become `phi_re_k<i>.bin` / `phi_im_k<i>.bin`; `rho` and
`v_local` are shared.  Grids are rebuilt from the model and k and checked
against the stored sizes.  Round trips are bit-exact; every write goes
through a temporary file and an atomic rename.  Archive plumbing only: no
device code.
"""

import json
import os
import tempfile

import numpy as np

from .errors import ArchiveError, ConfigurationError
from .groundstate import GaussianWell, GroundState, KGroundState, ModelSpec
from .pwbasis import Lattice, build_grids

FORMAT_VERSION = 1       # the reference's (Gamma)
FORMAT_VERSION_K = 2     # k-point extension


def model_to_dict(model):
    """reference config.py:74-88."""
    return {
        "lattice": np.asarray(model.lattice.a).tolist(),
        "e_cut": model.e_cut,
        "n_electrons": model.n_electrons,
        "temperature": model.temperature,
        "smearing": model.smearing,
        "occupation_threshold": model.occupation_threshold,
        "xc": model.xc,
        "gaussians": [{"center": list(g.center), "amplitude": g.amplitude, "width": g.width}
                      for g in model.gaussians],
    }


def model_from_dict(d):
    """reference config.py:51-71."""
    try:
        return ModelSpec(
            lattice=Lattice.from_vectors(*d["lattice"]), e_cut=float(d["e_cut"]),
            n_electrons=int(d["n_electrons"]), temperature=float(d["temperature"]),
            smearing=d.get("smearing", "fermi_dirac"),
            occupation_threshold=float(d.get("occupation_threshold", 1e-8)),
            xc=d.get("xc", "none"),
            gaussians=tuple(GaussianWell(center=tuple(g["center"]), amplitude=float(g["amplitude"]),
                                         width=float(g["width"])) for g in d.get("gaussians", [])))
    except KeyError as missing:
        raise ConfigurationError(f"model config misses required key {missing}") from None


def _atomic_write(path, data):
    fd, tmp = tempfile.mkstemp(dir=os.path.dirname(path) or ".")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(data)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _read_blob(path, count):
    if not os.path.exists(path):
        raise ArchiveError(f"missing blob {os.path.basename(path)}")
    data = np.fromfile(path, dtype="<f8")
    if len(data) != count:
        raise ArchiveError(f"{os.path.basename(path)}: expected {count} float64 values, "
                           f"found {len(data)}")
    return data


def _write_phi(path, phi, suffix=""):
    _atomic_write(os.path.join(path, f"phi_re{suffix}.bin"),
                  np.ascontiguousarray(phi.real, dtype="<f8").tobytes(order="F"))
    _atomic_write(os.path.join(path, f"phi_im{suffix}.bin"),
                  np.ascontiguousarray(phi.imag, dtype="<f8").tobytes(order="F"))


def _read_phi(path, n_b, n_kept, suffix=""):
    re = _read_blob(os.path.join(path, f"phi_re{suffix}.bin"), n_b * n_kept)
    im = _read_blob(os.path.join(path, f"phi_im{suffix}.bin"), n_b * n_kept)
    return (re + 1j * im).reshape((n_b, n_kept), order="F")


def save_ground_state(path, gs):
    """Write a GroundState (reference format) or a KGroundState (k extension)."""
    os.makedirs(path, exist_ok=True)
    meta = {"endianness": "little", "model": model_to_dict(gs.model),
            "cube_dims": [int(d) for d in gs.grids.cube_dims], "n_g": int(gs.grids.n_g),
            "fermi_level": float(gs.fermi_level),
            "scf_residual": float(getattr(gs, "scf_residual", 0.0))}
    if hasattr(gs, "blocks"):
        meta["format_version"] = FORMAT_VERSION_K
        meta["kpoints"] = [
            {"kfrac": [float(v) for v in k], "weight": float(w), "n_b": int(b.grids.n_b),
             "n_occ": int(b.n_occ), "n_kept": int(b.n_kept), "eps": b.eps.tolist(),
             "occ": b.occ.tolist()}
            for k, w, b in zip(gs.kfracs, gs.weights, gs.blocks)]
        for i, b in enumerate(gs.blocks):
            _write_phi(path, b.phi, f"_k{i}")
    else:
        meta.update({"format_version": FORMAT_VERSION, "n_b": int(gs.grids.n_b),
                     "n_occ": int(gs.n_occ), "n_kept": int(gs.n_kept), "eps": gs.eps.tolist(),
                     "occ": gs.occ.tolist()})
        _write_phi(path, gs.phi)
    _atomic_write(os.path.join(path, "meta.json"), json.dumps(meta, indent=1).encode())
    _atomic_write(os.path.join(path, "rho.bin"), np.asarray(gs.rho, dtype="<f8").tobytes())
    _atomic_write(os.path.join(path, "v_local.bin"),
                  np.asarray(gs.v_local, dtype="<f8").tobytes())


def load_ground_state(path):
    """Read either format; raises ArchiveError on any inconsistency (reference
    archive.py:83-120 checks: version, endianness, grid rebuild, blob sizes)."""
    meta_path = os.path.join(path, "meta.json")
    if not os.path.exists(meta_path):
        raise ArchiveError(f"no meta.json under {path}")
    with open(meta_path) as fh:
        meta = json.load(fh)
    version = meta.get("format_version")
    if version not in (FORMAT_VERSION, FORMAT_VERSION_K):
        raise ArchiveError(f"archive format version {version}, expected "
                           f"{FORMAT_VERSION} or {FORMAT_VERSION_K}")
    if meta.get("endianness") != "little":
        raise ArchiveError(f"unsupported endianness tag {meta.get('endianness')!r}")
    model = model_from_dict(meta["model"])
    fermi = float(meta["fermi_level"])
    res = float(meta.get("scf_residual", 0.0))

    def grids_for(kfrac, n_b):
        g = build_grids(model.lattice, model.e_cut, tuple(kfrac))
        if g.n_b != n_b or list(g.cube_dims) != list(meta["cube_dims"]):
            raise ArchiveError(f"grid rebuild disagrees with archive: n_b {g.n_b} vs {n_b}, "
                               f"dims {g.cube_dims} vs {tuple(meta['cube_dims'])}")
        return g

    n_g = int(np.prod(meta["cube_dims"]))
    rho = _read_blob(os.path.join(path, "rho.bin"), n_g)
    v_local = _read_blob(os.path.join(path, "v_local.bin"), n_g)

    def block(kfrac, m, phi_suffix):
        g = grids_for(kfrac, int(m["n_b"]))
        n_kept = int(m["n_kept"])
        eps = np.asarray(m["eps"], dtype=float)
        occ = np.asarray(m["occ"], dtype=float)
        if len(eps) != n_kept or len(occ) != n_kept:
            raise ArchiveError("eps/occ length disagrees with n_kept")
        return GroundState(model=model, grids=g, phi=_read_phi(path, g.n_b, n_kept, phi_suffix),
                           eps=eps, occ=occ, fermi_level=fermi, rho=rho,
                           n_occ=int(m["n_occ"]), v_local=v_local, scf_residual=res)

    if version == FORMAT_VERSION:
        return block((0.0, 0.0, 0.0), meta, "")
    kp = meta.get("kpoints") or []
    if not kp:
        raise ArchiveError("k-point archive without kpoints")
    blocks = [block(m["kfrac"], m, f"_k{i}") for i, m in enumerate(kp)]
    return KGroundState(model=model, blocks=blocks,
                        weights=np.array([m["weight"] for m in kp], dtype=float),
                        kfracs=np.array([m["kfrac"] for m in kp], dtype=float),
                        fermi_level=fermi, rho=rho, v_local=v_local, scf_residual=res)
