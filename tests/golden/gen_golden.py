"""Generate golden fixtures by running the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden.py

It imports `pwdyson` from /root/reference/pkg/src (read-only) and writes
small .npz files next to this script.  The fixtures pin the CPU oracle
(tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_*.py); the
GPU box never needs /root/reference.  Library versions used are recorded in
every file (`versions`), since bitwise outputs depend on numpy/scipy.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import scipy  # noqa: E402

import pwdyson.harness as H  # noqa: E402
from pwdyson import Lattice  # noqa: E402
from pwdyson.config import (ExperimentConfig, Perturbation, ResponseParams,  # noqa: E402
                            ScfParams, reference_config)
from pwdyson.groundstate import (GaussianWell, ModelSpec, apply_hamiltonian,  # noqa: E402
                                 ham_counter, run_scf)
from pwdyson.igmres import igmres_solve  # noqa: E402
from pwdyson.kernels import KerkerSpec, KernelSpec, apply_kerker, apply_kernel  # noqa: E402
from pwdyson.pwbasis import build_grids  # noqa: E402
from pwdyson.response import (_occupied_pair_weights, apply_chi0,  # noqa: E402
                              apply_dielectric, delta_eigen_occupations,
                              dielectric_error_bound, orbital_row_norm)
from pwdyson.sternheimer import project_out_occupied, solve_sternheimer  # noqa: E402
from pwdyson.strategies import StrategySpec, ToleranceContext, select_tolerances  # noqa: E402

from paper_2505_02319_b200 import synth  # noqa: E402  (seeded generators; numpy only)

VERSIONS = json.dumps({"numpy": np.__version__, "scipy": scipy.__version__,
                       "python": sys.version.split()[0]})


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, versions=VERSIONS, **arrays)
    print("wrote", path, os.path.getsize(path), "bytes")


def gs_arrays(gs, prefix="gs_"):
    m = gs.model
    return {
        prefix + "lattice": m.lattice.a, prefix + "e_cut": m.e_cut,
        prefix + "n_electrons": m.n_electrons, prefix + "temperature": m.temperature,
        prefix + "smearing": m.smearing, prefix + "xc": m.xc,
        prefix + "wells": np.array([[*g.center, g.amplitude, g.width] for g in m.gaussians]),
        prefix + "phi": gs.phi, prefix + "eps": gs.eps, prefix + "occ": gs.occ,
        prefix + "fermi": gs.fermi_level, prefix + "rho": gs.rho, prefix + "n_occ": gs.n_occ,
        prefix + "v_local": gs.v_local,
    }


def grids_fixture():
    cases = [("cubic4_e3", Lattice.cubic(4.0), 3.0),
             ("ortho_4_5_6_e4", Lattice.orthorhombic(4.0, 5.0, 6.0), 4.0),
             ("toy_insulator", Lattice.from_vectors([8, 0, 0], [0, 4, 0], [0, 0, 4]), 9.0),
             ("cfg0", Lattice.cubic(10.0), 6.0),
             ("skew", Lattice.from_vectors([4.0, 0.3, 0.0], [0.2, 4.5, 0.1], [0.0, 0.4, 5.0]), 3.0)]
    out = {}
    rng = np.random.default_rng(123)
    for name, lat, ecut in cases:
        g = build_grids(lat, ecut)
        out[name + "_a"] = lat.a
        out[name + "_ecut"] = ecut
        out[name + "_dims"] = np.array(g.cube_dims)
        out[name + "_g_int"] = g.g_int
        out[name + "_sphere_flat"] = g.sphere_flat
        out[name + "_g2_sphere"] = g.g2_sphere
        out[name + "_g2_cube"] = g.g2_cube
        x = rng.standard_normal((3, g.n_b)) + 1j * rng.standard_normal((3, g.n_b))
        u = rng.standard_normal((2, g.n_g)) + 1j * rng.standard_normal((2, g.n_g))
        v = rng.standard_normal(g.n_g)
        out[name + "_x"] = x
        out[name + "_to_real"] = g.to_real_many(x)
        out[name + "_to_real0"] = g.to_real(x[0])
        out[name + "_u"] = u
        out[name + "_to_fourier"] = g.to_fourier_many(u)
        out[name + "_v"] = v
        out[name + "_h"] = np.stack([apply_hamiltonian(g, v, xi) for xi in x])
        out[name + "_cube_fft"] = g.cube_fft(v)
    save("grids.npz", **out)


def tiny_models():
    metal = ModelSpec(lattice=Lattice.cubic(4.0), e_cut=3.0, n_electrons=4, temperature=5e-3,
                      smearing="fermi_dirac",
                      gaussians=(GaussianWell(center=(0.3, 0.4, 0.5), amplitude=-3.0, width=0.8),
                                 GaussianWell(center=(0.7, 0.6, 0.4), amplitude=-2.0, width=0.7)))
    insul = ModelSpec(lattice=Lattice.cubic(4.0), e_cut=3.0, n_electrons=2, temperature=1e-3,
                      smearing="fermi_dirac",
                      gaussians=(GaussianWell(center=(0.5, 0.5, 0.5), amplitude=-5.0, width=0.8),))
    return metal, insul


def response_fixture(name, gs, seed):
    rng = np.random.default_rng(seed)
    g = gs.grids
    out = gs_arrays(gs)
    nocc = gs.n_occ
    dv = rng.standard_normal((3, g.n_g))
    out["dv"] = dv
    out["fprime"] = gs.fprime_occ()
    out["pair_weights"] = _occupied_pair_weights(gs)
    de, def_, df = delta_eigen_occupations(gs, dv[0])
    out["delta_eps"], out["delta_eps_f"], out["delta_f"] = de, def_, df
    # projector
    x = rng.standard_normal((g.n_b, 4)) + 1j * rng.standard_normal((g.n_b, 4))
    out["proj_x"], out["proj_qx"] = x, project_out_occupied(gs.phi_occ, x)
    # Sternheimer: per band, two tolerances
    rhs = project_out_occupied(gs.phi_occ, rng.standard_normal((g.n_b, nocc))
                               + 1j * rng.standard_normal((g.n_b, nocc)))
    out["cg_rhs"] = rhs
    for tag, tol in (("t6", 1e-6), ("t10", 1e-10)):
        sols, its, res = [], [], []
        for n in range(nocc):
            r = solve_sternheimer(gs, gs.v_local, n, rhs[:, n], tol)
            sols.append(r.solution), its.append(r.cg_iterations), res.append(r.final_residual_norm)
        out[f"cg_{tag}_x"], out[f"cg_{tag}_its"], out[f"cg_{tag}_res"] = (
            np.stack(sols, 1), np.array(its), np.array(res))
    # chi0 at tight and loose tolerances
    for tag, tol in (("t13", 1e-13), ("t8", 1e-8), ("t4", 1e-4)):
        drho, st = apply_chi0(gs, dv[0], np.full(nocc, tol))
        out[f"chi0_{tag}"], out[f"chi0_{tag}_its"] = drho, np.array(st.cg_iterations_per_band)
    tols = 10.0 ** rng.uniform(-10, -5, nocc)
    drho, st = apply_chi0(gs, dv[1], tols)
    out["chi0_mixed_tols"], out["chi0_mixed"], out["chi0_mixed_its"] = (
        tols, drho, np.array(st.cg_iterations_per_band))
    # constant perturbation
    drho, _ = apply_chi0(gs, np.full(g.n_g, 2.4), np.full(nocc, 1e-13))
    out["chi0_const"] = drho
    # dielectric / kernels
    for xc in ("none", "lda_x"):
        k = KernelSpec(xc=xc)
        out[f"kernel_{xc}"] = apply_kernel(k, g, gs.rho, dv[2])
        app = apply_dielectric(gs, k, dv[2], np.full(nocc, 1e-12))
        out[f"diel_{xc}"], out[f"diel_{xc}_kv"] = app.output, app.kv_norm
        out[f"diel_{xc}_its"] = np.array(app.cg_iterations_per_band)
    out["kerker_08"] = apply_kerker(KerkerSpec(0.8), g, dv[2])
    out["row_norm_abs"] = orbital_row_norm(g, gs.phi_occ)
    out["row_norm_re"] = orbital_row_norm(g, gs.phi_occ, real_part=True)
    out["bound_tols"] = tols
    out["bound"] = dielectric_error_bound(gs, 1.7, tols)
    save(name, **out)


def strategies_fixture():
    rng = np.random.default_rng(7)
    out = {}
    occ = rng.uniform(0.5, 2.0, 6)
    gaps = rng.uniform(0.05, 0.5, 6)
    i = 0
    for kind in ("grt", "bal", "agr", "d10", "d100", "d10n"):
        for pre in (False, True):
            for use_gap in (False, True):
                spec = StrategySpec(kind, pre, 1e-8, 10, use_gap)
                for it, cf in ((0, None), (3, None), (3, 2.5e-9)):
                    ctx = ToleranceContext(iteration=it, n_occ=6, occ=occ, volume=1000.0,
                                           n_g=13824, est_res_prev=3e-3, s=0.4, kv_norm=1.3,
                                           row_norm=0.6, rhs_norm=0.25, eps_gap=gaps,
                                           common_factor=cf)
                    out[f"case{i}_spec"] = np.array([kind, str(pre), str(use_gap), str(it),
                                                     str(cf)])
                    out[f"case{i}_tol"] = select_tolerances(spec, ctx)
                    i += 1
    out["occ"], out["gaps"], out["n_cases"] = occ, gaps, i
    save("strategies.npz", **out)


def igmres_fixture():
    rng = np.random.default_rng(11)
    out = {}
    for tag, n, m, tau in (("a", 50, 25, 1e-9), ("b", 60, 5, 1e-8)):
        a = np.eye(n) + 0.5 * rng.standard_normal((n, n)) / np.sqrt(n)
        b = rng.standard_normal(n)
        rep = igmres_solve(lambda v, budget: (a @ v, 1), b, m=m, tau=tau)
        out[f"{tag}_a"], out[f"{tag}_b"], out[f"{tag}_m"], out[f"{tag}_tau"] = a, b, m, tau
        out[f"{tag}_x"], out[f"{tag}_its"] = rep.solution, rep.iterations
        out[f"{tag}_hist"] = np.array(rep.est_res_history)
        out[f"{tag}_budgets"] = np.array([r.budget for r in rep.budgets])
        out[f"{tag}_sigma"] = rep.sigma_final
    save("igmres.npz", **out)


def run_dyson(gs, dv0, strategy, tau, m, xc):
    """run_response on the reference with dV0 injected and per-op tolerances logged."""
    log = []
    orig = H.apply_dielectric

    def logged(*args, **kw):
        app = orig(*args, **kw)
        log.append((np.array(app.tolerances_used), np.array(app.cg_iterations_per_band)))
        return app

    H.apply_dielectric = logged
    H.external_potential_derivative = lambda model, grids, index, direction: dv0.copy()
    rhs_log = []
    orig_chi0 = H.apply_chi0

    def logged_chi0(gs_, dv, tols, threads=1):
        rhs_log.append(np.array(tols))
        return orig_chi0(gs_, dv, tols, threads=threads)

    H.apply_chi0 = logged_chi0
    try:
        cfg = ExperimentConfig(model=gs.model, scf=ScfParams(),
                               response=ResponseParams(strategy=strategy, tau=tau, m=m,
                                                       perturbation=Perturbation()))
        met = H.run_response(cfg, gs=gs)
    finally:
        H.apply_dielectric = orig
        H.apply_chi0 = orig_chi0
    rep = met.igmres
    tol_sched = [t for t, _ in log]
    return dict(solution=met.solution, rhs=met.rhs, iterations=rep.iterations, n_ham=met.n_ham,
                n_ham_rhs=met.n_ham_rhs, final_est=met.final_est_res,
                final_true=met.final_true_res, hist=np.array(rep.est_res_history),
                rhs_tols=rhs_log[0], op_tols=tol_sched,
                budgets=np.array([r.budget for r in rep.budgets]))


def dyson_fixture(name, gs, dv0, runs):
    out = gs_arrays(gs)
    out["dv0"] = dv0
    for strategy, tau, m, xc in runs:
        r = run_dyson(gs, dv0, strategy, tau, m, xc)
        p = f"{strategy}_"
        for k in ("solution", "rhs", "iterations", "n_ham", "n_ham_rhs", "final_est",
                  "final_true", "hist", "rhs_tols", "budgets"):
            out[p + k] = r[k]
        # per-op tolerance schedule: the first `iterations` logged E applications are the
        # GMRES steps; later ones are the final true-residual evaluations
        sched = r["op_tols"][: len(r["budgets"])]
        out[p + "op_tols"] = np.array(sched)
        out[p + "meta"] = np.array([strategy, str(tau), str(m), xc])
    save(name, **out)


def kpoint_fixture():
    """Gamma supercell run of the reference = the k-sampled unit cell."""
    wells = (GaussianWell(center=(0.3, 0.4, 0.5), amplitude=-3.0, width=0.8),
             GaussianWell(center=(0.75, 0.6, 0.35), amplitude=-2.0, width=0.7))
    unit = ModelSpec(lattice=Lattice.cubic(4.0), e_cut=3.5, n_electrons=4, temperature=5e-3,
                     gaussians=wells)
    sup_wells = tuple(GaussianWell(center=(0.5 * (w.center[0] + s), w.center[1], w.center[2]),
                                   amplitude=w.amplitude, width=w.width)
                      for s in (0, 1) for w in wells)
    sup = ModelSpec(lattice=Lattice.orthorhombic(8.0, 4.0, 4.0), e_cut=3.5, n_electrons=8,
                    temperature=5e-3, gaussians=sup_wells)
    gs_sup = run_scf(sup, tol=1e-12, max_iter=600, damping=0.3)
    gsu = build_grids(unit.lattice, unit.e_cut)
    rng = np.random.default_rng(5)
    dv_unit = rng.standard_normal(gsu.n_g)
    nx, ny, nz = gsu.cube_dims
    cube = dv_unit.reshape((nx, ny, nz), order="F")
    dv_sup = np.concatenate([cube, cube], axis=0).ravel(order="F")
    drho, st = apply_chi0(gs_sup, dv_sup, np.full(gs_sup.n_occ, 1e-13))
    out = gs_arrays(gs_sup, "sup_")
    out.update(unit_lattice=unit.lattice.a, unit_e_cut=unit.e_cut, unit_wells=np.array(
        [[*w.center, w.amplitude, w.width] for w in wells]), dv_unit=dv_unit, dv_sup=dv_sup,
        drho_sup=drho, unit_dims=np.array(gsu.cube_dims))
    save("kpoint_supercell.npz", **out)


def main():
    grids_fixture()
    strategies_fixture()
    igmres_fixture()
    metal, insul = tiny_models()
    gs_m = run_scf(metal, tol=1e-11, max_iter=400, damping=0.3)
    gs_i = run_scf(insul, tol=1e-11, max_iter=400, damping=0.3)
    response_fixture("metal.npz", gs_m, 1)
    response_fixture("insulator.npz", gs_i, 2)
    rng = np.random.default_rng(3)
    dv0 = synth.smoothed_noise(gs_m.grids.g2_cube, gs_m.grids.cube_dims, rng)
    dyson_fixture("dyson_metal.npz", gs_m, dv0,
                  [("pbal", 1e-8, 8, "none"), ("bal", 1e-8, 8, "none"),
                   ("d10", 1e-8, 8, "none"), ("pagr", 1e-8, 8, "none")])
    # config 0 (BASELINE configs[0]) with the reference's own SCF
    spec0 = synth.config0_model(Lattice, GaussianWell, ModelSpec)
    gs0 = run_scf(spec0["model"], tol=1e-10)
    print("cfg0 n_occ", gs0.n_occ, "n_b", gs0.grids.n_b)
    dv00 = synth.smoothed_noise(gs0.grids.g2_cube, gs0.grids.cube_dims, spec0["rng"])
    dyson_fixture("dyson_cfg0.npz", gs0, dv00, [("bal", 1e-8, 10, "lda_x")])
    kpoint_fixture()


if __name__ == "__main__":
    main()
