"""Executable-lemma verification suite on the GPU path (reference harness.py:387-543).

The reference checks its building blocks with eight "executable lemma" checks
(`verify_suite`, harness.py:517-543).  They are restated here on top of this
package's device operators so they run at BASELINE scale, including k-point
ground states:

  fft_roundtrip            harness.py:387-394  to_fourier(to_real(x)) = x, every k block
  orbital_orthonormality   harness.py:397-400  Phi^H Phi = I, every k block
  kerker_lemma             harness.py:403-425  dense T on a coarse grid: symmetric, spectrum in (0, 1]
  row_norm_bounds          harness.py:428-435  sqrt(N_occ/Omega) <= ||F^-1 Phi||_{2,inf} <= sqrt(N_g/Omega)
  chi0_gauge_invariance    harness.py:438-443  chi0(const) = 0
  error_bound_dominance    harness.py:446-461  ||(E - E~) v|| <= Lemma bound (Gamma: the lemma's setting)
  y_coefficient_bound      harness.py:464-490  |y_i| <= cycle_est_i / sigma_min on a converged solve
  sternheimer_error_bound  harness.py:493-514  CG error <= tol / gap vs a dense pseudo-inverse (small n_b)

The random draws follow the reference's order on one generator seeded with the
response seed, so on a Gamma ground state the checks see the same vectors as
the reference's.  Checks whose reference formulation is Gamma-only (the
dielectric error bound, the dense pseudo-inverse) report `skipped` for
k-sampled states or when the dense matrix would not fit (n_b > dense_limit).
"""

import numpy as np

from .device import device_state, state_blocks, torch_mod
from .errors import InvariantViolationError
from .harness import perturbation_from_config, solve_dyson
from .kernels import KernelSpec, KerkerSpec, apply_kerker
from .pwbasis import build_grids
from .response import apply_chi0, apply_dielectric, dielectric_error_bound, orbital_row_norm
from .sternheimer import project_out_occupied, solve_sternheimer

REPORT_FORMAT_VERSION = 1


def _skip(name, why):
    return {"name": name, "passed": True, "skipped": why, "margin": float("nan")}


def check_fft_roundtrip(gs, rng, draws=20):
    """harness.py:387-394, on the GPU transforms of every k block."""
    from . import ops
    worst = 0.0
    blocks, _ = state_blocks(gs)
    for blk in blocks:
        g = blk.grids
        xs = [rng.standard_normal(g.n_b) + 1j * rng.standard_normal(g.n_b) for _ in range(draws)]
        back = ops.to_fourier_many(g, ops.to_real_many(g, np.stack(xs)))
        for x, y in zip(xs, back):
            worst = max(worst, float(np.linalg.norm(y - x) / np.linalg.norm(x)))
    return {"name": "fft_roundtrip", "passed": worst <= 1e-14,
            "margin": 1e-14 / max(worst, 1e-300)}


def check_orthonormality(gs):
    """harness.py:397-400 (all kept orbitals of every k block)."""
    defect = 0.0
    blocks, _ = state_blocks(gs)
    for blk in blocks:
        phi = blk.phi
        defect = max(defect, float(np.max(np.abs(phi.conj().T @ phi - np.eye(phi.shape[1])))))
    return {"name": "orbital_orthonormality", "passed": defect <= 1e-10,
            "margin": 1e-10 / max(defect, 1e-300)}


def check_kerker_lemma(gs, alpha):
    """harness.py:403-425: dense Kerker matrix on an auxiliary grid with n_g <= 512,
    assembled column by column with the GPU Kerker filter."""
    e_cut = gs.model.e_cut
    grids = build_grids(gs.model.lattice, e_cut)
    while grids.n_g > 512:
        e_cut /= 2
        grids = build_grids(gs.model.lattice, e_cut)
    spec = KerkerSpec(alpha=alpha)
    t = np.zeros((grids.n_g, grids.n_g))
    for j in range(grids.n_g):
        e = np.zeros(grids.n_g)
        e[j] = 1.0
        t[:, j] = apply_kerker(spec, grids, e)
    herm = float(np.max(np.abs(t - t.T)))
    eig = np.linalg.eigvalsh(0.5 * (t + t.T))
    const = np.ones(grids.n_g)
    const_defect = float(np.max(np.abs(apply_kerker(spec, grids, const) - const)))
    passed = (herm <= 1e-12 and eig.min() > 0 and eig.max() <= 1 + 1e-12
              and abs(eig.max() - 1) <= 1e-12 and const_defect <= 1e-12)
    return {"name": "kerker_lemma", "passed": bool(passed),
            "margin": min(1e-12 / max(herm, 1e-300), 1e-12 / max(abs(eig.max() - 1), 1e-300)),
            "details": {"hermiticity": herm, "lambda_min": float(eig.min()),
                        "lambda_max": float(eig.max()), "const_defect": const_defect,
                        "n_g": grids.n_g}}


def check_row_norm_bounds(gs):
    """harness.py:428-435, per k block (GPU row norm)."""
    blocks, _ = state_blocks(gs)
    margin, passed, details = np.inf, True, []
    for blk in blocks:
        g = blk.grids
        val = orbital_row_norm(g, blk.phi_occ)
        vol = g.lattice.volume
        lo, hi = np.sqrt(blk.n_occ / vol), np.sqrt(g.n_g / vol)
        passed &= bool(lo * (1 - 1e-12) <= val <= hi * (1 + 1e-12))
        margin = min(margin, val / lo, hi / val)
        details.append({"lower": lo, "value": val, "upper": hi})
    return {"name": "row_norm_bounds", "passed": passed, "margin": margin,
            "details": details if len(details) > 1 else details[0]}


def check_chi0_const(gs):
    """harness.py:438-443: a constant potential shift produces no density response."""
    c = 1.0
    n_pairs = sum(b.n_occ for b in state_blocks(gs)[0])
    out, _ = apply_chi0(gs, np.full(gs.grids.n_g, c), np.full(n_pairs, 1e-14))
    rel = float(np.linalg.norm(out)) / (c * gs.model.n_electrons)
    return {"name": "chi0_gauge_invariance", "passed": rel <= 1e-10,
            "margin": 1e-10 / max(rel, 1e-300)}


def check_bound_dominance(gs, kernel, rng, draws=20):
    """harness.py:446-461 (Gamma: the dielectric error bound is the Gamma lemma)."""
    if hasattr(gs, "blocks"):
        return _skip("error_bound_dominance", "k-sampled ground state (Gamma-point lemma)")
    margins = []
    for _ in range(draws):
        v = rng.standard_normal(gs.grids.n_g)
        tols = 10.0 ** rng.uniform(-8, -4, gs.n_occ)
        approx = apply_dielectric(gs, kernel, v, tols)
        exact = apply_dielectric(gs, kernel, v, np.full(gs.n_occ, 1e-14))
        measured = float(np.linalg.norm(approx.output - exact.output))
        bound = dielectric_error_bound(gs, approx.kv_norm, tols)
        margins.append(bound / max(measured, 1e-300))
    worst = min(margins)
    return {"name": "error_bound_dominance", "passed": worst >= 1.0, "margin": worst,
            "details": {"draws": draws}}


def check_y_bound(gs, strategy, tau, m, xc, perturbation=None, dv0=None, kerker_alpha=0.8):
    """harness.py:464-490: every GMRES coefficient of a converged solve obeys
    |y_i| <= (cycle estimated residual)_i / sigma_min(H)."""
    if dv0 is None:
        dv0 = perturbation_from_config(gs, perturbation)
    res = solve_dyson(gs, dv0, strategy=strategy, tau=max(tau, 1e-7), m=m, xc=xc,
                      kerker_alpha=kerker_alpha)
    y = np.asarray(res.y_final)
    cycle = res.cycle_est_res[-1]
    worst = 0.0
    for i, yi in enumerate(y):
        bound = cycle[i] / res.sigma_final
        worst = max(worst, abs(yi) / bound if bound > 0 else np.inf)
    return {"name": "y_coefficient_bound", "passed": worst <= 1.0 + 1e-12,
            "margin": 1.0 / max(worst, 1e-300),
            "details": {"gmres_iterations": res.iterations, "n_ham": res.n_ham}}


def check_sternheimer_error_bound(gs, rng, dense_limit=3000):
    """harness.py:493-514: GPU CG solution vs the dense pseudo-inverse of the stored H."""
    if hasattr(gs, "blocks"):
        return _skip("sternheimer_error_bound", "k-sampled ground state (dense Gamma oracle)")
    grids = gs.grids
    if grids.n_b > dense_limit:
        return _skip("sternheimer_error_bound", f"n_b = {grids.n_b} > {dense_limit} (dense eigh)")
    from .scf import dense_hamiltonian
    eps_all, phi_all = np.linalg.eigh(dense_hamiltonian(grids, gs.v_local))
    worst = 0.0
    for n in (0, gs.n_occ - 1):
        rhs = rng.standard_normal(grids.n_b) + 1j * rng.standard_normal(grids.n_b)
        rhs = project_out_occupied(gs.phi_occ, rhs)
        tol = 1e-8
        res = solve_sternheimer(gs, gs.v_local, n, rhs, tol)
        perp = phi_all[:, gs.n_occ:]
        gaps = eps_all[gs.n_occ:] - gs.eps[n]
        x_ref = perp @ ((perp.conj().T @ rhs) / gaps)
        err = float(np.linalg.norm(res.solution - x_ref))
        bound = tol / (gs.eps_gap_ref - gs.eps[n])
        worst = max(worst, err / bound)
    return {"name": "sternheimer_error_bound", "passed": worst <= 1.0 + 1e-9,
            "margin": 1.0 / max(worst, 1e-300)}


def verify_suite(gs, strategy="pbal", tau=1e-9, m=10, kerker_alpha=0.8, seed=0, xc=None,
                 perturbation=None, dv0=None, draws=20, dense_limit=3000, raise_on_fail=True):
    """Run the checks (reference verify_suite, harness.py:517-543) on the GPU path.

    Returns {"format_version", "ok", "checks": [...]}; raises
    InvariantViolationError naming the failed checks, like the reference.
    `dv0` (or the reference's Gaussian-displacement `perturbation`) defines
    the y-bound solve's right-hand side.
    """
    torch_mod()
    device_state(gs)
    rng = np.random.default_rng(seed)
    xc = gs.model.xc if xc is None else xc
    kernel = KernelSpec(xc=xc)
    checks = [
        check_fft_roundtrip(gs, rng, draws),
        check_orthonormality(gs),
        check_kerker_lemma(gs, kerker_alpha),
        check_row_norm_bounds(gs),
        check_chi0_const(gs),
        check_bound_dominance(gs, kernel, rng, draws),
        check_y_bound(gs, strategy, tau, m, xc, perturbation, dv0, kerker_alpha),
        check_sternheimer_error_bound(gs, rng, dense_limit),
    ]
    ok = all(c["passed"] for c in checks)
    result = {"format_version": REPORT_FORMAT_VERSION, "ok": ok, "checks": checks}
    if not ok and raise_on_fail:
        failed = [c["name"] for c in checks if not c["passed"]]
        raise InvariantViolationError(f"verification failed: {', '.join(failed)}")
    return result
