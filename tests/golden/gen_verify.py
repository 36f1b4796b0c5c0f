"""Golden results of the reference's verification checks (harness.py:387-543).

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_verify.py

Builds the tiny metal model of gen_golden.py with the reference's own SCF and
runs its eight checks in verify_suite's order on one generator (seed 0), with
a Gaussian-displacement perturbation; writes verify_metal.npz (check names,
passed flags, margins, the response parameters).  The GPU suite
(paper_2505_02319_b200.verify) is compared against it in
tests/test_gpu_verify.py.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import gen_golden as G  # noqa: E402  (imports the reference from /root/reference)

PARAMS = dict(strategy="pbal", tau=1e-8, m=8, kerker_alpha=0.8, seed=0, gaussian=0,
              direction=(1.0, 0.0, 0.0))


def main():
    H = G.H
    metal, _ = G.tiny_models()
    gs = G.run_scf(metal, tol=1e-11, max_iter=400, damping=0.3)
    pert = G.Perturbation(gaussian=PARAMS["gaussian"], direction=PARAMS["direction"])
    resp = G.ResponseParams(strategy=PARAMS["strategy"], tau=PARAMS["tau"], m=PARAMS["m"],
                            kerker_alpha=PARAMS["kerker_alpha"], perturbation=pert,
                            seed=PARAMS["seed"])
    cfg = G.ExperimentConfig(model=metal, response=resp)
    rng = np.random.default_rng(PARAMS["seed"])
    kernel = G.KernelSpec(xc=metal.xc)
    checks = [
        H.check_fft_roundtrip(gs, rng),
        H.check_orthonormality(gs),
        H.check_kerker_lemma(gs, PARAMS["kerker_alpha"]),
        H.check_row_norm_bounds(gs),
        H.check_chi0_const(gs),
        H.check_bound_dominance(gs, kernel, rng),
        H.check_y_bound(gs, cfg),
        H.check_sternheimer_error_bound(gs, rng),
    ]
    for c in checks:
        print(f"{c['name']:26s} passed={c['passed']} margin={c['margin']:.4g}")
    G.save("verify_metal.npz", names=np.array([c["name"] for c in checks]),
           passed=np.array([bool(c["passed"]) for c in checks]),
           margins=np.array([float(c["margin"]) for c in checks]),
           params=np.array(repr(PARAMS)), **G.gs_arrays(gs))


if __name__ == "__main__":
    main()
