"""CPU oracle for the chi0 / Sternheimer hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain-numpy restatement of the reference package
`pwdyson` (arXiv 2505.02319, mounted read-only at /root/reference) for the
path named by BASELINE.json:north_star.  It is the *checker*: only
`tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl
reference` legs of `bench.py` may import it.  The product package
`paper_2505_02319_b200` never imports it and has no CPU fallback.

Pinning: `tests/golden/*.npz` are produced by running the unmodified
reference (`tests/golden/gen_golden.py`); `tests/test_oracle_golden.py`
checks every oracle function against them, so the oracle is "pinned"
(section Oracle).

Every function cites the reference file:line it restates.  The arithmetic
of the reference lives in numpy/scipy (scipy.fft ducc backend, OpenBLAS);
the oracle calls the same library routines in the same order so it matches
the reference to round-off (usually bit-for-bit).

Modules:
    basis      -- lattice, sphere/cube grids, normalised transforms (+ k-points)
    model      -- toy solid, smearing, Hamiltonian apply, dense diag, SCF
    response   -- projector, Sternheimer PCG, chi0, dielectric operator, kernels
    outer      -- tolerance strategies and the inexact GMRES
    dyson      -- run_response-equivalent driver (RHS build + GMRES solve)
"""
