"""CPU oracle for the pffmg hot path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference `fracmg` algorithms on
the hot path named by BASELINE.json:north_star (matrix-free Jacobian vmult,
its diagonal, the Chebyshev-Jacobi smoother, masked GMG transfers, GMRES and
the CG-Lanczos spectrum estimator).  Every function cites the reference
file:line it restates (paths relative to /root/reference/pkg/src/fracmg/).

Parity pin: the restatement is checked against golden vectors produced by
the reference itself (tests/golden/make_golden.py imports /root/reference in
the build container and commits tests/golden/*.npz); see
tests/test_oracle_golden.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  The product path
(paper_1902_08112_b200) never imports it and never falls back to it.
"""
