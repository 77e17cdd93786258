"""pffmg: B200-native matrix-free phase-field-fracture Jacobian + GMG (sm_100a).

Drop-in GPU twins of the hot path of the reference `fracmg` package
(arXiv 1902.08112 re-implementation):

* model.PhaseFieldOperator   -- fused matrix-free Jacobian vmult / block vmults / diagonal
* fem.Discretization         -- masked Q1 restriction / prolongation / injection kernels
* mgsolve.*                  -- Chebyshev-Jacobi smoother, level contexts, V(1,1) cycle
* krylov.*                   -- restarted GMRES, CG-Lanczos spectrum estimator

All compute runs in libpffmg.so (hand-written CUDA for sm_100a, C ABI in
include/pffmg.h).  `patch.install()` swaps these into an imported `fracmg`.
Submodules import lazily so host-only helpers work without a GPU.
"""

__version__ = "0.1.0"

__all__ = ["model", "fem", "mgsolve", "krylov", "lattice", "configs", "patch"]
