// Launch interface between operator.cu (C ABI) and the per-dimension
// instantiation units op2d.cu / op3d.cu.
#pragma once
#include "op_kernels.cuh"

namespace pffmg {

template <int MODE, int EPI>
int launch2d(const OpArgs& A, bool iso, cudaStream_t s);
template <int MODE, int EPI>
int launch3d(const OpArgs& A, bool iso, cudaStream_t s);

#define PFFMG_INST1(F, M, E) template int F<M, E>(const OpArgs&, bool, cudaStream_t);
#define PFFMG_INSTANTIATE_LAUNCH(F)                                                          \
    PFFMG_INST1(F, M_FULL, E_STORE) PFFMG_INST1(F, M_FULL, E_RESID)                          \
    PFFMG_INST1(F, M_FULL, E_CHEB) PFFMG_INST1(F, M_FULL, E_CHEB0)                           \
    PFFMG_INST1(F, M_UBLK, E_STORE) PFFMG_INST1(F, M_UBLK, E_RESID)                          \
    PFFMG_INST1(F, M_UBLK, E_CHEB) PFFMG_INST1(F, M_UBLK, E_CHEB0)                           \
    PFFMG_INST1(F, M_PBLK, E_STORE) PFFMG_INST1(F, M_PBLK, E_RESID)                          \
    PFFMG_INST1(F, M_PBLK, E_CHEB) PFFMG_INST1(F, M_PBLK, E_CHEB0)                           \
    PFFMG_INST1(F, M_DIAG, E_DIAG) PFFMG_INST1(F, M_RES, E_RESZ)

template <int MODE, int EPI>
int launch2q(const OpArgs& A, cudaStream_t s);    // Q2 lattices (op2q.cu)

int launch_phi_coef3(const OpArgs& A, double* tab, cudaStream_t s);   // op3d.cu
int launch_phi_coef2(const OpArgs& A, double* tab, cudaStream_t s);   // op2d.cu
int launch_phi_coefq(const OpArgs& A, double* tab, cudaStream_t s);   // op2q.cu

#define PFFMG_INST2(F, M, E) template int F<M, E>(const OpArgs&, cudaStream_t);
#define PFFMG_INSTANTIATE_LAUNCH2(F)                                                         \
    PFFMG_INST2(F, M_FULL, E_STORE) PFFMG_INST2(F, M_FULL, E_RESID)                          \
    PFFMG_INST2(F, M_FULL, E_CHEB) PFFMG_INST2(F, M_FULL, E_CHEB0)                           \
    PFFMG_INST2(F, M_UBLK, E_STORE) PFFMG_INST2(F, M_UBLK, E_RESID)                          \
    PFFMG_INST2(F, M_UBLK, E_CHEB) PFFMG_INST2(F, M_UBLK, E_CHEB0)                           \
    PFFMG_INST2(F, M_PBLK, E_STORE) PFFMG_INST2(F, M_PBLK, E_RESID)                          \
    PFFMG_INST2(F, M_PBLK, E_CHEB) PFFMG_INST2(F, M_PBLK, E_CHEB0)                           \
    PFFMG_INST2(F, M_DIAG, E_DIAG) PFFMG_INST2(F, M_RES, E_RESZ)

}  // namespace pffmg
