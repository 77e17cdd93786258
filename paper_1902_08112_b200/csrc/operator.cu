// C ABI of the fused matrix-free operator: argument checking and dispatch to
// the per-dimension kernel instantiations (op2d.cu, op3d.cu; kernels in
// op_kernels.cuh).  Replaces reference model.py:368-413 and the vector
// updates of mgsolve.py:82-113 / 227 (fused epilogues).
#include <cmath>

#include "op_launch.cuh"

namespace pffmg {

template <int MODE, int EPI>
static int launch(const OpArgs& A, cudaStream_t s, const char* what) {
    const Lat& L = A.L;
    const bool iso = L.hx == L.hy && (L.dim == 2 || L.hz == L.hx);
    if (L.dim == 2)
        launch2d<MODE, EPI>(A, iso, s);
    else
        launch3d<MODE, EPI>(A, iso, s);
    return check_launch(what);
}

static int fill_args(const pffmg_lattice* lat, const pffmg_state* st, OpArgs* A) {
    PFFMG_REQUIRE(lat && st, "null lattice/state");
    *A = OpArgs{};
    int rc = make_lat(lat, &A->L);
    if (rc) return rc;
    rc = make_consts(lat, st, &A->K);
    if (rc) return rc;
    A->I = make_iso_host(A->K);
    if (rc) return rc;
    if (st->split != 0 && st->split != 1) {
        set_error("unknown split kind %d (0 NoSplit, 1 Miehe)", st->split);
        return PFFMG_ERR_ARG;
    }
    PFFMG_REQUIRE(st->split_band >= 0.0 && std::isfinite(st->split_band), "split_band must be finite and >= 0");
    A->split = st->split;
    PFFMG_REQUIRE(st->flags, "state.flags is NULL");
    A->U = st->U;
    A->pt = st->phi_tilde;
    A->rho = st->rho;
    A->flags = st->flags;
    A->premasked = (st->hints & PFFMG_HINT_PREMASKED) ? 1 : 0;
    return PFFMG_OK;
}

template <int EPI>
static int dispatch_which(const OpArgs& A, int which, cudaStream_t s, const char* what) {
    if (which == PFFMG_FULL) {
        PFFMG_REQUIRE(A.U && A.pt, "%s: full operator needs U and phi_tilde", what);
        return launch<M_FULL, EPI>(A, s, what);
    }
    if (which == PFFMG_UBLOCK) {
        PFFMG_REQUIRE(A.pt, "%s: u block needs phi_tilde", what);
        return launch<M_UBLK, EPI>(A, s, what);
    }
    if (which == PFFMG_PBLOCK) {
        PFFMG_REQUIRE(A.U, "%s: phi block needs U", what);
        return launch<M_PBLK, EPI>(A, s, what);
    }
    set_error("%s: which must be -1, 0 or 1 (got %d)", what, which);
    return PFFMG_ERR_ARG;
}

}  // namespace pffmg

using namespace pffmg;

extern "C" int pffmg_apply(const pffmg_lattice* lat, const pffmg_state* st, int which,
                           const double* v, double* out, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(v && out && v != out, "pffmg_apply: bad v/out");
    A.v = v;
    A.out = out;
    return dispatch_which<E_STORE>(A, which, as_stream(stream), "pffmg_apply");
}

extern "C" int pffmg_residual(const pffmg_lattice* lat, const pffmg_state* st, int which,
                              const double* x, const double* b, double* out, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(x && b && out && x != out, "pffmg_residual: bad x/b/out");
    A.v = x;
    A.b = b;
    A.out = out;
    return dispatch_which<E_RESID>(A, which, as_stream(stream), "pffmg_residual");
}

extern "C" int pffmg_semilinear_residual(const pffmg_lattice* lat, const pffmg_state* st, double* out,
                                         void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(out && A.U && A.pt, "pffmg_semilinear_residual: needs out, U and phi_tilde");
    A.out = out;
    A.v = A.U;   // unused (no v fields in residual mode)
    return launch<M_RES, E_RESZ>(A, as_stream(stream), "pffmg_semilinear_residual");
}

extern "C" int pffmg_diagonal(const pffmg_lattice* lat, const pffmg_state* st, double* out,
                              void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(out && A.U && A.pt, "pffmg_diagonal: needs out, U and phi_tilde");
    A.out = out;
    return launch<M_DIAG, E_DIAG>(A, as_stream(stream), "pffmg_diagonal");
}

extern "C" int pffmg_cheb_step(const pffmg_lattice* lat, const pffmg_state* st, int which,
                               const double* d_in, double* d_out, double* r, double* x,
                               const double* invdiag, double c_dd, double c_dr, int x_add_din,
                               void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(d_in && d_out && r && x && invdiag && d_in != d_out && x != d_in,
                  "pffmg_cheb_step: bad pointers");
    A.v = d_in;
    A.dout = d_out;
    A.r = r;
    A.x = x;
    A.inv = invdiag;
    A.c1 = c_dd;
    A.c2 = c_dr;
    A.x_add_din = x_add_din;
    return dispatch_which<E_CHEB>(A, which, as_stream(stream), "pffmg_cheb_step");
}

extern "C" int pffmg_cheb_step_dc(const pffmg_lattice* lat, const pffmg_state* st, int which,
                                  const double* d_in, double* d_out, double* r, double* x,
                                  const double* invdiag, const double* coef, int x_add_din, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(d_in && d_out && r && x && invdiag && coef && d_in != d_out && x != d_in,
                  "pffmg_cheb_step_dc: bad pointers");
    A.v = d_in;
    A.dout = d_out;
    A.r = r;
    A.x = x;
    A.inv = invdiag;
    A.coef = coef;
    A.x_add_din = x_add_din;
    return dispatch_which<E_CHEB>(A, which, as_stream(stream), "pffmg_cheb_step_dc");
}

extern "C" int pffmg_cheb_init_dc(const pffmg_lattice* lat, const pffmg_state* st, int which,
                                  const double* x, const double* b, double* r, double* d,
                                  const double* invdiag, const double* theta, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(x && b && r && d && invdiag && theta && d != x && r != x, "pffmg_cheb_init_dc: bad pointers");
    A.v = x;
    A.b = b;
    A.r = r;
    A.dout = d;
    A.inv = invdiag;
    A.coef = theta;
    return dispatch_which<E_CHEB0>(A, which, as_stream(stream), "pffmg_cheb_init_dc");
}

extern "C" int pffmg_cheb_init(const pffmg_lattice* lat, const pffmg_state* st, int which,
                               const double* x, const double* b, double* r, double* d,
                               const double* invdiag, double theta, void* stream) {
    OpArgs A;
    int rc = fill_args(lat, st, &A);
    if (rc) return rc;
    PFFMG_REQUIRE(x && b && r && d && invdiag && d != x && r != x, "pffmg_cheb_init: bad pointers");
    A.v = x;
    A.b = b;
    A.r = r;
    A.dout = d;
    A.inv = invdiag;
    A.c1 = theta;
    return dispatch_which<E_CHEB0>(A, which, as_stream(stream), "pffmg_cheb_init");
}
