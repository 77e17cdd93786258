// Cell-local physics of the linearised phase-field Jacobian (NoSplit), the
// work one thread does for one cell.  Restates reference model.py:270-355
// (caches + local kernels) with the coefficient tables recomputed on the fly
// from the linearisation state ("model F").
#pragma once

#include "common.cuh"

namespace pffmg {

enum Mode { M_FULL = 0, M_UBLK = 1, M_PBLK = 2, M_DIAG = 3, M_RES = 4 };

// Number of staged fp64 fields per vertex and of output components.
template <int D, int MODE, bool SPLIT = false>
struct ModeInfo {
    // FULL: v[0..D], U[0..D], phi_tilde;  UBLK: v[0..D-1], phi_tilde
    // PBLK: v[D], U[0..D-1];              DIAG: U[0..D-1], phi_tilde
    // RES (semilinear form A(U), model.py:420-460): U[0..D], phi_tilde
    // With the spectral split (SPLIT) the u block also needs U[0..D-1]: its
    // tangent depends on the strain of the linearisation state.
    static constexpr int NU = MODE == M_FULL || MODE == M_RES ? D + 1 : (MODE == M_UBLK && !SPLIT ? 0 : D);
    static constexpr int NV = MODE == M_FULL ? D + 1 : (MODE == M_UBLK ? D : (MODE == M_PBLK ? 1 : 0));
    static constexpr int NF = NV + NU + (MODE != M_PBLK ? 1 : 0);
    static constexpr bool PT = MODE != M_PBLK;
    static constexpr int NCO =
        MODE == M_FULL || MODE == M_DIAG || MODE == M_RES ? D + 1 : (MODE == M_UBLK ? D : 1);
    static constexpr int COMP0 = MODE == M_PBLK ? D : 0;   // global component of v/out slot 0
    // field slots in the staged tile
    static constexpr int F_V = 0;
    static constexpr int F_U = NV;
    static constexpr int F_PT = NV + NU;
};

// Per-QP state coefficients of _build_caches (model.py:274-309), NoSplit.
struct QPCoef {
    double gkr;    // gk * rho
    double T[3][3];
    double a;      // a_phiphi
};

template <int D>
__device__ __forceinline__ void strain_stuff(const double (&gu)[D][D], double& div, double& Ep,
                                             double (&sp)[D][D], const Consts& K) {
    div = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) div += gu[i][i];
    double ee = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const double e = 0.5 * (gu[i][j] + gu[j][i]);
            ee = fma(e, e, ee);
            sp[i][j] = 2.0 * K.mu * e + (i == j ? K.lam * div : 0.0);
        }
    Ep = 0.5 * K.lam * div * div + K.mu * ee;   // model.py:163-165
}

// Compute the cell contributions o[k][n] (k = output component slot, n = corner).
// cv[f][n]: staged corner values (v masked already), rho_q: per-QP modulus or null.
template <int D, int MODE>
__device__ __forceinline__ void cell_kernel(const double (&cv)[ModeInfo<D, MODE>::NF][1 << D],
                                            const double* __restrict__ rho_q, const Consts& K,
                                            double (&o)[ModeInfo<D, MODE>::NCO][1 << D]) {
    using MI = ModeInfo<D, MODE>;
    constexpr int NP = 1 << D;
    using S = SF<D>;
    if (MODE == M_RES) {
        // semilinear form A(U), NoSplit, general box cells (model.py:420-460)
        double rho[NP], pt[D + 1][NP], ph[D + 1][NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) rho[q] = rho_q ? __ldg(rho_q + q) : 1.0;
        S::interp(cv[MI::F_PT], pt, K);
        S::interp(cv[MI::F_U + D], ph, K);
        double G[D][D][NP], f[NP], g[D][NP];
        {
            double gu[NP][D][D];
#pragma unroll
            for (int i = 0; i < D; ++i) {
                double t[D + 1][NP];
                S::interp(cv[MI::F_U + i], t, K, false);
#pragma unroll
                for (int q = 0; q < NP; ++q)
#pragma unroll
                    for (int j = 0; j < D; ++j) gu[q][i][j] = t[1 + j][q] * K.ih[j];
            }
            const double p = 0.5 * K.two_p;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                double div, Ep, sp[D][D];
                strain_stuff<D>(gu[q], div, Ep, sp, K);
                const double gk = (K.omk * (pt[0][q] * pt[0][q]) + K.kappa) * rho[q];
                const double pp = pt[0][q] * pt[0][q] * p;
#pragma unroll
                for (int i = 0; i < D; ++i)
#pragma unroll
                    for (int j = 0; j < D; ++j)
                        G[i][j][q] = K.jxw * (gk * sp[i][j] + (i == j ? pp : 0.0)) * K.ih[j];
                const double phi = ph[0][q];
                f[q] = K.jxw * (K.omk * phi * rho[q] * Ep + K.two_p * phi * div - K.gc_over_eps * (1.0 - phi));
#pragma unroll
                for (int j = 0; j < D; ++j) g[j][q] = K.jxw * K.k_phi * (ph[1 + j][q] * K.ih[j]) * K.ih[j];
            }
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double t[NP];
            S::template integrate<false>(t, G[i], K);
#pragma unroll
            for (int n = 0; n < NP; ++n) o[i][n] = t[n];
        }
        S::template integrate<true>(f, g, K);
#pragma unroll
        for (int n = 0; n < NP; ++n) o[D][n] = f[n];
        return;
    }

    // ---- state-dependent per-QP data
    double gkr[NP];      // gk * rho       (FULL, UBLK, DIAG)
    double rho[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) rho[q] = rho_q ? __ldg(rho_q + q) : 1.0;
    if (MI::PT) {
        double pv[D + 1][NP];
        S::interp(cv[MI::F_PT], pv, K);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double ph = pv[0][q];
            gkr[q] = (K.omk * (ph * ph) + K.kappa) * rho[q];   // degradation(), model.py:135-137
        }
    }

    // grad U (u components) -> strain quantities, phi_q
    double Tq[NP][D][D];
    double aq[NP];
    if (MI::NU > 0) {
        double gu[NP][D][D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double t[D + 1][NP];
            S::interp(cv[MI::F_U + i], t, K, false);
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int j = 0; j < D; ++j) gu[q][i][j] = t[1 + j][q] * K.ih[j];
        }
        double phq[NP];
        if (MODE == M_FULL) {
            double t[D + 1][NP];
            S::interp(cv[MI::F_U + D], t, K);
#pragma unroll
            for (int q = 0; q < NP; ++q) phq[q] = t[0][q];
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            double div, Ep, sp[D][D];
            strain_stuff<D>(gu[q], div, Ep, sp, K);
            aq[q] = K.omk * rho[q] * Ep + K.two_p * div + K.gc_over_eps;   // model.py:304-308
            if (MODE == M_FULL) {
                const double c = rho[q] * K.omk * phq[q];
#pragma unroll
                for (int i = 0; i < D; ++i)
#pragma unroll
                    for (int j = 0; j < D; ++j)
                        Tq[q][i][j] = c * sp[i][j] + (i == j ? K.two_p * phq[q] : 0.0);   // model.py:299-303
            }
        }
    }

    if (MODE == M_DIAG) {
        // du[i][n] = JxW sum_q gk rho (mu |gradN|^2 + (mu+lam) (d_i N)^2); dphi[n] =
        // JxW sum_q a N^2 + k_phi JxW sum_q |gradN|^2   (model.py:394-413, fem.py:242-261)
#pragma unroll
        for (int n = 0; n < NP; ++n) {
            double du[D];
#pragma unroll
            for (int i = 0; i < D; ++i) du[i] = 0.0;
            double dp = 0.0, g2 = 0.0;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                double Nv = 1.0;
                double gN[D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    const int nb = (n >> a) & 1, qb = (q >> a) & 1;
                    const double gq = qb ? K.g1 : K.g0;
                    const double fac = nb ? gq : (qb ? K.omg1 : K.omg0);
                    Nv *= fac;
                }
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    double gv = ((n >> a) & 1) ? K.ih[a] : -K.ih[a];
#pragma unroll
                    for (int b = 0; b < D; ++b) {
                        if (b == a) continue;
                        const int nb = (n >> b) & 1, qb = (q >> b) & 1;
                        const double gq = qb ? K.g1 : K.g0;
                        gv *= nb ? gq : (qb ? K.omg1 : K.omg0);
                    }
                    gN[a] = gv;
                }
                double gg = 0.0;
#pragma unroll
                for (int a = 0; a < D; ++a) gg = fma(gN[a], gN[a], gg);
#pragma unroll
                for (int i = 0; i < D; ++i)
                    du[i] = fma(gkr[q], K.mu * gg + (K.mu + K.lam) * (gN[i] * gN[i]), du[i]);
                dp = fma(aq[q], Nv * Nv, dp);
                g2 += gg;
            }
#pragma unroll
            for (int i = 0; i < D; ++i) o[i][n] = K.jxw * du[i];
            o[D][n] = K.jxw * dp + K.k_phi * (K.jxw * g2);
        }
        return;
    }

    // ---- apply to the input field(s)
    if (MODE == M_FULL || MODE == M_UBLK) {
        double gv[NP][D][D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double t[D + 1][NP];
            S::interp(cv[MI::F_V + i], t, K, false);
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int j = 0; j < D; ++j) gv[q][i][j] = t[1 + j][q] * K.ih[j];
        }
        // u rows: sum_q JxW s(q) : gradN   with s = gk rho (2 mu e + lam tr I) (model.py:313-330)
        double G[D][D][NP];   // [comp i][direction j][q]
        double coup[NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            double tr = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) tr += gv[q][i][i];
            const double w = K.jxw * gkr[q];
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    const double e = 0.5 * (gv[q][i][j] + gv[q][j][i]);
                    const double s = 2.0 * K.mu * e + (i == j ? K.lam * tr : 0.0);
                    G[i][j][q] = w * s * K.ih[j];
                }
            if (MODE == M_FULL) {
                double c = 0.0;
#pragma unroll
                for (int i = 0; i < D; ++i)
#pragma unroll
                    for (int j = 0; j < D; ++j) c = fma(Tq[q][i][j], gv[q][i][j], c);   // model.py:350
                coup[q] = c;
            }
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double f[NP];
            S::template integrate<false>(f, G[i], K);
#pragma unroll
            for (int n = 0; n < NP; ++n) o[i][n] = f[n];
        }
        if (MODE == M_FULL) {
            double t[D + 1][NP];
            S::interp(cv[MI::F_V + D], t, K);
            double f[NP], g[D][NP];
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                f[q] = K.jxw * (coup[q] + aq[q] * t[0][q]);                   // model.py:351-352
#pragma unroll
                for (int j = 0; j < D; ++j) g[j][q] = K.jxw * K.k_phi * (t[1 + j][q] * K.ih[j]) * K.ih[j];
            }
            S::template integrate<true>(f, g, K);
#pragma unroll
            for (int n = 0; n < NP; ++n) o[D][n] = f[n];
        }
    } else {   // M_PBLK  (model.py:332-338)
        double t[D + 1][NP];
        S::interp(cv[MI::F_V], t, K);
        double f[NP], g[D][NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            f[q] = K.jxw * (aq[q] * t[0][q]);
#pragma unroll
            for (int j = 0; j < D; ++j) g[j][q] = K.jxw * K.k_phi * (t[1 + j][q] * K.ih[j]) * K.ih[j];
        }
        S::template integrate<true>(f, g, K);
#pragma unroll
        for (int n = 0; n < NP; ++n) o[0][n] = f[n];
    }
}

}  // namespace pffmg
