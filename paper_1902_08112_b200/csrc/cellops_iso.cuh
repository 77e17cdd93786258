// Cell kernel for isotropic cells (h equal on every axis -- every BASELINE
// configuration and every reference test mesh).  Same physics as the generic
// cell_kernel in cellops.cuh (reference model.py:270-355), with the 1/h and
// JxW factors folded into per-level constants (IsoK, built on the host) and
// the symmetric tensor algebra written out.
//
// With raw reference derivatives r_ij = d_j^ref U_i, w_ij = d_j^ref v_i, and
// the raw "stress" of U   S_ii = 2 mu r_ii + lam tr r,  S_ij = mu (r_ij + r_ji):
//   E+ (model.py:163-165)        = ih^2 * 1/2 S : sym(r)
//   a_phiphi (model.py:304-308)  = (1-k) rho E+ + 2 p ih tr r + Gc/eps
//   T : grad v (model.py:299-303, 350)
//                                = ih^2 rho (1-k) phi S : w + 2 p phi ih tr w
//   u-row stress (model.py:313-330)
//     G_ii = JxW ih^2 gk rho (2 mu w_ii + lam tr w),  G_ij = JxW ih^2 gk rho mu (w_ij + w_ji)
// and the k_phi Laplacian (constant per cell) is applied at the corners as
// sum_j (D^T D)_j (x) (B^T B)_others (model.py:337, 353-354).
#pragma once

#include "cellops.cuh"

namespace pffmg {

struct IsoK {
    double gk_a, gk_b;     // JxW ih^2 (1-k), JxW ih^2 k      -> gk_s = (gk_a phi~ phi~ + gk_b) rho
    double cS;             // JxW ih^2 (1-k) / 2              -> E+ term of a (times rho)
    double cdiv;           // JxW 2 p ih
    double c0;             // JxW Gc / eps
    double cc;             // JxW ih^2 (1-k)                  -> coupling (times rho phi)
    double ctr;            // JxW 2 p ih                      -> pressure coupling (times phi)
    double clap;           // JxW k_phi ih^2
    double two_mu, lam, mu;
    double bb_lo, bb_hi;   // sum_q B_qa B_qb: (2/3, 1/3) for the 2-point Gauss rule
};

inline IsoK make_iso_host(const Consts& K) {
    IsoK I;
    const double ih2 = K.ih[0] * K.ih[0];
    const double jh2 = K.jxw * ih2;
    I.gk_a = jh2 * K.omk;
    I.gk_b = jh2 * K.kappa;
    I.cS = 0.5 * jh2 * K.omk;
    I.cdiv = K.jxw * K.two_p * K.ih[0];
    I.c0 = K.jxw * K.gc_over_eps;
    I.cc = jh2 * K.omk;
    I.ctr = K.jxw * K.two_p * K.ih[0];
    I.clap = K.jxw * K.k_phi * ih2;
    I.two_mu = 2.0 * K.mu;
    I.lam = K.lam;
    I.mu = K.mu;
    I.bb_lo = K.omg0 * K.omg0 + K.omg1 * K.omg1;
    I.bb_hi = K.omg0 * K.g0 + K.omg1 * K.g1;
    return I;
}

// out[n] += scale * sum_j ((D^T D)_j (x) (B^T B)_{other axes}) c   (Q1 cell Laplacian)
template <int D>
__device__ __forceinline__ void corner_laplacian(const double (&c)[1 << D], double scale,
                                                 const IsoK& I, double (&out)[1 << D]) {
    constexpr int NP = 1 << D;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        double t[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) t[i] = c[i];
#pragma unroll
        for (int a = 0; a < D; ++a) {
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                if (i & (1 << a)) continue;
                const int k = i | (1 << a);
                const double u0 = t[i], u1 = t[k];
                if (a == j) {            // D^T D = [[2, -2], [-2, 2]]
                    const double d = 2.0 * (u1 - u0);
                    t[i] = -d;
                    t[k] = d;
                } else {                 // B^T B = [[lo, hi], [hi, lo]]
                    t[i] = fma(I.bb_lo, u0, I.bb_hi * u1);
                    t[k] = fma(I.bb_hi, u0, I.bb_lo * u1);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < NP; ++i) out[i] = fma(scale, t[i], out[i]);
    }
}

// B^T along every axis (the N-weighted "mass" part of the phi-row integration).
template <int D>
__device__ __forceinline__ void mass_transpose(double (&f)[1 << D], const Consts& K) {
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
#pragma unroll
        for (int i = 0; i < (1 << D); ++i) {
            if (i & (1 << a)) continue;
            const int j = i | (1 << a);
            const double f0 = f[i], f1 = f[j];
            f[i] = fma(K.omg0, f0, K.omg1 * f1);
            f[j] = fma(K.g0, f0, K.g1 * f1);
        }
    }
}

template <int D, int MODE, bool RHO>
__device__ __forceinline__ void cell_kernel_iso(const double (&cv)[ModeInfo<D, MODE>::NF][1 << D],
                                                const double* __restrict__ rho_q, const Consts& K,
                                                const IsoK& I,
                                                double (&o)[ModeInfo<D, MODE>::NCO][1 << D]) {
    using MI = ModeInfo<D, MODE>;
    constexpr int NP = 1 << D;
    using S = SF<D>;

    double rho[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) rho[q] = RHO ? __ldg(rho_q + q) : 1.0;

    double gks[NP];                                 // JxW ih^2 gk rho   (model.py:282, 295)
    if (MI::PT) {
        double pv[D + 1][NP];
        S::interp(cv[MI::F_PT], pv, K);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double ph = pv[0][q];
            const double g = fma(I.gk_a * ph, ph, I.gk_b);
            gks[q] = RHO ? g * rho[q] : g;
        }
    }

    // raw gradient of U's displacement part -> stress S, a_phiphi * JxW
    double Sd[NP][D], So[NP][D * (D - 1) / 2], aj[NP];
    if (MI::NU > 0) {
        double r[NP][D][D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double t[D + 1][NP];
            S::interp(cv[MI::F_U + i], t, K, false);
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int j = 0; j < D; ++j) r[q][i][j] = t[1 + j][q];
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            double dv = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) dv += r[q][i][i];
            const double ld = I.lam * dv;
            double e2 = 0.0;                           // S : sym(r) = 2 E+ / ih^2
#pragma unroll
            for (int i = 0; i < D; ++i) {
                Sd[q][i] = fma(I.two_mu, r[q][i][i], ld);
                e2 = fma(Sd[q][i], r[q][i][i], e2);
            }
            int k = 0;
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = i + 1; j < D; ++j, ++k) {
                    const double s = r[q][i][j] + r[q][j][i];
                    So[q][k] = I.mu * s;
                    e2 = fma(So[q][k], s, e2);
                }
            const double ce = RHO ? I.cS * rho[q] : I.cS;
            aj[q] = fma(ce, e2, fma(I.cdiv, dv, I.c0));
        }
    }

    if (MODE == M_DIAG) {
        // exact diagonal (model.py:394-413, fem.py:242-261); not hot -- plain loops
#pragma unroll
        for (int n = 0; n < NP; ++n) {
            double du[D];
#pragma unroll
            for (int i = 0; i < D; ++i) du[i] = 0.0;
            double dp = 0.0, g2 = 0.0;
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                double Nv = 1.0, gN[D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    const int nb = (n >> a) & 1, qb = (q >> a) & 1;
                    Nv *= nb ? (qb ? K.g1 : K.g0) : (qb ? K.omg1 : K.omg0);
                }
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    double gv = ((n >> a) & 1) ? 1.0 : -1.0;
#pragma unroll
                    for (int b = 0; b < D; ++b) {
                        if (b == a) continue;
                        const int nb = (n >> b) & 1, qb = (q >> b) & 1;
                        gv *= nb ? (qb ? K.g1 : K.g0) : (qb ? K.omg1 : K.omg0);
                    }
                    gN[a] = gv;
                }
                double gg = 0.0;
#pragma unroll
                for (int a = 0; a < D; ++a) gg = fma(gN[a], gN[a], gg);
#pragma unroll
                for (int i = 0; i < D; ++i)
                    du[i] = fma(gks[q], fma(I.mu, gg, (I.mu + I.lam) * (gN[i] * gN[i])), du[i]);
                dp = fma(aj[q], Nv * Nv, dp);
                g2 += gg;
            }
#pragma unroll
            for (int i = 0; i < D; ++i) o[i][n] = du[i];
            o[D][n] = fma(I.clap, g2, dp);
        }
        return;
    }

    double coup[NP];
    if (MODE == M_FULL || MODE == M_UBLK) {
        double w[NP][D][D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double t[D + 1][NP];
            S::interp(cv[MI::F_V + i], t, K, false);
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int j = 0; j < D; ++j) w[q][i][j] = t[1 + j][q];
        }
        double phq[NP];
        if (MODE == M_FULL) {
            double t[D + 1][NP];
            S::interp(cv[MI::F_U + D], t, K);
#pragma unroll
            for (int q = 0; q < NP; ++q) phq[q] = t[0][q];
        }
        double G[D][D][NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            double trw = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) trw += w[q][i][i];
            const double lt = I.lam * trw;
            double Y = 0.0;                            // S : w
#pragma unroll
            for (int i = 0; i < D; ++i) {
                G[i][i][q] = gks[q] * fma(I.two_mu, w[q][i][i], lt);
                if (MODE == M_FULL) Y = fma(Sd[q][i], w[q][i][i], Y);
            }
            const double cm = gks[q] * I.mu;
            int k = 0;
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = i + 1; j < D; ++j, ++k) {
                    const double sw = w[q][i][j] + w[q][j][i];
                    const double g = cm * sw;
                    G[i][j][q] = g;
                    G[j][i][q] = g;
                    if (MODE == M_FULL) Y = fma(So[q][k], sw, Y);
                }
            if (MODE == M_FULL) {
                const double cc = RHO ? I.cc * rho[q] : I.cc;
                coup[q] = phq[q] * fma(cc, Y, I.ctr * trw);
            }
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double f[NP];
            S::template integrate<false>(f, G[i], K);
#pragma unroll
            for (int n = 0; n < NP; ++n) o[i][n] = f[n];
        }
    }
    if (MODE == M_FULL || MODE == M_PBLK) {
        const double(&cp)[NP] = cv[MODE == M_FULL ? MI::F_V + D : MI::F_V];
        double t[D + 1][NP];
        S::interp(cp, t, K);
        double f[NP];
#pragma unroll
        for (int q = 0; q < NP; ++q)
            f[q] = MODE == M_FULL ? fma(aj[q], t[0][q], coup[q]) : aj[q] * t[0][q];
        mass_transpose<D>(f, K);
        corner_laplacian<D>(cp, I.clap, I, f);
        constexpr int slot = MODE == M_FULL ? D : 0;
#pragma unroll
        for (int n = 0; n < NP; ++n) o[slot][n] = f[n];
    }
}

}  // namespace pffmg
