// Cell kernel for isotropic cells (h equal on every axis -- every BASELINE
// configuration and every reference test mesh).  Same physics as the generic
// cell_kernel in cellops.cuh (reference model.py:270-355), with the 1/h and
// JxW factors folded into per-level constants (IsoK, built on the host), the
// symmetric tensor algebra written out, gradients kept in reduced form (a
// derivative along j is constant along j) and the constant-coefficient
// k_phi Laplacian applied in closed form at the corners.
//
// With raw reference derivatives r_ij = d_j^ref U_i, w_ij = d_j^ref v_i, and
// the raw "stress" of U   S_ii = 2 mu r_ii + lam tr r,  S_ij = mu (r_ij + r_ji):
//   E+ (model.py:163-165)        = ih^2 * 1/2 S : sym(r)
//   a_phiphi (model.py:304-308)  = (1-k) rho E+ + 2 p ih tr r + Gc/eps
//   T : grad v (model.py:299-303, 350)
//                                = ih^2 rho (1-k) phi S : w + 2 p phi ih tr w
//   u-row stress (model.py:313-330)
//     G_ii = JxW ih^2 gk rho (2 mu w_ii + lam tr w),  G_ij = JxW ih^2 gk rho mu (w_ij + w_ji)
//   k_phi Laplacian (model.py:337, 353-354): sum_j (D^T D)_j (x) (B^T B)_others
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
    double cpres;          // JxW p ih                        -> residual pressure stress (times phi~^2)
    double two_mu, lam, mu;
    double lapA, lapB, lapK1;   // 2D Laplacian: out_n += A u_n + B u_{n^3} + K1 sum(u)
    double lam3[8];             // 3D Laplacian eigenvalues in the Walsh basis (scaled, / 8)
    double dlo, dhi;            // diagonal helpers: sum_q B_qa B_qb (same / different corner)
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
    I.cpres = 0.5 * K.jxw * K.two_p * K.ih[0];
    I.two_mu = 2.0 * K.mu;
    I.lam = K.lam;
    I.mu = K.mu;
    // 1D tensor factors of the Laplacian: D^T D = 2 [[1,-1],[-1,1]], B^T B = [[lo,hi],[hi,lo]]
    const double lo = K.omg0 * K.omg0 + K.omg1 * K.omg1;
    const double hi = K.omg0 * K.g0 + K.omg1 * K.g1;
    I.dlo = lo;
    I.dhi = hi;
    // 2D: K[n][m] = k_{popcount(n^m)}: k0 = 4 lo, k1 = 2 (hi - lo), k2 = -4 hi
    const double k0 = 4.0 * lo, k1 = 2.0 * (hi - lo), k2 = -4.0 * hi;
    I.lapA = I.clap * (k0 - k1);
    I.lapB = I.clap * (k2 - k1);
    I.lapK1 = I.clap * k1;
    // 3D: Walsh basis s (bit a = difference mode along a): lambda(s) =
    // sum_j [s_j] 4 prod_{a != j} (s_a ? lo - hi : lo + hi); scaled by clap / 8
    for (int s = 0; s < 8; ++s) {
        double lamv = 0.0;
        for (int j = 0; j < 3; ++j) {
            if (!((s >> j) & 1)) continue;
            double p = 4.0;
            for (int a = 0; a < 3; ++a)
                if (a != j) p *= ((s >> a) & 1) ? (lo - hi) : (lo + hi);
            lamv += p;
        }
        I.lam3[s] = I.clap * lamv * 0.125;
    }
    return I;
}

// out[n] += k_phi JxW ih^2 sum_q grad N_m . grad N_n  u_m   (Q1 cell Laplacian)
template <int D>
__device__ __forceinline__ void corner_laplacian(const double (&c)[1 << D], const IsoK& I,
                                                 double (&out)[1 << D]) {
    if (D == 2) {
        const double s = (c[0] + c[1]) + (c[2] + c[3]);
        const double ks = I.lapK1 * s;
#pragma unroll
        for (int n = 0; n < 4; ++n) out[n] = fma(I.lapA, c[n], fma(I.lapB, c[n ^ 3], out[n] + ks));
    } else {
        double t[1 << D];
#pragma unroll
        for (int i = 0; i < (1 << D); ++i) t[i] = c[i];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int i = 0; i < (1 << D); ++i) {
                if (i & (1 << a)) continue;
                const int k = i | (1 << a);
                const double u0 = t[i], u1 = t[k];
                t[i] = u0 + u1;
                t[k] = u0 - u1;
            }
        t[0] = 0.0;
#pragma unroll
        for (int s = 1; s < (1 << D); ++s) t[s] *= I.lam3[s];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int i = 0; i < (1 << D); ++i) {
                if (i & (1 << a)) continue;
                const int k = i | (1 << a);
                const double u0 = t[i], u1 = t[k];
                t[i] = u0 + u1;
                t[k] = u0 - u1;
            }
#pragma unroll
        for (int i = 0; i < (1 << D); ++i) out[i] += t[i];
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
            const double f0 = f[i], f1 = f[j], d = f1 - f0;   // symmetric Gauss points: see SFr::deriv_T
            f[i] = fma(K.g0, d, f0);
            f[j] = fma(-K.g0, d, f1);
        }
    }
}

template <int D, int MODE, bool RHO>
__device__ __forceinline__ void cell_kernel_iso(const double (&cv)[ModeInfo<D, MODE>::NF][1 << D],
                                                const double* __restrict__ rho_q, const Consts& K,
                                                const IsoK& I,
                                                double (&o)[ModeInfo<D, MODE>::NCO][1 << D]) {
    using MI = ModeInfo<D, MODE>;
    constexpr int NP = 1 << D, NR = 1 << (D - 1);
    using S = SFr<D>;

    double rho[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) rho[q] = RHO ? __ldg(rho_q + q) : 1.0;

    double gks[NP];                                 // JxW ih^2 gk rho   (model.py:282, 295)
    double pv[NP];                                  // phi_tilde at the QPs
    if (MI::PT) {
        S::value(cv[MI::F_PT], pv, K);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double g = fma(I.gk_a * pv[q], pv[q], I.gk_b);
            gks[q] = RHO ? g * rho[q] : g;
        }
    }

    // U's displacement gradient -> stress S, a_phiphi * JxW
    double Sd[NP][D], So[NP][D * (D - 1) / 2 > 0 ? D * (D - 1) / 2 : 1], aj[NP];
    if (MI::NU > 0) {
        double rr[D][D][NR];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) S::deriv(cv[MI::F_U + i], j, rr[i][j], K);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            double r[D][D];
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) r[i][j] = rr[i][j][drop_bit(q, j)];
            double dv = r[0][0];
#pragma unroll
            for (int i = 1; i < D; ++i) dv += r[i][i];
            const double ld = I.lam * dv;
            double e2 = 0.0;                           // S : sym(r) = 2 E+ / ih^2
#pragma unroll
            for (int i = 0; i < D; ++i) {
                Sd[q][i] = fma(I.two_mu, r[i][i], ld);
                e2 = fma(Sd[q][i], r[i][i], e2);
            }
            int k = 0;
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = i + 1; j < D; ++j, ++k) {
                    const double s = r[i][j] + r[j][i];
                    So[q][k] = I.mu * s;
                    e2 = fma(So[q][k], s, e2);
                }
            const double ce = RHO ? I.cS * rho[q] : I.cS;
            aj[q] = fma(ce, e2, MODE == M_RES ? I.cdiv * dv : fma(I.cdiv, dv, I.c0));
        }
    }

    if (MODE == M_RES) {
        // semilinear form A(U), NoSplit (model.py:420-460): u rows integrate
        // gk rho sigma+ + p phi~^2 I against grad N; the phi row integrates
        // (1-k) phi rho E+ + 2 p phi div u - Gc/eps (1 - phi) against N plus
        // the Gc eps Laplacian of phi.
        double G[D][D][NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double pp = I.cpres * (pv[q] * pv[q]);
#pragma unroll
            for (int i = 0; i < D; ++i) G[i][i][q] = fma(gks[q], Sd[q][i], pp);
            int k = 0;
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = i + 1; j < D; ++j, ++k) {
                    G[i][j][q] = gks[q] * So[q][k];
                    G[j][i][q] = G[i][j][q];
                }
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            S::template deriv_T<false>(G[i][0], 0, o[i], K);
#pragma unroll
            for (int j = 1; j < D; ++j) S::template deriv_T<true>(G[i][j], j, o[i], K);
        }
        const double(&cu)[NP] = cv[MI::F_U + D];
        double f[NP];
        S::value(cu, f, K);
#pragma unroll
        for (int q = 0; q < NP; ++q) f[q] = fma(f[q], aj[q], -I.c0 * (1.0 - f[q]));
        mass_transpose<D>(f, K);
        corner_laplacian<D>(cu, I, f);
#pragma unroll
        for (int n = 0; n < NP; ++n) o[D][n] = f[n];
        return;
    }

    if (MODE == M_DIAG) {
        // exact diagonal (model.py:394-413, fem.py:242-261); not hot -- plain loops
#pragma unroll
        for (int n = 0; n < NP; ++n) {
            double du[D];
#pragma unroll
            for (int i = 0; i < D; ++i) du[i] = 0.0;
            double dp = 0.0;
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
            }
#pragma unroll
            for (int i = 0; i < D; ++i) o[i][n] = du[i];
            // Laplacian diagonal: k_phi JxW ih^2 * D * 2 * lo^(D-1)
            double lap = 2.0 * D;
#pragma unroll
            for (int a = 1; a < D; ++a) lap *= I.dlo;
            o[D][n] = fma(I.clap, lap, dp);
        }
        return;
    }

    double coup[NP];
    if (MODE == M_FULL || MODE == M_UBLK) {
        double ww[D][D][NR];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) S::deriv(cv[MI::F_V + i], j, ww[i][j], K);
        double phq[NP];
        if (MODE == M_FULL) S::value(cv[MI::F_U + D], phq, K);
        double G[D][D][NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            double w[D][D];
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) w[i][j] = ww[i][j][drop_bit(q, j)];
            double trw = w[0][0];
#pragma unroll
            for (int i = 1; i < D; ++i) trw += w[i][i];
            const double lt = I.lam * trw;
            double Y = 0.0;                            // S : w
#pragma unroll
            for (int i = 0; i < D; ++i) {
                G[i][i][q] = gks[q] * fma(I.two_mu, w[i][i], lt);
                if (MODE == M_FULL) Y = fma(Sd[q][i], w[i][i], Y);
            }
            const double cm = gks[q] * I.mu;
            int k = 0;
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = i + 1; j < D; ++j, ++k) {
                    const double sw = w[i][j] + w[j][i];
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
            S::template deriv_T<false>(G[i][0], 0, o[i], K);
#pragma unroll
            for (int j = 1; j < D; ++j) S::template deriv_T<true>(G[i][j], j, o[i], K);
        }
    }
    if (MODE == M_FULL || MODE == M_PBLK) {
        const double(&cp)[NP] = cv[MODE == M_FULL ? MI::F_V + D : MI::F_V];
        double f[NP];
        S::value(cp, f, K);
#pragma unroll
        for (int q = 0; q < NP; ++q) f[q] = MODE == M_FULL ? fma(aj[q], f[q], coup[q]) : aj[q] * f[q];
        mass_transpose<D>(f, K);
        corner_laplacian<D>(cp, I, f);
        constexpr int slot = MODE == M_FULL ? D : 0;
#pragma unroll
        for (int n = 0; n < NP; ++n) o[slot][n] = f[n];
    }
}

// JxW-scaled a_phiphi of the 4 QPs of a 2D isotropic cell from the corners of
// U's displacement (cu0, cu1): the phi-block coefficient of _build_caches
// (model.py:304-308), with the exact arithmetic of cell_kernel_iso's state
// part (so a table of it reproduces the on-the-fly operator bit for bit).
template <bool RHO>
__device__ __forceinline__ void phi_coef2(const double (&cu0)[4], const double (&cu1)[4],
                                          const double* __restrict__ rho_q, const Consts& K, const IsoK& I,
                                          double (&aj)[4]) {
    constexpr int D = 2, NP = 4, NR = 2;
    using S = SFr<D>;
    double rr[D][D][NR];
#pragma unroll
    for (int j = 0; j < D; ++j) {
        S::deriv(cu0, j, rr[0][j], K);
        S::deriv(cu1, j, rr[1][j], K);
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        double r[D][D];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) r[i][j] = rr[i][j][drop_bit(q, j)];
        double dv = r[0][0];
#pragma unroll
        for (int i = 1; i < D; ++i) dv += r[i][i];
        const double ld = I.lam * dv;
        double e2 = 0.0;
#pragma unroll
        for (int i = 0; i < D; ++i) {
            const double sd = fma(I.two_mu, r[i][i], ld);
            e2 = fma(sd, r[i][i], e2);
        }
        {
            const double sv = r[0][1] + r[1][0];
            const double so = I.mu * sv;
            e2 = fma(so, sv, e2);
        }
        const double ce = RHO ? I.cS * __ldg(rho_q + q) : I.cS;
        aj[q] = fma(ce, e2, fma(I.cdiv, dv, I.c0));
    }
}

// Block-diagonal operator (FULL without G_phiu) of a 2D isotropic cell with
// the phi-block coefficient read from the per-QP table (tq[q * tstride]):
// cv = {v_0, v_1, v_phi, phi_tilde} -- U is not needed at all.  Same
// arithmetic as cell_kernel_iso<2, M_FULL> with nocoup.
template <bool RHO>
__device__ __forceinline__ void cell_bd_tab2(const double (&cv)[4][4], const double* __restrict__ rho_q,
                                             const double* __restrict__ tq, int64_t tstride, const Consts& K,
                                             const IsoK& I, double (&o)[3][4]) {
    using S = SFr<2>;
    {
        const double cu[3][4] = {{cv[0][0], cv[0][1], cv[0][2], cv[0][3]},
                                 {cv[1][0], cv[1][1], cv[1][2], cv[1][3]},
                                 {cv[3][0], cv[3][1], cv[3][2], cv[3][3]}};
        double ou[2][4];
        cell_kernel_iso<2, M_UBLK, RHO>(cu, rho_q, K, I, ou);
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int n = 0; n < 4; ++n) o[k][n] = ou[k][n];
    }
    double f[4];
    S::value(cv[2], f, K);
#pragma unroll
    for (int q = 0; q < 4; ++q) f[q] = fma(__ldg(tq + q * tstride), f[q], 0.0);
    mass_transpose<2>(f, K);
    corner_laplacian<2>(cv[2], I, f);
#pragma unroll
    for (int n = 0; n < 4; ++n) o[2][n] = f[n];
}

// Phi block of a 2D isotropic cell with a_phiphi from the per-QP table
// (same arithmetic as cell_kernel_iso<2, M_PBLK>): only v is staged.
__device__ __forceinline__ void cell_pblk_tab2(const double (&cv)[1][4], const double* __restrict__ tq,
                                               int64_t tstride, const Consts& K, const IsoK& I,
                                               double (&o)[1][4]) {
    using S = SFr<2>;
    double f[4];
    S::value(cv[0], f, K);
#pragma unroll
    for (int q = 0; q < 4; ++q) f[q] = __ldg(tq + q * tstride) * f[q];
    mass_transpose<2>(f, K);
    corner_laplacian<2>(cv[0], I, f);
#pragma unroll
    for (int n = 0; n < 4; ++n) o[0][n] = f[n];
}

}  // namespace pffmg

