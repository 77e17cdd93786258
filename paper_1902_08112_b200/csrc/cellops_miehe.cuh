// 2D cell kernel with the Miehe spectral tensile/compressive split and its
// C^1 blend (reference model.py:56-86, 148-219; operator model.py:270-413;
// residual model.py:420-460).  General box cells, physical gradients.
//
// Per quadrature point the strain e(U) of the linearisation state is
// diagonalised in closed form (2x2 symmetric), giving eigenvalues w0 <= w1
// (ascending, as numpy.linalg.eigh) and projectors M_a = n_a n_a^T.  The
// fourth-order tangent dsig+ of _split_batch is never formed: only its action
// on an increment strain is needed,
//   dsig+ : eps = lam H(tr e) tr(eps) I
//               + 2 mu [ H(w0) eps'_00 M0 + H(w1) eps'_11 M1 + 2 dd eps'_01 S01 ],
// with eps'_ab = n_a^T eps n_b, S01 = sym(n0 n1^T) and dd the divided
// difference (wp0 - wp1)/(w0 - w1) or its degenerate-gap limit (model.py:198-213).
#pragma once

#include "cellops.cuh"

namespace pffmg {

__device__ __forceinline__ double blend_pos(double x, double band) {        // model.py:65-70
    if (band <= 0.0) return fmax(x, 0.0);
    if (x >= band) return x;
    if (x <= -band) return 0.0;
    return (x + band) * (x + band) / (4.0 * band);
}
__device__ __forceinline__ double blend_pos_prime(double x, double band) {  // model.py:73-77
    if (band <= 0.0) return x > 0.0 ? 1.0 : 0.0;
    if (x >= band) return 1.0;
    if (x <= -band) return 0.0;
    return (x + band) / (2.0 * band);
}
__device__ __forceinline__ double blend_pos_sq(double x, double band) {     // model.py:80-86
    if (band <= 0.0) {
        const double p = fmax(x, 0.0);
        return p * p;
    }
    if (x >= band) return x * x + band * band / 3.0;
    if (x <= -band) return 0.0;
    const double t = x + band;
    return t * t * t / (6.0 * band);
}

// Spectral data of one 2x2 symmetric strain (model.py:174-219).
struct Spec2 {
    double w0, w1;          // eigenvalues, ascending
    double n0x, n0y, n1x, n1y;
    double tr, Ep, Em;      // trace, E+, E-
    double sp[2][2];        // sigma+
    double sm[2][2];        // sigma-
    double H0, H1, Htr, dd; // tangent coefficients
};

__device__ __forceinline__ void spectral2(double a, double b, double c, const Consts& K, Spec2& S) {
    const double band = K.band;
    const double hd = 0.5 * (a - c), mid = 0.5 * (a + c);
    const double rad = hypot(hd, b);
    S.w0 = mid - rad;
    S.w1 = mid + rad;
    // eigenvector of w1 from the better-conditioned row of (e - w1 I)
    double vx, vy;
    if (rad == 0.0) {
        vx = 1.0;
        vy = 0.0;
    } else if (a >= c) {
        vx = S.w1 - c;
        vy = b;
    } else {
        vx = b;
        vy = S.w1 - a;
    }
    const double inv = 1.0 / sqrt(vx * vx + vy * vy);
    S.n1x = vx * inv;
    S.n1y = vy * inv;
    S.n0x = -S.n1y;
    S.n0y = S.n1x;
    const double tr = a + c;
    S.tr = tr;
    const double wp0 = blend_pos(S.w0, band), wp1 = blend_pos(S.w1, band), trp = blend_pos(tr, band);
    const double Es = 0.5 * K.lam * tr * tr + K.mu * (S.w0 * S.w0 + S.w1 * S.w1);
    S.Ep = 0.5 * K.lam * blend_pos_sq(tr, band) + K.mu * (blend_pos_sq(S.w0, band) + blend_pos_sq(S.w1, band));
    S.Em = Es - S.Ep;
    // e+ = wp0 M0 + wp1 M1;  sigma+ = 2 mu e+ + lam trp I;  sigma- = sigma - sigma+
    const double ep00 = wp0 * S.n0x * S.n0x + wp1 * S.n1x * S.n1x;
    const double ep01 = wp0 * S.n0x * S.n0y + wp1 * S.n1x * S.n1y;
    const double ep11 = wp0 * S.n0y * S.n0y + wp1 * S.n1y * S.n1y;
    S.sp[0][0] = 2.0 * K.mu * ep00 + K.lam * trp;
    S.sp[1][1] = 2.0 * K.mu * ep11 + K.lam * trp;
    S.sp[0][1] = S.sp[1][0] = 2.0 * K.mu * ep01;
    S.sm[0][0] = 2.0 * K.mu * a + K.lam * tr - S.sp[0][0];
    S.sm[1][1] = 2.0 * K.mu * c + K.lam * tr - S.sp[1][1];
    S.sm[0][1] = S.sm[1][0] = 2.0 * K.mu * b - S.sp[0][1];
    S.H0 = blend_pos_prime(S.w0, band);
    S.H1 = blend_pos_prime(S.w1, band);
    S.Htr = blend_pos_prime(tr, band);
    const double scale = sqrt(a * a + 2.0 * b * b + c * c);
    const double gap = S.w0 - S.w1;
    const bool degenerate = fabs(gap) < 1e-8 * fmax(scale, 1e-300);     // _EIG_GAP_TOL, model.py:48
    S.dd = degenerate ? 0.5 * (S.H0 + S.H1) : (wp0 - wp1) / gap;
}

// dsig+ : eps for a symmetric increment (e00, e01, e11)
__device__ __forceinline__ void tangent_action(const Spec2& S, const Consts& K, double e00, double e01,
                                               double e11, double (&out)[2][2]) {
    const double p00 = S.n0x * (S.n0x * e00 + S.n0y * e01) + S.n0y * (S.n0x * e01 + S.n0y * e11);
    const double p11 = S.n1x * (S.n1x * e00 + S.n1y * e01) + S.n1y * (S.n1x * e01 + S.n1y * e11);
    const double p01 = S.n0x * (S.n1x * e00 + S.n1y * e01) + S.n0y * (S.n1x * e01 + S.n1y * e11);
    const double c0 = S.H0 * p00, c1 = S.H1 * p11, c2 = 2.0 * S.dd * p01;
    const double l = K.lam * S.Htr * (e00 + e11);
    out[0][0] = l + 2.0 * K.mu * (c0 * S.n0x * S.n0x + c1 * S.n1x * S.n1x + c2 * S.n0x * S.n1x);
    out[1][1] = l + 2.0 * K.mu * (c0 * S.n0y * S.n0y + c1 * S.n1y * S.n1y + c2 * S.n0y * S.n1y);
    out[0][1] = out[1][0] = 2.0 * K.mu * (c0 * S.n0x * S.n0y + c1 * S.n1x * S.n1y +
                                          c2 * 0.5 * (S.n0x * S.n1y + S.n1x * S.n0y));
}

// Physical-coordinate corner gradient factor of basis n at QP q, axis a
// (fem.py:44-60 restated for the 2-point rule): gN = +/- ih[a] * B_other.
__device__ __forceinline__ double q1_shape(const Consts& K, int n, int q, int a) {
    const int nb = (n >> a) & 1, qb = (q >> a) & 1;
    return nb ? (qb ? K.g1 : K.g0) : (qb ? K.omg1 : K.omg0);
}

template <int MODE>
__device__ __forceinline__ void cell_kernel_miehe2(const double (&cv)[ModeInfo<2, MODE, true>::NF][4],
                                                   const double* __restrict__ rho_q, const Consts& K,
                                                   double (&o)[ModeInfo<2, MODE, true>::NCO][4]) {
    constexpr int D = 2, NP = 4;
    using MI = ModeInfo<D, MODE, true>;
    using S = SF<D>;
    // strain of the linearisation state at the QPs (physical gradients)
    double ea[NP], eb[NP], ec[NP];
    {
        double g0[D + 1][NP], g1[D + 1][NP];
        S::interp(cv[MI::F_U + 0], g0, K, false);
        S::interp(cv[MI::F_U + 1], g1, K, false);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            ea[q] = g0[1][q] * K.ih[0];
            ec[q] = g1[2][q] * K.ih[1];
            eb[q] = 0.5 * (g0[2][q] * K.ih[1] + g1[1][q] * K.ih[0]);
        }
    }
    double gk[NP];
    if (MI::PT) {
        double t[D + 1][NP];
        S::interp(cv[MI::F_PT], t, K);
#pragma unroll
        for (int q = 0; q < NP; ++q) gk[q] = K.omk * (t[0][q] * t[0][q]) + K.kappa;   // model.py:135-137
    }

    if (MODE == M_DIAG) {
        // du = sum_q JxW [rho (2 mu e2 + lam tr^2) + (gk-1) rho E:dsig+:E], E = sym(e_i (x) gradN)
        // dphi = sum_q JxW a N^2 + k_phi JxW |gradN|^2            (model.py:394-413)
        double du[D][NP], dp[NP];
#pragma unroll
        for (int n = 0; n < NP; ++n) du[0][n] = du[1][n] = dp[n] = 0.0;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double rho = rho_q ? __ldg(rho_q + q) : 1.0;
            Spec2 sq;
            spectral2(ea[q], eb[q], ec[q], K, sq);
            const double am = K.omk * rho * sq.Ep + K.two_p * (ea[q] + ec[q]) + K.gc_over_eps;
            const double gm = (gk[q] - 1.0) * rho;
#pragma unroll
            for (int n = 0; n < NP; ++n) {
                const double gN0 = (((n >> 0) & 1) ? K.ih[0] : -K.ih[0]) * q1_shape(K, n, q, 1);
                const double gN1 = (((n >> 1) & 1) ? K.ih[1] : -K.ih[1]) * q1_shape(K, n, q, 0);
                const double Nv = q1_shape(K, n, q, 0) * q1_shape(K, n, q, 1);
                const double gg = gN0 * gN0 + gN1 * gN1;
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    const double gi = i == 0 ? gN0 : gN1, gj = i == 0 ? gN1 : gN0;
                    const double e00 = i == 0 ? gi : 0.0, e11 = i == 1 ? gi : 0.0, e01 = 0.5 * gj;
                    double T[2][2];
                    tangent_action(sq, K, e00, e01, e11, T);
                    const double edde = T[0][0] * e00 + 2.0 * T[0][1] * e01 + T[1][1] * e11;
                    const double iso = K.mu * gg + (K.mu + K.lam) * (gi * gi);
                    du[i][n] += K.jxw * (rho * iso + gm * edde);
                }
                dp[n] += K.jxw * (am * (Nv * Nv)) + K.k_phi * (K.jxw * gg);
            }
        }
#pragma unroll
        for (int n = 0; n < NP; ++n) {
            o[0][n] = du[0][n];
            o[1][n] = du[1][n];
            o[D][n] = dp[n];
        }
        return;
    }

    double G[D][D][NP], f[NP], g[D][NP];
    if (MODE == M_RES) {
        // stress = gk rho sigma+ + rho sigma- + phi~^2 p I ; vphi of model.py:450-452
        double ph[D + 1][NP], pt[D + 1][NP];
        S::interp(cv[MI::F_U + D], ph, K);
        S::interp(cv[MI::F_PT], pt, K);
        const double p = 0.5 * K.two_p;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double rho = rho_q ? __ldg(rho_q + q) : 1.0;
            Spec2 sq;
            spectral2(ea[q], eb[q], ec[q], K, sq);
            const double pp = pt[0][q] * pt[0][q] * p;
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    const double s = gk[q] * rho * sq.sp[i][j] + rho * sq.sm[i][j] + (i == j ? pp : 0.0);
                    G[i][j][q] = K.jxw * s * K.ih[j];
                }
            const double phi = ph[0][q];
            f[q] = K.jxw * (K.omk * phi * rho * sq.Ep + K.two_p * phi * sq.tr - K.gc_over_eps * (1.0 - phi));
#pragma unroll
            for (int j = 0; j < D; ++j) g[j][q] = K.jxw * K.k_phi * (ph[1 + j][q] * K.ih[j]) * K.ih[j];
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

    constexpr bool HAS_U = MODE == M_FULL || MODE == M_UBLK;
    constexpr bool HAS_P = MODE == M_FULL || MODE == M_PBLK;
    double gv0[D + 1][NP], gv1[D + 1][NP], tp[D + 1][NP], phq[NP];
    if (HAS_U) {
        S::interp(cv[MI::F_V + 0], gv0, K, false);
        S::interp(cv[MI::F_V + 1], gv1, K, false);
    }
    if (HAS_P) S::interp(cv[MODE == M_FULL ? MI::F_V + D : MI::F_V], tp, K);
    if (MODE == M_FULL) {
        double t[D + 1][NP];
        S::interp(cv[MI::F_U + D], t, K);
#pragma unroll
        for (int q = 0; q < NP; ++q) phq[q] = t[0][q];
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const double rho = rho_q ? __ldg(rho_q + q) : 1.0;
        Spec2 sq;
        spectral2(ea[q], eb[q], ec[q], K, sq);
        double coup = 0.0;
        if (HAS_U) {
            const double w00 = gv0[1][q] * K.ih[0], w01 = gv0[2][q] * K.ih[1];
            const double w10 = gv1[1][q] * K.ih[0], w11 = gv1[2][q] * K.ih[1];
            const double e00 = w00, e11 = w11, e01 = 0.5 * (w01 + w10), tre = e00 + e11;
            double T[2][2];
            tangent_action(sq, K, e00, e01, e11, T);
            // model.py:321-323: rho iso(e) + (gk - 1) rho dsig+:e
            const double gm = (gk[q] - 1.0) * rho;
            const double s00 = rho * (2.0 * K.mu * e00 + K.lam * tre) + gm * T[0][0];
            const double s11 = rho * (2.0 * K.mu * e11 + K.lam * tre) + gm * T[1][1];
            const double s01 = rho * (2.0 * K.mu * e01) + gm * T[0][1];
            G[0][0][q] = K.jxw * s00 * K.ih[0];
            G[0][1][q] = K.jxw * s01 * K.ih[1];
            G[1][0][q] = K.jxw * s01 * K.ih[0];
            G[1][1][q] = K.jxw * s11 * K.ih[1];
            if (MODE == M_FULL) {
                // T = rho (1-k) phi sigma+ + 2 p phi I ; coupling T : grad v (model.py:299-303, 350)
                const double cph = rho * K.omk * phq[q];
                const double t00 = cph * sq.sp[0][0] + K.two_p * phq[q];
                const double t11 = cph * sq.sp[1][1] + K.two_p * phq[q];
                const double t01 = cph * sq.sp[0][1];
                coup = t00 * w00 + t01 * (w01 + w10) + t11 * w11;
            }
        }
        if (HAS_P) {
            const double a = K.omk * rho * sq.Ep + K.two_p * sq.tr + K.gc_over_eps;   // model.py:304-308
            f[q] = K.jxw * (coup + a * tp[0][q]);
#pragma unroll
            for (int j = 0; j < D; ++j) g[j][q] = K.jxw * K.k_phi * (tp[1 + j][q] * K.ih[j]) * K.ih[j];
        }
    }
    if (HAS_U) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double t[NP];
            S::template integrate<false>(t, G[i], K);
#pragma unroll
            for (int n = 0; n < NP; ++n) o[i][n] = t[n];
        }
    }
    if (HAS_P) {
        S::template integrate<true>(f, g, K);
#pragma unroll
        for (int n = 0; n < NP; ++n) o[MODE == M_FULL ? D : 0][n] = f[n];
    }
}

}  // namespace pffmg
