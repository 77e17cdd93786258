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


// ====================================================================== 3D
// Symmetric 3x3 eigen-decomposition by cyclic Jacobi rotations: high absolute
// accuracy (|dw| ~ eps ||e||) like LAPACK's eigh.  Eigenvalue order does not
// matter below: every split quantity is symmetric in the eigen-pairs (the
// divided differences dd_ab = dd_ba), so no sort is needed.
struct Spec3 {
    double w[3];
    double n[3][3];          // n[a][i]: component i of eigenvector a
    double tr, Ep;
    double sp[6], sm[6];     // sigma+ / sigma- as (00, 11, 22, 01, 02, 12)
    double H[3], Htr, dd[3]; // dd for pairs (0,1), (0,2), (1,2)
};

template <int P, int Q, int R>
__device__ __forceinline__ void jacobi_rot(double (&a)[3][3], double (&v)[3][3]) {
    const double apq = a[P][Q];
    if (apq == 0.0) return;
    const double theta = 0.5 * (a[Q][Q] - a[P][P]) / apq;
    double t = 1.0 / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
    if (theta < 0.0) t = -t;
    const double c = 1.0 / sqrt(fma(t, t, 1.0)), s = t * c;
    a[P][P] -= t * apq;
    a[Q][Q] += t * apq;
    a[P][Q] = a[Q][P] = 0.0;
    const double arp = a[R][P], arq = a[R][Q];
    a[R][P] = a[P][R] = c * arp - s * arq;
    a[R][Q] = a[Q][R] = s * arp + c * arq;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double vp = v[k][P], vq = v[k][Q];
        v[k][P] = c * vp - s * vq;
        v[k][Q] = s * vp + c * vq;
    }
}

__device__ __forceinline__ void spectral3(const double (&e)[6], const Consts& K, Spec3& S) {
    const double band = K.band;
    double a[3][3] = {{e[0], e[3], e[4]}, {e[3], e[1], e[5]}, {e[4], e[5], e[2]}};
    double v[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
    const double fro2 = e[0] * e[0] + e[1] * e[1] + e[2] * e[2] + 2.0 * (e[3] * e[3] + e[4] * e[4] + e[5] * e[5]);
#pragma unroll 1
    for (int sweep = 0; sweep < 12; ++sweep) {
        const double off = a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2];
        if (off <= 1e-40 * fro2) break;
        jacobi_rot<0, 1, 2>(a, v);
        jacobi_rot<0, 2, 1>(a, v);
        jacobi_rot<1, 2, 0>(a, v);
    }
    double wp[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        S.w[k] = a[k][k];
#pragma unroll
        for (int i = 0; i < 3; ++i) S.n[k][i] = v[i][k];
        wp[k] = blend_pos(S.w[k], band);
        S.H[k] = blend_pos_prime(S.w[k], band);
    }
    const double tr = e[0] + e[1] + e[2];
    S.tr = tr;
    const double trp = blend_pos(tr, band);
    const double Es = 0.5 * K.lam * tr * tr + K.mu * (S.w[0] * S.w[0] + S.w[1] * S.w[1] + S.w[2] * S.w[2]);
    S.Ep = 0.5 * K.lam * blend_pos_sq(tr, band) +
           K.mu * (blend_pos_sq(S.w[0], band) + blend_pos_sq(S.w[1], band) + blend_pos_sq(S.w[2], band));
    (void)Es;
    constexpr int II[6] = {0, 1, 2, 0, 0, 1}, JJ[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int m = 0; m < 6; ++m) {
        double ep = 0.0;
#pragma unroll
        for (int k = 0; k < 3; ++k) ep = fma(wp[k] * S.n[k][II[m]], S.n[k][JJ[m]], ep);
        S.sp[m] = 2.0 * K.mu * ep + (m < 3 ? K.lam * trp : 0.0);
        S.sm[m] = 2.0 * K.mu * e[m] + (m < 3 ? K.lam * tr : 0.0) - S.sp[m];
    }
    S.Htr = blend_pos_prime(tr, band);
    const double scale = sqrt(fro2);
    constexpr int PA[3] = {0, 0, 1}, PB[3] = {1, 2, 2};
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        const double gap = S.w[PA[m]] - S.w[PB[m]];
        const bool degenerate = fabs(gap) < 1e-8 * fmax(scale, 1e-300);   // model.py:203-209
        S.dd[m] = degenerate ? 0.5 * (S.H[PA[m]] + S.H[PB[m]]) : (wp[PA[m]] - wp[PB[m]]) / gap;
    }
}

// out = dsig+ : eps (both as (00, 11, 22, 01, 02, 12))
__device__ __forceinline__ void tangent_action3(const Spec3& S, const Consts& K, const double (&ep)[6],
                                                double (&out)[6]) {
    constexpr int II[6] = {0, 1, 2, 0, 0, 1}, JJ[6] = {0, 1, 2, 1, 2, 2};
    double en[3][3];   // en[b] = eps n_b
#pragma unroll
    for (int b = 0; b < 3; ++b) {
        en[b][0] = ep[0] * S.n[b][0] + ep[3] * S.n[b][1] + ep[4] * S.n[b][2];
        en[b][1] = ep[3] * S.n[b][0] + ep[1] * S.n[b][1] + ep[5] * S.n[b][2];
        en[b][2] = ep[4] * S.n[b][0] + ep[5] * S.n[b][1] + ep[2] * S.n[b][2];
    }
    double c[3], cp[3];
    constexpr int PA[3] = {0, 0, 1}, PB[3] = {1, 2, 2};
#pragma unroll
    for (int a = 0; a < 3; ++a)
        c[a] = S.H[a] * (S.n[a][0] * en[a][0] + S.n[a][1] * en[a][1] + S.n[a][2] * en[a][2]);
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        const int a = PA[m], b = PB[m];
        cp[m] = 2.0 * S.dd[m] * (S.n[a][0] * en[b][0] + S.n[a][1] * en[b][1] + S.n[a][2] * en[b][2]);
    }
    const double l = K.lam * S.Htr * (ep[0] + ep[1] + ep[2]);
#pragma unroll
    for (int m = 0; m < 6; ++m) {
        const int i = II[m], j = JJ[m];
        double t = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) t = fma(c[a] * S.n[a][i], S.n[a][j], t);
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            const int a = PA[p], b = PB[p];
            t = fma(cp[p], 0.5 * (S.n[a][i] * S.n[b][j] + S.n[b][i] * S.n[a][j]), t);
        }
        out[m] = 2.0 * K.mu * t + (m < 3 ? l : 0.0);
    }
}

// Value and physical gradient of one Q1 field at a single QP (b[a][k]: 1D
// basis weight of corner bit k along axis a at this QP).
__device__ __forceinline__ void qp_eval3(const double (&c)[8], const double (&b)[3][2], const Consts& K,
                                         double& val, double (&g)[3]) {
    double vx[4], dx[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        vx[r] = b[0][0] * c[2 * r] + b[0][1] * c[2 * r + 1];
        dx[r] = c[2 * r + 1] - c[2 * r];
    }
    double vxy[2], dxy[2], dy[2];
#pragma unroll
    for (int z = 0; z < 2; ++z) {
        vxy[z] = b[1][0] * vx[2 * z] + b[1][1] * vx[2 * z + 1];
        dxy[z] = b[1][0] * dx[2 * z] + b[1][1] * dx[2 * z + 1];
        dy[z] = vx[2 * z + 1] - vx[2 * z];
    }
    val = b[2][0] * vxy[0] + b[2][1] * vxy[1];
    g[0] = (b[2][0] * dxy[0] + b[2][1] * dxy[1]) * K.ih[0];
    g[1] = (b[2][0] * dy[0] + b[2][1] * dy[1]) * K.ih[1];
    g[2] = (vxy[1] - vxy[0]) * K.ih[2];
}

// Adjoint of qp_eval3: o[n] += f N_n(q) + sum_a g[a] dN_n/dx_a(q)
__device__ __forceinline__ void qp_scatter3(double f, const double (&gin)[3], const double (&b)[3][2],
                                            const Consts& K, double (&o)[8]) {
    const double gx = gin[0] * K.ih[0], gy = gin[1] * K.ih[1], gz = gin[2] * K.ih[2];
    double Avxy[2], Adxy[2], Ady[2];
#pragma unroll
    for (int z = 0; z < 2; ++z) {
        Avxy[z] = b[2][z] * f + (z ? gz : -gz);
        Adxy[z] = b[2][z] * gx;
        Ady[z] = b[2][z] * gy;
    }
    double Avx[4], Adx[4];
#pragma unroll
    for (int z = 0; z < 2; ++z)
#pragma unroll
        for (int y = 0; y < 2; ++y) {
            Avx[2 * z + y] = b[1][y] * Avxy[z] + (y ? Ady[z] : -Ady[z]);
            Adx[2 * z + y] = b[1][y] * Adxy[z];
        }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int x = 0; x < 2; ++x) o[2 * r + x] += b[0][x] * Avx[r] + (x ? Adx[r] : -Adx[r]);
}

template <int MODE>
__device__ __forceinline__ void cell_kernel_miehe3(const double (&cv)[ModeInfo<3, MODE, true>::NF][8],
                                                   const double* __restrict__ rho_q, const Consts& K,
                                                   double (&o)[ModeInfo<3, MODE, true>::NCO][8]) {
    constexpr int D = 3, NP = 8;
    using MI = ModeInfo<D, MODE, true>;
#pragma unroll
    for (int k = 0; k < MI::NCO; ++k)
#pragma unroll
        for (int n = 0; n < NP; ++n) o[k][n] = 0.0;
    const double p = 0.5 * K.two_p;
#pragma unroll 1
    for (int q = 0; q < NP; ++q) {
        double b[3][2];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int qb = (q >> a) & 1;
            b[a][0] = qb ? K.omg1 : K.omg0;
            b[a][1] = qb ? K.g1 : K.g0;
        }
        const double rho = rho_q ? __ldg(rho_q + q) : 1.0;
        // strain of the linearisation state
        double gu[3][3], val;
#pragma unroll
        for (int i = 0; i < 3; ++i) qp_eval3(cv[MI::F_U + i], b, K, val, gu[i]);
        double e[6] = {gu[0][0], gu[1][1], gu[2][2], 0.5 * (gu[0][1] + gu[1][0]), 0.5 * (gu[0][2] + gu[2][0]),
                       0.5 * (gu[1][2] + gu[2][1])};
        Spec3 S;
        spectral3(e, K, S);
        double gk = 0.0, ptq = 0.0;
        if (MI::PT) {
            double gd[3];
            qp_eval3(cv[MI::F_PT], b, K, ptq, gd);
            gk = K.omk * (ptq * ptq) + K.kappa;
        }
        constexpr int II[6] = {0, 1, 2, 0, 0, 1}, JJ[6] = {0, 1, 2, 1, 2, 2};
        auto sym = [](const double (&s)[6], int i, int j) -> double {
            return i == j ? s[i] : s[i + j + 2];   // (0,1)->3, (0,2)->4, (1,2)->5
        };

        if (MODE == M_DIAG) {
            const double am = K.omk * rho * S.Ep + K.two_p * S.tr + K.gc_over_eps;
            const double gm = (gk - 1.0) * rho;
#pragma unroll
            for (int n = 0; n < NP; ++n) {
                double Nv = 1.0;
#pragma unroll
                for (int a = 0; a < 3; ++a) Nv *= b[a][(n >> a) & 1];
                double gN[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    double t = ((n >> a) & 1) ? K.ih[a] : -K.ih[a];
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        if (c != a) t *= b[c][(n >> c) & 1];
                    gN[a] = t;
                }
                const double gg = gN[0] * gN[0] + gN[1] * gN[1] + gN[2] * gN[2];
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    double E[6];
#pragma unroll
                    for (int m = 0; m < 6; ++m) {
                        const int a = II[m], c = JJ[m];
                        E[m] = (a == c) ? (a == i ? gN[i] : 0.0)
                                        : (a == i ? 0.5 * gN[c] : (c == i ? 0.5 * gN[a] : 0.0));
                    }
                    double T[6];
                    tangent_action3(S, K, E, T);
                    const double edde = T[0] * E[0] + T[1] * E[1] + T[2] * E[2] +
                                        2.0 * (T[3] * E[3] + T[4] * E[4] + T[5] * E[5]);
                    const double iso = K.mu * gg + (K.mu + K.lam) * (gN[i] * gN[i]);
                    o[i][n] += K.jxw * (rho * iso + gm * edde);
                }
                o[D][n] += K.jxw * (am * (Nv * Nv)) + K.k_phi * (K.jxw * gg);
            }
            continue;
        }
        if (MODE == M_RES) {
            double ph, gph[3];
            qp_eval3(cv[MI::F_U + D], b, K, ph, gph);
            const double pp = ptq * ptq * p;
            double s6[6];
#pragma unroll
            for (int m = 0; m < 6; ++m) s6[m] = gk * rho * S.sp[m] + rho * S.sm[m] + (m < 3 ? pp : 0.0);
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                double g[3];
#pragma unroll
                for (int j = 0; j < 3; ++j) g[j] = K.jxw * sym(s6, i, j);
                qp_scatter3(0.0, g, b, K, o[i]);
            }
            const double f = K.jxw * (K.omk * ph * rho * S.Ep + K.two_p * ph * S.tr - K.gc_over_eps * (1.0 - ph));
            double g[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) g[j] = K.jxw * K.k_phi * gph[j];
            qp_scatter3(f, g, b, K, o[D]);
            continue;
        }
        constexpr bool HAS_U = MODE == M_FULL || MODE == M_UBLK;
        constexpr bool HAS_P = MODE == M_FULL || MODE == M_PBLK;
        double coup = 0.0;
        if (HAS_U) {
            double gv[3][3];
#pragma unroll
            for (int i = 0; i < 3; ++i) qp_eval3(cv[MI::F_V + i], b, K, val, gv[i]);
            double ev[6] = {gv[0][0], gv[1][1], gv[2][2], 0.5 * (gv[0][1] + gv[1][0]),
                            0.5 * (gv[0][2] + gv[2][0]), 0.5 * (gv[1][2] + gv[2][1])};
            double T[6];
            tangent_action3(S, K, ev, T);
            const double tre = ev[0] + ev[1] + ev[2], gm = (gk - 1.0) * rho;   // model.py:321-323
            double s6[6];
#pragma unroll
            for (int m = 0; m < 6; ++m) s6[m] = rho * (2.0 * K.mu * ev[m] + (m < 3 ? K.lam * tre : 0.0)) + gm * T[m];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                double g[3];
#pragma unroll
                for (int j = 0; j < 3; ++j) g[j] = K.jxw * sym(s6, i, j);
                qp_scatter3(0.0, g, b, K, o[i]);
            }
            if (MODE == M_FULL) {
                double phq, gd[3];
                qp_eval3(cv[MI::F_U + D], b, K, phq, gd);
                const double cph = rho * K.omk * phq;
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        coup += (cph * sym(S.sp, i, j) + (i == j ? K.two_p * phq : 0.0)) * gv[i][j];
            }
        }
        if (HAS_P) {
            double vp, gvp[3];
            qp_eval3(cv[MODE == M_FULL ? MI::F_V + D : MI::F_V], b, K, vp, gvp);
            const double a = K.omk * rho * S.Ep + K.two_p * S.tr + K.gc_over_eps;   // model.py:304-308
            double g[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) g[j] = K.jxw * K.k_phi * gvp[j];
            qp_scatter3(K.jxw * (coup + a * vp), g, b, K, o[MODE == M_FULL ? D : 0]);
        }
    }
}

}  // namespace pffmg
