// Biquadratic (Q2, 9-node) cell physics for BASELINE configs[2]: the
// reference's operator / residual / diagonal (model.py:270-460) with the
// reference element replaced by Q2 and the 3x3 Gauss rule.  The reference
// has no Q2 element; the definitions follow oracle/q2.py (nodes a + 3b,
// x fastest; QPs qx + 3 qy).  Per QP the nine-node field values and
// gradients are evaluated by sum factorisation (x pass per node row, then y),
// the pointwise physics is the generic NoSplit / Miehe code, and the
// integration is the transposed pass.
#pragma once

#ifndef PFFMG_Q2_UNROLL_QY
#define PFFMG_Q2_UNROLL_QY 1
#endif

#include "cellops_miehe.cuh"

namespace pffmg {

struct Q2Tab {
    double B[3][3];   // B[q][a]: 1D Lagrange basis a on {0, 1/2, 1} at Gauss point q
    double D[3][3];   // reference derivatives
    double w[3];      // Gauss weights (5, 8, 5) / 18
    double vol;       // cell volume
    // folded on the host (the kernels use them as constant-bank operands
    // instead of re-multiplying in registers): physical derivatives and JxW
    double Dx[3][3], Dy[3][3];   // D / hx, D / hy
    double W[3][3];              // W[qy][qx] = (w[qy] vol) w[qx]
};

inline Q2Tab make_q2_host(double hx, double hy) {
    Q2Tab T;
    const double g[3] = {0.5 - 0.5 * 0.7745966692414834, 0.5, 0.5 + 0.5 * 0.7745966692414834};
    for (int q = 0; q < 3; ++q) {
        const double t = g[q];
        T.B[q][0] = 2.0 * (t - 0.5) * (t - 1.0);
        T.B[q][1] = -4.0 * t * (t - 1.0);
        T.B[q][2] = 2.0 * t * (t - 0.5);
        T.D[q][0] = 4.0 * t - 3.0;
        T.D[q][1] = -8.0 * t + 4.0;
        T.D[q][2] = 4.0 * t - 1.0;
    }
    T.w[0] = 5.0 / 18.0;
    T.w[1] = 8.0 / 18.0;
    T.w[2] = 5.0 / 18.0;
    T.vol = hx * hy;
    for (int q = 0; q < 3; ++q)
        for (int a = 0; a < 3; ++a) {
            T.Dx[q][a] = T.D[q][a] * (1.0 / hx);
            T.Dy[q][a] = T.D[q][a] * (1.0 / hy);
            T.W[q][a] = (T.w[q] * T.vol) * T.w[a];   // the row kernel's order: (w_qy vol) w_qx
        }
    return T;
}

struct Q2Point {
    double Bx[3], Dx[3], By[3], Dy[3];   // D already scaled by 1/h
    // value and physical gradient of a nine-node field at this QP
    __device__ __forceinline__ void eval(const double (&c)[9], double& val, double& gx, double& gy) const {
        double vx[3], dx[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            vx[b] = fma(Bx[0], c[3 * b], fma(Bx[1], c[3 * b + 1], Bx[2] * c[3 * b + 2]));
            dx[b] = fma(Dx[0], c[3 * b], fma(Dx[1], c[3 * b + 1], Dx[2] * c[3 * b + 2]));
        }
        val = fma(By[0], vx[0], fma(By[1], vx[1], By[2] * vx[2]));
        gx = fma(By[0], dx[0], fma(By[1], dx[1], By[2] * dx[2]));
        gy = fma(Dy[0], vx[0], fma(Dy[1], vx[1], Dy[2] * vx[2]));
    }
    // out[n] += f N_n + gx dN_n/dx + gy dN_n/dy
    __device__ __forceinline__ void scatter(double f, double gx, double gy, double (&out)[9]) const {
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const double r0 = fma(By[b], f, Dy[b] * gy), r1 = By[b] * gx;
#pragma unroll
            for (int a = 0; a < 3; ++a) out[3 * b + a] = fma(Bx[a], r0, fma(Dx[a], r1, out[3 * b + a]));
        }
    }
};

// NoSplit energy / stress of a 2x2 strain (model.py:160-172)
__device__ __forceinline__ void nosplit2(double a, double b, double c, const Consts& K, double& Ep,
                                         double (&sp)[2][2]) {
    const double tr = a + c;
    Ep = 0.5 * K.lam * tr * tr + K.mu * (a * a + 2.0 * b * b + c * c);
    sp[0][0] = 2.0 * K.mu * a + K.lam * tr;
    sp[1][1] = 2.0 * K.mu * c + K.lam * tr;
    sp[0][1] = sp[1][0] = 2.0 * K.mu * b;
}

template <int MODE, bool MIE>
__device__ __forceinline__ void cell_q2(const double (&cv)[ModeInfo<2, MODE, MIE>::NF][9],
                                        const double* __restrict__ rho_q, const Consts& K, const Q2Tab& T,
                                        double (&o)[ModeInfo<2, MODE, MIE>::NCO][9]) {
    using MI = ModeInfo<2, MODE, MIE>;
    constexpr int NCO = MI::NCO;
#pragma unroll
    for (int k = 0; k < NCO; ++k)
#pragma unroll
        for (int n = 0; n < 9; ++n) o[k][n] = 0.0;
#pragma unroll 1
    for (int q = 0; q < 9; ++q) {
        const int qx = q % 3, qy = q / 3;
        Q2Point P;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            P.Bx[a] = T.B[qx][a];
            P.Dx[a] = T.D[qx][a] * K.ih[0];
            P.By[a] = T.B[qy][a];
            P.Dy[a] = T.D[qy][a] * K.ih[1];
        }
        const double jxw = T.w[qx] * T.w[qy] * T.vol;
        const double rho = rho_q ? __ldg(rho_q + q) : 1.0;
        double val;
        // strain of the linearisation state (all modes but the u block of NoSplit)
        double ea = 0.0, eb = 0.0, ec = 0.0;
        if (MI::NU >= 2) {
            double g0[2], g1[2];
            P.eval(cv[MI::F_U + 0], val, g0[0], g0[1]);
            P.eval(cv[MI::F_U + 1], val, g1[0], g1[1]);
            ea = g0[0];
            ec = g1[1];
            eb = 0.5 * (g0[1] + g1[0]);
        }
        double gk = 0.0, ptq = 0.0;
        if (MI::PT) {
            double gx, gy;
            P.eval(cv[MI::F_PT], ptq, gx, gy);
            gk = fma(K.omk, ptq * ptq, K.kappa);                       // model.py:135-137
        }
        // split data of the state strain
        double Ep = 0.0, Em = 0.0, sp[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, sm[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        Spec2 S;
        if (MI::NU >= 2) {
            if (MIE) {
                spectral2(ea, eb, ec, K, S);
                Ep = S.Ep;
                Em = S.Em;
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        sp[i][j] = S.sp[i][j];
                        sm[i][j] = S.sm[i][j];
                    }
            } else {
                nosplit2(ea, eb, ec, K, Ep, sp);
            }
        }
        const double div = ea + ec;

        if (MODE == M_DIAG) {                                          // model.py:394-413
            const double am = K.omk * rho * Ep + K.two_p * div + K.gc_over_eps;
#pragma unroll
            for (int n = 0; n < 9; ++n) {
                const int a = n % 3, b = n / 3;
                const double Nv = P.Bx[a] * P.By[b];
                const double gN0 = P.Dx[a] * P.By[b], gN1 = P.Bx[a] * P.Dy[b];
                const double gg = gN0 * gN0 + gN1 * gN1;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const double gi = i == 0 ? gN0 : gN1;
                    const double iso = K.mu * gg + (K.mu + K.lam) * (gi * gi);
                    double du;
                    if (MIE) {
                        const double e00 = i == 0 ? gi : 0.0, e11 = i == 1 ? gi : 0.0;
                        const double e01 = 0.5 * (i == 0 ? gN1 : gN0);
                        double Tn[2][2];
                        tangent_action(S, K, e00, e01, e11, Tn);
                        const double edde = Tn[0][0] * e00 + 2.0 * Tn[0][1] * e01 + Tn[1][1] * e11;
                        du = rho * iso + (gk - 1.0) * rho * edde;
                    } else {
                        du = gk * rho * iso;
                    }
                    o[i][n] = fma(jxw, du, o[i][n]);
                }
                o[2][n] = fma(jxw, am * (Nv * Nv) + K.k_phi * gg, o[2][n]);
            }
            continue;
        }

        if (MODE == M_RES) {                                           // model.py:420-460
            double ph, gph[2];
            P.eval(cv[MI::F_U + 2], ph, gph[0], gph[1]);
            const double pp = ptq * ptq * (0.5 * K.two_p);
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                double g[2];
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    g[j] = jxw * (gk * rho * sp[i][j] + rho * sm[i][j] + (i == j ? pp : 0.0));
                P.scatter(0.0, g[0], g[1], o[i]);
            }
            const double f = jxw * (K.omk * ph * rho * Ep + K.two_p * ph * div - K.gc_over_eps * (1.0 - ph));
            P.scatter(f, jxw * K.k_phi * gph[0], jxw * K.k_phi * gph[1], o[2]);
            continue;
        }

        constexpr bool HAS_U = MODE == M_FULL || MODE == M_UBLK;
        constexpr bool HAS_P = MODE == M_FULL || MODE == M_PBLK;
        double coup = 0.0;
        if (HAS_U) {
            double w[2][2];
            P.eval(cv[MI::F_V + 0], val, w[0][0], w[0][1]);
            P.eval(cv[MI::F_V + 1], val, w[1][0], w[1][1]);
            const double e00 = w[0][0], e11 = w[1][1], e01 = 0.5 * (w[0][1] + w[1][0]), tre = e00 + e11;
            double s[2][2];
            if (MIE) {                                                 // model.py:321-323
                double Tn[2][2];
                tangent_action(S, K, e00, e01, e11, Tn);
                const double gm = (gk - 1.0) * rho;
                s[0][0] = rho * (2.0 * K.mu * e00 + K.lam * tre) + gm * Tn[0][0];
                s[1][1] = rho * (2.0 * K.mu * e11 + K.lam * tre) + gm * Tn[1][1];
                s[0][1] = s[1][0] = rho * (2.0 * K.mu * e01) + gm * Tn[0][1];
            } else {                                                   // model.py:316-319
                const double g = gk * rho;
                s[0][0] = g * (2.0 * K.mu * e00 + K.lam * tre);
                s[1][1] = g * (2.0 * K.mu * e11 + K.lam * tre);
                s[0][1] = s[1][0] = g * (2.0 * K.mu * e01);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) P.scatter(0.0, jxw * s[i][0], jxw * s[i][1], o[i]);
            if (MODE == M_FULL) {                                      // model.py:299-303, 350
                double phq, gx, gy;
                P.eval(cv[MI::F_U + 2], phq, gx, gy);
                const double cph = rho * K.omk * phq;
                const double t00 = cph * sp[0][0] + K.two_p * phq, t11 = cph * sp[1][1] + K.two_p * phq;
                const double t01 = cph * sp[0][1];
                coup = t00 * w[0][0] + t01 * (w[0][1] + w[1][0]) + t11 * w[1][1];
            }
        }
        if (HAS_P) {
            double vp, gx, gy;
            P.eval(cv[MODE == M_FULL ? MI::F_V + 2 : MI::F_V], vp, gx, gy);
            const double a = K.omk * rho * Ep + K.two_p * div + K.gc_over_eps;   // model.py:304-308
            P.scatter(jxw * (coup + a * vp), jxw * K.k_phi * gx, jxw * K.k_phi * gy,
                      o[MODE == M_FULL ? 2 : 0]);
        }
    }
}


// a_phiphi (model.py:304-308) of the 9 QPs of a Q2 cell from the nine-node
// U displacement (u0, u1): the arithmetic of cell_q2_rows' state part, so a
// table of it reproduces the on-the-fly phi block bit for bit.
__device__ __forceinline__ void phi_coef_q2(const double (&u0)[9], const double (&u1)[9],
                                            const double* __restrict__ rho_q, const Consts& K, const Q2Tab& T,
                                            double (&aq)[9]) {
#pragma unroll 1
    for (int qy = 0; qy < 3; ++qy) {
        double By[3], Dy[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            By[b] = T.B[qy][b];
            Dy[b] = T.Dy[qy][b];
        }
        double y0v[3], y0d[3], y1v[3], y1d[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            y0v[a] = fma(By[0], u0[a], fma(By[1], u0[a + 3], By[2] * u0[a + 6]));
            y0d[a] = fma(Dy[0], u0[a], fma(Dy[1], u0[a + 3], Dy[2] * u0[a + 6]));
            y1v[a] = fma(By[0], u1[a], fma(By[1], u1[a + 3], By[2] * u1[a + 6]));
            y1d[a] = fma(Dy[0], u1[a], fma(Dy[1], u1[a + 3], Dy[2] * u1[a + 6]));
        }
#pragma unroll
        for (int qx = 0; qx < 3; ++qx) {
            double u0x = 0, u0y = 0, u1x = 0, u1y = 0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double dx = T.Dx[qx][a], bx = T.B[qx][a];
                u0x = fma(dx, y0v[a], u0x);
                u0y = fma(bx, y0d[a], u0y);
                u1x = fma(dx, y1v[a], u1x);
                u1y = fma(bx, y1d[a], u1y);
            }
            const double ea = u0x, ec = u1y, eb = 0.5 * (u0y + u1x);
            const double rho = rho_q ? __ldg(rho_q + 3 * qy + qx) : 1.0;
            const double div = ea + ec;
            const double Ep = 0.5 * K.lam * div * div + K.mu * (ea * ea + 2.0 * eb * eb + ec * ec);
            aq[3 * qy + qx] = K.omk * rho * Ep + K.two_p * div + K.gc_over_eps;
        }
    }
}

// Row-factorised NoSplit cell kernel for the hot modes (FULL / UBLK / PBLK):
// the 9 QPs are processed one QP row (fixed qy) at a time; every nodal field
// is first contracted along y for that row (6 values), then evaluated at the
// row's 3 QPs, and the transposed pass accumulates x first, then y -- about
// half the flops of the per-QP evaluation, and no 9 x NF corner array held in
// registers (fields are re-read through `load(f, c)`, an L1 hit).
// nocoup: FULL without the G_phiu coupling (block-diagonal operator).
// TAB: a_phiphi of the 9 QPs from the per-QP table (tq[q * tstride], q = 3 qy + qx,
// pffmg_phi_coef) -- the phi block and the block-diagonal operator (nocoup)
// then need no state strain.
template <int MODE, bool TAB = false, class Load>
__device__ __forceinline__ void cell_q2_rows(Load&& load, const double* __restrict__ rho_q, const Consts& K,
                                             const Q2Tab& T, bool nocoup,
                                             double (&o)[ModeInfo<2, MODE>::NCO][9],
                                             const double* __restrict__ tq = nullptr, int64_t tstride = 0) {
    using MI = ModeInfo<2, MODE>;
    constexpr int NCO = MI::NCO;
    constexpr bool HAS_U = MODE == M_FULL || MODE == M_UBLK;
    constexpr bool HAS_P = MODE == M_FULL || MODE == M_PBLK;
    constexpr bool NEED_STRAIN = (MODE == M_FULL || MODE == M_PBLK) && !TAB;
#pragma unroll
    for (int k = 0; k < NCO; ++k)
#pragma unroll
        for (int n = 0; n < 9; ++n) o[k][n] = 0.0;
    const bool cpl = MODE == M_FULL && !nocoup;
#if PFFMG_Q2_UNROLL_QY
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int qy = 0; qy < 3; ++qy) {
        double By[3], Dy[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            By[b] = T.B[qy][b];
            Dy[b] = T.Dy[qy][b];
        }
        // y-contraction of field f for this QP row: yv[a], yd[a] per node column a
        auto ycon = [&](int f, double (&yv)[3], double (&yd)[3]) {
            double c[9];
            load(f, c);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                yv[a] = fma(By[0], c[a], fma(By[1], c[a + 3], By[2] * c[a + 6]));
                yd[a] = fma(Dy[0], c[a], fma(Dy[1], c[a + 3], Dy[2] * c[a + 6]));
            }
        };
        // ---- state coefficients at the row's 3 QPs (model.py:274-309)
        double gr[3], aq[3], t00[3], t11[3], t01[3];
#pragma unroll
        for (int qx = 0; qx < 3; ++qx) {
            gr[qx] = 1.0;
            aq[qx] = t00[qx] = t11[qx] = t01[qx] = 0.0;
        }
        double ea[3] = {0, 0, 0}, eb[3] = {0, 0, 0}, ec[3] = {0, 0, 0};
        if (NEED_STRAIN) {
            double y0v[3], y0d[3], y1v[3], y1d[3];
            ycon(MI::F_U + 0, y0v, y0d);
            ycon(MI::F_U + 1, y1v, y1d);
#pragma unroll
            for (int qx = 0; qx < 3; ++qx) {
                double u0x = 0, u0y = 0, u1x = 0, u1y = 0;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const double dx = T.Dx[qx][a], bx = T.B[qx][a];
                    u0x = fma(dx, y0v[a], u0x);
                    u0y = fma(bx, y0d[a], u0y);
                    u1x = fma(dx, y1v[a], u1x);
                    u1y = fma(bx, y1d[a], u1y);
                }
                ea[qx] = u0x;
                ec[qx] = u1y;
                eb[qx] = 0.5 * (u0y + u1x);
            }
        }
        if (MI::PT) {
            double yv[3], yd[3];
            ycon(MI::F_PT, yv, yd);
#pragma unroll
            for (int qx = 0; qx < 3; ++qx) {
                const double pt = fma(T.B[qx][0], yv[0], fma(T.B[qx][1], yv[1], T.B[qx][2] * yv[2]));
                gr[qx] = fma(K.omk, pt * pt, K.kappa);                    // model.py:135-137
            }
        }
        double phq[3] = {0, 0, 0};
        if (MODE == M_FULL && cpl) {
            double yv[3], yd[3];
            ycon(MI::F_U + 2, yv, yd);
#pragma unroll
            for (int qx = 0; qx < 3; ++qx)
                phq[qx] = fma(T.B[qx][0], yv[0], fma(T.B[qx][1], yv[1], T.B[qx][2] * yv[2]));
        }
#pragma unroll
        for (int qx = 0; qx < 3; ++qx) {
            const double rho = rho_q ? __ldg(rho_q + 3 * qy + qx) : 1.0;
            gr[qx] *= rho;
            if (TAB) aq[qx] = __ldg(tq + (3 * qy + qx) * tstride);
            if (NEED_STRAIN) {
                const double div = ea[qx] + ec[qx];
                const double Ep = 0.5 * K.lam * div * div +
                                  K.mu * (ea[qx] * ea[qx] + 2.0 * eb[qx] * eb[qx] + ec[qx] * ec[qx]);
                aq[qx] = K.omk * rho * Ep + K.two_p * div + K.gc_over_eps;    // model.py:304-308
                if (MODE == M_FULL && cpl) {                                  // model.py:299-303
                    const double c = rho * K.omk * phq[qx];
                    const double ld = K.lam * div;
                    t00[qx] = c * (2.0 * K.mu * ea[qx] + ld) + K.two_p * phq[qx];
                    t11[qx] = c * (2.0 * K.mu * ec[qx] + ld) + K.two_p * phq[qx];
                    t01[qx] = c * (2.0 * K.mu * eb[qx]);
                }
            }
        }
        // ---- increments and the transposed pass
        double tv[NCO][3], td[NCO][3];
#pragma unroll
        for (int k = 0; k < NCO; ++k)
#pragma unroll
            for (int a = 0; a < 3; ++a) tv[k][a] = td[k][a] = 0.0;
        double w00[3], w01[3], w10[3], w11[3];
        if (HAS_U) {
            double y0v[3], y0d[3], y1v[3], y1d[3];
            ycon(MI::F_V + 0, y0v, y0d);
            ycon(MI::F_V + 1, y1v, y1d);
#pragma unroll
            for (int qx = 0; qx < 3; ++qx) {
                w00[qx] = w01[qx] = w10[qx] = w11[qx] = 0.0;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const double dx = T.Dx[qx][a], bx = T.B[qx][a];
                    w00[qx] = fma(dx, y0v[a], w00[qx]);
                    w01[qx] = fma(bx, y0d[a], w01[qx]);
                    w10[qx] = fma(dx, y1v[a], w10[qx]);
                    w11[qx] = fma(bx, y1d[a], w11[qx]);
                }
                const double jxw = T.W[qy][qx];
                const double e01 = 0.5 * (w01[qx] + w10[qx]), tre = w00[qx] + w11[qx];
                const double g = jxw * gr[qx];                               // model.py:316-319
                const double s00 = g * (2.0 * K.mu * w00[qx] + K.lam * tre);
                const double s11 = g * (2.0 * K.mu * w11[qx] + K.lam * tre);
                const double s01 = g * (2.0 * K.mu * e01);
                // u rows: sum_j s_ij dN/dx_j -> x pass (F = 0)
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const double dx = T.Dx[qx][a], bx = T.B[qx][a];
                    tv[0][a] = fma(dx, s00, tv[0][a]);
                    td[0][a] = fma(bx, s01, td[0][a]);
                    tv[1][a] = fma(dx, s01, tv[1][a]);
                    td[1][a] = fma(bx, s11, td[1][a]);
                }
            }
        }
        if (HAS_P) {
            double yv[3], yd[3];
            ycon(MODE == M_FULL ? MI::F_V + 2 : MI::F_V, yv, yd);
            constexpr int kp = MODE == M_FULL ? 2 : 0;
#pragma unroll
            for (int qx = 0; qx < 3; ++qx) {
                double val = 0, gx = 0, gy = 0;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const double dx = T.Dx[qx][a], bx = T.B[qx][a];
                    val = fma(bx, yv[a], val);
                    gx = fma(dx, yv[a], gx);
                    gy = fma(bx, yd[a], gy);
                }
                const double jxw = T.W[qy][qx];
                double coup = 0.0;
                if (MODE == M_FULL && cpl)
                    coup = t00[qx] * w00[qx] + t01[qx] * (w01[qx] + w10[qx]) + t11[qx] * w11[qx];
                const double F = jxw * (coup + aq[qx] * val);
                const double Gx = jxw * K.k_phi * gx, Gy = jxw * K.k_phi * gy;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const double dx = T.Dx[qx][a], bx = T.B[qx][a];
                    tv[kp][a] = fma(bx, F, fma(dx, Gx, tv[kp][a]));
                    td[kp][a] = fma(bx, Gy, td[kp][a]);
                }
            }
        }
        // y pass of the transposed contraction
#pragma unroll
        for (int k = 0; k < NCO; ++k)
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    o[k][3 * b + a] = fma(By[b], tv[k][a], fma(Dy[b], td[k][a], o[k][3 * b + a]));
    }
}

}  // namespace pffmg
