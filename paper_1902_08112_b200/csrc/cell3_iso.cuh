// Register-lean 3D cell kernel for isotropic hexahedra (NoSplit).
//
// Same physics as cell_kernel_iso<3> (cellops_iso.cuh; reference
// model.py:270-355 for the Jacobian, model.py:420-460 for the residual
// mode), reorganised as a stream over gradient components so that only
// O(8)-sized per-QP arrays are live at a time: every reduced derivative array
// (4 values: d_j of a trilinear field is bilinear in the other two axes) is
// produced from the staged corners when it is needed, consumed by the u-row
// stress terms, the S:w coupling and the E+ energy, and dropped.  Outputs are
// handed to `emit(k, o[8])` component by component so the caller can start
// the vertex reduction (x-shuffle) early.
#pragma once

#include "cellops_iso.cuh"

namespace pffmg {

// JxW-scaled a_phiphi of the 8 QPs of one cell from the corners of U
// (fields 0..2 of `C`): the phi-block coefficient of _build_caches
// (model.py:304-308), the same expression cell3_iso evaluates in the PBLK /
// FULL modes.  Used to build the per-QP table of pffmg_phi_coef.
template <bool RHO, class Corners>
__device__ __forceinline__ void phi_coef3(const Corners& C, const double* __restrict__ rho_q, const Consts& K,
                                          const IsoK& I, double (&aj)[8]) {
    using S = SFr<3>;
    constexpr int NP = 8;
    auto expand = [](const double (&r)[4], int j, int q) { return r[drop_bit(q, j)]; };
    auto deriv = [&](int field, int j, double (&g)[4]) {
        double c[NP];
        C.load(field, c);
        S::deriv(c, j, g, K);
    };
    double rd[3][4], trr[NP], e2[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) trr[q] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        deriv(i, i, rd[i]);
#pragma unroll
        for (int q = 0; q < NP; ++q) trr[q] += expand(rd[i], i, q);
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const double ld = I.lam * trr[q];
        e2[q] = ld * trr[q];
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double r2 = I.two_mu * expand(rd[i], i, q);
            e2[q] = fma(r2, expand(rd[i], i, q), e2[q]);
        }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i + 1; j < 3; ++j) {
            double a[4], b[4];
            deriv(i, j, a);
            deriv(j, i, b);
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const double s = expand(a, j, q) + expand(b, i, q);
                const double ms = I.mu * s;
                e2[q] = fma(ms, s, e2[q]);
            }
        }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const double ce = RHO ? I.cS * __ldg(rho_q + q) : I.cS;
        aj[q] = fma(ce, e2[q], fma(I.cdiv, trr[q], I.c0));
    }
}

// TAB (PBLK only): a_phiphi read from the per-QP table (`tq[q * tstride]`)
// instead of being recomputed from U -- the phi block then stages v only.
template <int MODE, bool RHO, class Corners, class Emit, bool TAB = false>
__device__ __forceinline__ void cell3_iso(const Corners& C, const double* __restrict__ rho_q,
                                          const Consts& K, const IsoK& I, Emit&& emit,
                                          const double* __restrict__ tq = nullptr, int64_t tstride = 0) {
    using MI = ModeInfo<3, MODE>;
    using S = SFr<3>;
    constexpr int NP = 8;
    if constexpr (TAB) {
        static_assert(MODE == M_PBLK, "the a_phiphi table serves the phi block");
        double cp[NP], f[NP];
        C.load(MI::F_V, cp);
        S::value(cp, f, K);
#pragma unroll
        for (int q = 0; q < NP; ++q) f[q] = __ldg(tq + q * tstride) * f[q];
        mass_transpose<3>(f, K);
        corner_laplacian<3>(cp, I, f);
        emit(0, f);
        return;
    }
    constexpr bool RES = MODE == M_RES;
    constexpr bool HAS_W = MODE == M_FULL || MODE == M_UBLK;     // v displacement gradient
    constexpr bool HAS_R = MODE == M_FULL || MODE == M_PBLK || RES;   // U displacement gradient
    constexpr bool HAS_G = HAS_W || RES;                         // u rows

    double rho[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) rho[q] = RHO ? __ldg(rho_q + q) : 1.0;

    auto expand = [](const double (&r)[4], int j, int q) { return r[drop_bit(q, j)]; };
    auto deriv = [&](int field, int j, double (&g)[4]) {
        double c[NP];
        C.load(field, c);
        S::deriv(c, j, g, K);
    };

    // ------------------------------------------------------------ gk rho
    double gks[NP], pv[NP];
    if (MI::PT) {
        double c[NP];
        C.load(MI::F_PT, c);
        S::value(c, pv, K);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double g = fma(I.gk_a * pv[q], pv[q], I.gk_b);
            gks[q] = RHO ? g * rho[q] : g;
        }
    }

    // ----------------------------------------------- diagonal gradient terms
    double wd[3][4], rd[3][4];
    double trw[NP], trr[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        trw[q] = 0.0;
        trr[q] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (HAS_W) {
            deriv(MI::F_V + i, i, wd[i]);
#pragma unroll
            for (int q = 0; q < NP; ++q) trw[q] += expand(wd[i], i, q);
        }
        if (HAS_R) {
            deriv(MI::F_U + i, i, rd[i]);
#pragma unroll
            for (int q = 0; q < NP; ++q) trr[q] += expand(rd[i], i, q);
        }
    }

    double ou[3][NP];     // u-row outputs (accumulated)
    double Y[NP], e2[NP]; // S:w coupling and S:sym(r) energy
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        if (HAS_R) {
            const double ld = I.lam * trr[q];
            e2[q] = ld * trr[q];                      // lam (tr r)^2
            if (MODE == M_FULL) Y[q] = ld * trw[q];   // lam tr r tr w
        }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (HAS_W) {                                  // G_ii = gk (2 mu w_ii + lam tr w)
            double G[NP];
#pragma unroll
            for (int q = 0; q < NP; ++q) G[q] = gks[q] * fma(I.two_mu, expand(wd[i], i, q), I.lam * trw[q]);
            S::template deriv_T<false>(G, i, ou[i], K);
        }
        if (RES) {                                    // gk sigma+_ii + p phi~^2   (model.py:445-448)
            double G[NP];
#pragma unroll
            for (int q = 0; q < NP; ++q)
                G[q] = fma(gks[q], fma(I.two_mu, expand(rd[i], i, q), I.lam * trr[q]),
                           I.cpres * (pv[q] * pv[q]));
            S::template deriv_T<false>(G, i, ou[i], K);
        }
        if (HAS_R) {
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const double r2 = I.two_mu * expand(rd[i], i, q);
                e2[q] = fma(r2, expand(rd[i], i, q), e2[q]);            // 2 mu r_ii^2
                if (MODE == M_FULL) Y[q] = fma(r2, expand(wd[i], i, q), Y[q]);   // 2 mu r_ii w_ii
            }
        }
    }

    // ------------------------------------------- off-diagonal gradient terms
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = i + 1; j < 3; ++j) {
            double sw[NP], s[NP];
            if (HAS_W) {
                double a[4], b[4];
                deriv(MI::F_V + i, j, a);
                deriv(MI::F_V + j, i, b);
#pragma unroll
                for (int q = 0; q < NP; ++q) sw[q] = expand(a, j, q) + expand(b, i, q);
                double G[NP];                          // G_ij = G_ji = gk mu (w_ij + w_ji)
#pragma unroll
                for (int q = 0; q < NP; ++q) G[q] = (gks[q] * I.mu) * sw[q];
                S::template deriv_T<true>(G, j, ou[i], K);
                S::template deriv_T<true>(G, i, ou[j], K);
            }
            if (HAS_R) {
                double a[4], b[4];
                deriv(MI::F_U + i, j, a);
                deriv(MI::F_U + j, i, b);
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    s[q] = expand(a, j, q) + expand(b, i, q);
                    const double ms = I.mu * s[q];
                    e2[q] = fma(ms, s[q], e2[q]);                       // mu s_ij^2
                    if (MODE == M_FULL) Y[q] = fma(ms, sw[q], Y[q]);    // mu s_ij sw_ij
                }
                if (RES) {                             // gk sigma+_ij
                    double G[NP];
#pragma unroll
                    for (int q = 0; q < NP; ++q) G[q] = (gks[q] * I.mu) * s[q];
                    S::template deriv_T<true>(G, j, ou[i], K);
                    S::template deriv_T<true>(G, i, ou[j], K);
                }
            }
        }
    if (HAS_G) {
#pragma unroll
        for (int i = 0; i < 3; ++i) emit(i, ou[i]);
    }

    // ------------------------------------------------------------ phi row
    if (HAS_R) {
        double cp[NP], f[NP];
        C.load(MODE == M_FULL ? MI::F_V + 3 : (RES ? MI::F_U + 3 : MI::F_V), cp);
        S::value(cp, f, K);
        double phq[NP];
        if (MODE == M_FULL) {
            double cu[NP];
            C.load(MI::F_U + 3, cu);
            S::value(cu, phq, K);
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double ce = RHO ? I.cS * rho[q] : I.cS;
            if (RES) {                                  // model.py:450-452
                const double a = fma(ce, e2[q], I.cdiv * trr[q]);
                f[q] = fma(f[q], a, -I.c0 * (1.0 - f[q]));
                continue;
            }
            const double aj = fma(ce, e2[q], fma(I.cdiv, trr[q], I.c0));   // JxW a_phiphi
            if (MODE == M_FULL) {
                const double cc = RHO ? I.cc * rho[q] : I.cc;
                const double coup = phq[q] * fma(cc, Y[q], I.ctr * trw[q]);
                f[q] = fma(aj, f[q], coup);
            } else {
                f[q] = aj * f[q];
            }
        }
        mass_transpose<3>(f, K);
        corner_laplacian<3>(cp, I, f);
        emit(MODE == M_FULL || RES ? 3 : 0, f);
    }
}

}  // namespace pffmg
