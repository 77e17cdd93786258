// 3D instantiations of the fused operator kernels: the streaming isotropic
// kernel (op3dt.cuh) for FULL / UBLK / PBLK, the generic shared-memory kernel
// (op_kernels.cuh) for the diagonal and for anisotropic cells.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "op3dt.cuh"
#include "op_launch.cuh"

namespace pffmg {

constexpr int TY3D = 8;    // generic kernel
constexpr int TY3T = 8;    // streaming kernel

template <int MODE, int EPI, bool ISO, bool MIE = false>
static void set_smem(size_t smem) {
    static size_t done = 0;
    if (done < smem) {
        cudaFuncSetAttribute(op3d_kernel<MODE, EPI, TY3D, ISO, MIE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        done = smem;
    }
}

// Planes per CTA of the streaming kernel: each CTA marches `per` vertex
// planes after a one-plane warm-up, so the cost of a launch is about
//   ceil(active tiles x ceil(planes / per) / (SMs x resident CTAs)) x (per + c0)
// waves of plane steps (c0 = warm-up + ring fill, ~2 plane steps).  `frac`
// estimates the share of x-y tile columns that hold vertices (non-box
// lattices leave whole columns empty, and those CTAs exit at once).
static int planes_per_cta(int64_t columns, int planes, int occ, double frac) {
    static const int forced = [] {
        const char* e = getenv("PFFMG_3D_PLANES");
        return e ? atoi(e) : 0;
    }();
    if (forced > 0) return forced;
    const int64_t slots = (int64_t)sm_count() * (occ > 0 ? occ : 1);
    const int64_t active = (int64_t)std::ceil((double)columns * frac);
    int best = 32;
    double best_cost = 1e300;
    for (int per = 2; per <= 32; ++per) {
        const int64_t ctas = active * ((planes + per - 1) / per);
        const int64_t waves = (ctas + slots - 1) / slots;
        const double cost = (double)waves * (std::min(per, planes) + 2.0);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = per;
        }
    }
    return best;
}

template <int MODE, int EPI, bool RHO, bool BOX, bool PRE, bool TAB = false>
static void launch_t(const OpArgs& A0, int gx, int gy, int planes, double frac, size_t smem, cudaStream_t s) {
    auto kern = op3dt_kernel<MODE, EPI, TY3T, RHO, BOX, PRE, TAB>;
    static size_t done = 0;
    static int occ = 0;
    if (done < smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        done = smem;
        occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * TY3T, smem) != cudaSuccess) occ = 1;
    }
    OpArgs A = A0;
    int per;
    if (TAB) {
        // light, HBM-bound phi block (4 CTAs/SM): latency-bound unless the
        // grid fills the resident slots several times over
        per = planes_per_cta((int64_t)gx * gy, planes, occ, frac);
    } else {
        // FP64-bound modes: ~2 CTAs of work per SM per wave, strips of 1..32
        // planes (measured sweep)
        static const int forced = [] {
            const char* e = getenv("PFFMG_3D_PLANES");
            return e ? atoi(e) : 0;
        }();
        const int64_t sms = sm_count();
        int64_t p = ((int64_t)planes * gx * gy + 2LL * sms - 1) / (2LL * sms);
        per = (int)(p < 1 ? 1 : (p > 32 ? 32 : p));
        if (forced > 0) per = forced;
    }
    if (A.ends) per = 1;
    A.planes_per_cta = per;
    const dim3 grid(gx, gy, (unsigned)((planes + per - 1) / per));
    pdl_launch(kern, grid, dim3(32 * TY3T), smem, s, A);
}

template <int MODE, int EPI>
static int launch_stream(const OpArgs& A, cudaStream_t s) {
    const Lat& L = A.L;
    using MI = ModeInfo<3, MODE>;
    const int gx = (L.nx + 1 + 29) / 30;
    const int gy = (L.ny + 1 + TY3T - 2) / (TY3T - 1);
    const int planes = A.ends ? 2 : L.own_hi - L.own_lo;
    const double frac = std::min(1.0, (double)L.V / ((double)(L.nx + 1) * (L.ny + 1) * (L.nz + 1)));
    constexpr int ROWS = TY3T + 1;
    const bool tab = MODE == M_PBLK && A.ptab != nullptr;
    const size_t smem = sizeof(double) * (4 * (tab ? MI::NV : MI::NF) * ROWS * 32 + TY3T * MI::NCO * 2 * 32 +
                                          ((MODE == M_UBLK || (MODE == M_FULL && (EPI == E_CHEB || EPI == E_CHEB0)))
                                               ? 32 * TY3T * EpiIn<MI::NCO, EPI>::NL * MI::NCO : 0)) +
                        4 * ROWS * 48 + 4 * ROWS * sizeof(int);
    const bool rho = A.rho != nullptr, box = L.vrow_off == nullptr, pre = A.premasked != 0;
#define PFFMG_T(R, B, P, T) launch_t<MODE, EPI, R, B, P, T>(A, gx, gy, planes, frac, smem, s)
    if constexpr (MODE == M_PBLK) {
        if (tab) {                       // the table already holds rho
            if (box) { if (pre) PFFMG_T(false, true, true, true); else PFFMG_T(false, true, false, true); }
            else { if (pre) PFFMG_T(false, false, true, true); else PFFMG_T(false, false, false, true); }
            return PFFMG_OK;
        }
    }
    if (rho) {
        if (box) { if (pre) PFFMG_T(true, true, true, false); else PFFMG_T(true, true, false, false); }
        else { if (pre) PFFMG_T(true, false, true, false); else PFFMG_T(true, false, false, false); }
    } else {
        if (box) { if (pre) PFFMG_T(false, true, true, false); else PFFMG_T(false, true, false, false); }
        else { if (pre) PFFMG_T(false, false, true, false); else PFFMG_T(false, false, false, false); }
    }
#undef PFFMG_T
    return PFFMG_OK;
}

template <int MODE, int EPI>
int launch3d(const OpArgs& A0, bool iso, cudaStream_t s) {
    if (iso && MODE != M_DIAG && !A0.split) return launch_stream<MODE, EPI>(A0, s);
    OpArgs A = A0;
    const Lat& L = A.L;
    const int sms = sm_count();
    using MI = ModeInfo<3, MODE>;
    constexpr int TV = 33 * (TY3D + 1);
    const int nf = A.split ? ModeInfo<3, MODE, true>::NF : MI::NF;
    const size_t smem = sizeof(double) * (2 * nf * TV + TY3D * 2 * MI::NCO * 32) + 2 * TV;
    const int gx = (L.nx + 1 + 30) / 31;
    const int gy = (L.ny + 1 + TY3D - 2) / (TY3D - 1);
    const int planes = A.ends ? 2 : L.own_hi - L.own_lo;
    int per = (int)(((int64_t)planes * gx * gy + 2LL * sms - 1) / (2LL * sms));
    per = per < 4 ? 4 : (per > 32 ? 32 : per);
    if (A.ends) per = 1;
    A.planes_per_cta = per;
    dim3 grid(gx, gy, (planes + per - 1) / per);
    if (A.split) {   // Miehe spectral split: general cells, per-QP Jacobi eigen-solve
        set_smem<MODE, EPI, false, true>(smem);
        pdl_launch(op3d_kernel<MODE, EPI, TY3D, false, true>, dim3(grid), dim3(32 * TY3D), smem, s, A);
    } else if (iso) {
        set_smem<MODE, EPI, true>(smem);
        pdl_launch(op3d_kernel<MODE, EPI, TY3D, true>, dim3(grid), dim3(32 * TY3D), smem, s, A);
    } else {
        set_smem<MODE, EPI, false>(smem);
        pdl_launch(op3d_kernel<MODE, EPI, TY3D, false>, dim3(grid), dim3(32 * TY3D), smem, s, A);
    }
    return PFFMG_OK;
}

PFFMG_INSTANTIATE_LAUNCH(launch3d)

// Per-QP a_phiphi table of a 3D isotropic NoSplit level (model.py:304-308,
// the phi-block entry of _build_caches), QP-major: tab[q * C + c] for lattice
// cell c = cx + nx (cy + ny cz), C = nx ny nz.  One thread per lattice cell;
// cells absent from a non-box lattice get 0.
template <bool RHO>
__global__ void __launch_bounds__(256) phi_coef3_kernel(const OpArgs A, double* __restrict__ tab) {
    pdl_wait();
    const Lat& L = A.L;
    const int64_t C = (int64_t)L.nx * L.ny * L.nz;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int cx = (int)(c % L.nx);
        const int64_t r = c / L.nx;
        const int cy = (int)(r % L.ny), cz = (int)(r / L.ny);
        double aj[8];
        if (cell_exists<3>(L, cx, cy, cz)) {
            struct G {
                const double* U;
                int64_t V, vid[8];
                __device__ __forceinline__ void load(int f, double (&c)[8]) const {
#pragma unroll
                    for (int n = 0; n < 8; ++n) c[n] = __ldg(U + f * V + vid[n]);
                }
            } g;
            g.U = A.U;
            g.V = L.V;
#pragma unroll
            for (int n = 0; n < 8; ++n) g.vid[n] = vertex_id(L, cx + (n & 1), cy + ((n >> 1) & 1), cz + (n >> 2));
            phi_coef3<RHO>(g, RHO ? A.rho + c * 8 : nullptr, A.K, A.I, aj);
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) aj[q] = 0.0;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) tab[q * C + c] = aj[q];
    }
}

int launch_phi_coef3(const OpArgs& A, double* tab, cudaStream_t s) {
    const int64_t C = (int64_t)A.L.nx * A.L.ny * A.L.nz;
    int64_t blocks = (C + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (A.rho)
        pdl_launch(phi_coef3_kernel<true>, dim3((unsigned)blocks), dim3(256), 0, s, A, tab);
    else
        pdl_launch(phi_coef3_kernel<false>, dim3((unsigned)blocks), dim3(256), 0, s, A, tab);
    return PFFMG_OK;
}

}  // namespace pffmg
