// 3D instantiations of the fused operator kernels: the streaming isotropic
// kernel (op3dt.cuh) for FULL / UBLK / PBLK, the generic shared-memory kernel
// (op_kernels.cuh) for the diagonal and for anisotropic cells.
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

template <int MODE, int EPI, bool RHO, bool BOX, bool PRE>
static void launch_t(const OpArgs& A, dim3 grid, size_t smem, cudaStream_t s) {
    static size_t done = 0;
    if (done < smem) {
        cudaFuncSetAttribute(op3dt_kernel<MODE, EPI, TY3T, RHO, BOX, PRE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        done = smem;
    }
    pdl_launch(op3dt_kernel<MODE, EPI, TY3T, RHO, BOX, PRE>, dim3(grid), dim3(32 * TY3T), smem, s, A);
}

template <int MODE, int EPI>
static int launch_stream(const OpArgs& A0, cudaStream_t s) {
    OpArgs A = A0;
    const Lat& L = A.L;
    using MI = ModeInfo<3, MODE>;
    const int sms = sm_count();
    const int gx = (L.nx + 1 + 29) / 30;
    const int gy = (L.ny + 1 + TY3T - 2) / (TY3T - 1);
    const int planes = A.ends ? 2 : L.own_hi - L.own_lo;
    // ~2 CTAs of work per SM per wave, strips of 4..32 planes
    int64_t per = ((int64_t)planes * gx * gy + 2LL * sms - 1) / (2LL * sms);
    static const int minp = [] {
        const char* e = getenv("PFFMG_3D_MINPLANES");
        return e ? atoi(e) : 1;
    }();
    per = per < minp ? minp : (per > 32 ? 32 : per);
    static const int forced = [] {
        const char* e = getenv("PFFMG_3D_PLANES");
        return e ? atoi(e) : 0;
    }();
    if (forced > 0) per = forced;
    if (A.ends) per = 1;
    A.planes_per_cta = (int)per;
    dim3 grid(gx, gy, (unsigned)((planes + per - 1) / per));
    constexpr int ROWS = TY3T + 1;
    const size_t smem = sizeof(double) * (4 * MI::NF * ROWS * 32 + TY3T * MI::NCO * 2 * 32) +
                        4 * ROWS * 48 + 4 * ROWS * sizeof(int);
    const bool rho = A.rho != nullptr, box = L.vrow_off == nullptr, pre = A.premasked != 0;
#define PFFMG_T(R, B, P) launch_t<MODE, EPI, R, B, P>(A, grid, smem, s)
    if (rho) {
        if (box) { if (pre) PFFMG_T(true, true, true); else PFFMG_T(true, true, false); }
        else { if (pre) PFFMG_T(true, false, true); else PFFMG_T(true, false, false); }
    } else {
        if (box) { if (pre) PFFMG_T(false, true, true); else PFFMG_T(false, true, false); }
        else { if (pre) PFFMG_T(false, false, true); else PFFMG_T(false, false, false); }
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

}  // namespace pffmg
