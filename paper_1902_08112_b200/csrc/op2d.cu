// 2D instantiations of the fused operator kernels (see op_kernels.cuh).
#include <cstdlib>

#include "op_launch.cuh"

namespace pffmg {

constexpr int NW2D = 4;   // warps per CTA of the warp-independent 2D kernel

// Strips of `per` vertex rows per warp (the first cell row of a strip is
// recomputed for the y carry: overhead 1/per).  The warps are independent, so
// the strip height is chosen to give ONE wave of resident warps (occupancy of
// the instantiation x SMs): a partial second wave left ~30% of the SMs idle
// for a whole strip (cfg2 vmult 41 -> 39 us).
template <int MODE, int EPI, bool ISO, bool RHO, bool BOX, bool PRE, bool MIE, bool TAB = false>
static void launch_w(const OpArgs& A0, int nseg, int rows, size_t smem, cudaStream_t s) {
    auto kern = op2dw_kernel<MODE, EPI, NW2D, ISO, RHO, BOX, PRE, MIE, TAB>;
    static size_t done = 0;
    static int occ = 0;
    if (done < smem || occ == 0) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        done = smem;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * NW2D, smem) != cudaSuccess || occ < 1)
            occ = 1;
    }
    OpArgs A = A0;
    const int64_t slots = (int64_t)sm_count() * occ * NW2D;
    int64_t per = ((int64_t)rows * nseg + slots - 1) / slots;
    static const int minrows = [] {
        const char* e = getenv("PFFMG_2D_MINROWS");
        return e ? atoi(e) : 1;
    }();
    per = per < minrows ? minrows : (per > 64 ? 64 : per);
    static const int forced = [] {
        const char* e = getenv("PFFMG_2D_ROWS");
        return e ? atoi(e) : 0;
    }();
    if (forced > 0) per = forced;
    if (A.ends) per = 1;
    A.planes_per_cta = (int)per;
    A.nseg = nseg;
    const int64_t warps = (int64_t)nseg * ((rows + per - 1) / per);
    const dim3 grid((unsigned)((warps + NW2D - 1) / NW2D));
    pdl_launch(kern, grid, dim3(32 * NW2D), smem, s, A);
}

template <int MODE, int EPI, bool ISO, bool RHO, bool MIE = false, bool TAB = false>
static void launch_box(const OpArgs& A, bool pre, int nseg, int rows, size_t smem, cudaStream_t s) {
    const bool box = A.L.vrow_off == nullptr;
    if (box && pre)
        launch_w<MODE, EPI, ISO, RHO, true, true, MIE, TAB>(A, nseg, rows, smem, s);
    else if (box)
        launch_w<MODE, EPI, ISO, RHO, true, false, MIE, TAB>(A, nseg, rows, smem, s);
    else if (pre)
        launch_w<MODE, EPI, ISO, RHO, false, true, MIE, TAB>(A, nseg, rows, smem, s);
    else
        launch_w<MODE, EPI, ISO, RHO, false, false, MIE, TAB>(A, nseg, rows, smem, s);
}

template <int MODE, int EPI>
int launch2d(const OpArgs& A, bool iso, cudaStream_t s) {
    const Lat& L = A.L;
    using MI = ModeInfo<2, MODE>;
    const int nseg = (L.nx + 1 + 29) / 30;
    const int rows = A.ends ? 2 : L.own_hi - L.own_lo;
    const int nf = A.split ? ModeInfo<2, MODE, true>::NF : MI::NF;
    const size_t smem = NW2D * sizeof(double) * 4 * nf * 32;
    const bool rho = A.rho != nullptr;
    const bool pre = A.premasked != 0;
    if constexpr (MODE == M_FULL) {
        // block-diagonal smoother with the per-QP a_phiphi table: v and phi~ only
        if (A.nocoup && A.ptab && iso && !A.split) {
            const size_t smem_t = NW2D * sizeof(double) * 4 * (MI::NV + 1) * 32;
            if (rho)
                launch_box<MODE, EPI, true, true, false, true>(A, pre, nseg, rows, smem_t, s);
            else
                launch_box<MODE, EPI, true, false, false, true>(A, pre, nseg, rows, smem_t, s);
            return PFFMG_OK;
        }
    }
    if constexpr (MODE == M_PBLK) {
        // phi block with the table: v only (the table already holds rho)
        if (A.ptab && iso && !A.split) {
            const size_t smem_t = NW2D * sizeof(double) * 4 * MI::NV * 32;
            launch_box<MODE, EPI, true, false, false, true>(A, pre, nseg, rows, smem_t, s);
            return PFFMG_OK;
        }
    }
    if (A.split)   // Miehe split: general-cell kernel, modulus field resolved in-kernel
        launch_box<MODE, EPI, false, false, true>(A, pre, nseg, rows, smem, s);
    else if (iso && rho)
        launch_box<MODE, EPI, true, true>(A, pre, nseg, rows, smem, s);
    else if (iso)
        launch_box<MODE, EPI, true, false>(A, pre, nseg, rows, smem, s);
    else if (rho)
        launch_box<MODE, EPI, false, true>(A, pre, nseg, rows, smem, s);
    else
        launch_box<MODE, EPI, false, false>(A, pre, nseg, rows, smem, s);
    return PFFMG_OK;
}

PFFMG_INSTANTIATE_LAUNCH(launch2d)

// Per-QP a_phiphi table of a 2D isotropic NoSplit level (model.py:304-308, the
// phi-block entry of _build_caches), QP-major: tab[q * C + c] for lattice cell
// c = cx + nx cy, C = nx ny.  One thread per lattice cell; cells absent from a
// non-box lattice get 0.
template <bool RHO>
__global__ void __launch_bounds__(256) phi_coef2_kernel(const OpArgs A, double* __restrict__ tab) {
    pdl_wait();
    const Lat& L = A.L;
    const int64_t C = (int64_t)L.nx * L.ny;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int cx = (int)(c % L.nx), cy = (int)(c / L.nx);
        double aj[4] = {0.0, 0.0, 0.0, 0.0};
        if (cell_exists<2>(L, cx, cy, 0)) {
            double u0[4], u1[4];
#pragma unroll
            for (int n = 0; n < 4; ++n) {
                const int64_t vid = vertex_id(L, cx + (n & 1), cy + (n >> 1), 0);
                u0[n] = __ldg(A.U + vid);
                u1[n] = __ldg(A.U + L.V + vid);
            }
            phi_coef2<RHO>(u0, u1, RHO ? A.rho + c * 4 : nullptr, A.K, A.I, aj);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) tab[q * C + c] = aj[q];
    }
}

int launch_phi_coef2(const OpArgs& A, double* tab, cudaStream_t s) {
    const int64_t C = (int64_t)A.L.nx * A.L.ny;
    int64_t blocks = (C + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (A.rho)
        pdl_launch(phi_coef2_kernel<true>, dim3((unsigned)blocks), dim3(256), 0, s, A, tab);
    else
        pdl_launch(phi_coef2_kernel<false>, dim3((unsigned)blocks), dim3(256), 0, s, A, tab);
    return PFFMG_OK;
}

}  // namespace pffmg
