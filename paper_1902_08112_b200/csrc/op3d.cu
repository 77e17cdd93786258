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

template <int MODE, int EPI, bool ISO, bool MIE = false>
static void set_smem(size_t smem) {
    static size_t done = 0;
    if (done < smem) {
        cudaFuncSetAttribute(op3d_kernel<MODE, EPI, TY3D, ISO, MIE>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        done = smem;
    }
}

template <int MODE, int EPI, int TX, bool RHO, bool BOX, bool PRE, bool TAB = false>
static void launch_t(const OpArgs& A0, int planes, cudaStream_t s) {
    using MI = ModeInfo<3, MODE>;
    using TL = Tile3<TX>;
    constexpr int NCO = MI::NCO;
    constexpr bool STAGE = MODE == M_UBLK || (MODE == M_FULL && (EPI == E_CHEB || EPI == E_CHEB0));
    constexpr size_t smem = TL::template smem<TAB ? MI::NV : MI::NF, NCO, STAGE ? EpiIn<NCO, EPI>::NL : 0>();
    auto kern = op3dt_kernel<MODE, EPI, TX, RHO, BOX, PRE, TAB>;
    static int occ = 0;
    if (occ == 0) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, T3_NT, smem) != cudaSuccess || occ < 1)
            occ = 1;
    }
    // persistent grid: one wave of resident CTAs sharing the (tile, plane)
    // items equally (op3dt_kernel); never more CTAs than items
    const Lat& L = A0.L;
    const bool listed = TX - 1 == PFFMG_TILE3 && L.tiles3d != nullptr;
    const int64_t ntiles = listed ? L.n_tiles3d
                                  : (int64_t)((L.nx + 1 + TX - 2) / (TX - 1)) * ((L.ny + 1 + TL::TY - 2) / (TL::TY - 1));
    const int64_t items = ntiles * (A0.ends ? 2 : planes);
    static const int cap = [] {
        const char* e = getenv("PFFMG_3D_CTAS");      // tuning: CTAs per SM of the persistent grid
        return e ? atoi(e) : 0;
    }();
    int64_t g = (int64_t)sm_count() * (cap > 0 ? cap : occ);
    if (g > items) g = items;
    if (g < 1) g = 1;
    // schedule (op3dt_kernel): persistent tile-major for the FP64-bound full
    // operator and on listed (non-box) lattices; the strips x tiles grid,
    // whose concurrent CTAs share halo planes in L2, for the lighter modes of
    // box lattices (measured: cfg5 phi block 216 -> 163 us, u block 390 -> 373 us;
    // full operator and the cfg4 L-prism better persistent, 153 -> 136 us)
    static const int forced_sched = [] {
        const char* e = getenv("PFFMG_3D_SCHED");    // tuning: 1 persistent, 2 grid
        return e ? atoi(e) : 0;
    }();
    static const int forced = [] {
        const char* e = getenv("PFFMG_3D_PLANES");   // tuning: strip height of the grid schedule
        return e ? atoi(e) : 0;
    }();
    OpArgs A = A0;
    A.sched = forced_sched ? forced_sched : ((MODE == M_FULL || listed || A0.ends) ? 1 : 2);
    if (A0.ends) A.sched = 1;
    if (A.sched == 2) {
        // strips: about half a resident CTA's share of planes per tile, 8..32
        // planes, balanced so the last strip is not a sliver
        const int64_t share = items / g;
        int S = forced > 0 ? forced : (int)std::min<int64_t>(32, std::max<int64_t>(8, share / 2));
        S = std::max(1, std::min(S, planes));
        const int nstrips = (planes + S - 1) / S;
        S = (planes + nstrips - 1) / nstrips;
        A.planes_per_cta = S;
        g = (int64_t)nstrips * ntiles;
    }
    const dim3 grid((unsigned)g);
    pdl_launch(kern, grid, dim3(T3_NT), smem, s, A);
}

// Tile shape of the streaming kernel: 16 x 16 cells (default) or 32 x 8
// (PFFMG_3D_TX=32).
static int tile_tx() {
    static const int tx = [] {
        const char* e = getenv("PFFMG_3D_TX");
        return (e && atoi(e) == 32) ? 32 : 16;
    }();
    return tx;
}

template <int MODE, int EPI>
static int launch_stream(const OpArgs& A, cudaStream_t s) {
    const Lat& L = A.L;
    const int planes = A.ends ? 2 : L.own_hi - L.own_lo;
    const bool tab = MODE == M_PBLK && A.ptab != nullptr;
    const bool rho = A.rho != nullptr, box = L.vrow_off == nullptr, pre = A.premasked != 0;
    const bool t32 = tile_tx() == 32;
#define PFFMG_T(R, B, P, T)                                                        \
    (t32 ? launch_t<MODE, EPI, 32, R, B, P, T>(A, planes, s)                       \
         : launch_t<MODE, EPI, 16, R, B, P, T>(A, planes, s))
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
