// Coarse-level solve of the V-cycle in ONE kernel (reference mgsolve.py:209-218
// coarse_solve: per block, Chebyshev-Jacobi with the solver range and degree
// from the block spectrum, started from x = 0).
//
// The coarsest level has a few dozen cells, so the multi-kernel path spends its
// time in launch latency (up to ~40 dependent launches per V-cycle).  Here one
// CTA runs both blocks' recurrences: per Chebyshev step a cell pass (one
// thread per lattice cell, both diagonal blocks at once -- the block-diagonal
// operator, T_phiu = 0) into shared memory, a barrier, a vertex pass that sums
// each vertex's cell contributions in a fixed order and applies the
// recurrence (mgsolve.py:103-112), and a barrier.  Deterministic, no atomics.
// The recurrence of the shorter block simply stops updating.
#include "cell_q2.cuh"
#include "op_kernels.cuh"

namespace pffmg {

constexpr int CT = 256;   // threads = maximum lattice cells of a coarse level handled here

struct CoarseArgs {
    OpArgs A;                 // level operator (U, pt, rho, flags, constants)
    const double* b;          // right-hand side (full vector)
    double* x;
    double* r;
    double* d;
    const double* inv;
    const double* coef_u;     // [theta, c_dd_1, c_dr_1, ...] (mgsolve.py:103-112)
    const double* coef_p;
    int deg_u, deg_p;
    Q2Tab T;
};

// The level's vectors while the kernel runs: shared-memory copies.
struct CoarseData {
    const double* U;
    const double* pt;
    const uint8_t* fl;
    const double* d;
};

// KIND: 0 Q1 NoSplit (generic cell kernel), 1 Q1 Miehe, 2 Q2 NoSplit, 3 Q2 Miehe,
//       4 Q1 NoSplit on isotropic cells (folded-constant kernel)
template <int D, int KIND>
struct CoarseCell {
    static constexpr bool Q2 = KIND == 2 || KIND == 3;
    static constexpr bool MIE = KIND == 1 || KIND == 3;
    static constexpr bool ISO = KIND == 4;
    static constexpr int NPC = Q2 ? 9 : (1 << D);
    using MI = ModeInfo<D, M_FULL, MIE>;
    static constexpr int NF = MI::NF, NCO = MI::NCO;

    __device__ static int64_t node(const Lat& L, int cx, int cy, int cz, int n) {
        if (Q2) return (int64_t)(2 * cy + n / 3) * (2 * L.nx + 1) + 2 * cx + n % 3;
        return vertex_id(L, cx + (n & 1), cy + ((n >> 1) & 1), D == 3 ? cz + ((n >> 2) & 1) : 0);
    }

    __device__ static void compute(const CoarseArgs& C, const CoarseData& S, const int* ids, int64_t cell,
                                   double (&o)[NCO][NPC]) {
        const OpArgs& A = C.A;
        const Lat& L = A.L;
        const int64_t V = L.V;
        double cv[NF][NPC];
#pragma unroll
        for (int n = 0; n < NPC; ++n) {
            const int64_t id = ids[n];
            const unsigned fl = S.fl[id];
#pragma unroll
            for (int i = 0; i < MI::NV; ++i) cv[MI::F_V + i][n] = ((fl >> i) & 1) ? 0.0 : S.d[(int64_t)i * V + id];
#pragma unroll
            for (int i = 0; i < MI::NU; ++i) cv[MI::F_U + i][n] = S.U[(int64_t)i * V + id];
            cv[MI::F_PT][n] = S.pt[id];
            cv[MI::F_U + D][n] = 0.0;       // block-diagonal operator: no G_phiu coupling
        }
        const double* rq = A.rho ? A.rho + cell * NPC : nullptr;
        if constexpr (ISO) {
            if (rq)
                cell_kernel_iso<D, M_FULL, true>(cv, rq, A.K, A.I, o);
            else
                cell_kernel_iso<D, M_FULL, false>(cv, rq, A.K, A.I, o);
        } else if constexpr (Q2 && !MIE) {
            auto load = [&](int f, double (&c)[9]) {
#pragma unroll
                for (int n = 0; n < 9; ++n) c[n] = cv[f][n];
            };
            cell_q2_rows<M_FULL>(load, rq, A.K, C.T, true, o);   // block-diagonal: no coupling
        } else if constexpr (Q2) {
            cell_q2<M_FULL, MIE>(cv, rq, A.K, C.T, o);
        } else if constexpr (MIE) {
            if constexpr (D == 2)
                cell_kernel_miehe2<M_FULL>(cv, rq, A.K, o);
            else
                cell_kernel_miehe3<M_FULL>(cv, rq, A.K, o);
        } else {
            cell_kernel<D, M_FULL>(cv, rq, A.K, o);
        }
    }
};

template <int D, int KIND>
__global__ void __launch_bounds__(CT, 1) coarse_cheb_kernel(const CoarseArgs C) {
    pdl_wait();
    using CC = CoarseCell<D, KIND>;
    constexpr int NCO = CC::NCO, NPC = CC::NPC;
    extern __shared__ double smem[];
    const OpArgs& A = C.A;
    const Lat& L = A.L;
    const int64_t V = L.V;
    const int ncell = L.nx * L.ny * (D == 3 ? L.nz : 1);
    const int tid = threadIdx.x;
    const int nu = D;                                         // displacement components
    constexpr int NC = D + 1;
    // shared memory: cell outputs, then the level's vectors (the level is small)
    double* cellbuf = smem;                                   // [cells][NCO][NPC]
    double* sU = cellbuf + (int64_t)ncell * NCO * NPC;
    double* spt = sU + NC * V;
    double* sinv = spt + V;
    double* sr = sinv + NC * V;
    double* sd = sr + NC * V;
    double* sx = sd + NC * V;
    constexpr int MAXA = CC::Q2 ? 4 : (1 << D);               // cells sharing a vertex / node
    int* cnodes = reinterpret_cast<int*>(sx + NC * V);        // [cells][NPC] node ids, -1: no cell
    int* vadj = cnodes + ncell * NPC;                         // [V][MAXA] cell * NPC + corner, -1 pad
    uint8_t* sfl = reinterpret_cast<uint8_t*>(vadj + (int64_t)V * MAXA);
    for (int i = tid; i < NC * (int)V; i += CT) {
        sU[i] = A.U[i];
        sinv[i] = C.inv[i];
    }
    for (int i = tid; i < (int)V; i += CT) {
        spt[i] = A.pt[i];
        sfl[i] = A.flags[i];
    }
    const CoarseData S{sU, spt, sfl, sd};
    // lattice points of the vertex pass
    const int px = CC::Q2 ? 2 * L.nx + 1 : L.nx + 1;
    const int py = CC::Q2 ? 2 * L.ny + 1 : L.ny + 1;
    const int pz = D == 3 ? L.nz + 1 : 1;
    const int npts = px * py * pz;
    // index tables, once: the nodes of every cell, and for every vertex its
    // (cell, corner) pairs in increasing cell order (the fixed summation order)
    for (int c = tid; c < ncell; c += CT) {
        const int cx = c % L.nx, t = c / L.nx;
        const int cy = D == 3 ? t % L.ny : t, cz = D == 3 ? t / L.ny : 0;
        const bool ex = CC::Q2 || cell_exists<D>(L, cx, cy, cz);
#pragma unroll
        for (int n = 0; n < NPC; ++n) cnodes[c * NPC + n] = ex ? (int)CC::node(L, cx, cy, cz, n) : -1;
    }
    for (int p = tid; p < npts; p += CT) {
        const int X = p % px, t = p / px;
        const int Y = D == 3 ? t % py : t, Z = D == 3 ? t / py : 0;
        const int64_t vid = CC::Q2 ? (int64_t)Y * px + X : vertex_id(L, X, Y, Z);
        if (vid < 0) continue;
        int k = 0;
        if (CC::Q2) {
            const int cx0 = (X & 1) ? X >> 1 : (X >> 1) - 1, cx1 = X >> 1;
            const int cy0 = (Y & 1) ? Y >> 1 : (Y >> 1) - 1, cy1 = Y >> 1;
            for (int cy = cy0; cy <= min(cy1, L.ny - 1); ++cy) {
                if (cy < 0) continue;
                for (int cx = cx0; cx <= min(cx1, L.nx - 1); ++cx) {
                    if (cx < 0) continue;
                    vadj[vid * MAXA + k++] = (cx + L.nx * cy) * NPC + (X - 2 * cx) + 3 * (Y - 2 * cy);
                }
            }
        } else {
            for (int dz = (D == 3 ? 1 : 0); dz >= 0; --dz)
                for (int dy = 1; dy >= 0; --dy)
                    for (int dx = 1; dx >= 0; --dx) {
                        const int cx = X - dx, cy = Y - dy, cz = D == 3 ? Z - dz : 0;
                        if (!cell_exists<D>(L, cx, cy, cz)) continue;
                        vadj[vid * MAXA + k++] = (cx + L.nx * (cy + L.ny * cz)) * NPC + (dx | (dy << 1) | (dz << 2));
                    }
        }
        for (; k < MAXA; ++k) vadj[vid * MAXA + k] = -1;
    }

    // x = d = inv b / theta, r = b            (mgsolve.py:95, 103-106 from x = 0)
    const double thu = C.coef_u[0], thp = C.coef_p[0];
    for (int i = tid; i < (D + 1) * (int)V; i += CT) {
        const double ri = C.b[i];
        const double di = (C.inv[i] * ri) / (i < nu * V ? thu : thp);
        sr[i] = ri;
        sd[i] = di;
        sx[i] = 0.0 + di;
    }
    const int steps = max(C.deg_u, C.deg_p) - 1;
    for (int s = 0; s < steps; ++s) {
        __syncthreads();                                      // d of the previous step complete
        if (tid < ncell && cnodes[tid * NPC] >= 0) {
            double o[NCO][NPC];
            {
                CC::compute(C, S, cnodes + tid * NPC, tid, o);
#pragma unroll
                for (int k = 0; k < NCO; ++k)
#pragma unroll
                    for (int n = 0; n < NPC; ++n) cellbuf[((int64_t)tid * NCO + k) * NPC + n] = o[k][n];
            }
        }
        __syncthreads();
        const bool up_u = s < C.deg_u - 1, up_p = s < C.deg_p - 1;
        for (int vid = tid; vid < (int)V; vid += CT) {
            double acc[NCO];
#pragma unroll
            for (int k = 0; k < NCO; ++k) acc[k] = 0.0;
#pragma unroll
            for (int a = 0; a < MAXA; ++a) {
                const int e = vadj[vid * MAXA + a];
                if (e < 0) break;
                const int c = e / NPC, n = e - c * NPC;
#pragma unroll
                for (int k = 0; k < NCO; ++k) acc[k] += cellbuf[((int64_t)c * NCO + k) * NPC + n];
            }
            const unsigned fl = sfl[vid];
#pragma unroll
            for (int k = 0; k < NCO; ++k) {
                const bool phi = k == D;
                if (phi ? !up_p : !up_u) continue;
                const int64_t g = (int64_t)k * V + vid;
                const double dk = sd[g];
                const double Av = ((fl >> k) & 1) ? dk : acc[k];          // identity rows
                const double* cf = phi ? C.coef_p : C.coef_u;
                const double rr = sr[g] - Av;
                const double dn = cf[1 + 2 * s] * dk + cf[2 + 2 * s] * (sinv[g] * rr);
                sr[g] = rr;
                sd[g] = dn;
                sx[g] = sx[g] + dn;
            }
        }
    }
    __syncthreads();
    for (int i = tid; i < (D + 1) * (int)V; i += CT) C.x[i] = sx[i];    // the solve's result
}

template <int D, int KIND>
static int launch_coarse(const CoarseArgs& C, size_t smem, cudaStream_t s) {
    static size_t done = 0;
    if (smem > 48 * 1024 && smem > done) {
        cudaFuncSetAttribute(coarse_cheb_kernel<D, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        done = smem;
    }
    pdl_launch(coarse_cheb_kernel<D, KIND>, dim3(1), dim3(CT), smem, s, C);
    return check_launch("pffmg_coarse_cheb");
}

}  // namespace pffmg

using namespace pffmg;

extern "C" int pffmg_coarse_cheb(const pffmg_lattice* lat, const pffmg_state* st, const double* b, double* x,
                                 double* r, double* d, const double* invdiag, const double* coef_u,
                                 int deg_u, const double* coef_p, int deg_p, void* stream) {
    CoarseArgs C{};
    PFFMG_REQUIRE(lat && st && st->U && st->phi_tilde && st->flags, "pffmg_coarse_cheb: null lattice/state");
    int rc = make_lat(lat, &C.A.L);
    if (rc) return rc;
    rc = make_consts(lat, st, &C.A.K);
    if (rc) return rc;
    PFFMG_REQUIRE(b && x && r && d && invdiag && coef_u && coef_p && deg_u >= 1 && deg_p >= 1,
                  "pffmg_coarse_cheb: bad arguments");
    PFFMG_REQUIRE(st->split == 0 || st->split == 1, "pffmg_coarse_cheb: unknown split");
    const Lat& L = C.A.L;
    PFFMG_REQUIRE(L.own_lo == 0 && L.own_hi == (L.order == 2 ? 2 * L.ny + 1 : (L.dim == 3 ? L.nz : L.ny) + 1) &&
                      L.plane0 == 0,
                  "pffmg_coarse_cheb: whole lattices only");
    const int ncell = L.nx * L.ny * (L.dim == 3 ? L.nz : 1);
    if (ncell > CT) {
        set_error("pffmg_coarse_cheb: %d lattice cells > %d (use the per-step kernels)", ncell, CT);
        return PFFMG_ERR_UNSUPPORTED;
    }
    C.A.U = st->U;
    C.A.pt = st->phi_tilde;
    C.A.rho = st->rho;
    C.A.flags = st->flags;
    C.b = b;
    C.x = x;
    C.r = r;
    C.d = d;
    C.inv = invdiag;
    C.coef_u = coef_u;
    C.coef_p = coef_p;
    C.deg_u = deg_u;
    C.deg_p = deg_p;
    C.T = make_q2_host(L.hx, L.hy);
    const int nco = L.dim + 1;
    const int npc = L.order == 2 ? 9 : (1 << L.dim);
    const int maxa = L.order == 2 ? 4 : (1 << L.dim);
    const size_t smem = sizeof(double) * ((size_t)ncell * nco * npc + (size_t)L.V * (5 * nco + 1)) +
                        sizeof(int) * ((size_t)ncell * npc + (size_t)L.V * maxa) + (size_t)L.V + 16;
    if (smem > 200 * 1024) {
        set_error("pffmg_coarse_cheb: level needs %zu B of shared memory > 200 KiB (use the per-step kernels)", smem);
        return PFFMG_ERR_UNSUPPORTED;
    }
    C.A.I = make_iso_host(C.A.K);
    const cudaStream_t s = as_stream(stream);
    const bool iso = L.order == 1 && L.hx == L.hy && (L.dim == 2 || L.hz == L.hx);
    int kind = (L.order == 2 ? 2 : 0) + (st->split == 1 ? 1 : 0);
    if (kind == 0 && iso) kind = 4;
    if (L.dim == 2) {
        switch (kind) {
            case 0: return launch_coarse<2, 0>(C, smem, s);
            case 1: return launch_coarse<2, 1>(C, smem, s);
            case 2: return launch_coarse<2, 2>(C, smem, s);
            case 3: return launch_coarse<2, 3>(C, smem, s);
            default: return launch_coarse<2, 4>(C, smem, s);
        }
    }
    return kind == 0 ? launch_coarse<3, 0>(C, smem, s)
                     : (kind == 1 ? launch_coarse<3, 1>(C, smem, s) : launch_coarse<3, 4>(C, smem, s));
}
