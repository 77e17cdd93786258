// The fused matrix-free vmult of the linearised PFF Jacobian on a lattice
// level: stage vertex rows/planes in shared memory, one thread per cell
// (gather -> sum-factorised interpolation -> pointwise physics -> integrate),
// then a deterministic vertex sum (warp shuffles in x, shared memory in y,
// registers carried in the marching direction) and a fused epilogue
// (store / residual / Chebyshev step / diagonal).
//
// Kernel templates (included by op2d.cu / op3d.cu, which instantiate them).
// Replaces reference model.py:368-413 (apply, apply_block, diagonal) with
// fem.py:203-225 (masked gather, bincount scatter) and the vector updates of
// mgsolve.py:82-113 (chebyshev_apply) and 227 (residual) fused in.
#pragma once
#include <cmath>

#include "cellops_iso.cuh"
#include "cellops_miehe.cuh"

namespace pffmg {

enum Epi { E_STORE = 0, E_RESID = 1, E_CHEB = 2, E_CHEB0 = 3, E_DIAG = 4, E_RESZ = 5 };

struct OpArgs {
    Lat L;
    Consts K;
    IsoK I;                            // folded constants for isotropic cells (host-built)
    const double* __restrict__ v;      // block base of the input field (component stride V)
    double* __restrict__ out;          // STORE / RESID / DIAG output
    const double* __restrict__ U;
    const double* __restrict__ pt;
    const double* __restrict__ rho;
    const double* __restrict__ ptab;   // per-QP a_phiphi table (pffmg_phi_coef) or NULL
    const uint8_t* __restrict__ flags;
    // epilogue operands (block base pointers, component stride V)
    const double* __restrict__ b;
    double* __restrict__ r;
    double* __restrict__ x;            // CHEB: updated in place; CHEB0: x_out
    double* __restrict__ dout;
    const double* __restrict__ inv;
    double c1, c2;                     // CHEB: c_dd, c_dr   CHEB0: theta
    const double* __restrict__ coef;   // if set, c1/c2 are read from device memory (coef[0], coef[1])
    const double* __restrict__ coef2;  // block-diagonal mode: the phase-field component's coefficients
    int nocoup;                        // FULL mode without the G_phiu coupling (block-diagonal operator)
    int x_add_din;                     // CHEB: 1: x = (x + d_in) + d_out instead of x += d_out;
                                       // 2: first step after the x = 0 start: x_old = 0 + d_in, x is not read
    const double* __restrict__ r_in;   // CHEB: residual read from here (written to r) if set
    int planes_per_cta;
    int nseg;                          // 2D warp kernel: 30-column segments per row
    int sched;                         // work schedule of the streaming kernels (tuning, see launchers)
    int premasked;                     // PFFMG_HINT_PREMASKED
    int ends;                          // PFFMG_HINT_ENDS: strips = {own_lo}, {own_hi - 1}
    int split;                         // 0 NoSplit, 1 Miehe spectral split (2D)
};

// ------------------------------------------------------------ epilogue

// Epilogue operands loaded ahead of the cell work (their DRAM latency then
// overlaps the stencil arithmetic instead of stalling the epilogue).
template <int NCO, int EPI>
struct EpiIn {
    static constexpr int NL = EPI == E_CHEB ? 3 : (EPI == E_CHEB0 ? 2 : (EPI == E_RESID ? 1 : 0));
    double a[NL > 0 ? NL : 1][NCO];
};

template <int NCO, int EPI>
__device__ __forceinline__ void epi_load(const OpArgs& A, int64_t vid, EpiIn<NCO, EPI>& e) {
    const int64_t V = A.L.V;
#pragma unroll
    for (int k = 0; k < NCO; ++k) {
        const int64_t g = (int64_t)k * V + vid;
        if (EPI == E_CHEB) {
            e.a[0][k] = A.r_in ? __ldg(A.r_in + g) : A.r[g];
            e.a[1][k] = __ldg(A.inv + g);
            e.a[2][k] = A.x_add_din == 2 ? 0.0 : A.x[g];
        } else if (EPI == E_CHEB0) {
            e.a[0][k] = __ldg(A.b + g);
            e.a[1][k] = __ldg(A.inv + g);
        } else if (EPI == E_RESID) {
            e.a[0][k] = __ldg(A.b + g);
        }
    }
}

// The same operands staged into shared memory with cp.async (slot = NL x NCO
// doubles of the calling thread): the prefetch then holds no registers across
// the cell work (in the register-capped 3D kernels a register prefetch was
// spilled, and the spill store waited for the load).
template <int NCO, int EPI>
__device__ __forceinline__ void epi_stage(const OpArgs& A, int64_t vid, double* slot) {
    const int64_t V = A.L.V;
#pragma unroll
    for (int k = 0; k < NCO; ++k) {
        const int64_t g = (int64_t)k * V + vid;
        if (EPI == E_CHEB) {
            cp_async8(slot + 0 * NCO + k, (A.r_in ? A.r_in : A.r) + g, true);
            cp_async8(slot + 1 * NCO + k, A.inv + g, true);
            if (A.x_add_din != 2) cp_async8(slot + 2 * NCO + k, A.x + g, true);
        } else if (EPI == E_CHEB0) {
            cp_async8(slot + 0 * NCO + k, A.b + g, true);
            cp_async8(slot + 1 * NCO + k, A.inv + g, true);
        } else if (EPI == E_RESID) {
            cp_async8(slot + 0 * NCO + k, A.b + g, true);
        }
    }
}

template <int NCO, int EPI>
__device__ __forceinline__ void epi_unstage(const double* slot, EpiIn<NCO, EPI>& e) {
    constexpr int NL = EpiIn<NCO, EPI>::NL;
#pragma unroll
    for (int l = 0; l < NL; ++l)
#pragma unroll
        for (int k = 0; k < NCO; ++k) e.a[l][k] = slot[l * NCO + k];
}

// Vertex epilogue (model.py:373-374, 390-391, 412, 459; mgsolve.py:95-111, 227)
// with the operands from epi_load.
template <int NCO, int COMP0, int EPI>
__device__ __forceinline__ void epilogue(const OpArgs& A, int64_t vid, uint8_t fl, const double (&acc)[NCO],
                                             const double (&vin)[NCO], const EpiIn<NCO, EPI>& e) {
    const int64_t V = A.L.V;
#pragma unroll
    for (int k = 0; k < NCO; ++k) {
        const bool con = (fl >> (COMP0 + k)) & 1;
        const int64_t g = (int64_t)k * V + vid;
        if (EPI == E_DIAG) {
            A.out[g] = con ? 1.0 : acc[k];                       // model.py:412
            continue;
        }
        if (EPI == E_RESZ) {
            A.out[g] = con ? 0.0 : acc[k];                       // model.py:459
            continue;
        }
        const double Av = con ? vin[k] : acc[k];                 // model.py:373-374, 390-391
        if (EPI == E_STORE) {
            A.out[g] = Av;
        } else if (EPI == E_RESID) {
            A.out[g] = e.a[0][k] - Av;                           // mgsolve.py:227
        } else if (EPI == E_CHEB) {                              // mgsolve.py:108-111
            const double rr = e.a[0][k] - Av;
            const double* cf = (A.coef2 && COMP0 + k == A.L.dim) ? A.coef2 : A.coef;
            const double c1 = cf ? __ldg(cf) : A.c1, c2 = cf ? __ldg(cf + 1) : A.c2;
            const double dn = c1 * vin[k] + c2 * (e.a[1][k] * rr);
            A.r[g] = rr;
            A.dout[g] = dn;
            // (2: x was started as 0.0 + d_in by the x = 0 init, which did not store it)
            const double xo = A.x_add_din == 2 ? 0.0 + vin[k] : e.a[2][k];
            A.x[g] = A.x_add_din == 1 ? (xo + vin[k]) + dn : xo + dn;
        } else {                                                 // E_CHEB0: mgsolve.py:95, 105
            const double rr = e.a[0][k] - Av;
            A.r[g] = rr;
            const double* cf = (A.coef2 && COMP0 + k == A.L.dim) ? A.coef2 : A.coef;
            A.dout[g] = (e.a[1][k] * rr) / (cf ? __ldg(cf) : A.c1);
        }
    }
}

// Load one staged vertex: all NF fields (raw) + flags.
template <int D, int MODE, bool SPLIT = false>
__device__ __forceinline__ void load_vertex(const OpArgs& A, int64_t vid,
                                            double (&f)[ModeInfo<D, MODE, SPLIT>::NF], uint8_t& fl) {
    using MI = ModeInfo<D, MODE, SPLIT>;
    const int64_t V = A.L.V;
    if (vid < 0) {
#pragma unroll
        for (int i = 0; i < MI::NF; ++i) f[i] = 0.0;
        fl = 0;
        return;
    }
#pragma unroll
    for (int i = 0; i < MI::NV; ++i) f[MI::F_V + i] = __ldg(A.v + (int64_t)i * V + vid);
#pragma unroll
    for (int i = 0; i < MI::NU; ++i) f[MI::F_U + i] = __ldg(A.U + (int64_t)i * V + vid);
    if (MI::PT) f[MI::F_PT] = __ldg(A.pt + vid);
    fl = __ldg(A.flags + vid);
}

// ================================================================ 2D (warps)
// Warp-independent 2D kernel.  Each warp owns a segment of 30 vertex columns
// and a strip of vertex rows.  Lanes load columns x0..x0+31 (x0 = 30*seg - 1);
// lanes 0..30 compute cells cx = x0 + L (lane 0's cell is shared with the
// neighbouring segment), lanes 1..30 finalise their vertex column.  Rows are
// staged into a warp-private 4-slot shared-memory ring with cp.async three
// rows ahead (fp64 fields: one 8-byte copy per lane and field; constraint
// flags: the 9 aligned 32-bit words covering the row's 32 flag bytes, ids of a
// lattice row being contiguous).  No block-wide barriers.  Unless the caller
// promises pre-masked inputs (PFFMG_HINT_PREMASKED -- true inside the V-cycle,
// CG-Lanczos and GMRES, whose vectors are always zero at constrained dofs),
// every lane zeroes its own constrained entries once the row has landed
// (the masked gather of fem.py:205-206, once per vertex).

template <bool BOX>
struct RowAddr {
    // vertex id of (x, y) or -1 (32-bit: every supported level has < 2^31 dofs)
    __device__ __forceinline__ static int id(const Lat& L, int x, int y) {
        if (BOX) {
            if ((unsigned)x > (unsigned)L.nx || (unsigned)y > (unsigned)L.ny) return -1;
            return y * (L.nx + 1) + x;
        }
        return (int)vertex_id(L, x, y, 0);
    }
    // "virtual" id of column x in row y: ids of a row are contiguous, so this
    // extends the row's numbering to columns outside the row (flag staging)
    __device__ __forceinline__ static int vid_virtual(const Lat& L, int x, int y) {
        if (BOX) return y * (L.nx + 1) + x;
        if ((unsigned)y > (unsigned)L.ny) return 0;
        return (int)__ldg(L.vrow_off + y) + (x - __ldg(L.vrow_lo + y));
    }
};

// TAB (isotropic NoSplit; FULL mode only with nocoup): the block-diagonal
// operator / the phi block with a_phiphi read from the per-QP table A.ptab --
// U is not staged.
template <int MODE, int EPI, int NW, bool ISO, bool RHO, bool BOX, bool PRE, bool MIE = false, bool TAB = false>
#ifndef PFFMG_MINB_FULL
#define PFFMG_MINB_FULL 4
#endif
#ifndef PFFMG_MINB_BLK
#define PFFMG_MINB_BLK 8
#endif
__global__ void __launch_bounds__(32 * NW, MIE ? 2 : (MODE == M_FULL ? PFFMG_MINB_FULL : PFFMG_MINB_BLK))
op2dw_kernel(const OpArgs A) {
    pdl_wait();
    constexpr int D = 2, NP = 4;
    using MI = ModeInfo<D, MODE, MIE>;
    static_assert(!TAB || ((MODE == M_FULL || MODE == M_PBLK) && ISO && !MIE),
                  "the table path is the isotropic block-diagonal operator or phi block");
    constexpr int NF = TAB ? (MODE == M_FULL ? MI::NV + 1 : MI::NV) : MI::NF, NCO = MI::NCO, NV = MI::NV;
    constexpr int RING = 4, W = 32, SLOT = NF * W;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* sv = reinterpret_cast<double*>(smem_raw) + w * (RING * SLOT);

    const Lat& L = A.L;
    const int gw = (int)blockIdx.x * NW + w;
    const int seg = gw % A.nseg, strip = gw / A.nseg;
    if (A.ends && strip > 1) return;
    const int vy0 = A.ends ? (strip == 0 ? L.own_lo : L.own_hi - 1) : L.own_lo + strip * A.planes_per_cta;
    if (vy0 >= L.own_hi) return;
    const int vy1 = A.ends ? vy0 + 1 : min(vy0 + A.planes_per_cta, L.own_hi);
    const int x0 = 30 * seg - 1;
    const int cx = x0 + lane;
    const bool col_cell = lane <= 30 && cx >= 0 && cx < L.nx;
    const bool col_fin = lane >= 1 && lane <= 30;

    const double* fsrc[NF];
#pragma unroll
    for (int i = 0; i < NV; ++i) fsrc[MI::F_V + i] = A.v + (int64_t)i * L.V;
    if constexpr (TAB) {
        if constexpr (MODE == M_FULL) fsrc[NV] = A.pt;
    } else {
#pragma unroll
        for (int i = 0; i < MI::NU; ++i) fsrc[MI::F_U + i] = A.U + (int64_t)i * L.V;
        if (MI::PT) fsrc[MI::F_PT] = A.pt;
    }

    // Stage row y into the ring slot (one column per lane); the lane's own
    // constraint byte of that row comes back in a register (a plain load: it
    // is first read one to three iterations later, so its latency is hidden
    // and no shared-memory flag words / offsets are needed).
    auto issue = [&](int y, int slot) -> unsigned {
        double* dst = sv + slot * SLOT + lane;
        const int vid = RowAddr<BOX>::id(L, cx, y);
        const bool ok = vid >= 0;
        const int off = ok ? vid : 0;
#pragma unroll
        for (int f = 0; f < NF; ++f) cp_async8(dst + f * W, fsrc[f] + off, ok);
        cp_async_commit();
        return ok ? (unsigned)__ldg(A.flags + off) : 0u;
    };
    auto mask_row = [&](int slot, unsigned fl) {   // fem.py:205-206, once per vertex
        if (PRE || NV == 0) return;
        double* row = sv + slot * SLOT;
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if ((fl >> (MI::COMP0 + i)) & 1) row[i * W + lane] = 0.0;
    };

    // flags of rows cy (bottom), cy+1 (top), cy+2 (in flight)
    unsigned fl_bot = issue(vy0 - 1, 0);
    unsigned fl_top = issue(vy0, 1);
    unsigned fl_nxt = issue(vy0 + 1, 2);
    cp_async_wait<1>();                          // rows vy0-1, vy0 landed
    __syncwarp();
    double raw_bot[NV > 0 ? NV : 1];             // raw own-column v of the bottom row
#pragma unroll
    for (int i = 0; i < NV; ++i) raw_bot[i] = sv[0 * SLOT + i * W + lane];
    mask_row(0, fl_bot);
    double raw_top[NV > 0 ? NV : 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) raw_top[i] = sv[1 * SLOT + i * W + lane];
    mask_row(1, fl_top);

    double carry[NCO];
#pragma unroll
    for (int k = 0; k < NCO; ++k) carry[k] = 0.0;

    int it = 0;
    for (int cy = vy0 - 1; cy < vy1; ++cy, ++it) {
        const int s0 = it & 3, s1 = (it + 1) & 3;
        // vertex finalised this iteration and its epilogue operands (loaded early)
        const int vid_f = (cy >= vy0 && col_fin) ? RowAddr<BOX>::id(L, cx, cy) : -1;
        EpiIn<NCO, EPI> ein;
        if (vid_f >= 0) epi_load<NCO, EPI>(A, vid_f, ein);
        if (it > 0) {                            // row cy+1 becomes the top row
            cp_async_wait<1>();
            __syncwarp();
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                raw_bot[i] = raw_top[i];
                raw_top[i] = sv[s1 * SLOT + i * W + lane];
            }
            mask_row(s1, fl_top);
        }
        unsigned fl_new = 0;
        if (cy + 3 <= vy1)
            fl_new = issue(cy + 3, (it + 3) & 3);
        else
            cp_async_commit();
        if (!PRE) __syncwarp();                  // neighbour lanes' masking visible

        const double* r0 = sv + s0 * SLOT;
        const double* r1 = sv + s1 * SLOT;
        double o[NCO][NP];
        // FULL (operator / residual / block-diagonal smoother): every lane runs
        // the cell kernel (lane 31 and absent cells on a copy of a valid
        // column, outputs zeroed by a select) -- no divergent branch around
        // the cell work (cfg2 vmult 36.1 -> 34.5 us, ncu).  The register-capped
        // block modes keep the branch (the select costs them spills).
        constexpr bool BRANCHLESS = MODE == M_FULL;
        const bool cell = col_cell && (BOX ? (cy >= 0 && cy < L.ny) : cell_exists<D>(L, cx, cy, 0));
        if (BRANCHLESS || cell) {
            const int ll = lane < 31 ? lane : 30;
            double cv[NF][NP];
#pragma unroll
            for (int i = 0; i < NF; ++i) {
                cv[i][0] = r0[i * W + ll];
                cv[i][1] = r0[i * W + ll + 1];
                cv[i][2] = r1[i * W + ll];
                cv[i][3] = r1[i * W + ll + 1];
            }
            if constexpr (MODE == M_FULL && !TAB) {   // block-diagonal operator: no G_phiu coupling
                if (A.nocoup) {                  // (T_phiu = 0 when phi(U) reads 0, model.py:299-303)
#pragma unroll
                    for (int n = 0; n < NP; ++n) cv[MI::F_U + D][n] = 0.0;
                }
            }
            const int64_t lc = cell ? ((int64_t)cx + (int64_t)L.nx * cy) : 0;   // rho row of a real cell
            const double* rq = RHO ? A.rho + lc * NP : nullptr;
            if constexpr (TAB && MODE == M_FULL) {
                cell_bd_tab2<RHO>(cv, rq, A.ptab + lc, (int64_t)L.nx * L.ny, A.K, A.I, o);
            } else if constexpr (TAB) {
                cell_pblk_tab2(cv, A.ptab + lc, (int64_t)L.nx * L.ny, A.K, A.I, o);
            } else if constexpr (MIE) {   // spectral split: modulus field resolved at run time
                cell_kernel_miehe2<MODE>(cv, A.rho ? A.rho + lc * NP : nullptr, A.K, o);
            } else {
                if (ISO)
                    cell_kernel_iso<D, MODE, RHO>(cv, rq, A.K, A.I, o);
                else
                    cell_kernel<D, MODE>(cv, rq, A.K, o);
            }
            // Lane 31's outputs are never used (its left corners belong to a
            // vertex it does not finalise, its right corners are shuffled to
            // nobody), so only warps holding an absent cell in lanes 0..30 --
            // the lattice's edge columns / rows -- need the select: a
            // warp-uniform branch around it.
            if (BRANCHLESS && __any_sync(0xffffffffu, !cell && lane < 31)) {
#pragma unroll
                for (int k = 0; k < NCO; ++k)
#pragma unroll
                    for (int n = 0; n < NP; ++n) o[k][n] = cell ? o[k][n] : 0.0;
            }
        } else {
#pragma unroll
            for (int k = 0; k < NCO; ++k)
#pragma unroll
                for (int n = 0; n < NP; ++n) o[k][n] = 0.0;
        }

        double bot[NCO], top[NCO];
#pragma unroll
        for (int k = 0; k < NCO; ++k) {
            const double q0 = __shfl_up_sync(0xffffffffu, o[k][1], 1);
            const double q1 = __shfl_up_sync(0xffffffffu, o[k][3], 1);
            bot[k] = o[k][0] + q0;
            top[k] = o[k][2] + q1;
        }
        if (vid_f >= 0) {
            double acc[NCO], vin[NCO];
#pragma unroll
            for (int k = 0; k < NCO; ++k) {
                acc[k] = carry[k] + bot[k];
                vin[k] = (MODE == M_DIAG) ? 0.0 : raw_bot[k < NV ? k : 0];
            }
            epilogue<NCO, MI::COMP0, EPI>(A, vid_f, (uint8_t)fl_bot, acc, vin, ein);
        }
#pragma unroll
        for (int k = 0; k < NCO; ++k) carry[k] = top[k];
        fl_bot = fl_top;
        fl_top = fl_nxt;
        fl_nxt = fl_new;
        __syncwarp();                            // slot s0 free for the next issue
    }
    cp_async_wait<0>();
}

// ======================================================================= 3D
// CTA = TY warps; warp w <-> cell row cy0 + w, lane <-> cell column cx0 + lane.
// Finalises vertices (cx0 + lane, cy0 + w) for lane >= 1, w >= 1; marches in z.

template <int MODE, int EPI, int TY, bool ISO, bool MIE = false>
__global__ void __launch_bounds__(32 * TY) op3d_kernel(const OpArgs A) {
    pdl_wait();
    constexpr int D = 3, NP = 8;
    using MI = ModeInfo<D, MODE, MIE>;
    constexpr int NF = MI::NF, NCO = MI::NCO;
    constexpr int TXV = 33, TYV = TY + 1, TV = TXV * TYV;
    constexpr int NT = 32 * TY;
    constexpr int SLOTS = (TV + NT - 1) / NT;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sv = reinterpret_cast<double*>(smem_raw);                 // [2][NF][TV]
    double* sy = sv + 2 * NF * TV;                                     // [TY][2][NCO][32]
    uint8_t* sfl = reinterpret_cast<uint8_t*>(sy + TY * 2 * NCO * 32); // [2][TV]

    const Lat& L = A.L;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int cx0 = -1 + (int)blockIdx.x * 31;
    const int cy0 = -1 + (int)blockIdx.y * (TY - 1);
    const int vz0 = A.ends ? ((int)blockIdx.z == 0 ? L.own_lo : L.own_hi - 1)
                           : L.own_lo + (int)blockIdx.z * A.planes_per_cta;
    const int vz1 = A.ends ? vz0 + 1 : min(vz0 + A.planes_per_cta, L.own_hi);
    const int cx = cx0 + lane, cy = cy0 + w;

    auto SV = [&](int buf, int f, int j) -> double& { return sv[(buf * NF + f) * TV + j]; };
    auto stage_now = [&](int z, int buf) {
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            const int j = tid + s * NT;
            if (j < TV) {
                const int jx = j % TXV, jy = j / TXV;
                double f[NF];
                uint8_t fl;
                load_vertex<D, MODE, MIE>(A, vertex_id(L, cx0 + jx, cy0 + jy, z), f, fl);
#pragma unroll
                for (int i = 0; i < NF; ++i) SV(buf, i, j) = f[i];
                sfl[buf * TV + j] = fl;
            }
        }
    };

    stage_now(vz0 - 1, 0);
    stage_now(vz0, 1);
    __syncthreads();

    double carry[NCO];
#pragma unroll
    for (int k = 0; k < NCO; ++k) carry[k] = 0.0;

    int b0 = 0;
    for (int cz = vz0 - 1; cz < vz1; ++cz) {
        const int b1 = b0 ^ 1;
        const int64_t vid_f = (w >= 1 && cz >= vz0 && lane >= 1) ? vertex_id(L, cx, cy, cz) : -1;
        EpiIn<NCO, EPI> ein;
        if (vid_f >= 0) epi_load<NCO, EPI>(A, vid_f, ein);
        double pf[SLOTS][NF];
        uint8_t pfl[SLOTS];
        const bool need_next = (cz + 2 <= vz1);
        if (need_next) {
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const int j = tid + s * NT;
                const int64_t vid = j < TV ? vertex_id(L, cx0 + j % TXV, cy0 + j / TXV, cz + 2) : -1;
                load_vertex<D, MODE, MIE>(A, vid, pf[s], pfl[s]);
            }
        }

        double o[NCO][NP];
        if (cell_exists<D>(L, cx, cy, cz)) {
            double cv[NF][NP];
#pragma unroll
            for (int n = 0; n < NP; ++n) {
                const int bb = (n >> 2) ? b1 : b0;
                const int j = (lane + (n & 1)) + TXV * (w + ((n >> 1) & 1));
                const uint8_t fl = sfl[bb * TV + j];
#pragma unroll
                for (int i = 0; i < NF; ++i) {
                    double val = SV(bb, i, j);
                    if (i < MI::NV && ((fl >> (MI::COMP0 + i)) & 1)) val = 0.0;
                    cv[i][n] = val;
                }
            }
            if constexpr (MODE == M_FULL) {      // block-diagonal operator: no G_phiu coupling
                if (A.nocoup) {
#pragma unroll
                    for (int n = 0; n < NP; ++n) cv[MI::F_U + D][n] = 0.0;
                }
            }
            const double* rq =
                A.rho ? A.rho + ((int64_t)cx + (int64_t)L.nx * (cy + (int64_t)L.ny * cz)) * NP : nullptr;
            if constexpr (MIE) {
                cell_kernel_miehe3<MODE>(cv, rq, A.K, o);
            } else {
                if (ISO && rq) cell_kernel_iso<D, MODE, true>(cv, rq, A.K, A.I, o);
                else if (ISO) cell_kernel_iso<D, MODE, false>(cv, rq, A.K, A.I, o);
                else cell_kernel<D, MODE>(cv, rq, A.K, o);
            }
        } else {
#pragma unroll
            for (int k = 0; k < NCO; ++k)
#pragma unroll
                for (int n = 0; n < NP; ++n) o[k][n] = 0.0;
        }

        // x-combine -> part[yb][zb][k] at vertex column x = cx
        double part[2][2][NCO];
#pragma unroll
        for (int yb = 0; yb < 2; ++yb)
#pragma unroll
            for (int zb = 0; zb < 2; ++zb)
#pragma unroll
                for (int k = 0; k < NCO; ++k) {
                    const int nl = (yb << 1) | (zb << 2);
                    const double rr = __shfl_up_sync(0xffffffffu, o[k][nl | 1], 1);
                    part[yb][zb][k] = o[k][nl] + rr;
                }
        // y-combine through shared memory: row w publishes its y=1 partials
#pragma unroll
        for (int zb = 0; zb < 2; ++zb)
#pragma unroll
            for (int k = 0; k < NCO; ++k) sy[((w * 2 + zb) * NCO + k) * 32 + lane] = part[1][zb][k];
        __syncthreads();
        if (w >= 1) {
            double vp[2][NCO];
#pragma unroll
            for (int zb = 0; zb < 2; ++zb)
#pragma unroll
                for (int k = 0; k < NCO; ++k)
                    vp[zb][k] = part[0][zb][k] + sy[(((w - 1) * 2 + zb) * NCO + k) * 32 + lane];
            if (vid_f >= 0) {
                const int j = lane + TXV * w;
                const uint8_t fl = sfl[b0 * TV + j];
                double acc[NCO], vin[NCO];
#pragma unroll
                for (int k = 0; k < NCO; ++k) {
                    acc[k] = carry[k] + vp[0][k];
                    vin[k] = (MODE == M_DIAG) ? 0.0 : SV(b0, MI::F_V + k, j);
                }
                epilogue<NCO, MI::COMP0, EPI>(A, vid_f, fl, acc, vin, ein);
            }
#pragma unroll
            for (int k = 0; k < NCO; ++k) carry[k] = vp[1][k];
        }
        __syncthreads();
        if (need_next) {
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const int j = tid + s * NT;
                if (j < TV) {
#pragma unroll
                    for (int i = 0; i < NF; ++i) SV(b0, i, j) = pf[s][i];
                    sfl[b0 * TV + j] = pfl[s];
                }
            }
        }
        __syncthreads();
        b0 = b1;
    }
}


}  // namespace pffmg
