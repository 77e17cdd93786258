// 3D fused operator for isotropic hexahedra: a CTA of 256 threads owns a tile
// of TX (x) x TY (y) cells (TX TY = 256, one cell per thread: tx = tid % TX,
// ty = tid / TX) and marches it in z.  The staged vertex plane is
// (TY + 1) x (TX + 1), so every thread computes a real cell; the vertices
// (x0 + tx, y0 + ty) with tx, ty >= 1 are finalised by the tile (its four
// cells are all in it), i.e. neighbouring tiles overlap by one cell row /
// column.  A 16 x 16 tile computes 256 cells per 225 finalised vertices
// (32 x 8: 256 per 217), and its 15-vertex granularity fits lattices of
// 2^k + 1 vertices far better than a 30-column warp segment.
// Vertex planes are staged with cp.async into a 4-slot shared-memory ring two
// planes ahead; the cell work is the streaming cell3_iso kernel; vertex sums:
// x by shuffles, y through shared memory, z by a register carry.  Replaces
// reference model.py:368-392 (+ the fused epilogues of mgsolve.py:82-113,
// 227) for 3D levels.
#pragma once

#include "cell3_iso.cuh"
#include "op_kernels.cuh"

namespace pffmg {

constexpr int T3_NT = 256;                        // threads per CTA of the streaming kernel
constexpr int T3_RING = 5;                        // staged vertex planes: cz, cz+1 read, cz+2 ready, cz+3 landing

template <int TX>
struct Tile3 {
    static constexpr int TY = T3_NT / TX;
    static constexpr int ROWS = TY + 1, COLS = TX + 1, PL = ROWS * COLS;
    static constexpr int EPT = (PL + T3_NT - 1) / T3_NT;   // staged vertices per thread and plane
    // dynamic shared memory of one instantiation (doubles / bytes)
    template <int NF, int NCO, int NLE>
    static constexpr size_t smem() {
        return sizeof(double) * (T3_RING * NF * PL + 2 * TY * NCO * 2 * TX + (size_t)T3_NT * NLE * NCO) +
               T3_RING * PL;
    }
};

// TAB (phi block only): a_phiphi comes from the per-QP table A.ptab, so only
// v is staged (no U planes) -- the phi block becomes an HBM-bound stencil.
template <int MODE, int EPI, int TX, bool RHO, bool BOX, bool PRE, bool TAB = false>
#ifndef PFFMG_3D_FULL_MINB
#define PFFMG_3D_FULL_MINB 1
#endif
__global__ void __launch_bounds__(T3_NT, MODE == M_FULL ? PFFMG_3D_FULL_MINB : (TAB ? 4 : 2)) op3dt_kernel(const OpArgs A) {
    pdl_wait();
    using MI = ModeInfo<3, MODE>;
    using TL = Tile3<TX>;
    constexpr int NF = TAB ? MI::NV : MI::NF, NCO = MI::NCO, NV = MI::NV;
    constexpr int TY = TL::TY, ROWS = TL::ROWS, COLS = TL::COLS, PL = TL::PL, EPT = TL::EPT;
    constexpr int SLOT = NF * PL;                // doubles per staged plane

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sv = reinterpret_cast<double*>(smem_raw);                          // [T3_RING][NF][ROWS][COLS]
    double* sy0 = sv + T3_RING * SLOT;                                          // [2][TY][NCO][2][TX]
    // epilogue operands staged in shared memory where a register prefetch
    // spills (u block, and the Chebyshev variants of FULL); elsewhere they
    // stay in registers (ncu: staging costs the table phi block and RESID ~4%)
    constexpr bool STAGE = MODE == M_UBLK || (MODE == M_FULL && (EPI == E_CHEB || EPI == E_CHEB0));
    constexpr int NLE = STAGE ? EpiIn<NCO, EPI>::NL : 0;                        // staged epilogue operands
    double* sepi = sy0 + 2 * TY * NCO * 2 * TX;                                 // [T3_NT][NLE][NCO]
    unsigned char* sfl = reinterpret_cast<unsigned char*>(sepi + T3_NT * NLE * NCO);   // [T3_RING][PL]

    const Lat& L = A.L;
    const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
    const int V = (int)L.V;

    // Work distribution.  The work items are the (tile, plane) pairs of the
    // occupied tiles (L.tiles3d; every tile of the bounding lattice when
    // absent).  A.sched = 1 (persistent, tile-major): a grid of one wave of
    // resident CTAs, CTA b takes the contiguous items [b W / G, (b + 1) W / G)
    // and marches them as runs of consecutive planes of one tile (one warm-up
    // plane per run) -- equal shares, no wave quantisation: the FP64-bound
    // modes.  A.sched = 2 (grid): CTA = one strip of S = planes_per_cta planes
    // of one tile, strip-major, tiles fastest, so the CTAs running side by side
    // are neighbouring tiles of one strip and their shared halo columns are
    // read while in L2: the bandwidth-bound modes.
    const int ntx = (L.nx + 1 + TX - 2) / (TX - 1);
    const bool listed = TX - 1 == PFFMG_TILE3 && L.tiles3d != nullptr;
    const int ntiles = listed ? L.n_tiles3d : ntx * ((L.ny + 1 + TY - 2) / (TY - 1));
    const int P = A.ends ? 2 : L.own_hi - L.own_lo;          // plane slots per tile
    const int64_t W = (int64_t)ntiles * P;
    int64_t item = W * (int64_t)blockIdx.x / gridDim.x, item_hi = W * ((int64_t)blockIdx.x + 1) / gridDim.x;
    if (A.sched == 2) {
        const int S = A.planes_per_cta;
        const int st = (int)(blockIdx.x / ntiles), t = (int)(blockIdx.x % ntiles);
        item = (int64_t)t * P + (int64_t)st * S;
        item_hi = item + max(0, min(S, P - st * S));
    }
    while (item < item_hi) {
    const int tix = (int)(item / P), kz = (int)(item % P);
    const int len = A.ends ? 1 : (int)min((int64_t)(P - kz), item_hi - item);
    item += len;
    const int tile = listed ? __ldg(L.tiles3d + tix) : tix;
    const int x0 = (TX - 1) * (tile % ntx) - 1;
    const int y0 = (TY - 1) * (tile / ntx) - 1;
    const int vz0 = A.ends ? (kz == 0 ? L.own_lo : L.own_hi - 1) : L.own_lo + kz;
    const int vz1 = vz0 + len;
    const int cx = x0 + tx, cy = y0 + ty;
    __syncthreads();                             // the previous strip's shared memory is free

    if (!BOX && !listed) {
        // tiles of the bounding lattice that hold no vertex (e.g. the missing
        // quadrant of an L-shape) are skipped at once
        int any = 0;
        const int np = vz1 - vz0 + 2;
        for (int e = tid; e < ROWS * np; e += T3_NT) {
            const int y = y0 + e % ROWS, z = vz0 - 1 + e / ROWS;
            if ((unsigned)y > (unsigned)L.ny || (unsigned)z > (unsigned)L.nz) continue;
            const int r = y + (L.ny + 1) * z;
            const int lo = __ldg(L.vrow_lo + r), hi = __ldg(L.vrow_hi + r);
            if (hi > lo && hi > x0 && lo <= x0 + TX) any = 1;
        }
        if (!__syncthreads_or(any)) continue;
    }

    const double* fsrc[NF];
#pragma unroll
    for (int i = 0; i < NV; ++i) fsrc[MI::F_V + i] = A.v + (int64_t)i * V;
    if constexpr (!TAB) {
#pragma unroll
        for (int i = 0; i < MI::NU; ++i) fsrc[MI::F_U + i] = A.U + (int64_t)i * V;
        if (MI::PT) fsrc[MI::F_PT] = A.pt;
    }

    // Non-box lattices: the row tables of the tile's vertex rows (off, lo, hi)
    // and cell rows (lo, hi) are staged per plane into a ring of RR slots, four
    // planes ahead of the cell work, so vertex ids come from shared memory
    // (the dependent global row-table loads were the kernel's top stall).
    constexpr int RR = 8;
    struct RowI {
        long long off;
        int lo, hi;
    };
    __shared__ RowI srow[BOX ? 1 : RR][ROWS];
    __shared__ int2 scell[BOX ? 1 : RR][TY];
    const int zbase = vz0 - 1;
    auto rslot = [&](int z) { return (z - zbase) & (RR - 1); };
    auto fetch_rows = [&](int z) {
        if (BOX) return;
        const int sl = rslot(z);
        if (tid < ROWS) {
            const int y = y0 + tid;
            const bool ok = (unsigned)y <= (unsigned)L.ny && (unsigned)z <= (unsigned)L.nz;
            const int r = ok ? y + (L.ny + 1) * z : 0;
            cp_async8(&srow[sl][tid].off, L.vrow_off + r, ok);
            cp_async4(&srow[sl][tid].lo, L.vrow_lo + r, ok);
            cp_async4(&srow[sl][tid].hi, L.vrow_hi + r, ok);
        } else if (tid < ROWS + TY) {
            const int k = tid - ROWS, y = y0 + k;
            const bool ok = (unsigned)y < (unsigned)L.ny && (unsigned)z < (unsigned)L.nz;
            const int c = ok ? y + L.ny * z : 0;
            cp_async4(&scell[sl][k].x, L.crow_lo + c, ok);
            cp_async4(&scell[sl][k].y, L.crow_hi + c, ok);
        }
    };
    // vertex (x, y0 + rr, z) of the tile
    auto vid_of = [&](int x, int rr, int z) -> int {
        if (BOX) {
            const int y = y0 + rr;
            if ((unsigned)x > (unsigned)L.nx || (unsigned)y > (unsigned)L.ny || (unsigned)z > (unsigned)L.nz)
                return -1;
            return (z * (L.ny + 1) + y) * (L.nx + 1) + x;
        }
        const RowI& R = srow[rslot(z)][rr];
        return (x >= R.lo && x < R.hi) ? (int)(R.off + (x - R.lo)) : -1;
    };

    // Stage plane z into slot (one thread per staged vertex, EPT passes).  The
    // vertex's flag byte comes back in a register (a plain load issued with
    // the copies); once this thread's copies have landed, `finish` writes the
    // flags to shared memory and -- without PRE -- zeroes the constrained v
    // entries it copied itself (fem.py:205-206, once per vertex); the next
    // plane barrier publishes both.
    unsigned ifl[EPT];                                          // flags of the last issued plane
    auto issue = [&](int z, int slot) {
        double* dst = sv + slot * SLOT;
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
            const int e = tid + j * T3_NT;
            ifl[j] = 0u;
            if (e >= PL) break;
            const int rr = e / COLS, col = e % COLS;
            const int vid = vid_of(x0 + col, rr, z);
            const bool ok = vid >= 0;
            const int off = ok ? vid : 0;
#pragma unroll
            for (int f = 0; f < NF; ++f) cp_async8(dst + f * PL + e, fsrc[f] + off, ok);
            ifl[j] = ok ? (unsigned)__ldg(A.flags + off) : 0u;
        }
    };
    auto finish = [&](int slot, const unsigned (&fl)[EPT]) {   // after this thread's cp.async wait
        double* p = sv + slot * SLOT;
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
            const int e = tid + j * T3_NT;
            if (e >= PL) break;
            sfl[slot * PL + e] = (unsigned char)fl[j];
            if (!PRE) {
#pragma unroll
                for (int i = 0; i < NV; ++i)
                    if ((fl[j] >> (MI::COMP0 + i)) & 1) p[i * PL + e] = 0.0;
            }
        }
    };

    if (!BOX) {
        for (int z = vz0 - 1; z <= vz0 + 3; ++z) fetch_rows(z);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
    }
    {
        // planes vz0-1, vz0 and (if the run has it) vz0+1 into slots 0, 1, 2
        issue(vz0 - 1, 0);
        unsigned fl0[EPT], fl1[EPT];
#pragma unroll
        for (int j = 0; j < EPT; ++j) fl0[j] = ifl[j];
        issue(vz0, 1);
#pragma unroll
        for (int j = 0; j < EPT; ++j) fl1[j] = ifl[j];
        const bool third = vz0 + 1 <= vz1;
        if (third) issue(vz0 + 1, 2);
        cp_async_commit();
        cp_async_wait<0>();
        finish(0, fl0);
        finish(1, fl1);
        if (third) finish(2, ifl);
        __syncthreads();
    }
    double carry[NCO];
#pragma unroll
    for (int k = 0; k < NCO; ++k) carry[k] = 0.0;

    // One barrier per plane step.  Step `it` reads planes cz (slot s0) and
    // cz+1 (s1), writes its y partials to sy[it & 1], and lands + finishes
    // plane cz+3 (slot s3, the slot of plane cz-2); the single barrier between
    // the y-partial writes and reads also orders every thread's finish of
    // plane cz+2 (previous step) before the next step reads it, and every read
    // of a slot before it is refilled two steps later.
    int it = 0, s0 = 0;
    for (int cz = vz0 - 1; cz < vz1; ++cz, ++it, s0 = s0 == T3_RING - 1 ? 0 : s0 + 1) {
        const int s1 = s0 == T3_RING - 1 ? 0 : s0 + 1;
        const int s3 = s0 >= 2 ? s0 - 2 : s0 + 3;
        double* sy = sy0 + (it & 1) * (TY * NCO * 2 * TX);
        // vertex finalised this iteration and its epilogue operands (loaded early)
        const int vid_f = (ty >= 1 && tx >= 1 && cz >= vz0) ? vid_of(cx, ty, cz) : -1;
        double* eslot = sepi + tid * (NLE * NCO);
        EpiIn<NCO, EPI> ein;
        if (STAGE && vid_f >= 0) epi_stage<NCO, EPI>(A, vid_f, eslot);   // committed with the plane below
        if (!STAGE && vid_f >= 0) epi_load<NCO, EPI>(A, vid_f, ein);
        if (cz + 5 <= vz1 + 1) fetch_rows(cz + 5);     // committed with the plane below
        const bool issued = cz + 3 <= vz1;
        if (issued) issue(cz + 3, s3);
        cp_async_commit();

        const double* p0 = sv + s0 * SLOT;
        const double* p1 = sv + s1 * SLOT;
        struct Corners {
            const double* p0;
            const double* p1;
            int e;                               // staged index of the cell's (0, 0) corner
            bool zphi;                           // block-diagonal operator: phi(U) reads 0 (no G_phiu)
            __device__ __forceinline__ void load(int f, double (&c)[8]) const {
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    const double* p = (n >> 2) ? p1 : p0;
                    c[n] = p[f * PL + e + ((n >> 1) & 1) * COLS + (n & 1)];
                    if (MODE == M_FULL && f == MI::F_U + 3 && zphi) c[n] = 0.0;
                }
            }
        } C{p0, p1, ty * COLS + tx, A.nocoup != 0};

        const bool cell = BOX ? ((unsigned)cx < (unsigned)L.nx && (unsigned)cy < (unsigned)L.ny &&
                                 (unsigned)cz < (unsigned)L.nz)
                              : (cx >= scell[rslot(cz)][ty].x && cx < scell[rslot(cz)][ty].y);
        const int64_t lcell = (int64_t)cx + (int64_t)L.nx * (cy + (int64_t)L.ny * cz);
        const double* rq = (RHO && cell) ? A.rho + lcell * 8 : A.rho;
        const double* tq = (TAB && cell) ? A.ptab + lcell : A.ptab;
        double vp[NCO][2];                       // this vertex column's (y=0) partials, per z corner
        // absent cells (lattice edges, the L-prism's missing quadrant) contribute
        // nothing; warps holding none skip the selects (a warp-uniform branch)
        const bool any_absent = __any_sync(0xffffffffu, !cell);
        auto emit = [&](int k, double (&o)[8]) {
            if (any_absent) {
#pragma unroll
                for (int n = 0; n < 8; ++n) o[n] = cell ? o[n] : 0.0;
            }
#pragma unroll
            for (int zb = 0; zb < 2; ++zb)
#pragma unroll
                for (int yb = 0; yb < 2; ++yb) {
                    const int nl = (yb << 1) | (zb << 2);
                    // tx = 0 reads a neighbour row's value: that column is not finalised
                    const double part = o[nl] + __shfl_up_sync(0xffffffffu, o[nl | 1], 1);
                    if (yb)
                        sy[((ty * NCO + k) * 2 + zb) * TX + tx] = part;
                    else
                        vp[k][zb] = part;
                }
        };
        cell3_iso<MODE, RHO, Corners, decltype(emit)&, TAB>(C, rq, A.K, A.I, emit, tq,
                                                            (int64_t)L.nx * L.ny * L.nz);
        __syncthreads();                         // y partials visible (see the loop head)

        if (ty >= 1) {
            double acc[NCO], top[NCO];
#pragma unroll
            for (int k = 0; k < NCO; ++k) {
                acc[k] = carry[k] + (vp[k][0] + sy[(((ty - 1) * NCO + k) * 2 + 0) * TX + tx]);
                top[k] = vp[k][1] + sy[(((ty - 1) * NCO + k) * 2 + 1) * TX + tx];
            }
            if (vid_f >= 0) {
                const int vid = vid_f;
                const int e = ty * COLS + tx;
                const unsigned fl = sfl[s0 * PL + e];
                if (STAGE && NLE > 0) {
                    cp_async_wait<0>();          // this thread's staged operands (issued at the step's start)
                    epi_unstage<NCO, EPI>(eslot, ein);
                }
                double vin[NCO];
#pragma unroll
                for (int k = 0; k < NCO; ++k) {
                    // raw v (for identity rows): the staged copy was masked unless PRE
                    vin[k] = PRE ? p0[(MI::F_V + k) * PL + e]
                                 : (((fl >> (MI::COMP0 + k)) & 1) ? A.v[(int64_t)k * V + vid]
                                                                  : p0[(MI::F_V + k) * PL + e]);
                }
                epilogue<NCO, MI::COMP0, EPI>(A, vid, (uint8_t)fl, acc, vin, ein);
            }
#pragma unroll
            for (int k = 0; k < NCO; ++k) carry[k] = top[k];
        }
        if (issued) {                            // plane cz+3: flags + masking before the next step's barrier
            cp_async_wait<0>();
            finish(s3, ifl);
        }
    }
    cp_async_wait<0>();
    }                                            // next strip
}

}  // namespace pffmg
