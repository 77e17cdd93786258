// 3D fused operator for isotropic hexahedra: CTA = TY warps, a tile of
// 31 (x) x TY (y) cells marching in z.  Lanes load lattice columns
// x0..x0+31 (x0 = 30*bx - 1); lanes 0..30 compute cells, lanes 1..30 /
// warps 1..TY-1 finalise vertices.  Vertex planes are staged with cp.async
// into a 4-slot shared-memory ring two planes ahead; the cell work is the
// streaming cell3_iso kernel; vertex sums: x by shuffles, y through shared
// memory, z by a register carry.  Replaces reference model.py:368-392 (+ the
// fused epilogues of mgsolve.py:82-113, 227) for 3D levels.
#pragma once

#include "cell3_iso.cuh"
#include "op_kernels.cuh"

namespace pffmg {

// TAB (phi block only): a_phiphi comes from the per-QP table A.ptab, so only
// v is staged (no U planes) -- the phi block becomes an HBM-bound stencil.
template <int MODE, int EPI, int TY, bool RHO, bool BOX, bool PRE, bool TAB = false>
#ifndef PFFMG_3D_FULL_MINB
#define PFFMG_3D_FULL_MINB 1
#endif
__global__ void __launch_bounds__(32 * TY, MODE == M_FULL ? PFFMG_3D_FULL_MINB : (TAB ? 4 : 2)) op3dt_kernel(const OpArgs A) {
    pdl_wait();
    using MI = ModeInfo<3, MODE>;
    constexpr int NF = TAB ? MI::NV : MI::NF, NCO = MI::NCO, NV = MI::NV;
    constexpr int RING = 4, ROWS = TY + 1, W = 32;
    constexpr int SLOT = NF * ROWS * W;          // doubles per staged plane
    constexpr int FB = 48;                       // flag bytes per staged row

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* sv = reinterpret_cast<double*>(smem_raw);                          // [RING][NF][ROWS][W]
    double* sy = sv + RING * SLOT;                                              // [TY][NCO][2][W]
    // epilogue operands staged in shared memory where a register prefetch
    // spills (u block, and the Chebyshev variants of FULL); elsewhere they
    // stay in registers (ncu: staging costs the table phi block and RESID ~4%)
    constexpr bool STAGE = MODE == M_UBLK || (MODE == M_FULL && (EPI == E_CHEB || EPI == E_CHEB0));
    constexpr int NLE = STAGE ? EpiIn<NCO, EPI>::NL : 0;                        // staged epilogue operands
    double* sepi = sy + TY * NCO * 2 * W;                                       // [32 TY][NLE][NCO]
    unsigned char* sfl = reinterpret_cast<unsigned char*>(sepi + 32 * TY * NLE * NCO);  // [RING][ROWS][FB]
    int* sfo = reinterpret_cast<int*>(sfl + RING * ROWS * FB);                 // [RING][ROWS]

    const Lat& L = A.L;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int x0 = 30 * (int)blockIdx.x - 1;
    const int y0 = (TY - 1) * (int)blockIdx.y - 1;
    const int vz0 = A.ends ? ((int)blockIdx.z == 0 ? L.own_lo : L.own_hi - 1)
                           : L.own_lo + (int)blockIdx.z * A.planes_per_cta;
    const int vz1 = A.ends ? vz0 + 1 : min(vz0 + A.planes_per_cta, L.own_hi);
    const int cx = x0 + lane, cy = y0 + w;
    const int V = (int)L.V;
    const int nwords = (V + 3) / 4 + 8;
    const bool lane_cell = lane <= 30;

    if (!BOX) {
        // tiles of the bounding lattice that hold no vertex (e.g. the missing
        // quadrant of an L-shape) leave at once
        int any = 0;
        const int np = vz1 - vz0 + 2;
        for (int e = tid; e < ROWS * np; e += 32 * TY) {
            const int y = y0 + e % ROWS, z = vz0 - 1 + e / ROWS;
            if ((unsigned)y > (unsigned)L.ny || (unsigned)z > (unsigned)L.nz) continue;
            const int r = y + (L.ny + 1) * z;
            const int lo = __ldg(L.vrow_lo + r), hi = __ldg(L.vrow_hi + r);
            if (hi > lo && hi > x0 && lo <= x0 + 31) any = 1;
        }
        if (!__syncthreads_or(any)) return;
    }

    const double* fsrc[NF];
#pragma unroll
    for (int i = 0; i < NV; ++i) fsrc[MI::F_V + i] = A.v + (int64_t)i * V;
    if constexpr (!TAB) {
#pragma unroll
        for (int i = 0; i < MI::NU; ++i) fsrc[MI::F_U + i] = A.U + (int64_t)i * V;
        if (MI::PT) fsrc[MI::F_PT] = A.pt;
    }
    const uint32_t* fw = reinterpret_cast<const uint32_t*>(A.flags);

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
    auto vid_virtual = [&](int x, int rr, int z) -> int {
        if (BOX) return (z * (L.ny + 1) + y0 + rr) * (L.nx + 1) + x;
        const RowI& R = srow[rslot(z)][rr];
        return (int)(R.off + (x - R.lo));
    };

    // stage plane z into slot: row rr of the tile (rr = 0..TY), column = lane
    // Without PRE the staged v entries of constrained dofs read 0 (fem.py:205-206).
    // Each thread masks exactly the entries it copied itself, with their flag
    // bytes loaded into registers at issue time: the masking then needs only the
    // thread's own cp.async wait, and the next plane barrier publishes it.
    constexpr bool OWNMASK = !PRE && NV > 0;
    constexpr int EPT = (ROWS * W + 32 * TY - 1) / (32 * TY);   // staged entries per thread
    unsigned ifl[EPT];                                          // flags of the last issued plane
    auto issue = [&](int z, int slot) {
        double* dst = sv + slot * SLOT;
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
            const int e = tid + j * 32 * TY;
            if (e >= ROWS * W) break;
            const int rr = e / W, col = e % W;
            const int vid = vid_of(x0 + col, rr, z);
            const bool ok = vid >= 0;
            const int off = ok ? vid : 0;
#pragma unroll
            for (int f = 0; f < NF; ++f) cp_async8(dst + (f * ROWS + rr) * W + col, fsrc[f] + off, ok);
            if (OWNMASK) ifl[j] = ok ? (unsigned)__ldg(A.flags + off) : 0u;
        }
        for (int e = tid; e < ROWS * 9; e += 32 * TY) {
            const int rr = e / 9, k = e % 9;
            const int v0 = vid_virtual(x0, rr, z);
            const int w0 = v0 >> 2;
            const int wi = w0 + k;
            const bool okw = wi >= 0 && wi < nwords && (unsigned)(y0 + rr) <= (unsigned)L.ny &&
                             (unsigned)z <= (unsigned)L.nz;
            cp_async4(sfl + (slot * ROWS + rr) * FB + 4 * k, fw + (okw ? wi : 0), okw);
            if (k == 0) sfo[slot * ROWS + rr] = v0 - 4 * w0;
        }
        cp_async_commit();
    };
    auto flag = [&](int slot, int rr, int col) -> unsigned {
        return sfl[(slot * ROWS + rr) * FB + sfo[slot * ROWS + rr] + col];
    };
    auto mask_own = [&](int slot, const unsigned (&fl)[EPT]) {   // after this thread's cp.async wait
        if (!OWNMASK) return;
        double* p = sv + slot * SLOT;
#pragma unroll
        for (int j = 0; j < EPT; ++j) {
            const int e = tid + j * 32 * TY;
            if (e >= ROWS * W) break;
            const int rr = e / W, col = e % W;
#pragma unroll
            for (int i = 0; i < NV; ++i)
                if ((fl[j] >> (MI::COMP0 + i)) & 1) p[(i * ROWS + rr) * W + col] = 0.0;
        }
    };

    if (!BOX) {
        for (int z = vz0 - 1; z <= vz0 + 2; ++z) fetch_rows(z);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
    }
    issue(vz0 - 1, 0);
    if (OWNMASK) {
        unsigned fl0[EPT];
#pragma unroll
        for (int j = 0; j < EPT; ++j) fl0[j] = ifl[j];
        issue(vz0, 1);
        cp_async_wait<0>();
        mask_own(0, fl0);
        mask_own(1, ifl);
    } else {
        issue(vz0, 1);
    }
    double carry[NCO];
#pragma unroll
    for (int k = 0; k < NCO; ++k) carry[k] = 0.0;

    int it = 0;
    for (int cz = vz0 - 1; cz < vz1; ++cz, ++it) {
        const int s0 = it & 3, s1 = (it + 1) & 3;
        // vertex finalised this iteration and its epilogue operands (loaded early)
        const int vid_f = (w >= 1 && cz >= vz0 && lane >= 1 && lane <= 30) ? vid_of(cx, w, cz) : -1;
        double* eslot = sepi + tid * (NLE * NCO);
        EpiIn<NCO, EPI> ein;
        if (STAGE && vid_f >= 0) epi_stage<NCO, EPI>(A, vid_f, eslot);   // committed with the plane below
        if (!STAGE && vid_f >= 0) epi_load<NCO, EPI>(A, vid_f, ein);
        if (cz + 4 <= vz1 + 1) fetch_rows(cz + 4);     // committed with the plane below
        const bool issued = cz + 2 <= vz1;
        if (issued)
            issue(cz + 2, (it + 2) & 3);
        else
            cp_async_commit();
        cp_async_wait<1>();                      // planes cz, cz+1 landed (this thread's copies)
        __syncthreads();                         // ... and everyone else's (masked: see the loop end)

        const double* p0 = sv + s0 * SLOT;
        const double* p1 = sv + s1 * SLOT;
        struct Corners {
            const double* p0;
            const double* p1;
            int lane, w;
            bool zphi;                           // block-diagonal operator: phi(U) reads 0 (no G_phiu)
            __device__ __forceinline__ void load(int f, double (&c)[8]) const {
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    const double* p = (n >> 2) ? p1 : p0;
                    c[n] = p[(f * ROWS + w + ((n >> 1) & 1)) * W + lane + (n & 1)];
                    if (MODE == M_FULL && f == MI::F_U + 3 && zphi) c[n] = 0.0;
                }
            }
        } C{p0, p1, lane < 31 ? lane : 30, w, A.nocoup != 0};

        const bool cell = lane_cell && (BOX ? ((unsigned)cx < (unsigned)L.nx && (unsigned)cy < (unsigned)L.ny &&
                                               (unsigned)cz < (unsigned)L.nz)
                                            : (cx >= scell[rslot(cz)][w].x && cx < scell[rslot(cz)][w].y));
        const int64_t lcell = (int64_t)cx + (int64_t)L.nx * (cy + (int64_t)L.ny * cz);
        const double* rq = (RHO && cell) ? A.rho + lcell * 8 : A.rho;
        const double* tq = (TAB && cell) ? A.ptab + lcell : A.ptab;
        double vp[NCO][2];                       // this vertex column's (y=0) partials, per z corner
        auto emit = [&](int k, double (&o)[8]) {
#pragma unroll
            for (int n = 0; n < 8; ++n) o[n] = cell ? o[n] : 0.0;
#pragma unroll
            for (int zb = 0; zb < 2; ++zb)
#pragma unroll
                for (int yb = 0; yb < 2; ++yb) {
                    const int nl = (yb << 1) | (zb << 2);
                    const double part = o[nl] + __shfl_up_sync(0xffffffffu, o[nl | 1], 1);
                    if (yb)
                        sy[((w * NCO + k) * 2 + zb) * W + lane] = part;
                    else
                        vp[k][zb] = part;
                }
        };
        cell3_iso<MODE, RHO, Corners, decltype(emit)&, TAB>(C, rq, A.K, A.I, emit, tq,
                                                            (int64_t)L.nx * L.ny * L.nz);
        __syncthreads();                         // y partials visible; planes fully read

        if (w >= 1) {
            double acc[NCO], top[NCO];
#pragma unroll
            for (int k = 0; k < NCO; ++k) {
                acc[k] = carry[k] + (vp[k][0] + sy[(((w - 1) * NCO + k) * 2 + 0) * W + lane]);
                top[k] = vp[k][1] + sy[(((w - 1) * NCO + k) * 2 + 1) * W + lane];
            }
            if (vid_f >= 0) {
                const int vid = vid_f;
                const unsigned fl = flag(s0, w, lane);
                if (STAGE && NLE > 0) {
                    cp_async_wait<0>();          // this thread's staged operands (issued at the step's start)
                    epi_unstage<NCO, EPI>(eslot, ein);
                }
                double vin[NCO];
#pragma unroll
                for (int k = 0; k < NCO; ++k) {
                    // raw v (for identity rows): the staged copy was masked unless PRE
                    vin[k] = PRE ? p0[((MI::F_V + k) * ROWS + w) * W + lane]
                                 : (((fl >> (MI::COMP0 + k)) & 1) ? A.v[(int64_t)k * V + vid]
                                                                  : p0[((MI::F_V + k) * ROWS + w) * W + lane]);
                }
                epilogue<NCO, MI::COMP0, EPI>(A, vid, (uint8_t)fl, acc, vin, ein);
            }
#pragma unroll
            for (int k = 0; k < NCO; ++k) carry[k] = top[k];
        }
        if (OWNMASK && issued) {                 // plane cz+2: masked before the next step's barrier
            cp_async_wait<0>();
            mask_own((it + 2) & 3, ifl);
        }
    }
    cp_async_wait<0>();
}

}  // namespace pffmg
