// Q2 (9-node) 2D fused operator kernels (BASELINE configs[2]).
//
// One thread = one Q2 cell; a warp = 32 consecutive cells of a cell row
// (lane 0 is the halo cell of the previous segment: it only feeds its right
// node column to lane 1) marching up a strip of cell rows.  A cell row cy
// owns node rows 2cy (finished with the carry of the row below) and 2cy+1
// (interior to the row); node row 2cy+2 is carried.  Node columns likewise:
// column 2cx gets the left neighbour's right column by one shuffle, column
// 2cx+1 is interior.  Every node is summed in a fixed order -- deterministic,
// no atomics.  Epilogues are the ones of the Q1 kernels (op_kernels.cuh).
#include <cstdlib>

#include "cell_q2.cuh"
#include "op_launch.cuh"

namespace pffmg {

#ifndef PFFMG_Q2_MINB
#define PFFMG_Q2_MINB 3
#endif

// TAB: the phi block / block-diagonal operator with a_phiphi from the per-QP table.
template <int MODE, int EPI, bool MIE, bool TAB = false>
__global__ void __launch_bounds__(128, MODE == M_FULL ? 2 : PFFMG_Q2_MINB) op2q_kernel(const OpArgs A, const Q2Tab T) {
    pdl_wait();
    using MI = ModeInfo<2, MODE, MIE>;
    constexpr int NF = MI::NF, NCO = MI::NCO, NV = MI::NV;
    const Lat& L = A.L;
    const int lane = threadIdx.x & 31;
    const int gw = (int)blockIdx.x * 4 + (threadIdx.x >> 5);
    const int seg = gw % A.nseg, strip = gw / A.nseg;
    // cell row cy finalises node rows 2cy and 2cy+1 (those inside the owned
    // node rows [own_lo, own_hi) of a slab); cy = ny only its bottom row
    const int cyA = L.own_lo >> 1, cyB = (L.own_hi + 1) >> 1;
    const int cy0 = cyA + strip * A.planes_per_cta;
    if (cy0 >= cyB) return;
    const int cy1 = min(cy0 + A.planes_per_cta, cyB);
    const int cx = 31 * seg - 1 + lane;
    const int nxn = 2 * L.nx + 1;
    const int64_t V = L.V;

    const double* fsrc[NF];
#pragma unroll
    for (int i = 0; i < NV; ++i) fsrc[MI::F_V + i] = A.v + (int64_t)i * V;
#pragma unroll
    for (int i = 0; i < MI::NU; ++i) fsrc[MI::F_U + i] = A.U + (int64_t)i * V;
    if (MI::PT) fsrc[MI::F_PT] = A.pt;

    double carry_s[NCO], carry_m[NCO];     // node row 2cy from the row below: columns 2cx, 2cx+1
#pragma unroll
    for (int k = 0; k < NCO; ++k) carry_s[k] = carry_m[k] = 0.0;

    for (int cy = cy0 - 1; cy < cy1; ++cy) {
        double o[NCO][9];
        const bool cell = cx >= 0 && cx < L.nx && cy >= 0 && cy < L.ny;
        constexpr bool ROWS = !MIE && (MODE == M_FULL || MODE == M_UBLK || MODE == M_PBLK);
        if (ROWS && cell) {
            // row-factorised kernel: nodal fields re-read per QP row (L1 hits)
            const int64_t id0 = (int64_t)(2 * cy) * nxn + 2 * cx;
            unsigned fl[9];
#pragma unroll
            for (int n = 0; n < 9; ++n)
                fl[n] = (NV > 0 && !A.premasked) ? __ldg(A.flags + id0 + (n / 3) * nxn + n % 3) : 0u;
            auto load = [&](int f, double (&c)[9]) {
#pragma unroll
                for (int n = 0; n < 9; ++n) {
                    double x = __ldg(fsrc[f] + id0 + (n / 3) * nxn + n % 3);
                    if (f < NV && ((fl[n] >> (MI::COMP0 + f)) & 1)) x = 0.0;   // fem.py:205-206
                    c[n] = x;
                }
            };
            const double* rq = A.rho ? A.rho + ((int64_t)cx + (int64_t)L.nx * cy) * 9 : nullptr;
            if constexpr (ROWS)
                cell_q2_rows<MODE, TAB>(load, rq, A.K, T, A.nocoup != 0, o,
                                        TAB ? A.ptab + ((int64_t)cx + (int64_t)L.nx * cy) : nullptr,
                                        (int64_t)L.nx * L.ny);
        } else if (cell) {
            double cv[NF][9];
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const int64_t id = (int64_t)(2 * cy + b) * nxn + 2 * cx + a;
                    const unsigned fl = (NV > 0 && !A.premasked) ? __ldg(A.flags + id) : 0u;
#pragma unroll
                    for (int f = 0; f < NF; ++f) {
                        double x = __ldg(fsrc[f] + id);
                        if (f < NV && ((fl >> (MI::COMP0 + f)) & 1)) x = 0.0;   // fem.py:205-206
                        cv[f][3 * b + a] = x;
                    }
                }
            if constexpr (MODE == M_FULL) {
                if (A.nocoup) {                  // block-diagonal operator: phi(U) reads 0
#pragma unroll
                    for (int n = 0; n < 9; ++n) cv[MI::F_U + 2][n] = 0.0;
                }
            }
            const double* rq = A.rho ? A.rho + ((int64_t)cx + (int64_t)L.nx * cy) * 9 : nullptr;
            cell_q2<MODE, MIE>(cv, rq, A.K, T, o);
        } else {
#pragma unroll
            for (int k = 0; k < NCO; ++k)
#pragma unroll
                for (int n = 0; n < 9; ++n) o[k][n] = 0.0;
        }
        // node column 2cx: own left column + the left neighbour's right column
        double s[NCO][3], m[NCO][3];
#pragma unroll
        for (int k = 0; k < NCO; ++k)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                s[k][b] = o[k][3 * b] + __shfl_up_sync(0xffffffffu, o[k][3 * b + 2], 1);
                m[k][b] = o[k][3 * b + 1];
            }
        if (cy >= cy0 && lane >= 1 && cx >= 0 && cx <= L.nx) {
            // (column offset, row offset, value source) of the up to four nodes
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int dx = t & 1, dy = t >> 1;
                if (dx == 1 && cx >= L.nx) continue;
                if (dy == 1 && cy >= L.ny) continue;
                if (2 * cy + dy < L.own_lo || 2 * cy + dy >= L.own_hi) continue;
                const int64_t id = (int64_t)(2 * cy + dy) * nxn + 2 * cx + dx;
                double acc[NCO], vin[NCO];
#pragma unroll
                for (int k = 0; k < NCO; ++k) {
                    acc[k] = dy == 0 ? (dx == 0 ? carry_s[k] + s[k][0] : carry_m[k] + m[k][0])
                                     : (dx == 0 ? s[k][1] : m[k][1]);
                    vin[k] = (MODE == M_DIAG || MODE == M_RES) ? 0.0 : __ldg(A.v + (int64_t)k * V + id);
                }
                EpiIn<NCO, EPI> ein;
                epi_load<NCO, EPI>(A, id, ein);
                epilogue<NCO, MI::COMP0, EPI>(A, id, __ldg(A.flags + id), acc, vin, ein);
            }
        }
#pragma unroll
        for (int k = 0; k < NCO; ++k) {
            carry_s[k] = s[k][2];
            carry_m[k] = m[k][2];
        }
    }
}

// ---------------------------------------------------------------------------
// Staged Q2 kernel for the hot modes (FULL / UBLK / PBLK, NoSplit): same cells,
// node sums and epilogues as op2q_kernel, but the node rows a warp needs are
// staged into a warp-private shared-memory ring with cp.async one cell row
// ahead (two node rows per cell row), instead of 9 x NF dependent __ldg per
// QP row.  A warp covers node columns nc0 .. nc0+64 (nc0 = 62 seg - 2); a
// staged row keeps the even columns E[0..32] and the odd columns O[0..31]
// apart, so lane L's cell reads E[L], O[L], E[L+1] without bank conflicts.
// Ring of 5 node rows: cell row cy reads rows 2cy..2cy+2 while rows 2cy+3,
// 2cy+4 land.  Epilogue operands of the RESID / Chebyshev variants are staged
// with cp.async at the start of the iteration that finalises their nodes.
// Unless PRE, every lane zeroes the constrained entries it copied itself once
// they have landed (fem.py:205-206, once per node).
template <int MODE, bool TAB>
struct Q2Fields {
    using MI = ModeInfo<2, MODE>;
    // fields the row kernel reads (TAB: a_phiphi comes from the table, no U)
    __host__ __device__ static constexpr bool used(int f) {
        return !TAB || f < MI::NV || (MI::PT && f == MI::F_PT);
    }
    __host__ __device__ static constexpr int slot(int f) {
        int s = 0;
        for (int g = 0; g < f; ++g) s += used(g) ? 1 : 0;
        return s;
    }
    static constexpr int NFS = slot(MI::NF);
};

constexpr int Q2_RING = 5, Q2_ROW = 66;    // node rows in the ring; doubles per staged field row (E 0..32, O 33..64)

#ifndef PFFMG_Q2S_FULL_MINB
#define PFFMG_Q2S_FULL_MINB 2
#endif
template <int MODE, int EPI, bool TAB, bool PRE>
__global__ void __launch_bounds__(128, MODE == M_FULL ? PFFMG_Q2S_FULL_MINB : PFFMG_Q2_MINB) op2qs_kernel(const OpArgs A, const Q2Tab T) {
    pdl_wait();
    using MI = ModeInfo<2, MODE>;
    using FS = Q2Fields<MODE, TAB>;
    constexpr int NF = MI::NF, NCO = MI::NCO, NV = MI::NV, NFS = FS::NFS;
    constexpr int SLOT = NFS * Q2_ROW;                       // doubles per staged node row
    constexpr int NL = EpiIn<NCO, EPI>::NL;
    constexpr bool STAGE = NL > 0 && (EPI == E_RESID || EPI == E_CHEB || EPI == E_CHEB0);
    constexpr int ESZ = STAGE ? 4 * NL * NCO : 0;            // staged epilogue doubles per lane
    constexpr int WSM = Q2_RING * SLOT + 32 * ESZ;           // doubles per warp

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* sv = reinterpret_cast<double*>(smem_raw) + wib * WSM;
    double* se = sv + Q2_RING * SLOT + lane * ESZ;

    const Lat& L = A.L;
    const int cyA = L.own_lo >> 1, cyB = (L.own_hi + 1) >> 1;
    const int nxn = 2 * L.nx + 1, nyn = 2 * L.ny + 1;
    const int64_t V = L.V;
    // Work: warp gw = seg + nseg * strip marches cell rows
    // [cyA + strip * per, + per) of segment seg (one warm-up cell row); the
    // launcher picks per for one wave of resident warps.  (A persistent
    // contiguous-share schedule, as in the 3D kernel, measured slower here:
    // cfg3 phi block 22.8 -> 27.0 us.)
    const int R = cyB - cyA;
    int item, item_hi;
    {
        const int gw = (int)blockIdx.x * 4 + wib;
        const int seg = gw % A.nseg, k0 = (gw / A.nseg) * A.planes_per_cta;
        item = seg * R + min(k0, R);
        item_hi = seg * R + min(k0 + A.planes_per_cta, R);
    }
    while (item < item_hi) {
    const int seg = item / R, kr = item % R;
    const int len = min(R - kr, item_hi - item);
    item += len;
    const int cy0 = cyA + kr, cy1 = cy0 + len;
    const int cx = 31 * seg - 1 + lane;
    const int nc0 = 62 * seg - 2;

    const double* fsrc[NFS];
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        if (!FS::used(f)) continue;
        const double* p = f < NV ? A.v + (int64_t)f * V
                                 : (f == MI::F_PT && MI::PT ? A.pt : A.U + (int64_t)(f - MI::F_U) * V);
        fsrc[FS::slot(f)] = p;
    }
    auto rslot = [](int r) { return (r + 10) % Q2_RING; };   // node rows >= -2

    // Stage node row r: lane L copies columns nc0 + 2L (E[L]) and nc0 + 2L + 1
    // (O[L]); lane 0 also nc0 + 64 (E[32]).  The lane's flag bytes come back
    // raw (a plain load issued with the copies) and are packed by `pack`
    // (E | O << 8 | E[32] << 16) only after the cell work of the iteration,
    // so their latency is hidden (packing them at issue stalled on the load).
    struct RawFl {
        unsigned e, o, x;
        __device__ __forceinline__ unsigned pack() const { return e | (o << 8) | (x << 16); }
    };
    auto issue = [&](int r) -> RawFl {
        double* dst = sv + rslot(r) * SLOT;
        const bool rok = (unsigned)r < (unsigned)nyn;
        const int64_t rb = (int64_t)r * nxn;
        const int ce = nc0 + 2 * lane, co = ce + 1, cx2 = nc0 + 64;
        const bool oke = rok && (unsigned)ce < (unsigned)nxn, oko = rok && (unsigned)co < (unsigned)nxn;
        const bool okx = lane == 0 && rok && (unsigned)cx2 < (unsigned)nxn;
        const int64_t ie = oke ? rb + ce : 0, io = oko ? rb + co : 0, ix = okx ? rb + cx2 : 0;
#pragma unroll
        for (int s = 0; s < NFS; ++s) {
            cp_async8(dst + s * Q2_ROW + lane, fsrc[s] + ie, oke);
            cp_async8(dst + s * Q2_ROW + 33 + lane, fsrc[s] + io, oko);
            if (lane == 0) cp_async8(dst + s * Q2_ROW + 32, fsrc[s] + ix, okx);
        }
        RawFl f;
        f.e = oke ? (unsigned)__ldg(A.flags + ie) : 0u;
        f.o = oko ? (unsigned)__ldg(A.flags + io) : 0u;
        f.x = okx ? (unsigned)__ldg(A.flags + ix) : 0u;
        return f;
    };
    auto mask_row = [&](int r, unsigned fl) {                // after the row landed
        if (PRE || NV == 0) return;
        double* p = sv + rslot(r) * SLOT;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int b = MI::COMP0 + i;
            if ((fl >> b) & 1) p[i * Q2_ROW + lane] = 0.0;
            if ((fl >> (8 + b)) & 1) p[i * Q2_ROW + 33 + lane] = 0.0;
            if ((fl >> (16 + b)) & 1) p[i * Q2_ROW + 32] = 0.0;
        }
    };

    // flags of node rows 2cy .. 2cy+4
    RawFl raw0 = issue(2 * cy0 - 2), raw1 = issue(2 * cy0 - 1), raw2 = issue(2 * cy0);
    cp_async_commit();
    unsigned fr0 = raw0.pack(), fr1 = raw1.pack(), fr2 = raw2.pack();
    RawFl raw3 = {0u, 0u, 0u}, raw4 = {0u, 0u, 0u};
    bool first = true;

    double carry_s[NCO], carry_m[NCO];     // node row 2cy from the row below: columns 2cx, 2cx+1
#pragma unroll
    for (int k = 0; k < NCO; ++k) carry_s[k] = carry_m[k] = 0.0;

    for (int cy = cy0 - 1; cy < cy1; ++cy) {
        const bool fin_row = cy >= cy0 && lane >= 1 && cx >= 0 && cx <= L.nx;
        // epilogue operands of the (up to) four nodes this lane finalises
        if (STAGE && fin_row) {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int dx = t & 1, dy = t >> 1;
                const bool ok = !(dx == 1 && cx >= L.nx) && !(dy == 1 && cy >= L.ny);
                const int64_t id = (int64_t)(2 * cy + dy) * nxn + 2 * cx + dx;
                if (ok) epi_stage<NCO, EPI>(A, id, se + t * NL * NCO);
            }
        }
        cp_async_commit();
        if (cy + 1 < cy1) {
            raw3 = issue(2 * cy + 3);
            raw4 = issue(2 * cy + 4);
        }
        cp_async_commit();
        cp_async_wait<2>();                     // rows 2cy .. 2cy+2 landed (this lane's copies)
        __syncwarp();
        if (first) mask_row(2 * cy, fr0);
        first = false;
        mask_row(2 * cy + 1, fr1);
        mask_row(2 * cy + 2, fr2);
        if (!PRE) __syncwarp();

        double o[NCO][9];
        const bool cell = cx >= 0 && cx < L.nx && cy >= 0 && cy < L.ny;
        if (cell) {
            const double* rw[3] = {sv + rslot(2 * cy) * SLOT, sv + rslot(2 * cy + 1) * SLOT,
                                   sv + rslot(2 * cy + 2) * SLOT};
            auto load = [&](int f, double (&c)[9]) {
                const int s = FS::slot(f);
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    const double* p = rw[b] + s * Q2_ROW;
                    c[3 * b] = p[lane];
                    c[3 * b + 1] = p[33 + lane];
                    c[3 * b + 2] = p[lane + 1];
                }
            };
            const double* rq = A.rho ? A.rho + ((int64_t)cx + (int64_t)L.nx * cy) * 9 : nullptr;
            cell_q2_rows<MODE, TAB>(load, rq, A.K, T, A.nocoup != 0, o,
                                    TAB ? A.ptab + ((int64_t)cx + (int64_t)L.nx * cy) : nullptr,
                                    (int64_t)L.nx * L.ny);
        } else {
#pragma unroll
            for (int k = 0; k < NCO; ++k)
#pragma unroll
                for (int n = 0; n < 9; ++n) o[k][n] = 0.0;
        }
        double s[NCO][3], m[NCO][3];
#pragma unroll
        for (int k = 0; k < NCO; ++k)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                s[k][b] = o[k][3 * b] + __shfl_up_sync(0xffffffffu, o[k][3 * b + 2], 1);
                m[k][b] = o[k][3 * b + 1];
            }
        if (fin_row) {
            if (STAGE) cp_async_wait<1>();      // this lane's epilogue operands
            const double* rw0 = sv + rslot(2 * cy) * SLOT;
            const double* rw1 = sv + rslot(2 * cy + 1) * SLOT;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int dx = t & 1, dy = t >> 1;
                if (dx == 1 && cx >= L.nx) continue;
                if (dy == 1 && cy >= L.ny) continue;
                if (2 * cy + dy < L.own_lo || 2 * cy + dy >= L.own_hi) continue;
                const int64_t id = (int64_t)(2 * cy + dy) * nxn + 2 * cx + dx;
                const unsigned fl = ((dy ? fr1 : fr0) >> (dx ? 8 : 0)) & 0xffu;
                const double* src = (dy ? rw1 : rw0) + (dx ? 33 : 0) + lane;
                double acc[NCO], vin[NCO];
#pragma unroll
                for (int k = 0; k < NCO; ++k) {
                    acc[k] = dy == 0 ? (dx == 0 ? carry_s[k] + s[k][0] : carry_m[k] + m[k][0])
                                     : (dx == 0 ? s[k][1] : m[k][1]);
                    // raw v (identity rows, Chebyshev d_in): the staged copy was masked unless PRE
                    vin[k] = PRE ? src[FS::slot(MI::F_V + k) * Q2_ROW]
                                 : (((fl >> (MI::COMP0 + k)) & 1) ? A.v[(int64_t)k * V + id]
                                                                  : src[FS::slot(MI::F_V + k) * Q2_ROW]);
                }
                EpiIn<NCO, EPI> ein;
                if (STAGE) epi_unstage<NCO, EPI>(se + t * NL * NCO, ein);
                epilogue<NCO, MI::COMP0, EPI>(A, id, (uint8_t)fl, acc, vin, ein);
            }
        }
#pragma unroll
        for (int k = 0; k < NCO; ++k) {
            carry_s[k] = s[k][2];
            carry_m[k] = m[k][2];
        }
        fr0 = fr2;
        fr1 = raw3.pack();
        fr2 = raw4.pack();
        __syncwarp();                           // rows 2cy, 2cy+1 and the epilogue slots free
    }
    cp_async_wait<0>();
    __syncwarp();                               // the ring is free for the next run
    }                                           // next run
}

template <int MODE, int EPI, bool TAB, bool PRE>
static void launch_qs(const OpArgs& A0, int nseg, int rows, const Q2Tab& T, cudaStream_t s) {
    auto kern = op2qs_kernel<MODE, EPI, TAB, PRE>;
    using FS = Q2Fields<MODE, TAB>;
    constexpr int NCO = ModeInfo<2, MODE>::NCO, NL = EpiIn<NCO, EPI>::NL;
    constexpr bool STAGE = NL > 0 && (EPI == E_RESID || EPI == E_CHEB || EPI == E_CHEB0);
    constexpr size_t smem = 4 * sizeof(double) * (Q2_RING * FS::NFS * Q2_ROW + 32 * (STAGE ? 4 * NL * NCO : 0));
    static int occ = 0;
    if (occ == 0) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem) != cudaSuccess || occ < 1) occ = 1;
    }
    // one wave of resident warps: strips of `per` cell rows
    OpArgs A = A0;
    A.nseg = nseg;
    const int64_t slots = (int64_t)sm_count() * occ * 4;
    int64_t per = ((int64_t)rows * nseg + slots - 1) / slots;
    per = per < 1 ? 1 : (per > 32 ? 32 : per);
    static const int forced = [] {
        const char* e = getenv("PFFMG_Q2_ROWS");
        return e ? atoi(e) : 0;
    }();
    if (forced > 0) per = forced;
    A.planes_per_cta = (int)per;
    const int64_t warps = (int64_t)nseg * ((rows + per - 1) / per);
    pdl_launch(kern, dim3((unsigned)((warps + 3) / 4)), dim3(128), smem, s, A, T);
}

static bool q2_staged() {
    static const int on = [] {
        const char* e = getenv("PFFMG_Q2_STAGED");
        return e ? atoi(e) : 1;
    }();
    return on != 0;
}

// One wave of resident warps (see op2d.cu): strips of `per` cell rows.
template <int MODE, int EPI, bool MIE, bool TAB = false>
static void launch_q(const OpArgs& A0, int nseg, int rows, const Q2Tab& T, cudaStream_t s) {
    if constexpr (!MIE && (MODE == M_FULL || MODE == M_UBLK || MODE == M_PBLK)) {
        if (q2_staged()) {
            if (A0.premasked)
                launch_qs<MODE, EPI, TAB, true>(A0, nseg, rows, T, s);
            else
                launch_qs<MODE, EPI, TAB, false>(A0, nseg, rows, T, s);
            return;
        }
    }
    auto kern = op2q_kernel<MODE, EPI, MIE, TAB>;
    static int occ = 0;
    if (occ == 0 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, 0) != cudaSuccess || occ < 1))
        occ = 1;
    OpArgs A = A0;
    const int64_t slots = (int64_t)sm_count() * occ * 4;
    int64_t per = ((int64_t)rows * nseg + slots - 1) / slots;
    per = per < 1 ? 1 : (per > 32 ? 32 : per);
    static const int forced = [] {
        const char* e = getenv("PFFMG_Q2_ROWS");
        return e ? atoi(e) : 0;
    }();
    if (forced > 0) per = forced;
    A.planes_per_cta = (int)per;
    A.nseg = nseg;
    const int64_t warps = (int64_t)nseg * ((rows + per - 1) / per);
    pdl_launch(kern, dim3((unsigned)((warps + 3) / 4)), dim3(128), 0, s, A, T);
}

template <int MODE, int EPI>
int launch2q(const OpArgs& A, cudaStream_t s) {
    const Lat& L = A.L;
    const int nseg = (L.nx + 1 + 30) / 31;
    const int rows = ((L.own_hi + 1) >> 1) - (L.own_lo >> 1);
    const Q2Tab T = make_q2_host(L.hx, L.hy);
    if constexpr (MODE == M_PBLK || MODE == M_FULL) {
        // phi block / block-diagonal operator: a_phiphi from the table (no state strain)
        if (!A.split && A.ptab && (MODE == M_PBLK || A.nocoup)) {
            launch_q<MODE, EPI, false, true>(A, nseg, rows, T, s);
            return PFFMG_OK;
        }
    }
    if (A.split)
        launch_q<MODE, EPI, true>(A, nseg, rows, T, s);
    else
        launch_q<MODE, EPI, false>(A, nseg, rows, T, s);
    return PFFMG_OK;
}

// Per-QP a_phiphi table of a Q2 level (model.py:304-308), QP-major:
// tab[q * C + c], q = 3 qy + qx, c = cx + nx cy, C = nx ny.
__global__ void __launch_bounds__(256) phi_coefq_kernel(const OpArgs A, const Q2Tab T, double* __restrict__ tab) {
    pdl_wait();
    const Lat& L = A.L;
    const int64_t C = (int64_t)L.nx * L.ny;
    const int nxn = 2 * L.nx + 1;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int cx = (int)(c % L.nx), cy = (int)(c / L.nx);
        const int64_t id0 = (int64_t)(2 * cy) * nxn + 2 * cx;
        double u0[9], u1[9], aq[9];
#pragma unroll
        for (int n = 0; n < 9; ++n) {
            const int64_t id = id0 + (n / 3) * nxn + n % 3;
            u0[n] = __ldg(A.U + id);
            u1[n] = __ldg(A.U + L.V + id);
        }
        phi_coef_q2(u0, u1, A.rho ? A.rho + c * 9 : nullptr, A.K, T, aq);
#pragma unroll
        for (int q = 0; q < 9; ++q) tab[q * C + c] = aq[q];
    }
}

int launch_phi_coefq(const OpArgs& A, double* tab, cudaStream_t s) {
    const int64_t C = (int64_t)A.L.nx * A.L.ny;
    int64_t blocks = (C + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const Q2Tab T = make_q2_host(A.L.hx, A.L.hy);
    pdl_launch(phi_coefq_kernel, dim3((unsigned)blocks), dim3(256), 0, s, A, T, tab);
    return PFFMG_OK;
}

PFFMG_INSTANTIATE_LAUNCH2(launch2q)

}  // namespace pffmg
