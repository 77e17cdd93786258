// Geometric-multigrid transfers between nested lattice levels l (coarse) and
// l+1 (fine): Q1 prolongation P, its transpose, nodal injection of states and
// of packed constraint flags.  Restates reference fem.py:308-411 (the scipy
// CSR built from lattice keys) as gather stencils -- no atomics, each output
// written by exactly one thread, summation in increasing input-id order like
// the CSR products -- and fuses the V-cycle masking of mgsolve.py:228-234.
#include <cstdlib>

#include "common.cuh"

namespace pffmg {

// Slab-aware indexing.  The cut axis is the last one (y in 2D, z in 3D);
// local plane p of a lattice is global plane p + plane0.  Kernels iterate over
// the owned planes [own_lo, own_hi) of their output lattice only.

// Launch geometry of the point kernels: x = block column, grid.y / grid.z = the
// owned rows / planes (no 64-bit index divisions per point).
__device__ __forceinline__ bool grid_point(const Lat& L, int& x, int& y, int& z) {
    x = (int)(blockIdx.x * blockDim.x + threadIdx.x);
    if (x > L.nx) return false;
    if (L.dim == 3) {
        y = (int)blockIdx.y;
        z = (int)blockIdx.z + L.own_lo;
    } else {
        y = (int)blockIdx.y + L.own_lo;
        z = 0;
    }
    return true;
}

// Component-parallel variant: gridDim.x = gx * ncomp blocks, component k = blockIdx.x / gx
// (a coarse vertex's gather of 9 / 27 fine values per component is then one
// thread's work: 3-4x more threads in flight on the small coarse grids).
__device__ __forceinline__ bool grid_point_comp(const Lat& L, int gx, int& x, int& y, int& z, int& k) {
    k = (int)blockIdx.x / gx;
    x = (int)(((int)blockIdx.x - k * gx) * blockDim.x + threadIdx.x);
    if (x > L.nx) return false;
    if (L.dim == 3) {
        y = (int)blockIdx.y;
        z = (int)blockIdx.z + L.own_lo;
    } else {
        y = (int)blockIdx.y + L.own_lo;
        z = 0;
    }
    return true;
}

static dim3 grid_points(const Lat& L, int threads) {
    const unsigned gx = (unsigned)((L.nx + 1 + threads - 1) / threads);
    const int own = L.own_hi - L.own_lo;
    if (L.dim == 3) return dim3(gx, (unsigned)(L.ny + 1), (unsigned)own);
    return dim3(gx, (unsigned)own, 1);
}

// fine local coordinates of the fine lattice point 2*(coarse point) + (a, b, c)
__device__ __forceinline__ void fine_of(const Lat& Lc, const Lat& Lf, int x, int y, int z, int a, int b, int c,
                                        int& fx, int& fy, int& fz) {
    fx = 2 * x + a;
    if (Lc.dim == 3) {
        fy = 2 * y + b;
        fz = 2 * (z + Lc.plane0) + c - Lf.plane0;
    } else {
        fy = 2 * (y + Lc.plane0) + b - Lf.plane0;
        fz = 0;
    }
}

// (P^T vf)[c] of one component (vfk = that component's fine vector): fine
// neighbours in increasing id order, the CSR product order of fem.py:323-339.
template <int D>
__device__ __forceinline__ double restrict_gather(const Lat& Lc, const Lat& Lf, int x, int y, int z,
                                                  const double* __restrict__ vfk) {
    constexpr int zlo = D == 3 ? -1 : 0, zhi = D == 3 ? 1 : 0;
    constexpr int NT = D == 3 ? 27 : 9;
    double val[NT];
    int t = 0;
#pragma unroll
    for (int c = zlo; c <= zhi; ++c)
#pragma unroll
        for (int b = -1; b <= 1; ++b)
#pragma unroll
            for (int a = -1; a <= 1; ++a, ++t) {
                int fx, fy, fz;
                fine_of(Lc, Lf, x, y, z, a, b, c, fx, fy, fz);
                const int64_t fid = vertex_id(Lf, fx, fy, fz);
                val[t] = fid >= 0 ? __ldg(vfk + fid) : 0.0;      // all loads in flight before the sum
            }
    double acc = 0.0;
    t = 0;
#pragma unroll
    for (int c = zlo; c <= zhi; ++c)
#pragma unroll
        for (int b = -1; b <= 1; ++b)
#pragma unroll
            for (int a = -1; a <= 1; ++a, ++t) {
                const double w = (a ? 0.5 : 1.0) * (b ? 0.5 : 1.0) * (c ? 0.5 : 1.0);
                acc += w * val[t];
            }
    return acc;
}

// vc[k] = sum_{fine f} P[f, c] vf[k][f]  for owned coarse vertices c, then masking.
template <int D>
__global__ void restrict_kernel(Lat Lc, Lat Lf, int gx, int comp0, const double* __restrict__ vf,
                                double* __restrict__ vc, const uint8_t* __restrict__ cflags) {
    pdl_wait();
    int x, y, z, k;
    if (!grid_point_comp(Lc, gx, x, y, z, k)) return;
    const int64_t cid = vertex_id(Lc, x, y, z);
    if (cid < 0) return;
    const uint8_t fl = cflags ? cflags[cid] : 0;
    const double acc = restrict_gather<D>(Lc, Lf, x, y, z, vf + (int64_t)k * Lf.V);
    vc[(int64_t)k * Lc.V + cid] = ((fl >> (comp0 + k)) & 1) ? 0.0 : acc;
}

// Restriction of all components into the coarse level's right-hand side fused
// with the start of its block-diagonal Chebyshev smoother from x = 0
// (mgsolve.py:95, 103-106; the arithmetic of cheb_init_zero_bd_k): per coarse
// dof rc = (P^T vf)[masked]; vc = r = rc; d = inv rc / theta_block; x = d.
template <int D>
__global__ void restrict_init_bd_kernel(Lat Lc, Lat Lf, int gx, const double* __restrict__ vf,
                                        double* __restrict__ vc, const uint8_t* __restrict__ cflags,
                                        const double* __restrict__ inv, const double* __restrict__ tu,
                                        const double* __restrict__ tp, double* __restrict__ r,
                                        double* __restrict__ d, double* __restrict__ x) {
    pdl_wait();
    int X, Y, Z, k;
    if (!grid_point_comp(Lc, gx, X, Y, Z, k)) return;
    const int64_t cid = vertex_id(Lc, X, Y, Z);
    if (cid < 0) return;
    const uint8_t fl = cflags[cid];
    const int64_t g = (int64_t)k * Lc.V + cid;
    const double iv = __ldg(inv + g);
    const double th = k < D ? *tu : *tp;
    const double acc = restrict_gather<D>(Lc, Lf, X, Y, Z, vf + (int64_t)k * Lf.V);
    const double ri = ((fl >> k) & 1) ? 0.0 : acc;
    const double di = (iv * ri) / th;
    vc[g] = ri;
    d[g] = di;
    if (r) {                                     // (NULL: the first step is pffmg_cheb_first_bd)
        r[g] = ri;
        x[g] = 0.0 + di;
    }
}

// All components of a coarse vertex in one thread (large levels, 3D: the
// 9 / 27 fine ids of the vertex are looked up once).
// vc[k] = sum_{fine f} P[f, c] vf[k][f]  for owned coarse vertices c, then masking.
template <int D>
__global__ void restrict_all_kernel(Lat Lc, Lat Lf, int ncomp, int comp0, const double* __restrict__ vf,
                                double* __restrict__ vc, const uint8_t* __restrict__ cflags) {
    pdl_wait();
    int x, y, z;
    if (!grid_point(Lc, x, y, z)) return;
    {
        const int64_t cid = vertex_id(Lc, x, y, z);
        if (cid < 0) return;
        const uint8_t fl = cflags ? cflags[cid] : 0;
        constexpr int zlo = D == 3 ? -1 : 0, zhi = D == 3 ? 1 : 0;
        // fine neighbours in increasing id order (the CSR product order); each
        // neighbour's id is looked up once for all components
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int c = zlo; c <= zhi; ++c)
#pragma unroll
            for (int b = -1; b <= 1; ++b)
#pragma unroll
                for (int a = -1; a <= 1; ++a) {
                    int fx, fy, fz;
                    fine_of(Lc, Lf, x, y, z, a, b, c, fx, fy, fz);
                    const int64_t fid = vertex_id(Lf, fx, fy, fz);
                    if (fid < 0) continue;
                    const double w = (a ? 0.5 : 1.0) * (b ? 0.5 : 1.0) * (c ? 0.5 : 1.0);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (k < ncomp) acc[k] += w * __ldg(vf + (int64_t)k * Lf.V + fid);
                }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k >= ncomp) break;
            vc[(int64_t)k * Lc.V + cid] = ((fl >> (comp0 + k)) & 1) ? 0.0 : acc[k];
        }
    }
}

// Restriction of all components into the coarse level's right-hand side fused
// with the start of its block-diagonal Chebyshev smoother from x = 0
// (mgsolve.py:95, 103-106; the arithmetic of cheb_init_zero_bd_k): per coarse
// dof rc = (P^T vf)[masked]; vc = r = rc; d = inv rc / theta_block; x = d.
template <int D>
__global__ void restrict_init_bd_all_kernel(Lat Lc, Lat Lf, const double* __restrict__ vf, double* __restrict__ vc,
                                        const uint8_t* __restrict__ cflags, const double* __restrict__ inv,
                                        const double* __restrict__ tu, const double* __restrict__ tp,
                                        double* __restrict__ r, double* __restrict__ d, double* __restrict__ x) {
    pdl_wait();
    int X, Y, Z;
    if (!grid_point(Lc, X, Y, Z)) return;
    const int64_t cid = vertex_id(Lc, X, Y, Z);
    if (cid < 0) return;
    constexpr int NC = D + 1;
    const uint8_t fl = cflags[cid];
    constexpr int zlo = D == 3 ? -1 : 0, zhi = D == 3 ? 1 : 0;
    double acc[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) acc[k] = 0.0;
#pragma unroll
    for (int c = zlo; c <= zhi; ++c)
#pragma unroll
        for (int b = -1; b <= 1; ++b)
#pragma unroll
            for (int a = -1; a <= 1; ++a) {
                int fx, fy, fz;
                fine_of(Lc, Lf, X, Y, Z, a, b, c, fx, fy, fz);
                const int64_t fid = vertex_id(Lf, fx, fy, fz);
                if (fid < 0) continue;
                const double w = (a ? 0.5 : 1.0) * (b ? 0.5 : 1.0) * (c ? 0.5 : 1.0);
#pragma unroll
                for (int k = 0; k < NC; ++k) acc[k] += w * __ldg(vf + (int64_t)k * Lf.V + fid);
            }
    const double thu = *tu, thp = *tp;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        const int64_t g = (int64_t)k * Lc.V + cid;
        const double ri = ((fl >> k) & 1) ? 0.0 : acc[k];
        const double di = (__ldg(inv + g) * ri) / (k < D ? thu : thp);
        vc[g] = ri;
        d[g] = di;
        if (r) {                                 // (NULL: the first step is pffmg_cheb_first_bd)
            r[g] = ri;
            x[g] = 0.0 + di;
        }
    }
}

// vf[k][f] (=|+=) sum_c P[f, c] vc[k][c] for owned fine vertices, zeroed where
// the fine dof is constrained.  Coarse corners in bit order (x fastest), as
// the COO entries of fem.py:323-339; corners with a zero weight are skipped.
template <int D, int NC>
__global__ void prolongate_kernel(Lat Lc, Lat Lf, int comp0, const double* __restrict__ vc,
                                  double* __restrict__ vf, const uint8_t* __restrict__ fflags,
                                  int accumulate) {
    pdl_wait();
    int X, Y, Z;
    if (!grid_point(Lf, X, Y, Z)) return;
    const int64_t fid = vertex_id(Lf, X, Y, Z);
    if (fid < 0) return;
    const uint8_t fl = fflags ? fflags[fid] : 0;
    double cur[NC];                              // the fine values first: the long (DRAM) loads
#pragma unroll
    for (int k = 0; k < NC; ++k) cur[k] = accumulate ? vf[(int64_t)k * Lf.V + fid] : 0.0;
    // global coordinate along the cut axis decides the parity
    const int Yg = D == 3 ? Y : Y + Lf.plane0, Zg = D == 3 ? Z + Lf.plane0 : 0;
    const int shY = D == 3 ? 0 : Lc.plane0, shZ = D == 3 ? Lc.plane0 : 0;
    const int lox = X >> 1, hix = (X + 1) >> 1;
    const int loy = (Yg >> 1) - shY, hiy = ((Yg + 1) >> 1) - shY;
    const int loz = (Zg >> 1) - shZ, hiz = ((Zg + 1) >> 1) - shZ;
    const bool ox = X & 1, oy = Yg & 1, oz = Zg & 1;
    const double w = (ox ? 0.5 : 1.0) * (oy ? 0.5 : 1.0) * (D == 3 && oz ? 0.5 : 1.0);
    int64_t cid[1 << D];
#pragma unroll
    for (int bits = 0; bits < (1 << D); ++bits) {
        const bool bx = bits & 1, by = (bits >> 1) & 1, bz = (bits >> 2) & 1;
        const bool used = !((bx && !ox) || (by && !oy) || (bz && !oz));
        cid[bits] = used ? vertex_id(Lc, bx ? hix : lox, by ? hiy : loy, D == 3 ? (bz ? hiz : loz) : 0) : -1;
    }
    double cval[NC][1 << D];
#pragma unroll
    for (int k = 0; k < NC; ++k)
#pragma unroll
        for (int bits = 0; bits < (1 << D); ++bits)
            cval[k][bits] = cid[bits] >= 0 ? __ldg(vc + (int64_t)k * Lc.V + cid[bits]) : 0.0;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int bits = 0; bits < (1 << D); ++bits)
            if (cid[bits] >= 0) acc += w * cval[k][bits];
        const int64_t g = (int64_t)k * Lf.V + fid;
        if ((fl >> (comp0 + k)) & 1) acc = 0.0;
        vf[g] = accumulate ? cur[k] + acc : acc;
    }
}

template <int D>
static void launch_prolongate(const Lat& Lc, const Lat& Lf, int n_comp, int comp0, const double* vc, double* vf,
                              const uint8_t* fine_flags, int accumulate, cudaStream_t s) {
    const dim3 g = grid_points(Lf, 128), b(128);
    switch (n_comp) {
        case 1: pdl_launch(prolongate_kernel<D, 1>, g, b, 0, s, Lc, Lf, comp0, vc, vf, fine_flags, accumulate); break;
        case 2: pdl_launch(prolongate_kernel<D, 2>, g, b, 0, s, Lc, Lf, comp0, vc, vf, fine_flags, accumulate); break;
        case 3: pdl_launch(prolongate_kernel<D, 3>, g, b, 0, s, Lc, Lf, comp0, vc, vf, fine_flags, accumulate); break;
        default: pdl_launch(prolongate_kernel<D, 4>, g, b, 0, s, Lc, Lf, comp0, vc, vf, fine_flags, accumulate); break;
    }
}

// ---- Q2 levels (2D boxes; node lattices, see oracle/q2.py) ----------------
// 1D Q2 interpolation of a coarse function at the fine nodes: fine node j
// even -> coarse node j/2; j = 4c+1 / 4c+3 -> coarse nodes 2c, 2c+1, 2c+2 with
// weights (3/8, 3/4, -1/8) / (-1/8, 3/4, 3/8).  Restriction = its transpose:
// coarse node i even gathers fine 2i + {-3,-1,0,1,3} with (-1/8, 3/8, 1, 3/8,
// -1/8); i odd gathers 2i + {-1,0,1} with (3/4, 1, 3/4).
__device__ __forceinline__ int q2_restrict_taps(int i, int (&off)[5], double (&w)[5]) {
    if ((i & 1) == 0) {
        off[0] = -3; off[1] = -1; off[2] = 0; off[3] = 1; off[4] = 3;
        w[0] = -0.125; w[1] = 0.375; w[2] = 1.0; w[3] = 0.375; w[4] = -0.125;
        return 5;
    }
    off[0] = -1; off[1] = 0; off[2] = 1;
    w[0] = 0.75; w[1] = 1.0; w[2] = 0.75;
    return 3;
}

__device__ __forceinline__ int q2_prolong_taps(int j, int (&idx)[3], double (&w)[3]) {
    if ((j & 1) == 0) {
        idx[0] = j >> 1;
        w[0] = 1.0;
        return 1;
    }
    const int c = j >> 2;
    const bool first = (j & 3) == 1;
    idx[0] = 2 * c; idx[1] = 2 * c + 1; idx[2] = 2 * c + 2;
    w[0] = first ? 0.375 : -0.125;
    w[1] = 0.75;
    w[2] = first ? -0.125 : 0.375;
    return 3;
}

// Lc / Lf are the NODE lattices (nx = 2 * cells): nxn = nx + 1 nodes per row.
// Slabs: the output lattice's owned node rows only; tap parities and the
// coarse/fine row pairing use global rows (local row + plane0).
// One thread per (coarse node, component): blockIdx.y = owned coarse row,
// blockIdx.z = component; the (up to 5 x 5) fine values are loaded before the
// sum, which keeps the increasing-fine-id order of the CSR product.
// With d set (pffmg_restrict_init_bd on Q2 levels): all components from comp0 =
// 0, fused with the coarse level's block-diagonal Chebyshev start from x = 0
// (the arithmetic of cheb_init_zero_bd_k; r / x optional as there).
__global__ void restrict_q2_kernel(Lat Lc, Lat Lf, int comp0, const double* __restrict__ vf,
                                   double* __restrict__ vc, const uint8_t* __restrict__ cflags,
                                   const double* __restrict__ inv, const double* __restrict__ tu,
                                   const double* __restrict__ tp, double* __restrict__ r,
                                   double* __restrict__ d, double* __restrict__ xs) {
    pdl_wait();
    const int nxc = Lc.nx + 1, nxf = Lf.nx + 1, nyf = Lf.ny + 1;
    const int x = (int)(blockIdx.x * blockDim.x + threadIdx.x);
    if (x >= nxc) return;
    const int y = Lc.own_lo + (int)blockIdx.y, k = (int)blockIdx.z;
    const int yg = y + Lc.plane0;
    int ox[5], oy[5];
    double wx[5], wy[5];
    const int nx5 = q2_restrict_taps(x, ox, wx), ny5 = q2_restrict_taps(yg, oy, wy);
    const double* __restrict__ vfk = vf + (int64_t)k * Lf.V;
    double val[25];
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        const int fy = 2 * yg + oy[b < ny5 ? b : 0] - Lf.plane0;
        const bool oky = b < ny5 && fy >= 0 && fy < nyf;
#pragma unroll
        for (int a = 0; a < 5; ++a) {
            const int fx = 2 * x + ox[a < nx5 ? a : 0];
            const bool ok = oky && a < nx5 && fx >= 0 && fx < nxf;
            val[5 * b + a] = ok ? __ldg(vfk + (int64_t)fy * nxf + fx) : 0.0;
        }
    }
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        const int fy = 2 * yg + oy[b < ny5 ? b : 0] - Lf.plane0;
        if (!(b < ny5 && fy >= 0 && fy < nyf)) continue;
#pragma unroll
        for (int a = 0; a < 5; ++a) {
            const int fx = 2 * x + ox[a < nx5 ? a : 0];
            if (!(a < nx5 && fx >= 0 && fx < nxf)) continue;
            acc += (wx[a] * wy[b]) * val[5 * b + a];
        }
    }
    const int64_t cid = (int64_t)y * nxc + x;
    const uint8_t fl = cflags ? cflags[cid] : 0;
    const int64_t g = (int64_t)k * Lc.V + cid;
    const double ri = ((fl >> (comp0 + k)) & 1) ? 0.0 : acc;
    vc[g] = ri;
    if (d) {
        const double di = (__ldg(inv + g) * ri) / (k < 2 ? *tu : *tp);
        d[g] = di;
        if (r) {
            r[g] = ri;
            xs[g] = 0.0 + di;
        }
    }
}

// blockIdx.y = owned fine row; NC components per thread, the fine values and
// the (up to 3 x 3) coarse values loaded before the sums.
template <int NC>
__global__ void prolongate_q2_kernel(Lat Lc, Lat Lf, int comp0, const double* __restrict__ vc,
                                     double* __restrict__ vf, const uint8_t* __restrict__ fflags,
                                     int accumulate) {
    pdl_wait();
    const int nxc = Lc.nx + 1, nxf = Lf.nx + 1;
    const int X = (int)(blockIdx.x * blockDim.x + threadIdx.x);
    if (X >= nxf) return;
    const int Y = Lf.own_lo + (int)blockIdx.y;
    const int64_t fid = (int64_t)Y * nxf + X;
    double cur[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) cur[k] = accumulate ? vf[(int64_t)k * Lf.V + fid] : 0.0;
    int ix[3], iy[3];
    double wx[3], wy[3];
    const int nx3 = q2_prolong_taps(X, ix, wx), ny3 = q2_prolong_taps(Y + Lf.plane0, iy, wy);
    const uint8_t fl = fflags ? fflags[fid] : 0;
    double cv[NC][9];
#pragma unroll
    for (int k = 0; k < NC; ++k)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int a = 0; a < 3; ++a)
                cv[k][3 * b + a] = (b < ny3 && a < nx3)
                                       ? __ldg(vc + (int64_t)k * Lc.V + (int64_t)(iy[b] - Lc.plane0) * nxc + ix[a])
                                       : 0.0;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int a = 0; a < 3; ++a)
                if (b < ny3 && a < nx3) acc += (wx[a] * wy[b]) * cv[k][3 * b + a];
        const int64_t g = (int64_t)k * Lf.V + fid;
        if ((fl >> (comp0 + k)) & 1) acc = 0.0;
        vf[g] = accumulate ? cur[k] + acc : acc;
    }
}

__global__ void inject_f64_kernel(Lat Lc, Lat Lf, int ncomp, const double* __restrict__ vf,
                                  double* __restrict__ vc) {
    pdl_wait();
    int x, y, z;
    if (!grid_point(Lc, x, y, z)) return;
    {
        const int64_t cid = vertex_id(Lc, x, y, z);
        if (cid < 0) return;
        int fx, fy, fz;
        fine_of(Lc, Lf, x, y, z, 0, 0, 0, fx, fy, fz);
        const int64_t fid = vertex_id(Lf, fx, fy, fz);
        for (int k = 0; k < ncomp; ++k) vc[(int64_t)k * Lc.V + cid] = vf[(int64_t)k * Lf.V + fid];
    }
}

__global__ void inject_u8_kernel(Lat Lc, Lat Lf, const uint8_t* __restrict__ ff, uint8_t* __restrict__ fc,
                                 int64_t* __restrict__ map) {
    pdl_wait();
    int x, y, z;
    if (!grid_point(Lc, x, y, z)) return;
    {
        const int64_t cid = vertex_id(Lc, x, y, z);
        if (cid < 0) return;
        int fx, fy, fz;
        fine_of(Lc, Lf, x, y, z, 0, 0, 0, fx, fy, fz);
        const int64_t fid = vertex_id(Lf, fx, fy, fz);
        if (fc) fc[cid] = ff[fid];
        if (map) map[cid] = fid;
    }
}

// Q2 levels are handled on their node lattices (a Q1-shaped lattice of twice
// the cells): injection is then the Q1 vertex injection.
static void to_node_lattice(Lat* L) {
    if (L->order != 2) return;
    L->nx *= 2;
    L->ny *= 2;
    L->hx *= 0.5;
    L->hy *= 0.5;
    L->order = 1;
}

static int check_pair(const pffmg_lattice* c, const pffmg_lattice* f, Lat* Lc, Lat* Lf, bool* q2 = nullptr) {
    int rc = make_lat(c, Lc);
    if (rc) return rc;
    rc = make_lat(f, Lf);
    if (rc) return rc;
    PFFMG_REQUIRE(Lc->order == Lf->order, "levels of different element order");
    if (q2) *q2 = Lc->order == 2;
    to_node_lattice(Lc);
    to_node_lattice(Lf);
    // the cut axis (last) may be a slab of the level: only the others must nest
    PFFMG_REQUIRE(Lc->dim == Lf->dim && Lf->nx == 2 * Lc->nx && (Lc->dim == 2 || Lf->ny == 2 * Lc->ny),
                  "levels are not nested lattices (coarse %dx%dx%d, fine %dx%dx%d)", Lc->nx, Lc->ny,
                  Lc->nz, Lf->nx, Lf->ny, Lf->nz);
    return PFFMG_OK;
}


// Restriction into small 2D levels runs one thread per (coarse vertex,
// component): the launch then has 3x the threads to hide the latency of the
// gather (cfg2 V-cycle 621 -> 609 us, cfg1 159 -> 152 us).  Large 2D levels
// (full-size restriction 16.4 -> 20.5 us) and 3D levels (27 taps: cfg4 37 ->
// 70 us) keep all components of a vertex in one thread.
static bool comp_parallel(const Lat& Lc) {
    static const int64_t maxv = [] {
        const char* e = getenv("PFFMG_RESTRICT_CP_MAXV");       // tuning: largest coarse level taking it
        return e ? (int64_t)atoll(e) : (int64_t)1 << 17;
    }();
    return Lc.dim == 2 && Lc.V <= maxv;
}

}  // namespace pffmg

using namespace pffmg;

extern "C" int pffmg_restrict(const pffmg_lattice* coarse, const pffmg_lattice* fine, int n_comp,
                              int comp0, const double* vf, double* vc, const uint8_t* coarse_flags,
                              void* stream) {
    Lat Lc, Lf;
    bool q2 = false;
    int rc = check_pair(coarse, fine, &Lc, &Lf, &q2);
    if (rc) return rc;
    PFFMG_REQUIRE(vf && vc && n_comp >= 1 && comp0 >= 0 && comp0 + n_comp <= Lc.dim + 1,
                  "pffmg_restrict: bad arguments");
    if (q2) {
        pdl_launch(restrict_q2_kernel,
                   dim3((unsigned)((Lc.nx + 1 + 127) / 128), (unsigned)(Lc.own_hi - Lc.own_lo), (unsigned)n_comp),
                   dim3(128), 0, as_stream(stream), Lc, Lf, comp0, vf, vc, coarse_flags, (const double*)nullptr,
                   (const double*)nullptr, (const double*)nullptr, (double*)nullptr, (double*)nullptr,
                   (double*)nullptr);
        return check_launch("pffmg_restrict");
    }
    dim3 g = grid_points(Lc, 128);
    if (Lc.dim == 3) {
        pdl_launch(restrict_all_kernel<3>, g, dim3(128), 0, as_stream(stream), Lc, Lf, n_comp, comp0, vf, vc,
                   coarse_flags);
    } else if (comp_parallel(Lc)) {
        const int gx = (int)g.x;
        g.x *= (unsigned)n_comp;                 // one thread per (coarse vertex, component)
        pdl_launch(restrict_kernel<2>, g, dim3(128), 0, as_stream(stream), Lc, Lf, gx, comp0, vf, vc, coarse_flags);
    } else {
        pdl_launch(restrict_all_kernel<2>, g, dim3(128), 0, as_stream(stream), Lc, Lf, n_comp, comp0, vf, vc,
                   coarse_flags);
    }
    return check_launch("pffmg_restrict");
}

extern "C" int pffmg_prolongate(const pffmg_lattice* coarse, const pffmg_lattice* fine, int n_comp,
                                int comp0, const double* vc, double* vf, const uint8_t* fine_flags,
                                int accumulate, void* stream) {
    Lat Lc, Lf;
    bool q2 = false;
    int rc = check_pair(coarse, fine, &Lc, &Lf, &q2);
    if (rc) return rc;
    PFFMG_REQUIRE(vf && vc && n_comp >= 1 && comp0 >= 0 && comp0 + n_comp <= Lc.dim + 1,
                  "pffmg_prolongate: bad arguments");
    if (q2) {
        const dim3 g((unsigned)((Lf.nx + 1 + 127) / 128), (unsigned)(Lf.own_hi - Lf.own_lo)), b(128);
        const cudaStream_t s = as_stream(stream);
        switch (n_comp) {
            case 1: pdl_launch(prolongate_q2_kernel<1>, g, b, 0, s, Lc, Lf, comp0, vc, vf, fine_flags, accumulate); break;
            case 2: pdl_launch(prolongate_q2_kernel<2>, g, b, 0, s, Lc, Lf, comp0, vc, vf, fine_flags, accumulate); break;
            default: pdl_launch(prolongate_q2_kernel<3>, g, b, 0, s, Lc, Lf, comp0, vc, vf, fine_flags, accumulate); break;
        }
        return check_launch("pffmg_prolongate");
    }
    if (Lf.dim == 3)
        launch_prolongate<3>(Lc, Lf, n_comp, comp0, vc, vf, fine_flags, accumulate, as_stream(stream));
    else
        launch_prolongate<2>(Lc, Lf, n_comp, comp0, vc, vf, fine_flags, accumulate, as_stream(stream));
    return check_launch("pffmg_prolongate");
}

extern "C" int pffmg_inject_f64(const pffmg_lattice* coarse, const pffmg_lattice* fine, int n_comp,
                                const double* vf, double* vc, void* stream) {
    Lat Lc, Lf;
    int rc = check_pair(coarse, fine, &Lc, &Lf);
    if (rc) return rc;
    PFFMG_REQUIRE(vf && vc && n_comp >= 1, "pffmg_inject_f64: bad arguments");
    pdl_launch(inject_f64_kernel, dim3(grid_points(Lc, 128)), dim3(128), 0, as_stream(stream), Lc, Lf, n_comp, vf, vc);
    return check_launch("pffmg_inject_f64");
}

extern "C" int pffmg_inject_flags(const pffmg_lattice* coarse, const pffmg_lattice* fine,
                                  const uint8_t* ff, uint8_t* fc, void* stream) {
    Lat Lc, Lf;
    int rc = check_pair(coarse, fine, &Lc, &Lf);
    if (rc) return rc;
    PFFMG_REQUIRE(ff && fc, "pffmg_inject_flags: bad arguments");
    pdl_launch(inject_u8_kernel, dim3(grid_points(Lc, 128)), dim3(128), 0, as_stream(stream), Lc, Lf, ff, fc, nullptr);
    return check_launch("pffmg_inject_flags");
}

extern "C" int pffmg_injection_map(const pffmg_lattice* coarse, const pffmg_lattice* fine,
                                   int64_t* out, void* stream) {
    Lat Lc, Lf;
    int rc = check_pair(coarse, fine, &Lc, &Lf);
    if (rc) return rc;
    PFFMG_REQUIRE(out, "pffmg_injection_map: null out");
    pdl_launch(inject_u8_kernel, dim3(grid_points(Lc, 128)), dim3(128), 0, as_stream(stream), Lc, Lf, nullptr, nullptr, out);
    return check_launch("pffmg_injection_map");
}

extern "C" int pffmg_restrict_init_bd(const pffmg_lattice* coarse, const pffmg_lattice* fine, const double* vf,
                                      double* vc, const uint8_t* coarse_flags, const double* invdiag,
                                      const double* theta_u, const double* theta_p, double* r, double* d,
                                      double* x, void* stream) {
    Lat Lc, Lf;
    bool q2 = false;
    int rc = check_pair(coarse, fine, &Lc, &Lf, &q2);
    if (rc) return rc;
    PFFMG_REQUIRE(vf && vc && coarse_flags && invdiag && theta_u && theta_p && d && !r == !x,
                  "pffmg_restrict_init_bd: bad arguments");
    if (q2) {
        pdl_launch(restrict_q2_kernel,
                   dim3((unsigned)((Lc.nx + 1 + 127) / 128), (unsigned)(Lc.own_hi - Lc.own_lo), 3u), dim3(128), 0,
                   as_stream(stream), Lc, Lf, 0, vf, vc, coarse_flags, invdiag, theta_u, theta_p, r, d, x);
        return check_launch("pffmg_restrict_init_bd");
    }
    dim3 g = grid_points(Lc, 128);
    if (Lc.dim == 3) {
        pdl_launch(restrict_init_bd_all_kernel<3>, g, dim3(128), 0, as_stream(stream), Lc, Lf, vf, vc, coarse_flags,
                   invdiag, theta_u, theta_p, r, d, x);
    } else if (comp_parallel(Lc)) {
        const int gx = (int)g.x;
        g.x *= (unsigned)(Lc.dim + 1);           // one thread per (coarse vertex, component)
        pdl_launch(restrict_init_bd_kernel<2>, g, dim3(128), 0, as_stream(stream), Lc, Lf, gx, vf, vc, coarse_flags,
                   invdiag, theta_u, theta_p, r, d, x);
    } else {
        pdl_launch(restrict_init_bd_all_kernel<2>, g, dim3(128), 0, as_stream(stream), Lc, Lf, vf, vc, coarse_flags,
                   invdiag, theta_u, theta_p, r, d, x);
    }
    return check_launch("pffmg_restrict_init_bd");
}
