// Geometric-multigrid transfers between nested lattice levels l (coarse) and
// l+1 (fine): Q1 prolongation P, its transpose, nodal injection of states and
// of packed constraint flags.  Restates reference fem.py:308-411 (the scipy
// CSR built from lattice keys) as gather stencils -- no atomics, each output
// written by exactly one thread, summation in increasing input-id order like
// the CSR products -- and fuses the V-cycle masking of mgsolve.py:228-234.
#include "common.cuh"

namespace pffmg {

// Slab-aware indexing.  The cut axis is the last one (y in 2D, z in 3D);
// local plane p of a lattice is global plane p + plane0.  Kernels iterate over
// the owned planes [own_lo, own_hi) of their output lattice only.

// i-th point of the owned planes of L (x fastest) -> local lattice coordinates
__device__ __forceinline__ void owned_coords(const Lat& L, int64_t i, int& x, int& y, int& z) {
    const int64_t nxv = L.nx + 1;
    x = (int)(i % nxv);
    const int64_t t = i / nxv;
    if (L.dim == 3) {
        const int64_t nyv = L.ny + 1;
        y = (int)(t % nyv);
        z = (int)(t / nyv) + L.own_lo;
    } else {
        y = (int)t + L.own_lo;
        z = 0;
    }
}

__host__ __device__ __forceinline__ int64_t owned_points(const Lat& L) {
    const int64_t plane = L.dim == 3 ? (int64_t)(L.nx + 1) * (L.ny + 1) : (int64_t)(L.nx + 1);
    return plane * (L.own_hi - L.own_lo);
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

// vc[k] = sum_{fine f} P[f, c] vf[k][f]  for owned coarse vertices c, then masking.
__global__ void restrict_kernel(Lat Lc, Lat Lf, int ncomp, int comp0, const double* __restrict__ vf,
                                double* __restrict__ vc, const uint8_t* __restrict__ cflags) {
    const int64_t npts = owned_points(Lc);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts;
         i += (int64_t)gridDim.x * blockDim.x) {
        int x, y, z;
        owned_coords(Lc, i, x, y, z);
        const int64_t cid = vertex_id(Lc, x, y, z);
        if (cid < 0) continue;
        const uint8_t fl = cflags ? cflags[cid] : 0;
        const int zlo = Lc.dim == 3 ? -1 : 0, zhi = Lc.dim == 3 ? 1 : 0;
        // fine neighbours in increasing id order (the CSR product order); each
        // neighbour's id is looked up once for all components
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
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

// vf[k][f] (=|+=) sum_c P[f, c] vc[k][c] for owned fine vertices, zeroed where
// the fine dof is constrained.
__global__ void prolongate_kernel(Lat Lc, Lat Lf, int ncomp, int comp0, const double* __restrict__ vc,
                                  double* __restrict__ vf, const uint8_t* __restrict__ fflags,
                                  int accumulate) {
    const int64_t npts = owned_points(Lf);
    const int D = Lf.dim;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts;
         i += (int64_t)gridDim.x * blockDim.x) {
        int X, Y, Z;
        owned_coords(Lf, i, X, Y, Z);
        const int64_t fid = vertex_id(Lf, X, Y, Z);
        if (fid < 0) continue;
        const uint8_t fl = fflags ? fflags[fid] : 0;
        // global coordinate along the cut axis decides the parity
        const int Yg = D == 3 ? Y : Y + Lf.plane0, Zg = D == 3 ? Z + Lf.plane0 : 0;
        const int shY = D == 3 ? 0 : Lc.plane0, shZ = D == 3 ? Lc.plane0 : 0;
        // corners in bit order (x fastest), as the COO entries of fem.py:323-339
        int64_t cid[8];
        double wt[8];
        int nn = 0;
        const int lox = X >> 1, hix = (X + 1) >> 1;
        const int loy = (Yg >> 1) - shY, hiy = ((Yg + 1) >> 1) - shY;
        const int loz = (Zg >> 1) - shZ, hiz = ((Zg + 1) >> 1) - shZ;
        const bool ox = X & 1, oy = Yg & 1, oz = Zg & 1;
        for (int bits = 0; bits < (1 << D); ++bits) {
            const bool bx = bits & 1, by = (bits >> 1) & 1, bz = (bits >> 2) & 1;
            if ((bx && !ox) || (by && !oy) || (bz && !oz)) continue;
            const double w = (ox ? 0.5 : 1.0) * (oy ? 0.5 : 1.0) * (D == 3 && oz ? 0.5 : 1.0);
            cid[nn] = vertex_id(Lc, bx ? hix : lox, by ? hiy : loy, D == 3 ? (bz ? hiz : loz) : 0);
            wt[nn] = w;
            ++nn;
        }
        for (int k = 0; k < ncomp; ++k) {
            double acc = 0.0;
            for (int t = 0; t < nn; ++t)
                if (cid[t] >= 0) acc += wt[t] * vc[(int64_t)k * Lc.V + cid[t]];
            const int64_t g = (int64_t)k * Lf.V + fid;
            if ((fl >> (comp0 + k)) & 1) acc = 0.0;
            if (accumulate)
                vf[g] += acc;
            else
                vf[g] = acc;
        }
    }
}

__global__ void inject_f64_kernel(Lat Lc, Lat Lf, int ncomp, const double* __restrict__ vf,
                                  double* __restrict__ vc) {
    const int64_t npts = owned_points(Lc);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts;
         i += (int64_t)gridDim.x * blockDim.x) {
        int x, y, z;
        owned_coords(Lc, i, x, y, z);
        const int64_t cid = vertex_id(Lc, x, y, z);
        if (cid < 0) continue;
        int fx, fy, fz;
        fine_of(Lc, Lf, x, y, z, 0, 0, 0, fx, fy, fz);
        const int64_t fid = vertex_id(Lf, fx, fy, fz);
        for (int k = 0; k < ncomp; ++k) vc[(int64_t)k * Lc.V + cid] = vf[(int64_t)k * Lf.V + fid];
    }
}

__global__ void inject_u8_kernel(Lat Lc, Lat Lf, const uint8_t* __restrict__ ff, uint8_t* __restrict__ fc,
                                 int64_t* __restrict__ map) {
    const int64_t npts = owned_points(Lc);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts;
         i += (int64_t)gridDim.x * blockDim.x) {
        int x, y, z;
        owned_coords(Lc, i, x, y, z);
        const int64_t cid = vertex_id(Lc, x, y, z);
        if (cid < 0) continue;
        int fx, fy, fz;
        fine_of(Lc, Lf, x, y, z, 0, 0, 0, fx, fy, fz);
        const int64_t fid = vertex_id(Lf, fx, fy, fz);
        if (fc) fc[cid] = ff[fid];
        if (map) map[cid] = fid;
    }
}

static int check_pair(const pffmg_lattice* c, const pffmg_lattice* f, Lat* Lc, Lat* Lf) {
    int rc = make_lat(c, Lc);
    if (rc) return rc;
    rc = make_lat(f, Lf);
    if (rc) return rc;
    // the cut axis (last) may be a slab of the level: only the others must nest
    PFFMG_REQUIRE(Lc->dim == Lf->dim && Lf->nx == 2 * Lc->nx && (Lc->dim == 2 || Lf->ny == 2 * Lc->ny),
                  "levels are not nested lattices (coarse %dx%dx%d, fine %dx%dx%d)", Lc->nx, Lc->ny,
                  Lc->nz, Lf->nx, Lf->ny, Lf->nz);
    return PFFMG_OK;
}

static int64_t box_points_host(const Lat& L) { return owned_points(L); }

static dim3 grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return dim3((unsigned)b);
}

}  // namespace pffmg

using namespace pffmg;

extern "C" int pffmg_restrict(const pffmg_lattice* coarse, const pffmg_lattice* fine, int n_comp,
                              int comp0, const double* vf, double* vc, const uint8_t* coarse_flags,
                              void* stream) {
    Lat Lc, Lf;
    int rc = check_pair(coarse, fine, &Lc, &Lf);
    if (rc) return rc;
    PFFMG_REQUIRE(vf && vc && n_comp >= 1 && comp0 >= 0 && comp0 + n_comp <= Lc.dim + 1,
                  "pffmg_restrict: bad arguments");
    restrict_kernel<<<grid_for(box_points_host(Lc)), 256, 0, as_stream(stream)>>>(Lc, Lf, n_comp, comp0, vf,
                                                                                vc, coarse_flags);
    return check_launch("pffmg_restrict");
}

extern "C" int pffmg_prolongate(const pffmg_lattice* coarse, const pffmg_lattice* fine, int n_comp,
                                int comp0, const double* vc, double* vf, const uint8_t* fine_flags,
                                int accumulate, void* stream) {
    Lat Lc, Lf;
    int rc = check_pair(coarse, fine, &Lc, &Lf);
    if (rc) return rc;
    PFFMG_REQUIRE(vf && vc && n_comp >= 1 && comp0 >= 0 && comp0 + n_comp <= Lc.dim + 1,
                  "pffmg_prolongate: bad arguments");
    prolongate_kernel<<<grid_for(box_points_host(Lf)), 256, 0, as_stream(stream)>>>(
        Lc, Lf, n_comp, comp0, vc, vf, fine_flags, accumulate);
    return check_launch("pffmg_prolongate");
}

extern "C" int pffmg_inject_f64(const pffmg_lattice* coarse, const pffmg_lattice* fine, int n_comp,
                                const double* vf, double* vc, void* stream) {
    Lat Lc, Lf;
    int rc = check_pair(coarse, fine, &Lc, &Lf);
    if (rc) return rc;
    PFFMG_REQUIRE(vf && vc && n_comp >= 1, "pffmg_inject_f64: bad arguments");
    inject_f64_kernel<<<grid_for(box_points_host(Lc)), 256, 0, as_stream(stream)>>>(Lc, Lf, n_comp, vf, vc);
    return check_launch("pffmg_inject_f64");
}

extern "C" int pffmg_inject_flags(const pffmg_lattice* coarse, const pffmg_lattice* fine,
                                  const uint8_t* ff, uint8_t* fc, void* stream) {
    Lat Lc, Lf;
    int rc = check_pair(coarse, fine, &Lc, &Lf);
    if (rc) return rc;
    PFFMG_REQUIRE(ff && fc, "pffmg_inject_flags: bad arguments");
    inject_u8_kernel<<<grid_for(box_points_host(Lc)), 256, 0, as_stream(stream)>>>(Lc, Lf, ff, fc, nullptr);
    return check_launch("pffmg_inject_flags");
}

extern "C" int pffmg_injection_map(const pffmg_lattice* coarse, const pffmg_lattice* fine,
                                   int64_t* out, void* stream) {
    Lat Lc, Lf;
    int rc = check_pair(coarse, fine, &Lc, &Lf);
    if (rc) return rc;
    PFFMG_REQUIRE(out, "pffmg_injection_map: null out");
    inject_u8_kernel<<<grid_for(box_points_host(Lc)), 256, 0, as_stream(stream)>>>(Lc, Lf, nullptr, nullptr, out);
    return check_launch("pffmg_injection_map");
}
