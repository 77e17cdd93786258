// Error state, device queries and host-side construction of the kernel
// argument structs for libpffmg.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <cstdlib>

#include "common.cuh"

namespace pffmg {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: CUDA launch failed: %s", what, cudaGetErrorString(e));
        return PFFMG_ERR_CUDA;
    }
    return PFFMG_OK;
}

static std::atomic<int> g_pdl_on{1};

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("PFFMG_PDL");
        return !(e && e[0] == '0');
    }();
    return on && g_pdl_on.load(std::memory_order_relaxed) != 0;
}

int pdl_set(int on) { return g_pdl_on.exchange(on ? 1 : 0); }

int sm_count() {
    static int cached = 0;
    if (!cached) {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        cached = n;
    }
    return cached;
}

int check_device() {
    static int first = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        set_error("cudaGetDevice failed");
        return PFFMG_ERR_CUDA;
    }
    if (first < 0) first = dev;
    PFFMG_REQUIRE(dev == first,
                  "libpffmg serves one GPU per process: it was first used on device %d, now called on device %d",
                  first, dev);
    return PFFMG_OK;
}

int make_lat(const pffmg_lattice* in, Lat* out) {
    PFFMG_REQUIRE(in, "null lattice");
    PFFMG_REQUIRE(in->struct_size == (int32_t)sizeof(pffmg_lattice),
                  "pffmg_lattice.struct_size = %d, this library expects %d (ABI version %d)",
                  in->struct_size, (int)sizeof(pffmg_lattice), PFFMG_ABI_VERSION);
    PFFMG_REQUIRE(in->dim == 2 || in->dim == 3, "lattice dim must be 2 or 3 (got %d)", in->dim);
    PFFMG_REQUIRE(in->nx >= 1 && in->ny >= 1 && (in->dim == 2 ? in->nz == 0 : in->nz >= 1),
                  "bad lattice extents %d x %d x %d", in->nx, in->ny, in->nz);
    PFFMG_REQUIRE(in->n_vertices > 0, "n_vertices must be positive");
    const int order = in->order <= 1 ? 1 : in->order;
    PFFMG_REQUIRE(order == 1 || order == 2, "lattice order must be 1 (Q1) or 2 (Q2), got %d", in->order);
    if (order == 2) {
        PFFMG_REQUIRE(in->dim == 2 && in->vrow_off == nullptr, "Q2 lattices must be 2D boxes");
        PFFMG_REQUIRE((int64_t)(2 * in->nx + 1) * (2 * in->ny + 1) == in->n_vertices,
                      "Q2 box has %lld nodes, n_vertices=%lld",
                      (long long)(2 * in->nx + 1) * (2 * in->ny + 1), (long long)in->n_vertices);
        // slabs of a Q2 level start on a cell boundary: plane0 (a node row) is even
        PFFMG_REQUIRE(in->plane0 % 2 == 0, "Q2 slab must start on an even node row (plane0=%d)", in->plane0);
    }
    const bool has_rows = in->vrow_off != nullptr;
    PFFMG_REQUIRE(has_rows == (in->vrow_lo != nullptr) && has_rows == (in->vrow_hi != nullptr) &&
                      has_rows == (in->crow_lo != nullptr) && has_rows == (in->crow_hi != nullptr),
                  "row tables must be all NULL (box) or all set");
    if (!has_rows && order == 1) {
        const int64_t Vbox = (int64_t)(in->nx + 1) * (in->ny + 1) * (in->dim == 3 ? in->nz + 1 : 1);
        PFFMG_REQUIRE(Vbox == in->n_vertices, "box lattice has %lld vertices, n_vertices=%lld",
                      (long long)Vbox, (long long)in->n_vertices);
    }
    out->dim = in->dim;
    out->nx = in->nx;
    out->ny = in->ny;
    out->nz = in->nz;
    out->hx = in->hx;
    out->hy = in->hy;
    out->hz = in->hz;
    out->V = in->n_vertices;
    out->vrow_off = in->vrow_off;
    out->vrow_lo = in->vrow_lo;
    out->vrow_hi = in->vrow_hi;
    out->crow_lo = in->crow_lo;
    out->crow_hi = in->crow_hi;
    out->plane0 = in->plane0;
    PFFMG_REQUIRE(in->tiles3d == nullptr || in->n_tiles3d > 0, "tiles3d given with n_tiles3d = %d",
                  in->n_tiles3d);
    out->tiles3d = in->tiles3d;
    out->n_tiles3d = in->tiles3d ? in->n_tiles3d : 0;
    out->order = order;
    const int nplanes = order == 2 ? 2 * in->ny + 1 : (in->dim == 3 ? in->nz : in->ny) + 1;
    if (in->own_lo == 0 && in->own_hi == 0) {
        out->own_lo = 0;
        out->own_hi = nplanes;
    } else {
        PFFMG_REQUIRE(in->own_lo >= 0 && in->own_lo < in->own_hi && in->own_hi <= nplanes,
                      "bad owned plane range [%d, %d) of %d planes", in->own_lo, in->own_hi, nplanes);
        out->own_lo = in->own_lo;
        out->own_hi = in->own_hi;
    }
    return PFFMG_OK;
}

int make_consts(const pffmg_lattice* lat, const pffmg_state* st, Consts* K) {
    PFFMG_REQUIRE(st, "null state");
    PFFMG_REQUIRE(st->struct_size == (int32_t)sizeof(pffmg_state),
                  "pffmg_state.struct_size = %d, this library expects %d (ABI version %d)",
                  st->struct_size, (int)sizeof(pffmg_state), PFFMG_ABI_VERSION);
    PFFMG_REQUIRE(lat->hx > 0 && lat->hy > 0 && (lat->dim == 2 || lat->hz > 0), "cell sizes must be > 0");
    PFFMG_REQUIRE(st->eps > 0, "eps must be > 0");
    // fem.py:33-34
    K->g0 = 0.5 - 0.5 / std::sqrt(3.0);
    K->g1 = 0.5 + 0.5 / std::sqrt(3.0);
    K->omg0 = 1.0 - K->g0;
    K->omg1 = 1.0 - K->g1;
    K->ih[0] = 1.0 / lat->hx;
    K->ih[1] = 1.0 / lat->hy;
    K->ih[2] = lat->dim == 3 ? 1.0 / lat->hz : 0.0;
    // JxW = w_q * cell volume, w_q = 0.5^dim (fem.py:179)
    const double vol = lat->dim == 3 ? lat->hx * lat->hy * lat->hz : lat->hx * lat->hy;
    K->jxw = (lat->dim == 3 ? 0.125 : 0.25) * vol;
    K->mu = st->mu;
    K->lam = st->lam;
    K->kappa = st->kappa;
    K->omk = 1.0 - st->kappa;
    K->two_p = 2.0 * st->pressure;
    K->gc_over_eps = st->g_c / st->eps;
    K->k_phi = st->g_c * st->eps;
    K->band = st->split_band;
    K->eps = st->eps;
    PFFMG_ONE_DEVICE();                 // after the argument checks (they need no GPU)
    return PFFMG_OK;
}

}  // namespace pffmg

using namespace pffmg;

extern "C" const char* pffmg_last_error(void) { return g_err; }

extern "C" int pffmg_version(void) { return PFFMG_ABI_VERSION; }

extern "C" int pffmg_set_pdl(int on, int* previous) {
    const int prev = pdl_set(on);
    if (previous) *previous = prev;
    return PFFMG_OK;
}

extern "C" int pffmg_device_sm_count(int* out) {
    PFFMG_REQUIRE(out, "null out");
    *out = sm_count();
    return PFFMG_OK;
}
