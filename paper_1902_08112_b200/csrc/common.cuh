// Shared device-side helpers of libpffmg: lattice addressing, error state,
// and the 2-point tensor-product (sum-factorised) Q1 kernels.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include <utility>

#include "../../include/pffmg.h"

namespace pffmg {

// ------------------------------------------------------------------ errors

void set_error(const char* fmt, ...);
int check_launch(const char* what);

#define PFFMG_REQUIRE(cond, ...)                                  \
    do {                                                          \
        if (!(cond)) {                                            \
            ::pffmg::set_error(__VA_ARGS__);                      \
            return PFFMG_ERR_ARG;                                 \
        }                                                         \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// libpffmg serves ONE GPU per process (the launch-shape, occupancy and
// reduction-scratch caches are set up for the first device used): every
// entry point that touches device state checks the current device against
// that first one and fails loudly instead of mixing devices.
int check_device();
#define PFFMG_ONE_DEVICE()                          \
    do {                                            \
        const int rc_ = ::pffmg::check_device();    \
        if (rc_) return rc_;                        \
    } while (0)

// ----------------------------------------------------------------- lattice

// Kernel-side copy of pffmg_lattice (passed by value).
struct Lat {
    int dim, nx, ny, nz;
    double hx, hy, hz;
    int64_t V;
    const int64_t* __restrict__ vrow_off;
    const int32_t* __restrict__ vrow_lo;
    const int32_t* __restrict__ vrow_hi;
    const int32_t* __restrict__ crow_lo;
    const int32_t* __restrict__ crow_hi;
    int own_lo, own_hi;    // finalised vertex planes of the last axis (always set by make_lat)
    int plane0;            // global index of local plane 0 along the last axis
    int order;             // 1 = Q1, 2 = Q2 (2D box, nodes on the half-spacing lattice)
    const int32_t* __restrict__ tiles3d;   // occupied PFFMG_TILE3^2-column x-y tiles (NULL: all)
    int n_tiles3d;
};

int make_lat(const pffmg_lattice* in, Lat* out);

// Vertex id of lattice point (x, y, z) or -1 when absent (reference vertex
// numbering, mesh.py:163-194: x fastest, rows contiguous).
__device__ __forceinline__ int64_t vertex_id(const Lat& L, int x, int y, int z) {
    if (x < 0 || y < 0 || z < 0 || x > L.nx || y > L.ny || z > L.nz) return -1;
    if (L.vrow_off == nullptr)
        return (int64_t)x + (int64_t)(L.nx + 1) * ((int64_t)y + (int64_t)(L.ny + 1) * z);
    const int r = y + (L.ny + 1) * z;
    const int lo = __ldg(L.vrow_lo + r), hi = __ldg(L.vrow_hi + r);
    if (x < lo || x >= hi) return -1;
    return __ldg(L.vrow_off + r) + (x - lo);
}

template <int D>
__device__ __forceinline__ bool cell_exists(const Lat& L, int x, int y, int z) {
    if (x < 0 || y < 0 || x >= L.nx || y >= L.ny) return false;
    if (D == 3 && (z < 0 || z >= L.nz)) return false;
    if (L.crow_lo == nullptr) return true;
    const int s = y + L.ny * z;
    return x >= __ldg(L.crow_lo + s) && x < __ldg(L.crow_hi + s);
}

// ------------------------------------------------------- element constants

// Everything the cell kernels need besides the fields.  Built on the host
// with the same double expressions as the reference tables (fem.py:33-34,
// 174-179, model.py:270-309) so results agree to rounding.
struct Consts {
    double g0, g1;        // 2-pt Gauss points 0.5 -/+ 0.5/sqrt(3)
    double omg0, omg1;    // 1 - g
    double ih[3];         // 1 / cell_size
    double jxw;           // quadrature weight * cell volume (identical for all QPs)
    double mu, lam, kappa, omk, two_p, gc_over_eps, k_phi;
    double band;          // C^1 blend half-width of the spectral split (0 = hard)
    double eps;           // regularisation length (QoIs)
};

int make_consts(const pffmg_lattice* lat, const pffmg_state* st, Consts* K);

// ----------------------------------------------- sum factorisation (2-pt Q1)
//
// Arrays of 2^D doubles are indexed by bit patterns: bit a of the index is the
// corner offset (or quadrature-point index) along axis a, x fastest -- the
// corner order of mesh.py:36-39 and the QP order of fem.py:44-51.

template <int D>
struct SF {
    static constexpr int NP = 1 << D;

    // value (p = 0) and raw derivatives (p = 1 + a, not yet scaled by 1/h)
    // of one nodal field at the 2^D Gauss points (fem.py:229-238 einsums,
    // factorised along the axes).  CSE merges the shared passes.
    __device__ __forceinline__ static void interp(const double (&c)[NP], double (&out)[D + 1][NP],
                                                  const Consts& K, bool need_val = true) {
#pragma unroll
        for (int p = 0; p <= D; ++p)
#pragma unroll
            for (int i = 0; i < NP; ++i) out[p][i] = c[i];
#pragma unroll
        for (int a = 0; a < D; ++a) {
#pragma unroll
            for (int p = 0; p <= D; ++p) {
                if (p == 0 && !need_val) continue;
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    if (i & (1 << a)) continue;
                    const int j = i | (1 << a);
                    const double u0 = out[p][i], u1 = out[p][j];
                    const double d = u1 - u0;
                    if (p == a + 1) {
                        out[p][i] = d;
                        out[p][j] = d;
                    } else {
                        out[p][i] = fma(K.g0, d, u0);
                        out[p][j] = fma(K.g1, d, u0);
                    }
                }
            }
        }
    }

    // out[n] = sum_q f[q] N_q(n) + sum_{q,a} g[a][q] dN_q(n)/dref_a
    // (the transposed contraction of model.py:347-354).  f / g are consumed.
    template <bool HAS_F>
    __device__ __forceinline__ static void integrate(double (&f)[NP], double (&g)[D][NP],
                                                     const Consts& K) {
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                if (i & (1 << a)) continue;
                const int j = i | (1 << a);
                // S <- B_a^T S + D_a^T G_a
                const double s = g[a][i] + g[a][j];
                if (HAS_F || a != D - 1) {
                    const double f0 = f[i], f1 = f[j];
                    f[i] = fma(K.omg0, f0, fma(K.omg1, f1, -s));
                    f[j] = fma(K.g0, f0, fma(K.g1, f1, s));
                } else {
                    f[i] = -s;
                    f[j] = s;
                }
                // G_b <- B_a^T G_b for b < a
#pragma unroll
                for (int b = 0; b < a; ++b) {
                    const double q0 = g[b][i], q1 = g[b][j];
                    g[b][i] = fma(K.omg0, q0, K.omg1 * q1);
                    g[b][j] = fma(K.g0, q0, K.g1 * q1);
                }
            }
        }
    }
};

// cp.async (LDGSTS) helpers: asynchronous global -> shared copies, zero-filled
// when `valid` is false (src must still be a mapped address).
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    const int n = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(gsrc), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Leaner factorisations used by the isotropic kernels.  A derivative along j
// of a Q1 field is constant along j, so it is stored "reduced": an array of
// 2^(D-1) values indexed by the other axes' bits (compile-time helpers
// below).  Gradients take the pair difference first and interpolate the
// reduced array; transposed gradient terms sum the pairs first.
__host__ __device__ constexpr int drop_bit(int i, int j) {       // remove bit j
    return (i & ((1 << j) - 1)) | ((i >> (j + 1)) << j);
}
__host__ __device__ constexpr int put_bit(int r, int j, int b) {  // insert bit b at j
    return (r & ((1 << j) - 1)) | (b << j) | ((r >> j) << (j + 1));
}

template <int D>
struct SFr {
    static constexpr int NP = 1 << D, NR = 1 << (D - 1);

    // values at the QPs (B along every axis)
    __device__ __forceinline__ static void value(const double (&c)[NP], double (&v)[NP], const Consts& K) {
#pragma unroll
        for (int i = 0; i < NP; ++i) v[i] = c[i];
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                if (i & (1 << a)) continue;
                const int k = i | (1 << a);
                const double u0 = v[i], d = v[k] - u0;
                v[i] = fma(K.g0, d, u0);
                v[k] = fma(K.g1, d, u0);
            }
    }

    // raw derivative along j, reduced: g[r] = d_j^ref c at QPs with other bits r
    __device__ __forceinline__ static void deriv(const double (&c)[NP], int j, double (&g)[NR],
                                                 const Consts& K) {
#pragma unroll
        for (int r = 0; r < NR; ++r) g[r] = c[put_bit(r, j, 1)] - c[put_bit(r, j, 0)];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            if (a == j) continue;
            const int ab = a < j ? a : a - 1;     // bit position in the reduced index
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                if (r & (1 << ab)) continue;
                const int k = r | (1 << ab);
                const double u0 = g[r], d = g[k] - u0;
                g[r] = fma(K.g0, d, u0);
                g[k] = fma(K.g1, d, u0);
            }
        }
    }

    // out[n] (=|+=) sum_q G[q] dN_n/dref_j (q): pairs summed along j, then B^T on the others
    template <bool ACC>
    __device__ __forceinline__ static void deriv_T(const double (&G)[NP], int j, double (&out)[NP],
                                                   const Consts& K) {
        double r[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) r[i] = G[put_bit(i, j, 0)] + G[put_bit(i, j, 1)];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            if (a == j) continue;
            const int ab = a < j ? a : a - 1;
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                if (i & (1 << ab)) continue;
                const int k = i | (1 << ab);
                // B^T of a pair; the Gauss points are symmetric (omg0 = g1, omg1 = g0,
                // g0 + g1 = 1), so (g1 f0 + g0 f1, g0 f0 + g1 f1) = (f0 + g0 d, f1 - g0 d)
                const double f0 = r[i], f1 = r[k], d = f1 - f0;
                r[i] = fma(K.g0, d, f0);
                r[k] = fma(-K.g0, d, f1);
            }
        }
#pragma unroll
        for (int n = 0; n < NP; ++n) {
            const double t = r[drop_bit(n, j)];
            if (ACC)
                out[n] = ((n >> j) & 1) ? out[n] + t : out[n] - t;
            else
                out[n] = ((n >> j) & 1) ? t : -t;
        }
    }
};

// Programmatic dependent launch ---------------------------------------------
// Every libpffmg kernel is launched with the programmatic-stream-serialization
// attribute (pdl_launch) and begins with pdl_wait(): the next kernel of a
// chain (a V-cycle, a CG run) is scheduled while the previous one drains, and
// waits for its completion (and memory flush) before touching data.  The wait
// returns at once when there is no prerequisite grid.  PFFMG_PDL=0 disables it.
//
// PFFMG_PDL_EARLY (compile time): right after its own wait a kernel lets its
// dependents launch (griddepcontrol.launch_dependents); they park in their
// wait until this grid has completed and flushed, so a single-stream chain
// overlaps every launch with the previous kernel.  Parked dependents hold SM
// slots, which costs a multi-stream graph its concurrency: pffmg_set_pdl(0)
// switches the launch attribute off for such sections (the setup graph).
__device__ __forceinline__ void pdl_wait() {
#ifdef PFFMG_PDL_EARLY
    asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
#else
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Deterministic block reduction helpers --------------------------------------

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace pffmg
