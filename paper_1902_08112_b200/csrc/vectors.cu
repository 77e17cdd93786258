// Krylov BLAS-1 and deterministic reductions (reference krylov.py:50-198 and
// the vector updates of mgsolve.py:82-113).
//
// Every reduction runs on a grid whose size is a fixed function of n, sums
// each thread's grid-stride slice in order, reduces the block with a fixed
// shuffle/shared-memory tree, and lets the last block to finish add the block
// partials in index order -- so results are bitwise reproducible run to run
// (the reference guarantees thread-count independent results, README.md:92-97).
// Scalars that steer later kernels (GMRES H entries, CG alpha/beta, stop
// flags) stay in device memory so no host round trip is needed between steps.
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>
#include <mutex>
#include <unordered_map>

#include "cellops_miehe.cuh"

namespace pffmg {

constexpr int RT = 256;         // reduction block size
constexpr int RMAXB = 1024;     // max reduction blocks

struct Scratch {
    double partial[2 * RMAXB];
    unsigned int counter;
};

// One scratch block per stream: reductions on different streams (e.g. the
// concurrent per-level CG-Lanczos branches of the recorded setup graph) must
// not share the partials / last-block counter.
static int scratch(cudaStream_t stream, Scratch** out) {
    PFFMG_ONE_DEVICE();
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, Scratch*> table;
    std::lock_guard<std::mutex> lock(mu);
    auto it = table.find(stream);
    if (it != table.end()) {
        *out = it->second;
        return PFFMG_OK;
    }
    Scratch* S = nullptr;
    if (cudaMalloc(&S, sizeof(Scratch)) != cudaSuccess || cudaMemset(S, 0, sizeof(Scratch)) != cudaSuccess) {
        set_error("cannot allocate reduction scratch");
        return PFFMG_ERR_CUDA;
    }
    table[stream] = S;
    *out = S;
    return PFFMG_OK;
}

static int red_blocks(int64_t n) {
    int64_t b = (n + RT * 8 - 1) / (RT * 8);
    if (b < 1) b = 1;
    if (b > RMAXB) b = RMAXB;
    return (int)b;
}

__device__ __forceinline__ void block_sum2(double& a0, double& a1) {
    __shared__ double s0[RT / 32], s1[RT / 32];
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        s0[w] = a0;
        s1[w] = a1;
    }
    __syncthreads();
    if (w == 0) {
        a0 = lane < RT / 32 ? s0[lane] : 0.0;
        a1 = lane < RT / 32 ? s1[lane] : 0.0;
        a0 = warp_sum(a0);
        a1 = warp_sum(a1);
    }
}

// Generic fused "elementwise update + up to two sums + scalar finisher".
template <class Op>
__global__ void __launch_bounds__(RT) fused_kernel(Op op, int64_t n, Scratch* S) {
    pdl_wait();
    if (op.skip()) return;
    op.prepare();
    double a0 = 0.0, a1 = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)RT + threadIdx.x; i < n; i += (int64_t)gridDim.x * RT)
        op.elem(i, a0, a1);
    if (!Op::REDUCES) return;
    block_sum2(a0, a1);
    __shared__ bool last;
    if (threadIdx.x == 0) {
        S->partial[2 * blockIdx.x] = a0;
        S->partial[2 * blockIdx.x + 1] = a1;
        __threadfence();
        const unsigned t = atomicAdd(&S->counter, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {
        // the last block adds the block partials with a fixed tree: thread t
        // sums partials t, t+RT, t+2RT, ... in order, then the block tree
        __threadfence();
        double s0 = 0.0, s1 = 0.0;
        volatile double* p = S->partial;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += RT) {
            s0 += p[2 * b];
            s1 += p[2 * b + 1];
        }
        block_sum2(s0, s1);
        if (threadIdx.x == 0) {
            op.finish(s0, s1);
            S->counter = 0;
        }
    }
}

template <class Op>
static int run_fused(const Op& op, int64_t n, cudaStream_t s, const char* what) {
    Scratch* S;
    int rc = scratch(s, &S);
    if (rc) return rc;
    pdl_launch(fused_kernel<Op>, dim3(red_blocks(n)), dim3(RT), 0, s, op, n, S);
    return check_launch(what);
}

// ---------------------------------------------------------------- ops

struct DotOp {
    static constexpr bool REDUCES = true;
    const double* x;
    const double* y;
    const double* s;   // optional elementwise scale: sum x*y*s
    double* result;
    __device__ bool skip() const { return false; }
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double& a0, double&) const {
        a0 = s ? fma(x[i], y[i] * s[i], a0) : fma(x[i], y[i], a0);
    }
    __device__ void finish(double s0, double) const { *result = s0; }
};

// One modified Gram-Schmidt pass (krylov.py:97-107):
//   w -= (*hprev) * Vprev   (if Vprev)
//   s0 = Vcur . w           (if Vcur)
//   s1 = w . w              (if NRM)
struct MgsOp {
    static constexpr bool REDUCES = true;
    const double* Vprev;
    const double* hprev;
    const double* Vcur;
    double* w;
    double* ctl;       // [0] w0n2, [1] wn2, [2] reorth flag, [3..] corrections
    double* hcol;      // H[:, j] (device)
    int i;             // index of Vcur
    int kind;          // 0: first pass, 1: middle, 2: last (norm), 3..5: re-orth variants
    int gate;          // 1: only run when ctl[2] != 0
    double hp;
    __device__ bool skip() const { return gate && ctl[2] == 0.0; }
    __device__ void prepare() { hp = Vprev ? *hprev : 0.0; }
    __device__ void elem(int64_t k, double& a0, double& a1) const {
        double wk = w[k];
        if (Vprev) {
            wk = fma(-hp, Vprev[k], wk);
            w[k] = wk;
        }
        if (Vcur) a0 = fma(Vcur[k], wk, a0);
        if (kind == 0 || kind == 2 || kind == 5) a1 = fma(wk, wk, a1);
    }
    __device__ void finish(double s0, double s1) const {
        switch (kind) {
            case 0: hcol[i] = s0; ctl[0] = s1; break;                 // first pass: H[0,j], ||w0||^2
            case 1: hcol[i] = s0; break;                              // H[i,j]
            case 2: {                                                 // after the last update
                ctl[1] = s1;
                const double wn = sqrt(s1), w0 = sqrt(ctl[0]);
                ctl[2] = (wn < 1e-3 * w0) ? 1.0 : 0.0;                // krylov.py:101
                hcol[i] = wn;                                         // H[j+1, j] (krylov.py:107)
                break;
            }
            case 3: ctl[3 + i] = s0; hcol[i] += s0; break;            // re-orth first
            case 4: ctl[3 + i] = s0; hcol[i] += s0; break;            // re-orth middle
            case 5: ctl[1] = s1; hcol[i] = sqrt(s1); break;           // re-orth final norm
        }
    }
};

struct ScaleByInvOp {      // V_{j+1} = w / h  when h != 0 (krylov.py:108-110)
    static constexpr bool REDUCES = false;
    double* w;
    const double* h;
    double hv;
    __device__ bool skip() const { return *h == 0.0; }
    __device__ void prepare() { hv = *h; }
    __device__ void elem(int64_t k, double&, double&) const { w[k] = w[k] / hv; }
    __device__ void finish(double, double) const {}
};

// ------------------------------------------------ CG-Lanczos (krylov.py:146-185)
// scal layout
enum { C_RZ = 0, C_STOP = 1, C_ALPHA = 2, C_BETA = 3, C_K = 4, C_NB = 5, C_PAP = 6, C_RZN = 7, C_HIST = 8 };
constexpr int CG_MAXIT = 64;

struct CgStartOp {
    static constexpr bool REDUCES = true;
    const double *b, *diag;
    double *r, *z, *p, *scal;
    __device__ bool skip() const { return false; }
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double& a0, double&) const {
        const double ri = b[i];
        const double zi = ri / diag[i];
        r[i] = ri;
        z[i] = zi;
        p[i] = zi;
        a0 = fma(ri, zi, a0);
    }
    __device__ void finish(double s0, double) const {
        scal[C_RZ] = s0;
        scal[C_STOP] = (s0 > 0.0 && isfinite(s0)) ? 0.0 : 1.0;
        scal[C_K] = 0.0;
        scal[C_NB] = 0.0;
    }
};

struct CgPApOp {
    static constexpr bool REDUCES = true;
    const double *p, *Ap;
    double* scal;
    __device__ bool skip() const { return scal[C_STOP] != 0.0; }
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double& a0, double&) const { a0 = fma(p[i], Ap[i], a0); }
    __device__ void finish(double s0, double) const {
        scal[C_PAP] = s0;
        if (!(s0 > 0.0 && isfinite(s0))) {
            scal[C_STOP] = 1.0;
            return;
        }
        const double alpha = scal[C_RZ] / s0;
        const int k = (int)scal[C_K];
        scal[C_ALPHA] = alpha;
        if (k < CG_MAXIT) scal[C_HIST + k] = alpha;
        scal[C_K] = k + 1;
    }
};

struct CgUpdateOp {
    static constexpr bool REDUCES = true;
    const double *Ap, *diag;
    double *r, *z, *scal;
    double alpha;
    __device__ bool skip() const { return scal[C_STOP] != 0.0; }
    __device__ void prepare() { alpha = scal[C_ALPHA]; }
    __device__ void elem(int64_t i, double& a0, double&) const {
        const double ri = r[i] - alpha * Ap[i];
        const double zi = ri / diag[i];
        r[i] = ri;
        z[i] = zi;
        a0 = fma(ri, zi, a0);
    }
    __device__ void finish(double s0, double) const {
        const double rz = scal[C_RZ];
        if (s0 <= 1e-28 * rz || !isfinite(s0)) {
            scal[C_STOP] = 1.0;
            return;
        }
        const double beta = s0 / rz;
        const int nb = (int)scal[C_NB];
        scal[C_BETA] = beta;
        if (nb < CG_MAXIT) scal[C_HIST + CG_MAXIT + nb] = beta;
        scal[C_NB] = nb + 1;
        scal[C_RZ] = s0;
    }
};

struct CgPOp {
    static constexpr bool REDUCES = false;
    const double* z;
    double *p, *scal;
    double beta;
    __device__ bool skip() const { return scal[C_STOP] != 0.0; }
    __device__ void prepare() { beta = scal[C_BETA]; }
    __device__ void elem(int64_t i, double&, double&) const { p[i] = z[i] + beta * p[i]; }
    __device__ void finish(double, double) const {}
};

// -------------------------------------------------------- plain vector kernels

#define GRID_STRIDE(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

static dim3 vgrid(int64_t n) {
    int64_t b = (n + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 32;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return dim3((unsigned)b);
}

__global__ void pack_flags_k(const uint8_t* m, int nc, int64_t V, uint8_t* f) {
    pdl_wait();
    GRID_STRIDE(v, V) {
        uint8_t b = 0;
        for (int c = 0; c < nc; ++c) b |= (uint8_t)((m[(int64_t)c * V + v] != 0) << c);
        f[v] = b;
    }
}
__global__ void unpack_flags_k(const uint8_t* f, int nc, int64_t V, uint8_t* m) {
    pdl_wait();
    GRID_STRIDE(v, V) {
        const uint8_t b = f[v];
        for (int c = 0; c < nc; ++c) m[(int64_t)c * V + v] = (b >> c) & 1;
    }
}
__global__ void masked_copy_k(const uint8_t* f, int64_t V, int comp0, int nc, const double* in, double* out) {
    pdl_wait();
    GRID_STRIDE(i, V * nc) {
        const int c = (int)(i / V);
        const int64_t v = i - (int64_t)c * V;
        out[i] = ((f[v] >> (comp0 + c)) & 1) ? 0.0 : in[i];
    }
}
// V-cycle entry (mgsolve.py:271-272 then 95, 103-106): the masked right-hand
// side and the fine level's block-diagonal Chebyshev start from x = 0 in one
// pass (the arithmetic of masked_copy_k then cheb_init_zero_bd_k).
__global__ void masked_copy_init_bd_k(const uint8_t* f, int64_t V, int nc, const double* in, double* rhs,
                                      const double* inv, const double* tu, const double* tp, double* r,
                                      double* d, double* x) {
    pdl_wait();
    const double thu = *tu, thp = *tp;
    GRID_STRIDE(i, V * nc) {
        const int c = (int)(i / V);
        const int64_t v = i - (int64_t)c * V;
        const double ri = ((f[v] >> c) & 1) ? 0.0 : in[i];
        const double di = (inv[i] * ri) / (c < nc - 1 ? thu : thp);
        rhs[i] = ri;
        d[i] = di;
        if (r) {                                   // (NULL: the first step is pffmg_cheb_first_*)
            r[i] = ri;
            x[i] = 0.0 + di;
        }
    }
}
__global__ void reciprocal_k(const double* d, double* o, int64_t n) {
    pdl_wait();
    GRID_STRIDE(i, n) o[i] = 1.0 / d[i];
}
__global__ void cheb_init_zero_k(const double* b, const double* inv, double theta_v, const double* theta_p,
                                 double* r, double* d, double* x, int64_t n) {
    pdl_wait();
    const double theta = theta_p ? *theta_p : theta_v;
    GRID_STRIDE(i, n) {
        const double ri = b[i];
        const double di = (inv[i] * ri) / theta;   // mgsolve.py:105
        d[i] = di;
        if (r) {
            r[i] = ri;
            x[i] = 0.0 + di;                       // x = zeros; x += d
        }
    }
}
__global__ void jacobi_update_k(const double* r, const double* inv, double theta_v, const double* theta_p,
                                double* x, int64_t n) {
    pdl_wait();
    const double theta = theta_p ? *theta_p : theta_v;
    GRID_STRIDE(i, n) x[i] += (inv[i] * r[i]) / theta;   // mgsolve.py:99
}
__global__ void axpby_k(double a, const double* x, double b, double* y, int64_t n, int mode) {
    pdl_wait();
    GRID_STRIDE(i, n) {
        if (mode == 0) y[i] = fma(a, x[i], y[i]);
        else if (mode == 1) y[i] = a * x[i] + b * y[i];
        else if (mode == 2) y[i] = a * y[i];
        else y[i] = x[i];
    }
}
__global__ void sub_k(const double* x, const double* y, double* o, int64_t n) {
    pdl_wait();
    GRID_STRIDE(i, n) o[i] = x[i] - y[i];
}
// Primal-dual active set of the phase field (nonlinear.py:75-89):
//   active_phi[v] = (minv[v] * R[v] + c * (U[v] - phi_old[v])) > 0  and not Dirichlet.
// Explicit _rn intrinsics keep the reference's rounding (no FMA contraction),
// so the set is bit-exact for identical inputs.
__global__ void active_set_k(const double* R, const double* U, const double* phi_old, const double* minv,
                             double c, const uint8_t* dflags, int comp, int64_t V, uint8_t* active) {
    pdl_wait();
    GRID_STRIDE(v, V) {
        const double ind = __dadd_rn(__dmul_rn(minv[v], R[v]), __dmul_rn(c, __dsub_rn(U[v], phi_old[v])));
        bool a = ind > 0.0;
        if (dflags && ((dflags[v] >> comp) & 1)) a = false;
        active[v] = a ? 1 : 0;
    }
}

// x += sum_k y[k] * Z_k   (krylov.py:132: x + Z[:j].T @ y)
__global__ void multi_axpy_k(const double* Z, int64_t ld, int k, const double* y, double* x, int64_t n) {
    pdl_wait();
    __shared__ double ys[64];
    if (threadIdx.x < k) ys[threadIdx.x] = y[threadIdx.x];
    __syncthreads();
    GRID_STRIDE(i, n) {
        double s = 0.0;
        for (int t = 0; t < k; ++t) s = fma(ys[t], Z[(int64_t)t * ld + i], s);
        x[i] += s;
    }
}

}  // namespace pffmg

using namespace pffmg;

#define VCHECK(what) return check_launch(what)

extern "C" int pffmg_pack_flags(const uint8_t* mask, int n_comp, int64_t V, uint8_t* flags, void* stream) {
    PFFMG_REQUIRE(mask && flags && n_comp >= 1 && n_comp <= 8 && V >= 0, "pffmg_pack_flags: bad args");
    pdl_launch(pack_flags_k, dim3(vgrid(V)), dim3(256), 0, as_stream(stream), mask, n_comp, V, flags);
    VCHECK("pffmg_pack_flags");
}
extern "C" int pffmg_unpack_flags(const uint8_t* flags, int n_comp, int64_t V, uint8_t* mask, void* stream) {
    PFFMG_REQUIRE(mask && flags && n_comp >= 1 && n_comp <= 8 && V >= 0, "pffmg_unpack_flags: bad args");
    pdl_launch(unpack_flags_k, dim3(vgrid(V)), dim3(256), 0, as_stream(stream), flags, n_comp, V, mask);
    VCHECK("pffmg_unpack_flags");
}
extern "C" int pffmg_masked_copy(const uint8_t* flags, int64_t V, int comp0, int n_comp, const double* in,
                                 double* out, void* stream) {
    PFFMG_REQUIRE(flags && in && out && n_comp >= 1 && comp0 >= 0, "pffmg_masked_copy: bad args");
    pdl_launch(masked_copy_k, dim3(vgrid(V * n_comp)), dim3(256), 0, as_stream(stream), flags, V, comp0, n_comp, in, out);
    VCHECK("pffmg_masked_copy");
}
extern "C" int pffmg_masked_copy_init_bd(const uint8_t* flags, int64_t V, int n_comp, const double* in,
                                         double* rhs, const double* invdiag, const double* theta_u,
                                         const double* theta_p, double* r, double* d, double* x, void* stream) {
    PFFMG_REQUIRE(flags && in && rhs && invdiag && theta_u && theta_p && d && !r == !x && V >= 0 && n_comp >= 2 &&
                      n_comp <= 4,
                  "pffmg_masked_copy_init_bd: bad args");
    pdl_launch(masked_copy_init_bd_k, dim3(vgrid(V * n_comp)), dim3(256), 0, as_stream(stream), flags, V, n_comp, in,
               rhs, invdiag, theta_u, theta_p, r, d, x);
    VCHECK("pffmg_masked_copy_init_bd");
}
extern "C" int pffmg_reciprocal(const double* diag, double* out, int64_t n, void* stream) {
    PFFMG_REQUIRE(diag && out, "pffmg_reciprocal: bad args");
    pdl_launch(reciprocal_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), diag, out, n);
    VCHECK("pffmg_reciprocal");
}
extern "C" int pffmg_cheb_init_zero(const double* b, const double* invdiag, double theta, double* r,
                                    double* d, double* x, int64_t n, void* stream) {
    PFFMG_REQUIRE(b && invdiag && r && d && x, "pffmg_cheb_init_zero: bad args");
    pdl_launch(cheb_init_zero_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), b, invdiag, theta, nullptr, r, d, x, n);
    VCHECK("pffmg_cheb_init_zero");
}
extern "C" int pffmg_cheb_init_zero_dc(const double* b, const double* invdiag, const double* theta, double* r,
                                       double* d, double* x, int64_t n, void* stream) {
    PFFMG_REQUIRE(b && invdiag && theta && d && !r == !x, "pffmg_cheb_init_zero_dc: bad args");
    pdl_launch(cheb_init_zero_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), b, invdiag, 0.0, theta, r, d, x, n);
    VCHECK("pffmg_cheb_init_zero_dc");
}
__global__ void cheb_init_zero_bd_k(const double* b, const double* inv, const double* tu, const double* tp,
                                    int64_t n_u, double* r, double* d, double* x, int64_t n) {
    pdl_wait();
    const double thu = *tu, thp = *tp;
    GRID_STRIDE(i, n) {
        const double ri = b[i];
        const double di = (inv[i] * ri) / (i < n_u ? thu : thp);
        d[i] = di;
        if (r) {
            r[i] = ri;
            x[i] = 0.0 + di;
        }
    }
}
extern "C" int pffmg_cheb_init_zero_bd(const double* b, const double* invdiag, const double* theta_u,
                                       const double* theta_p, int64_t n_u, double* r, double* d, double* x,
                                       int64_t n, void* stream) {
    PFFMG_REQUIRE(b && invdiag && theta_u && theta_p && d && !r == !x && n_u >= 0 && n_u <= n,
                  "pffmg_cheb_init_zero_bd: bad args");
    pdl_launch(cheb_init_zero_bd_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), b, invdiag, theta_u, theta_p, n_u, r, d, x, n);
    VCHECK("pffmg_cheb_init_zero_bd");
}
extern "C" int pffmg_jacobi_update(const double* r, const double* invdiag, double theta, double* x,
                                   int64_t n, void* stream) {
    PFFMG_REQUIRE(r && invdiag && x, "pffmg_jacobi_update: bad args");
    pdl_launch(jacobi_update_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), r, invdiag, theta, nullptr, x, n);
    VCHECK("pffmg_jacobi_update");
}
extern "C" int pffmg_jacobi_update_dc(const double* r, const double* invdiag, const double* theta, double* x,
                                      int64_t n, void* stream) {
    PFFMG_REQUIRE(r && invdiag && theta && x, "pffmg_jacobi_update_dc: bad args");
    pdl_launch(jacobi_update_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), r, invdiag, 0.0, theta, x, n);
    VCHECK("pffmg_jacobi_update_dc");
}
extern "C" int pffmg_axpy(double a, const double* x, double* y, int64_t n, void* stream) {
    PFFMG_REQUIRE(x && y, "pffmg_axpy: bad args");
    pdl_launch(axpby_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), a, x, 1.0, y, n, 0);
    VCHECK("pffmg_axpy");
}
extern "C" int pffmg_axpby(double a, const double* x, double b, double* y, int64_t n, void* stream) {
    PFFMG_REQUIRE(x && y, "pffmg_axpby: bad args");
    pdl_launch(axpby_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), a, x, b, y, n, 1);
    VCHECK("pffmg_axpby");
}
extern "C" int pffmg_scale(double a, double* x, int64_t n, void* stream) {
    PFFMG_REQUIRE(x, "pffmg_scale: bad args");
    pdl_launch(axpby_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), a, x, 0.0, x, n, 2);
    VCHECK("pffmg_scale");
}
extern "C" int pffmg_copy(const double* x, double* y, int64_t n, void* stream) {
    PFFMG_REQUIRE(x && y, "pffmg_copy: bad args");
    pdl_launch(axpby_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), 0.0, x, 0.0, y, n, 3);
    VCHECK("pffmg_copy");
}
extern "C" int pffmg_sub(const double* x, const double* y, double* out, int64_t n, void* stream) {
    PFFMG_REQUIRE(x && y && out, "pffmg_sub: bad args");
    pdl_launch(sub_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), x, y, out, n);
    VCHECK("pffmg_sub");
}
// ------------------------------------------------------------ QoIs
// Cell integrals of reference model.py:472-506 (crack_energy, bulk_energy,
// fracture_volume): one thread per lattice cell, 2^D Gauss points, the same
// deterministic block/last-block reduction as the dots.

// value and physical gradient of a Q1 field at QP q
template <int D>
__device__ __forceinline__ void q1_eval(const double (&c)[1 << D], int q, const Consts& K, double& val,
                                        double (&g)[D]) {
    val = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) g[a] = 0.0;
#pragma unroll
    for (int n = 0; n < (1 << D); ++n) {
        double B[D];
#pragma unroll
        for (int a = 0; a < D; ++a) B[a] = q1_shape(K, n, q, a);
        double N = 1.0;
#pragma unroll
        for (int a = 0; a < D; ++a) N *= B[a];
        val = fma(N, c[n], val);
#pragma unroll
        for (int a = 0; a < D; ++a) {
            double t = ((n >> a) & 1) ? K.ih[a] : -K.ih[a];
#pragma unroll
            for (int b = 0; b < D; ++b)
                if (b != a) t *= B[b];
            g[a] = fma(t, c[n], g[a]);
        }
    }
}

template <int D>
struct QoiOp {
    static constexpr bool REDUCES = true;
    Lat L;
    Consts K;
    const double* U;
    const double* rho;
    int kind;      // 0 crack energy, 1 bulk energy, 2 fracture volume
    int split;
    double scale;
    double* result;
    __device__ bool skip() const { return false; }
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double& a0, double&) const {
        constexpr int NP = 1 << D;
        const int cx = (int)(i % L.nx);
        const int64_t t = i / L.nx;
        const int cy = D == 3 ? (int)(t % L.ny) : (int)t;
        const int cz = D == 3 ? (int)(t / L.ny) : 0;
        if (!cell_exists<D>(L, cx, cy, cz)) return;
        double c[D + 1][NP];
#pragma unroll
        for (int n = 0; n < NP; ++n) {
            const int64_t vid = vertex_id(L, cx + (n & 1), cy + ((n >> 1) & 1), D == 3 ? cz + ((n >> 2) & 1) : 0);
#pragma unroll
            for (int k = 0; k <= D; ++k) c[k][n] = U[(int64_t)k * L.V + vid];
        }
        double sum = 0.0;
        for (int q = 0; q < NP; ++q) {
            double phi, gphi[D];
            q1_eval<D>(c[D], q, K, phi, gphi);
            double dens;
            if (kind == 2) {                                    // model.py:500-504
                dens = 1.0 - phi;
            } else if (kind == 0) {                             // model.py:472-480
                double gg = 0.0;
#pragma unroll
                for (int a = 0; a < D; ++a) gg = fma(gphi[a], gphi[a], gg);
                dens = (1.0 - phi) * (1.0 - phi) / K.eps + K.eps * gg;
            } else {                                            // model.py:483-497
                double gu[D][D], v;
#pragma unroll
                for (int k = 0; k < D; ++k) q1_eval<D>(c[k], q, K, v, gu[k]);
                double div = 0.0;
#pragma unroll
                for (int a = 0; a < D; ++a) div += gu[a][a];
                double Ep, Em;
                if (split == 0) {
                    double ee = 0.0;
#pragma unroll
                    for (int a = 0; a < D; ++a)
#pragma unroll
                        for (int b = 0; b < D; ++b) {
                            const double e = 0.5 * (gu[a][b] + gu[b][a]);
                            ee = fma(e, e, ee);
                        }
                    Ep = 0.5 * K.lam * div * div + K.mu * ee;
                    Em = 0.0;
                } else if (D == 2) {
                    Spec2 S;
                    spectral2(gu[0][0], 0.5 * (gu[0][1] + gu[1][0]), gu[D - 1][D - 1], K, S);
                    Ep = S.Ep;
                    Em = S.Em;
                } else {
                    const double e6[6] = {gu[0][0], gu[1 % D][1 % D], gu[D - 1][D - 1],
                                          0.5 * (gu[0][1 % D] + gu[1 % D][0]),
                                          0.5 * (gu[0][D - 1] + gu[D - 1][0]),
                                          0.5 * (gu[1 % D][D - 1] + gu[D - 1][1 % D])};
                    Spec3 S;
                    spectral3(e6, K, S);
                    const double Es = 0.5 * K.lam * S.tr * S.tr +
                                      K.mu * (S.w[0] * S.w[0] + S.w[1] * S.w[1] + S.w[2] * S.w[2]);
                    Ep = S.Ep;
                    Em = Es - S.Ep;
                }
                const double r = rho ? rho[i * NP + q] : 1.0;
                const double g = K.omk * (phi * phi) + K.kappa;
                dens = g * r * Ep + r * Em + phi * phi * (0.5 * K.two_p) * div;
            }
            sum = fma(K.jxw, dens, sum);
        }
        a0 += sum;
    }
    __device__ void finish(double s0, double) const { *result = scale * s0; }
};

// Boundary load (reference model.py:511-547): traction component `dir` of the
// transmitted stress g(phi) rho sigma+ + rho sigma- integrated over a list of
// boundary faces (lattice cell, face f = 2 axis + side) with the 2^(D-1)-point
// Gauss rule on each face (fem.py:265-292); one thread per face, the dots'
// deterministic reduction.
template <int D>
struct BoundaryLoadOp {
    static constexpr bool REDUCES = true;
    Lat L;
    Consts K;
    const double* U;
    const double* rho;      // NULL or (n_faces, 2^(D-1)) modulus at the face points
    const int64_t* fcell;   // lattice cell index cx + nx (cy + ny cz)
    const int32_t* fface;   // 2 axis + side
    int dir;
    int split;
    double vol;             // cell volume (LevelMesh.cell_volume)
    double* result;
    __device__ bool skip() const { return false; }
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double& a0, double&) const {
        constexpr int NP = 1 << D, NQ = 1 << (D - 1);
        const int64_t c = fcell[i];
        const int f = fface[i];
        const int axis = f >> 1, side = f & 1;
        const int cx = (int)(c % L.nx);
        const int64_t t = c / L.nx;
        const int cy = D == 3 ? (int)(t % L.ny) : (int)t;
        const int cz = D == 3 ? (int)(t / L.ny) : 0;
        double cv[D + 1][NP];
#pragma unroll
        for (int n = 0; n < NP; ++n) {
            const int64_t vid = vertex_id(L, cx + (n & 1), cy + ((n >> 1) & 1), D == 3 ? cz + ((n >> 2) & 1) : 0);
#pragma unroll
            for (int k = 0; k <= D; ++k) cv[k][n] = U[(int64_t)k * L.V + vid];
        }
        const double h[3] = {L.hx, L.hy, L.hz};
        const double wq = (D == 2 ? 0.5 : 0.25) * (vol / h[axis]);     // w * area (fem.py:286-290)
        const double sign = side == 1 ? 1.0 : -1.0;
        int other[2] = {0, 0};
        for (int a = 0, o = 0; a < D; ++a)
            if (a != axis) other[o++] = a;
        double sum = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double x[3] = {0.0, 0.0, 0.0};
            x[axis] = (double)side;
            x[other[0]] = (D == 3 ? (q >> 1) : q) ? K.g1 : K.g0;       // meshgrid(pts, pts, "ij").ravel()
            if (D == 3) x[other[1]] = (q & 1) ? K.g1 : K.g0;
            double gu[D][D], phi = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
                for (int b = 0; b < D; ++b) gu[a][b] = 0.0;
#pragma unroll
            for (int n = 0; n < NP; ++n) {
                double B[D];
#pragma unroll
                for (int a = 0; a < D; ++a) B[a] = ((n >> a) & 1) ? x[a] : 1.0 - x[a];
                double N = 1.0;
#pragma unroll
                for (int a = 0; a < D; ++a) N *= B[a];
                phi = fma(N, cv[D][n], phi);
#pragma unroll
                for (int b = 0; b < D; ++b) {
                    double g = ((n >> b) & 1) ? 1.0 : -1.0;
#pragma unroll
                    for (int a = 0; a < D; ++a)
                        if (a != b) g *= B[a];
                    g /= h[b];
#pragma unroll
                    for (int k = 0; k < D; ++k) gu[k][b] = fma(cv[k][n], g, gu[k][b]);
                }
            }
            double sp, sm;   // sigma+[dir][axis], sigma-[dir][axis]
            if (split == 0) {
                double tr = 0.0;
#pragma unroll
                for (int a = 0; a < D; ++a) tr += gu[a][a];
                const double e = 0.5 * (gu[dir][axis] + gu[axis][dir]);
                sp = 2.0 * K.mu * e + (dir == axis ? K.lam * tr : 0.0);
                sm = 0.0;
            } else if (D == 2) {
                Spec2 S;
                spectral2(gu[0][0], 0.5 * (gu[0][1] + gu[1][0]), gu[D - 1][D - 1], K, S);
                sp = S.sp[dir][axis];
                sm = S.sm[dir][axis];
            } else {
                const double e6[6] = {gu[0][0], gu[1 % D][1 % D], gu[D - 1][D - 1],
                                      0.5 * (gu[0][1 % D] + gu[1 % D][0]),
                                      0.5 * (gu[0][D - 1] + gu[D - 1][0]),
                                      0.5 * (gu[1 % D][D - 1] + gu[D - 1][1 % D])};
                Spec3 S;
                spectral3(e6, K, S);
                const int lo = dir < axis ? dir : axis, hi = dir < axis ? axis : dir;
                const int m = lo == hi ? lo : (lo == 0 ? (hi == 1 ? 3 : 4) : 5);   // (00,11,22,01,02,12)
                sp = S.sp[m];
                sm = S.sm[m];
            }
            const double r = rho ? rho[i * NQ + q] : 1.0;
            const double g = K.omk * (phi * phi) + K.kappa;
            sum = fma(wq, sign * (g * r * sp + r * sm), sum);
        }
        a0 += sum;
    }
    __device__ void finish(double s0, double) const { *result = s0; }
};

extern "C" int pffmg_boundary_load(const pffmg_lattice* lat, const pffmg_state* st, const int64_t* face_cell,
                                   const int32_t* face_id, int64_t n_faces, int direction, const double* rho_face,
                                   double* result, void* stream) {
    PFFMG_REQUIRE(lat && st && st->U && result && n_faces >= 0 && (n_faces == 0 || (face_cell && face_id)),
                  "pffmg_boundary_load: bad args");
    PFFMG_REQUIRE(st->split == 0 || st->split == 1, "pffmg_boundary_load: unknown split %d", st->split);
    Lat L;
    Consts K;
    int rc = make_lat(lat, &L);
    if (rc) return rc;
    rc = make_consts(lat, st, &K);
    if (rc) return rc;
    PFFMG_REQUIRE(L.order == 1, "pffmg_boundary_load: Q1 lattices only (reference model.py:511-547)");
    PFFMG_REQUIRE(direction >= 0 && direction < L.dim, "pffmg_boundary_load: direction %d", direction);
    const double vol = L.dim == 3 ? L.hx * L.hy * L.hz : L.hx * L.hy;
    const cudaStream_t s = as_stream(stream);
    if (L.dim == 2)
        return run_fused(BoundaryLoadOp<2>{L, K, st->U, rho_face, face_cell, face_id, direction, st->split, vol,
                                           result},
                         n_faces, s, "pffmg_boundary_load");
    return run_fused(BoundaryLoadOp<3>{L, K, st->U, rho_face, face_cell, face_id, direction, st->split, vol, result},
                     n_faces, s, "pffmg_boundary_load");
}

extern "C" int pffmg_qoi(const pffmg_lattice* lat, const pffmg_state* st, int kind, double* result,
                         void* stream) {
    PFFMG_REQUIRE(lat && st && st->U && result && kind >= 0 && kind <= 2, "pffmg_qoi: bad args");
    PFFMG_REQUIRE(st->split == 0 || st->split == 1, "pffmg_qoi: unknown split %d", st->split);
    Lat L;
    Consts K;
    int rc = make_lat(lat, &L);
    if (rc) return rc;
    rc = make_consts(lat, st, &K);
    if (rc) return rc;
    const int64_t ncell = (int64_t)L.nx * L.ny * (L.dim == 3 ? L.nz : 1);
    const double scale = kind == 0 ? 0.5 * st->g_c : 1.0;
    const cudaStream_t s = as_stream(stream);
    if (L.dim == 2)
        return run_fused(QoiOp<2>{L, K, st->U, st->rho, kind, st->split, scale, result}, ncell, s, "pffmg_qoi");
    return run_fused(QoiOp<3>{L, K, st->U, st->rho, kind, st->split, scale, result}, ncell, s, "pffmg_qoi");
}

extern "C" int pffmg_dot(const double* x, const double* y, int64_t n, double* result, void* stream) {
    PFFMG_REQUIRE(x && y && result && n >= 0, "pffmg_dot: bad args");
    return run_fused(DotOp{x, y, nullptr, result}, n, as_stream(stream), "pffmg_dot");
}
extern "C" int pffmg_dot_scaled(const double* x, const double* y, const double* s, int64_t n, double* result,
                                void* stream) {
    PFFMG_REQUIRE(x && y && s && result && n >= 0, "pffmg_dot_scaled: bad args");
    return run_fused(DotOp{x, y, s, result}, n, as_stream(stream), "pffmg_dot_scaled");
}

// ------------------------------------------------- one-launch Arnoldi step
// The whole MGS step of krylov.py:97-110 (sweep, norm, conditional second
// sweep, V_{j+1} = w / h) as ONE cooperative launch: CTA b keeps its slice of
// w in shared memory for the whole step, so w crosses HBM twice (load, final
// store) instead of four vector passes per basis vector; every inner product
// is a deterministic two-level sum (fixed per-CTA tree, then every CTA adds the
// CTA partials in index order after one grid barrier).  Same arithmetic order
// per element as the multi-launch path: w -= h_{i-1} V_{i-1} fused with the
// dot against V_i.
constexpr int MGS_T = 1024;
constexpr int MGS_MAXJ = 64;   // largest Arnoldi index of the one-launch form (larger j: multi-launch path)

__device__ __forceinline__ double mgs_block_sum(double a, double* red) {
    a = warp_sum(a);
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    if (lane == 0) red[wi] = a;
    __syncthreads();
    if (wi == 0) {
        a = lane < MGS_T / 32 ? red[lane] : 0.0;
        a = warp_sum(a);
    }
    return a;   // valid in warp 0
}

struct MgsSums {   // grid-wide fixed-order sums of up to two per-CTA partials
    double* part;  // [2 buffers][2 sums][gridDim.x]
    int phase;
    __device__ void post(double a0, double a1, double* red) {
        const double s0 = mgs_block_sum(a0, red);
        __syncthreads();
        const double s1 = mgs_block_sum(a1, red);
        double* p = part + (phase & 1) * 2 * gridDim.x;
        if (threadIdx.x == 0) {
            p[blockIdx.x] = s0;
            p[gridDim.x + blockIdx.x] = s1;
        }
    }
    // after the grid barrier: the same totals in every CTA
    __device__ void fetch(double& t0, double& t1, double* red) {
        const double* p = part + (phase & 1) * 2 * gridDim.x;
        if (threadIdx.x < 32) {
            double a = 0.0, b = 0.0;
            for (unsigned k = threadIdx.x; k < gridDim.x; k += 32) {
                a += __ldcg(p + k);
                b += __ldcg(p + gridDim.x + k);
            }
            a = warp_sum(a);
            b = warp_sum(b);
            if (threadIdx.x == 0) {
                red[32] = a;
                red[33] = b;
            }
        }
        __syncthreads();
        t0 = red[32];
        t1 = red[33];
        __syncthreads();
        ++phase;
    }
};

__global__ void __launch_bounds__(MGS_T, 1) mgs_coop_kernel(const double* __restrict__ Vb, int64_t ld, int j,
                                                            double* w, int64_t n, int64_t chunk, double* h,
                                                            double* ctl, double* part) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double sw[];
    __shared__ double red[40];
    const int64_t c0 = (int64_t)blockIdx.x * chunk;
    const int64_t c1 = c0 + chunk < n ? c0 + chunk : n;
    const int m = c1 > c0 ? (int)(c1 - c0) : 0;
    for (int k = threadIdx.x; k < m; k += MGS_T) sw[k] = w[c0 + k];
    __syncthreads();
    MgsSums S{part, 0};
    auto V = [&](int i) { return Vb + (int64_t)i * ld + c0; };
    double hv[MGS_MAXJ + 2];   // H[0..j+1, j] (local memory; indexed by the uniform pass counter)
    double w0n2 = 0.0;
    bool reorth = false;
    for (int sweep = 0; sweep < 2; ++sweep) {
        if (sweep == 1 && !reorth) break;
        double hprev = 0.0;
        for (int i = 0; i <= j + 1; ++i) {
            const double* vp = i ? V(i - 1) : nullptr;
            const double* vc = i <= j ? V(i) : nullptr;
            const bool nrm = (sweep == 0 && i == 0) || i == j + 1;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
            for (int k = threadIdx.x; k < m; k += MGS_T) {
                double wk = sw[k];
                if (vp) {
                    wk = fma(-hprev, __ldcg(vp + k), wk);
                    sw[k] = wk;
                }
                if (vc) a0 = fma(__ldcg(vc + k), wk, a0);
                if (nrm) a1 = fma(wk, wk, a1);
            }
            S.post(a0, a1, red);
            grid.sync();
            double t0, t1;
            S.fetch(t0, t1, red);
            if (i <= j) {
                if (sweep == 0) {
                    hv[i] = t0;                       // H[i, j]
                    if (i == 0) w0n2 = t1;            // ||w0||^2
                    hprev = t0;
                } else {
                    hv[i] += t0;                      // H[i, j] += correction (krylov.py:103-105)
                    hprev = t0;
                    if (blockIdx.x == 0 && threadIdx.x == 0) ctl[3 + i] = t0;
                }
            } else {
                const double wn = sqrt(t1);
                hv[j + 1] = wn;                       // H[j+1, j]
                if (sweep == 0) reorth = wn < 1e-3 * sqrt(w0n2);   // krylov.py:101
                if (blockIdx.x == 0 && threadIdx.x == 0) ctl[1] = t1;
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl[0] = w0n2;
        ctl[2] = reorth ? 1.0 : 0.0;
        for (int i = 0; i <= j + 1; ++i) h[i] = hv[i];
    }
    const double hn = hv[j + 1];
    for (int k = threadIdx.x; k < m; k += MGS_T) w[c0 + k] = hn != 0.0 ? sw[k] / hn : sw[k];   // krylov.py:108-110
}

static int mgs_coop(const double* Vb, int64_t ld, int j, double* w, int64_t n, double* h, double* ctl,
                    cudaStream_t s) {
    PFFMG_ONE_DEVICE();
    static int grid = -1;
    static int64_t cap = 0;
    static double* part = nullptr;
    if (grid < 0) {
        grid = 0;
        int dev = 0, sms = 0, coop = 0, maxsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        const int smem = maxsm - 2048;
        if (coop && smem > 0 &&
            cudaFuncSetAttribute(mgs_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess &&
            cudaMalloc(&part, sizeof(double) * 4 * sms) == cudaSuccess) {
            int occ = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, mgs_coop_kernel, MGS_T, smem) == cudaSuccess &&
                occ >= 1) {
                grid = sms;
                cap = (int64_t)sms * (smem / (int64_t)sizeof(double));
            }
        }
        cudaGetLastError();
    }
    if (grid <= 0 || n > cap || n < (int64_t)grid * MGS_T) return 1;   // not applicable: multi-launch path
    int64_t chunk = (n + grid - 1) / grid;
    const size_t smem = (size_t)chunk * sizeof(double);
    void* args[] = {(void*)&Vb, (void*)&ld, (void*)&j, (void*)&w, (void*)&n, (void*)&chunk, (void*)&h,
                    (void*)&ctl, (void*)&part};
    if (cudaLaunchCooperativeKernel((void*)mgs_coop_kernel, dim3(grid), dim3(MGS_T), args, smem, s) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    return 0;
}

extern "C" int pffmg_arnoldi_mgs(double* Vb, int64_t ld, int j, double* w, int64_t n, double* h,
                                 double* ctl, void* stream) {
    PFFMG_REQUIRE(Vb && w && h && ctl && j >= 0 && ld >= n, "pffmg_arnoldi_mgs: bad args");
    cudaStream_t s = as_stream(stream);
    static const bool coop_off = [] {
        const char* e = getenv("PFFMG_MGS_COOP");
        return e && e[0] == '0';
    }();
    // the one-launch form keeps H[0..j+1, j] in registers/local memory: j < MGS_MAXJ
    if (!coop_off && j < MGS_MAXJ && mgs_coop(Vb, ld, j, w, n, h, ctl, s) == 0) return check_launch("arnoldi_mgs");
    auto V = [&](int i) { return (const double*)(Vb + (int64_t)i * ld); };
    int rc;
    // modified Gram-Schmidt sweep
    for (int i = 0; i <= j; ++i) {
        MgsOp op{i ? V(i - 1) : nullptr, i ? h + (i - 1) : nullptr, V(i), w, ctl, h, i, i ? 1 : 0, 0, 0.0};
        if ((rc = run_fused(op, n, s, "arnoldi_mgs"))) return rc;
    }
    {
        MgsOp op{V(j), h + j, nullptr, w, ctl, h, j + 1, 2, 0, 0.0};
        if ((rc = run_fused(op, n, s, "arnoldi_mgs"))) return rc;
    }
    // conditional second pass (krylov.py:101-106), gated on ctl[2] on the device
    for (int i = 0; i <= j; ++i) {
        MgsOp op{i ? V(i - 1) : nullptr, i ? ctl + 3 + (i - 1) : nullptr, V(i), w, ctl, h, i, i ? 4 : 3, 1, 0.0};
        if ((rc = run_fused(op, n, s, "arnoldi_mgs"))) return rc;
    }
    {
        MgsOp op{V(j), ctl + 3 + j, nullptr, w, ctl, h, j + 1, 5, 1, 0.0};
        if ((rc = run_fused(op, n, s, "arnoldi_mgs"))) return rc;
    }
    // V_{j+1} = w / H[j+1, j]
    return run_fused(ScaleByInvOp{w, h + j + 1, 0.0}, n, s, "arnoldi_mgs");
}

extern "C" int pffmg_multi_axpy(const double* Z, int64_t ld, int k, const double* y, double* x, int64_t n,
                                void* stream) {
    PFFMG_REQUIRE(Z && y && x && k >= 0 && ld >= n, "pffmg_multi_axpy: bad args");
    // groups of up to 64 basis vectors per launch (restart lengths above 64 take several)
    for (int k0 = 0; k0 < k; k0 += 64) {
        const int kk = k - k0 < 64 ? k - k0 : 64;
        pdl_launch(multi_axpy_k, dim3(vgrid(n)), dim3(256), 0, as_stream(stream), Z + (int64_t)k0 * ld, ld, kk,
                   y + k0, x, n);
        const int rc = check_launch("pffmg_multi_axpy");
        if (rc) return rc;
    }
    return PFFMG_OK;
}

extern "C" int pffmg_active_set(const double* R_phi, const double* U_phi, const double* phi_old,
                                const double* mass_inv_phi, double c, const uint8_t* dirichlet_flags,
                                int phi_comp, int64_t V, uint8_t* active_phi, void* stream) {
    PFFMG_REQUIRE(R_phi && U_phi && phi_old && mass_inv_phi && active_phi && V >= 0 && phi_comp >= 0 &&
                      phi_comp < 8,
                  "pffmg_active_set: bad args");
    pdl_launch(active_set_k, dim3(vgrid(V)), dim3(256), 0, as_stream(stream), R_phi, U_phi, phi_old, mass_inv_phi, c,
                                                          dirichlet_flags, phi_comp, V, active_phi);
    VCHECK("pffmg_active_set");
}

extern "C" int pffmg_cg_start(const double* b, const double* diag, double* r, double* z, double* p, int64_t n,
                              double* scal, void* stream) {
    PFFMG_REQUIRE(b && diag && r && z && p && scal, "pffmg_cg_start: bad args");
    return run_fused(CgStartOp{b, diag, r, z, p, scal}, n, as_stream(stream), "pffmg_cg_start");
}

// phase 0: pAp + alpha; phase 1: r/z update + beta; phase 2: p update
extern "C" int pffmg_cg_step(const double* Ap, const double* diag, double* r, double* z, double* p, int64_t n,
                             double* scal, int phase, void* stream) {
    PFFMG_REQUIRE(Ap && diag && r && z && p && scal && phase >= 0 && phase <= 2, "pffmg_cg_step: bad args");
    cudaStream_t s = as_stream(stream);
    if (phase == 0) return run_fused(CgPApOp{p, Ap, scal}, n, s, "pffmg_cg_step");
    if (phase == 1) return run_fused(CgUpdateOp{Ap, diag, r, z, scal, 0.0}, n, s, "pffmg_cg_step");
    return run_fused(CgPOp{z, p, scal, 0.0}, n, s, "pffmg_cg_step");
}

// ================================================== slab-sharded Krylov (§8e)
namespace pffmg {

// owned-row predicate of a block vector with component stride V
struct Own {
    int64_t V, a, b;
    __device__ __forceinline__ bool in(int64_t i) const {
        if (a <= 0 && b >= V) return true;
        const int64_t v = i % V;
        return v >= a && v < b;
    }
};

struct DotOwnOp {
    static constexpr bool REDUCES = true;
    const double *x, *y;
    Own own;
    double* result;
    __device__ bool skip() const { return false; }
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double& a0, double&) const {
        if (own.in(i)) a0 = fma(x[i], y[i], a0);
    }
    __device__ void finish(double s0, double) const { *result = s0; }
};

// CG-Lanczos phases with owned partials (finish deferred to cg_dist_finish_k)
struct CgDistOp {
    static constexpr bool REDUCES = true;
    int phase;
    const double *in, *diag;
    double *r, *z, *p, *scal;
    Own own;
    double alpha, beta;
    __device__ bool skip() const { return phase != 0 && scal[C_STOP] != 0.0; }
    __device__ void prepare() {
        if (phase == 2) alpha = scal[C_ALPHA];
        if (phase == 3) beta = scal[C_BETA];
    }
    __device__ void elem(int64_t i, double& a0, double&) const {
        if (phase == 0) {                                   // krylov.py:163-166
            const double ri = in[i];
            const double zi = ri / diag[i];
            r[i] = ri;
            z[i] = zi;
            p[i] = zi;
            if (own.in(i)) a0 = fma(ri, zi, a0);
        } else if (phase == 1) {
            if (own.in(i)) a0 = fma(p[i], in[i], a0);
        } else if (phase == 2) {
            const double ri = r[i] - alpha * in[i];
            const double zi = ri / diag[i];
            r[i] = ri;
            z[i] = zi;
            if (own.in(i)) a0 = fma(ri, zi, a0);
        } else {
            p[i] = z[i] + beta * p[i];
        }
    }
    __device__ void finish(double s0, double) const {
        if (phase == 0) scal[C_RZ] = s0;
        else if (phase == 1) scal[C_PAP] = s0;
        else if (phase == 2) scal[C_RZN] = s0;
    }
};

// the finish logic of CgStartOp / CgPApOp / CgUpdateOp on all-reduced sums
__global__ void cg_dist_finish_k(double* scal, int phase) {
    pdl_wait();
    if (phase == 0) {
        const double s0 = scal[C_RZ];
        scal[C_STOP] = (s0 > 0.0 && isfinite(s0)) ? 0.0 : 1.0;
        scal[C_K] = 0.0;
        scal[C_NB] = 0.0;
        return;
    }
    if (scal[C_STOP] != 0.0) return;
    if (phase == 1) {
        const double s0 = scal[C_PAP];
        if (!(s0 > 0.0 && isfinite(s0))) {
            scal[C_STOP] = 1.0;
            return;
        }
        const double alpha = scal[C_RZ] / s0;
        const int k = (int)scal[C_K];
        scal[C_ALPHA] = alpha;
        if (k < CG_MAXIT) scal[C_HIST + k] = alpha;
        scal[C_K] = k + 1;
    } else {
        const double s0 = scal[C_RZN], rz = scal[C_RZ];
        if (s0 <= 1e-28 * rz || !isfinite(s0)) {
            scal[C_STOP] = 1.0;
            return;
        }
        const double beta = s0 / rz;
        const int nb = (int)scal[C_NB];
        scal[C_BETA] = beta;
        if (nb < CG_MAXIT) scal[C_HIST + CG_MAXIT + nb] = beta;
        scal[C_NB] = nb + 1;
        scal[C_RZ] = s0;
    }
}

// up to two dots of V_i . w (and w . w) per launch: the fused two-sum kernel
struct Dot2Op {
    static constexpr bool REDUCES = true;
    const double *v0, *v1, *w;   // v1 == nullptr -> the second sum is w . w (when norm) or unused
    int norm;
    Own own;
    double *o0, *o1;
    __device__ bool skip() const { return false; }
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double& a0, double& a1) const {
        if (!own.in(i)) return;
        const double wi = w[i];
        if (v0) a0 = fma(v0[i], wi, a0);
        if (v1) a1 = fma(v1[i], wi, a1);
        else if (norm) a1 = fma(wi, wi, a1);
    }
    __device__ void finish(double s0, double s1) const {
        if (o0) *o0 = s0;
        if (o1) *o1 = s1;
    }
};

struct GsSubOp {
    static constexpr bool REDUCES = true;
    const double* Vb;
    int64_t ld;
    int k;
    const double* c;
    double* w;
    double* hacc;
    Own own;
    double* norm2;
    __device__ bool skip() const { return false; }
    __device__ void prepare() {}
    __device__ void elem(int64_t i, double& a0, double&) const {
        double s = 0.0;
        for (int t = 0; t < k; ++t) s = fma(__ldg(c + t), Vb[(int64_t)t * ld + i], s);
        const double wi = w[i] - s;
        w[i] = wi;
        if (norm2 && own.in(i)) a0 = fma(wi, wi, a0);
    }
    __device__ void finish(double s0, double) const {
        if (norm2) *norm2 = s0;
        if (hacc)
            for (int t = 0; t < k; ++t) hacc[t] += c[t];
    }
};

struct NormalizeOp {
    static constexpr bool REDUCES = true;    // (for the finisher: *hout)
    const double* src;
    double* dst;
    const double* s2;
    double* hout;
    double hv;
    __device__ bool skip() const { return false; }
    __device__ void prepare() { hv = sqrt(*s2); }
    __device__ void elem(int64_t i, double&, double&) const { dst[i] = hv != 0.0 ? src[i] / hv : src[i]; }
    __device__ void finish(double, double) const {
        if (hout) *hout = hv;
    }
};

__global__ void pack_rows_k(double* vec, int64_t V, int nc, int64_t a, int64_t len, double* buf, int unpack) {
    pdl_wait();
    const int64_t n = len * nc;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i / len, t = i - c * len;
        double* g = vec + c * V + a + t;
        if (unpack)
            *g = buf[i];
        else
            buf[i] = *g;
    }
}

}  // namespace pffmg

extern "C" int pffmg_dot_owned(const double* x, const double* y, int64_t n, int64_t V, int64_t own_a,
                               int64_t own_b, double* result, void* stream) {
    PFFMG_REQUIRE(x && y && result && n >= 0 && V > 0, "pffmg_dot_owned: bad args");
    return run_fused(DotOwnOp{x, y, Own{V, own_a, own_b}, result}, n, as_stream(stream), "pffmg_dot_owned");
}

extern "C" int pffmg_cg_dist(int phase, const double* b_or_Ap, const double* diag, double* r, double* z, double* p,
                             int64_t n, int64_t V, int64_t own_a, int64_t own_b, double* scal, void* stream) {
    PFFMG_REQUIRE(phase >= 0 && phase <= 3 && r && z && p && scal && V > 0 &&
                      (phase == 3 || b_or_Ap) && (phase == 1 || phase == 3 || diag),
                  "pffmg_cg_dist: bad args");
    CgDistOp op{phase, b_or_Ap, diag, r, z, p, scal, Own{V, own_a, own_b}, 0.0, 0.0};
    return run_fused(op, n, as_stream(stream), "pffmg_cg_dist");
}

extern "C" int pffmg_cg_dist_finish(double* scal, int phase, void* stream) {
    PFFMG_REQUIRE(scal && phase >= 0 && phase <= 2, "pffmg_cg_dist_finish: bad args");
    pdl_launch(cg_dist_finish_k, dim3(1), dim3(1), 0, as_stream(stream), scal, phase);
    return check_launch("pffmg_cg_dist_finish");
}

extern "C" int pffmg_multi_dot_owned(const double* Vb, int64_t ld, int i0, int cnt, const double* w, int with_norm,
                                     int64_t n, int64_t V, int64_t own_a, int64_t own_b, double* out,
                                     void* stream) {
    PFFMG_REQUIRE(Vb && w && out && i0 >= 0 && cnt >= 0 && ld >= n && V > 0, "pffmg_multi_dot_owned: bad args");
    const Own own{V, own_a, own_b};
    const cudaStream_t s = as_stream(stream);
    // pairs of dots per launch; the norm rides in the free second slot of the last one
    bool norm_done = !with_norm;
    for (int t = 0; t < cnt; t += 2) {
        const double* v0 = Vb + (int64_t)(i0 + t) * ld;
        const double* v1 = t + 1 < cnt ? Vb + (int64_t)(i0 + t + 1) * ld : nullptr;
        const bool nrm = !v1 && !norm_done;
        Dot2Op op{v0, v1, w, nrm ? 1 : 0, own, out + t, v1 ? out + t + 1 : (nrm ? out + cnt : nullptr)};
        if (nrm) norm_done = true;
        const int rc = run_fused(op, n, s, "pffmg_multi_dot_owned");
        if (rc) return rc;
    }
    if (!norm_done) {
        Dot2Op op{nullptr, nullptr, w, 1, own, nullptr, out + cnt};
        return run_fused(op, n, s, "pffmg_multi_dot_owned");
    }
    return PFFMG_OK;
}

extern "C" int pffmg_gs_subtract(const double* Vb, int64_t ld, int k, const double* c, double* w, int64_t n,
                                 double* hacc, int64_t V, int64_t own_a, int64_t own_b, double* norm2,
                                 void* stream) {
    PFFMG_REQUIRE(Vb && c && w && k >= 0 && ld >= n && V > 0, "pffmg_gs_subtract: bad args");
    return run_fused(GsSubOp{Vb, ld, k, c, w, hacc, Own{V, own_a, own_b}, norm2}, n, as_stream(stream),
                     "pffmg_gs_subtract");
}

extern "C" int pffmg_normalize(const double* src, double* dst, int64_t n, const double* s2, double* hout,
                               void* stream) {
    PFFMG_REQUIRE(src && dst && s2 && n >= 0, "pffmg_normalize: bad args");
    return run_fused(NormalizeOp{src, dst, s2, hout, 0.0}, n, as_stream(stream), "pffmg_normalize");
}

extern "C" int pffmg_pack_rows(double* vec, int64_t V, int n_comp, int64_t a, int64_t len, double* buf, int unpack,
                               void* stream) {
    PFFMG_REQUIRE(vec && buf && n_comp >= 1 && a >= 0 && len >= 0 && a + len <= V, "pffmg_pack_rows: bad args");
    if (len == 0) return PFFMG_OK;
    pdl_launch(pack_rows_k, dim3(vgrid(len * n_comp)), dim3(256), 0, as_stream(stream), vec, V, n_comp, a, len, buf,
               unpack);
    return check_launch("pffmg_pack_rows");
}
