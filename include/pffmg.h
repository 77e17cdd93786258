/*
 * pffmg — B200-native matrix-free phase-field-fracture Jacobian + GMG kernels.
 *
 * Flat C ABI of libpffmg.so (built for sm_100a).  Every entry point takes
 * plain device pointers (fp64 vectors in the reference's component-major dof
 * layout gid = c*V + v, reference fem.py:1-4 / fem.py:91-126), sizes, and a
 * cudaStream_t passed as void*.  Every call returns an int status
 * (0 = ok); pffmg_last_error() returns the message of the last failure on the
 * calling thread.  No C++ exceptions cross this boundary.  All work is
 * enqueued asynchronously on the given stream; the library never
 * synchronises except in the functions documented as returning host data.
 *
 * The reference (fracmg, pure Python) binds these through ctypes; the host
 * twins live in paper_1902_08112_b200/ and INTEGRATION.md shows the binding.
 * Reference paths below are relative to /root/reference/pkg/src/fracmg/.
 */
#ifndef PFFMG_H
#define PFFMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFFMG_OK 0
#define PFFMG_ERR_ARG 1
#define PFFMG_ERR_CUDA 2
#define PFFMG_ERR_UNSUPPORTED 3

/* Which part of the Jacobian a vmult applies (reference model.py:368-392). */
#define PFFMG_FULL (-1)     /* PhaseFieldOperator.apply          model.py:368-375 */
#define PFFMG_UBLOCK 0      /* apply_block(0, .) displacement    model.py:377-392 */
#define PFFMG_PBLOCK 1      /* apply_block(1, .) phase field     model.py:377-392 */
#define PFFMG_BLOCKDIAG 2   /* both diagonal blocks at once on a full vector (u rows = apply_block(0),
                               phi row = apply_block(1)): the operator of the block smoother */

#define PFFMG_HINT_PREMASKED 1
#define PFFMG_HINT_ENDS 2       /* finalise only the first and the last owned plane (slab
                                   boundary rows once the halo has landed) */

/*
 * Level geometry: a (possibly non-box) lattice of congruent cells.  Vertex
 * numbering follows the reference mesh (mesh.py:163-194): x fastest, rows of
 * constant (y, z) contiguous.  For a box lattice the row tables are NULL and
 * vertex id = x + (nx+1)*(y + (ny+1)*z).  Otherwise, for vertex row
 * r = y + (ny+1)*z the vertices x in [vrow_lo[r], vrow_hi[r]) have ids
 * vrow_off[r] + (x - vrow_lo[r]); for cell row s = y + ny*z the cells
 * x in [crow_lo[s], crow_hi[s]) exist.  All table pointers are DEVICE pointers.
 */
typedef struct {
    int32_t struct_size;    /* = sizeof(pffmg_lattice); checked by every entry point (ABI guard) */
    int32_t dim;            /* 2 or 3 */
    int32_t nx, ny, nz;     /* cells per axis of the bounding lattice (nz = 0 in 2D) */
    double hx, hy, hz;      /* cell edge lengths (LevelMesh.cell_size) */
    int64_t n_vertices;     /* V: component stride of every dof vector */
    const int64_t* vrow_off;
    const int32_t* vrow_lo;
    const int32_t* vrow_hi;
    const int32_t* crow_lo;
    const int32_t* crow_hi;
    /* Slab decomposition (multi-GPU): operator kernels finalise only vertex
     * planes [own_lo, own_hi) of the last axis (y in 2D, z in 3D); the planes
     * own_lo-1 and own_hi, if inside the lattice, are ghost planes that must
     * hold the neighbours' values.  own_lo = own_hi = 0 means the whole lattice. */
    int32_t own_lo, own_hi;
    /* Global index of local plane 0 along the cut axis (0 unless this is a
     * slab of a larger level); transfers use it to pair coarse and fine slabs. */
    int32_t plane0;
    /* Element order: 0 or 1 = trilinear/bilinear Q1 (the reference's element,
     * fem.py:1-8); 2 = biquadratic Q2 (2D box lattices): dofs live on the
     * nodes of the half-spacing lattice, (2nx+1)(2ny+1) of them, x fastest;
     * 3x3 Gauss points (BASELINE configs[2]).  For Q2 the "planes" of
     * own_lo/own_hi/plane0 are NODE rows (2ny+1 of them); a slab starts on a
     * cell boundary (plane0 even) and a sharded operator needs two ghost node
     * rows below own_lo (four for restriction) and one above. */
    int32_t order;
    /* Optional work list of the 3D streaming kernels (NULL: every tile of the
     * bounding lattice).  The x-y plane of vertex columns is cut into tiles of
     * PFFMG_TILE3 x PFFMG_TILE3 columns, (nx+1+T-1)/T x (ny+1+T-1)/T of them
     * (x fastest); tiles3d lists, ascending, the n_tiles3d tile indices
     * bx + ntx*by that hold at least one vertex of the lattice.  A DEVICE
     * pointer.  Non-box lattices (the L-shapes) pass it so that the kernels
     * distribute only occupied tiles over the SMs; listing an empty tile or
     * every tile is always correct, omitting an occupied one is not. */
    const int32_t* tiles3d;
    int32_t n_tiles3d;
} pffmg_lattice;

#define PFFMG_TILE3 15

/*
 * Linearisation state + material of one level (model.py:89-119, 270-309).
 * The per-quadrature-point coefficient tables of _build_caches are NOT
 * stored: the kernels recompute gk, T_phiu, a_phiphi on the fly from U and
 * phi_tilde (SURVEY §8d "model F").
 */
typedef struct {
    int32_t struct_size;        /* = sizeof(pffmg_state); checked by every entry point (ABI guard) */
    double mu, lam, g_c, kappa, eps;
    double pressure;            /* MaterialParams.pressure(state.t) */
    int32_t split;              /* 0 = NOSPLIT; 1 = MIEHE spectral split */
    int32_t hints;              /* bit 0 (PFFMG_HINT_PREMASKED): every input vector of the
                                   call is already zero at constrained dofs, so the masked
                                   gather (fem.py:205-206) can be skipped.  Results are
                                   identical; a wrong hint gives wrong results.
                                   bit 1 (PFFMG_HINT_ENDS): operator calls finalise only
                                   planes own_lo and own_hi-1 (one launch for both slab
                                   boundary rows of an overlapped halo exchange). */
    const double* U;            /* (dim+1)*V linearisation point (may be NULL for the u block) */
    const double* phi_tilde;    /* V extrapolated phase field (may be NULL for the phi block) */
    const double* rho;          /* NULL (rho == 1) or modulus field per lattice cell x QP */
    const uint8_t* flags;       /* (see below) */
    double split_band;          /* MaterialParams.split_band: C^1 blend half-width of the
                                   spectral split (model.py:56-86); 0 = hard split */
    const double* phi_coef;     /* NULL, or the per-QP a_phiphi table of pffmg_phi_coef built
                                   from this state's U (NoSplit: isotropic Q1 or Q2
                                   lattices): the phi block (which = 1) and, in 2D, the
                                   block-diagonal operator (which = 2) then read it instead
                                   of re-deriving a_phiphi from U (model.py:304-308 cached,
                                   as _build_caches does).  Ignored elsewhere. */
    /* flags: V packed constraint bits: bit c <=> dof c*V+v constrained; the
     * buffer must stay readable (any content) up to 4*ceil(V/4) + 40 bytes:
     * kernels read aligned 32-bit words.
     * split = 1 (Miehe spectral split, model.py:174-219): per-QP closed-form
     * (2D) or Jacobi (3D) eigen-solve, tangent applied without forming it. */
} pffmg_state;

const char* pffmg_last_error(void);
/* ABI version: 3 (struct_size guards; pffmg_state.phi_coef; pffmg_lattice.tiles3d). */
#define PFFMG_ABI_VERSION 3
int pffmg_version(void);
int pffmg_device_sm_count(int* out);
/* Programmatic dependent launch of the library's kernels (on by default;
 * PFFMG_PDL=0 in the environment disables it for good): on = 0 makes every
 * later launch of this process fully stream-ordered, on = 1 restores it.
 * *previous (optional) receives the old setting.  Used around multi-stream
 * graph captures, where early-launched dependents would hold SM slots. */
int pffmg_set_pdl(int on, int* previous);

/* ---------------------------------------------------------------- operator */

/* out = G~ v restricted to `which` (model.py:368-392): constrained entries of
 * v read as 0, constrained rows copy v.  v/out point at the block's first
 * component (component stride = lattice->n_vertices). */
int pffmg_apply(const pffmg_lattice* lat, const pffmg_state* st, int which,
                const double* v, double* out, void* stream);

/* out = b - A x (mgsolve.py:95, 100, 227): fused residual. out != x. */
int pffmg_residual(const pffmg_lattice* lat, const pffmg_state* st, int which,
                   const double* x, const double* b, double* out, void* stream);

/* Semilinear form A(U) of the linearisation state (NoSplit), constrained
 * rows zeroed (model.py:420-460): the Newton right-hand side is -out. */
int pffmg_semilinear_residual(const pffmg_lattice* lat, const pffmg_state* st, double* out,
                              void* stream);

/* Per-QP phi-block coefficient table of a NoSplit lattice (isotropic Q1 in 2D
 * or 3D, or Q2): out[q * C + c] = a_phiphi at QP q of lattice cell c (c = cx +
 * nx (cy + ny cz), C = lattice cells; Q1: JxW and rho included, Q2: rho
 * included), the a_phiphi entry of the reference's _build_caches
 * (model.py:270-309, 304-308).  2^dim * C (Q1) or 9 * C (Q2) doubles; cells
 * absent from a non-box lattice get 0.  Point state.phi_coef at it afterwards. */
int pffmg_phi_coef(const pffmg_lattice* lat, const pffmg_state* st, double* out, void* stream);

/* Exact operator diagonal, constrained entries = 1.0 (model.py:394-413). */
int pffmg_diagonal(const pffmg_lattice* lat, const pffmg_state* st, double* out, void* stream);

/* One fused Chebyshev step of chebyshev_apply's recurrence (mgsolve.py:107-112):
 *   r -= A d_in;  d_out = c_dd*d_in + c_dr*(invdiag*r);  x += d_out
 * or, with x_add_din = 1 (first step after pffmg_cheb_init),
 *   x = (x + d_in) + d_out   -- the same rounding as the reference's two updates.
 * d_out != d_in; x is not read by the stencil so it is updated in place. */
int pffmg_cheb_step(const pffmg_lattice* lat, const pffmg_state* st, int which,
                    const double* d_in, double* d_out, double* r, double* x,
                    const double* invdiag, double c_dd, double c_dr, int x_add_din,
                    void* stream);

/* Start of chebyshev_apply from a non-zero x (mgsolve.py:95, 103-105):
 *   r = b - A x;  d = (invdiag*r)/theta.
 * The update x += d is deferred to the first pffmg_cheb_step (x_add_din = 1)
 * or done by pffmg_axpy when the degree is 1, so x is never written while
 * other CTAs still read it through the stencil. */
int pffmg_cheb_init(const pffmg_lattice* lat, const pffmg_state* st, int which,
                    const double* x, const double* b, double* r, double* d,
                    const double* invdiag, double theta, void* stream);

/* Device-coefficient forms ("_dc") of the Chebyshev entry points: the
 * recurrence scalars are read from device memory at kernel run time
 * (coef[0] = c_dd, coef[1] = c_dr; theta[0] = theta), so a CUDA graph that
 * captures a V-cycle stays valid when the spectra of the next Newton step
 * change its coefficients.  Results are bit-identical to the scalar forms. */
int pffmg_cheb_step_dc(const pffmg_lattice* lat, const pffmg_state* st, int which,
                       const double* d_in, double* d_out, double* r, double* x,
                       const double* invdiag, const double* coef, int x_add_din, void* stream);
int pffmg_cheb_init_dc(const pffmg_lattice* lat, const pffmg_state* st, int which,
                       const double* x, const double* b, double* r, double* d,
                       const double* invdiag, const double* theta, void* stream);

/* pffmg_apply with HOST v / out (pinned for overlap): the copies in, the
 * stencil and the copies out are pipelined over n_strips strips of planes of
 * the last axis on two internal copy streams.  d_v / d_out are device scratch
 * vectors of the block's size.  When the call returns the work is enqueued on
 * `stream`; synchronise it before reading h_out.  h_plane_off (n_planes + 1
 * host entries: first vertex id of every plane, then V) is required for
 * non-box lattices, NULL for boxes.  Whole (non-slab) lattices only. */
int pffmg_apply_host(const pffmg_lattice* lat, const pffmg_state* st, int which,
                     const double* h_v, double* h_out, double* d_v, double* d_out,
                     const int64_t* h_plane_off, int n_strips, void* stream);

/* The same for ORDINARY (pageable) host memory, e.g. the numpy arrays the
 * reference's drivers pass to PhaseFieldOperator.apply (model.py:368-375):
 * host threads (PFFMG_COPY_THREADS, default half the cores, at most 16) stage
 * the strips through page-locked buffers the library keeps, overlapped with
 * the link copies and the stencil.  Synchronous: h_out is complete on return. */
int pffmg_apply_pageable(const pffmg_lattice* lat, const pffmg_state* st, int which,
                         const double* h_v, double* h_out, double* d_v, double* d_out,
                         const int64_t* h_plane_off, int n_strips, void* stream);

/* Copies between ORDINARY (pageable) host memory and device memory for the
 * numpy-facing twins: 4 MiB chunks through a ring of page-locked slots, filled /
 * drained by host threads (PFFMG_COPY_THREADS) while earlier chunks are on the
 * link.  Ordered after prior work on `stream`; synchronous (complete on return). */
int pffmg_copy_h2d(const void* host, void* device, size_t bytes, void* stream);
int pffmg_copy_d2h(const void* device, void* host, size_t bytes, void* stream);

/* Boundary load (model.py:511-547): sum over the n_faces boundary faces
 * (face_cell[i] = lattice cell index cx + nx (cy + ny cz), face_id[i] =
 * 2 axis + side, LevelMesh.bf_face) of the face-Gauss integral of
 * sign(side) * (g(phi) rho sigma+ + rho sigma-)[direction, axis]; rho_face is
 * NULL (rho = 1) or the modulus field at the 2^(dim-1) face points of each
 * face (fem.py:265-292 order).  Q1 lattices; deterministic reduction into
 * the DEVICE double *result. */
int pffmg_boundary_load(const pffmg_lattice* lat, const pffmg_state* st, const int64_t* face_cell,
                        const int32_t* face_id, int64_t n_faces, int direction,
                        const double* rho_face, double* result, void* stream);
/* Quantities of interest (model.py:472-506) as one deterministic cell-integral
 * reduction into the device scalar *result: kind 0 = crack_energy (uses eps,
 * g_c), 1 = bulk_energy (split, band, modulus field, pressure; U's own phi
 * degrades), 2 = fracture_volume.  st->U is the full (dim+1)*V state. */
int pffmg_qoi(const pffmg_lattice* lat, const pffmg_state* st, int kind, double* result,
              void* stream);

/* Block-diagonal ("_bd") forms: one kernel runs the Chebyshev recurrences of
 * both diagonal blocks on full vectors (the blocks are independent in
 * _smooth_blockwise, mgsolve.py:200-206), with per-block scalars read from
 * device memory: coef_u/theta_u for the displacement components, coef_p /
 * theta_p for the phase field.  n_u = dim*V in pffmg_cheb_init_zero_bd. */
int pffmg_cheb_step_bd(const pffmg_lattice* lat, const pffmg_state* st, const double* d_in, double* d_out,
                       double* r, double* x, const double* invdiag, const double* coef_u,
                       const double* coef_p, int x_add_din, void* stream);
int pffmg_cheb_init_bd(const pffmg_lattice* lat, const pffmg_state* st, const double* x, const double* b,
                       double* r, double* d, const double* invdiag, const double* theta_u,
                       const double* theta_p, void* stream);
int pffmg_cheb_init_zero_bd(const double* b, const double* invdiag, const double* theta_u,
                            const double* theta_p, int64_t n_u, double* r, double* d, double* x,
                            int64_t n, void* stream);

/* "Lean" x = 0 start: the start's residual is the right-hand side and its
 * iterate is d, so pffmg_cheb_init_zero(_dc/_bd), pffmg_masked_copy_init_bd and
 * pffmg_restrict_init_bd accept r = x = NULL (only d is stored), and the FIRST
 * step of the recurrence (mgsolve.py:108-111) then goes through these entry
 * points: the residual is read from `rhs`, x is not read (x_old = 0 + d_in), and
 * r, d_out, x are written.  Bit-identical to the full init + pffmg_cheb_step_*. */
int pffmg_cheb_first_dc(const pffmg_lattice* lat, const pffmg_state* st, int which,
                        const double* d_in, const double* rhs, double* d_out, double* r, double* x,
                        const double* invdiag, const double* coef, void* stream);
int pffmg_cheb_first_bd(const pffmg_lattice* lat, const pffmg_state* st, const double* d_in,
                        const double* rhs, double* d_out, double* r, double* x, const double* invdiag,
                        const double* coef_u, const double* coef_p, void* stream);

/* The whole coarse_solve of the V-cycle (mgsolve.py:209-218) in one launch for
 * small whole levels (<= 256 lattice cells): both blocks' Chebyshev
 * recurrences from x = 0 with degrees deg_u / deg_p and the coefficient
 * tables coef_u / coef_p = [theta, c_dd_1, c_dr_1, ...] (device memory, as
 * for the _dc entry points).  b, x, r, d, invdiag: full vectors of the level.
 * Returns PFFMG_ERR_UNSUPPORTED for larger levels. */
int pffmg_coarse_cheb(const pffmg_lattice* lat, const pffmg_state* st, const double* b, double* x,
                      double* r, double* d, const double* invdiag, const double* coef_u, int deg_u,
                      const double* coef_p, int deg_p, void* stream);

/* ---------------------------------------------------------------- transfers */
/* fem.py:308-411 with the V-cycle masking of mgsolve.py:228-234.
 * `coarse`/`fine` are consecutive levels l and l+1; n_comp components. */

/* vc = P^T vf per component; if coarse_flags != NULL, constrained coarse
 * entries are set to 0 (mgsolve.py:228-229). */
int pffmg_restrict(const pffmg_lattice* coarse, const pffmg_lattice* fine, int n_comp,
                   int comp0, const double* vf, double* vc, const uint8_t* coarse_flags,
                   void* stream);

/* V-cycle descent (mgsolve.py:228-229 then 95, 103-106): vc = P^T vf over all
 * dim+1 components with constrained coarse entries 0, fused with the coarse
 * level's block-diagonal Chebyshev start from x = 0: r = vc, d = invdiag vc /
 * theta (theta_u for the displacement block, theta_p for phi; device scalars),
 * x = d. */
int pffmg_restrict_init_bd(const pffmg_lattice* coarse, const pffmg_lattice* fine, const double* vf,
                           double* vc, const uint8_t* coarse_flags, const double* invdiag,
                           const double* theta_u, const double* theta_p, double* r, double* d,
                           double* x, void* stream);

/* vf = P vc per component (fine_flags == NULL, accumulate == 0) or
 * vf += (fine constrained ? 0 : P vc) (mgsolve.py:232-234, accumulate = 1). */
int pffmg_prolongate(const pffmg_lattice* coarse, const pffmg_lattice* fine, int n_comp,
                     int comp0, const double* vc, double* vf, const uint8_t* fine_flags,
                     int accumulate, void* stream);

/* Nodal injection of n_comp fp64 components (fem.py:361-363, 394-401). */
int pffmg_inject_f64(const pffmg_lattice* coarse, const pffmg_lattice* fine, int n_comp,
                     const double* vf, double* vc, void* stream);
/* Injection of packed constraint flags (mgsolve.py:182-186): bit-exact. */
int pffmg_inject_flags(const pffmg_lattice* coarse, const pffmg_lattice* fine,
                       const uint8_t* ff, uint8_t* fc, void* stream);
/* Injection map coarse vertex -> fine vertex id (fem.py:346-351, 365-367). */
int pffmg_injection_map(const pffmg_lattice* coarse, const pffmg_lattice* fine,
                        int64_t* out, void* stream);

/* ----------------------------------------------------------- masks / vectors */

/* flags[v] = OR_c (mask[c*V+v] != 0) << c. */
int pffmg_pack_flags(const uint8_t* mask, int n_comp, int64_t V, uint8_t* flags, void* stream);
int pffmg_unpack_flags(const uint8_t* flags, int n_comp, int64_t V, uint8_t* mask, void* stream);
/* out = constrained ? 0 : in over components [comp0, comp0+n_comp). */
int pffmg_masked_copy(const uint8_t* flags, int64_t V, int comp0, int n_comp,
                      const double* in, double* out, void* stream);

/* V-cycle entry (mgsolve.py:271-272 then 95, 103-106): rhs = in with the dofs
 * constrained in flags set to 0 (n_comp = dim+1 components), fused with the
 * block-diagonal Chebyshev start from x = 0: r = rhs, d = invdiag rhs / theta
 * (theta_u for the displacement components, theta_p for phi; device scalars),
 * x = d. */
int pffmg_masked_copy_init_bd(const uint8_t* flags, int64_t V, int n_comp, const double* in,
                              double* rhs, const double* invdiag, const double* theta_u,
                              const double* theta_p, double* r, double* d, double* x, void* stream);
/* invdiag = 1 / diag. */
int pffmg_reciprocal(const double* diag, double* out, int64_t n, void* stream);
/* Chebyshev start from x = 0 (mgsolve.py:95, 103-106): r = b; d = (inv*r)/theta; x = d. */
int pffmg_cheb_init_zero(const double* b, const double* invdiag, double theta,
                         double* r, double* d, double* x, int64_t n, void* stream);
/* Degenerate-range update (mgsolve.py:99): x += (inv*r)/theta. */
int pffmg_jacobi_update(const double* r, const double* invdiag, double theta,
                        double* x, int64_t n, void* stream);
/* Device-coefficient forms (theta read from device memory, see pffmg_cheb_step_dc). */
int pffmg_cheb_init_zero_dc(const double* b, const double* invdiag, const double* theta,
                            double* r, double* d, double* x, int64_t n, void* stream);
int pffmg_jacobi_update_dc(const double* r, const double* invdiag, const double* theta,
                           double* x, int64_t n, void* stream);

/* y = a*x + y ; x = a*x ; y = x - y etc. */
int pffmg_axpy(double a, const double* x, double* y, int64_t n, void* stream);
int pffmg_axpby(double a, const double* x, double b, double* y, int64_t n, void* stream);
int pffmg_scale(double a, double* x, int64_t n, void* stream);
int pffmg_copy(const double* x, double* y, int64_t n, void* stream);
/* out = x - y */
int pffmg_sub(const double* x, const double* y, double* out, int64_t n, void* stream);

/* Deterministic reductions: fixed grid, fixed per-block tree, fixed-order
 * final sum -> bitwise reproducible for a given n.  Result written to the
 * DEVICE double *result. */
int pffmg_dot(const double* x, const double* y, int64_t n, double* result, void* stream);
int pffmg_dot_scaled(const double* x, const double* y, const double* s, int64_t n,
                     double* result, void* stream);   /* sum x*(s*y) ... see docs */

/* GMRES Arnoldi (krylov.py:93-107), device-resident H column:
 *   for i in 0..j: h[i] = V_i . w ; w -= h[i] V_i      (modified Gram-Schmidt)
 * with the conditional second pass when ||w|| < 1e-3 ||w0||, then
 * h[j+1] = ||w||, V_{j+1} = w / h[j+1] (if nonzero).  Vb is the (m+1) x ld
 * row-major basis, h is a device array of length >= j+2, scratch a device
 * array of length >= j+4 (any j >= 0: restart lengths are not limited).
 * Returns nothing on the host; the caller reads h. */
int pffmg_arnoldi_mgs(double* Vb, int64_t ld, int j, double* w, int64_t n, double* h,
                      double* scratch, void* stream);
/* x += sum_i y[i] * Z_i, i < k (krylov.py:132); y is a DEVICE array; any k >= 0. */
int pffmg_multi_axpy(const double* Z, int64_t ld, int k, const double* y, double* x,
                     int64_t n, void* stream);

/* Primal-dual active set of the phase-field dofs (nonlinear.py:75-89):
 * active[v] = (mass_inv[v]*R[v] + c*(U[v] - phi_old[v]) > 0) && !(dirichlet bit phi_comp),
 * evaluated with the reference's rounding (no FMA contraction): bit-exact for
 * identical inputs.  Pointers are the phase-field parts (length V);
 * dirichlet_flags (packed per-vertex bits) may be NULL. */
int pffmg_active_set(const double* R_phi, const double* U_phi, const double* phi_old,
                     const double* mass_inv_phi, double c, const uint8_t* dirichlet_flags,
                     int phi_comp, int64_t V, uint8_t* active_phi, void* stream);

/* Jacobi-PCG Lanczos for estimate_spectrum (krylov.py:146-185), device part.
 * State vector layout: see pffmg_cg_* in csrc/vectors.cu. */
int pffmg_cg_start(const double* b, const double* diag, double* r, double* z, double* p,
                   int64_t n, double* scal, void* stream);
int pffmg_cg_step(const double* Ap, const double* diag, double* r, double* z, double* p,
                  int64_t n, double* scal, int phase, void* stream);

/* ------------------------------------------ slab-sharded (multi-GPU) Krylov
 * Reductions over a rank's OWNED rows only: element i of a block vector
 * (component stride V) counts iff own_a <= i mod V < own_b (own_a = 0,
 * own_b = V: every element).  Each returns the rank-local partial sum; the
 * caller all-reduces it (one scalar / short vector per pass) before the next
 * step consumes it.  Deterministic like pffmg_dot. */

/* result = sum over owned rows of x*y. */
int pffmg_dot_owned(const double* x, const double* y, int64_t n, int64_t V, int64_t own_a,
                    int64_t own_b, double* result, void* stream);

/* Jacobi-PCG Lanczos of estimate_spectrum (krylov.py:146-185) with owned-row
 * partial reductions.  phase 0: r = b, z = D^-1 r, p = z, partial r.z ->
 * scal[0]; 1: partial p.Ap -> scal[6]; 2: r -= alpha Ap, z = D^-1 r, partial
 * r.z -> scal[7]; 3: p = z + beta p.  After all-reducing the partial,
 * pffmg_cg_dist_finish(scal, phase) (phases 0..2) applies the reference's
 * breakdown rules and records alpha / beta (scal layout of pffmg_cg_step). */
int pffmg_cg_dist(int phase, const double* b_or_Ap, const double* diag, double* r, double* z, double* p,
                  int64_t n, int64_t V, int64_t own_a, int64_t own_b, double* scal, void* stream);
int pffmg_cg_dist_finish(double* scal, int phase, void* stream);

/* Classical Gram-Schmidt passes of the distributed Arnoldi step (CGS2; the
 * single-GPU path keeps the reference's MGS, pffmg_arnoldi_mgs).
 * multi_dot: out[t] = owned V_{i0+t} . w for t < cnt, and (with_norm)
 * out[cnt] = owned w . w;  gs_subtract: w -= sum_{t<k} c[t] V_t, hacc[t] +=
 * c[t] (hacc may be NULL), and (norm2 != NULL) the owned partial of the new
 * w . w into *norm2;  normalize: h = sqrt(*s2), *hout = h, dst = src / h
 * (dst = src when h == 0, krylov.py:108-110). */
int pffmg_multi_dot_owned(const double* Vb, int64_t ld, int i0, int cnt, const double* w, int with_norm,
                          int64_t n, int64_t V, int64_t own_a, int64_t own_b, double* out, void* stream);
int pffmg_gs_subtract(const double* Vb, int64_t ld, int k, const double* c, double* w, int64_t n,
                      double* hacc, int64_t V, int64_t own_a, int64_t own_b, double* norm2, void* stream);
int pffmg_normalize(const double* src, double* dst, int64_t n, const double* s2, double* hout,
                    void* stream);

/* Halo packing: pack (unpack = 0) buf[c len + t] = vec[c V + a + t] for
 * c < n_comp, t < len, or unpack (unpack = 1) the reverse -- one contiguous
 * message per neighbour instead of one per component. */
int pffmg_pack_rows(double* vec, int64_t V, int n_comp, int64_t a, int64_t len, double* buf, int unpack,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PFFMG_H */
