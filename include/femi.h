/*
 * femi.h -- C ABI of the B200-native FEM harmonic-inpainting hot path
 * (Chizhov & Weickert, "Efficient Data Optimisation for Harmonic Inpainting with Finite
 * Elements", arXiv 2105.01586). Library: paper_2105_01586_b200/libfemi.so (sm_100a).
 *
 * Citations "PAPER.md:Lx-y" refer to the paper's LaTeX source; readings A1..A18 are the
 * interpretations frozen in DESIGN.md where the paper is silent.
 *
 * Conventions (all calls):
 *  - Pixel index pix = y*W + x; pixel centres at integer (x, y); Omega = [0,W-1]x[0,H-1]
 *    (reading A1). Images are row-major fp64 arrays of W*H values on the 0..255 scale.
 *  - Vertex numbering is canonical: unknown vertices first (ascending pix), then mask
 *    vertices (ascending pix). A vertex-value vector u_vert has n_vert = n_unknown +
 *    n_mask entries in that order; a mask-value vector g has n_mask entries in ascending
 *    mask-pix order.
 *  - Handles (femi_mesh, femi_system) are created and freed only by the library and are
 *    immutable after creation, EXCEPT that a femi_system caches device scratch for its
 *    solves. A femi_system may be shared across host threads and streams: calls on one
 *    system are serialised -- host side by a per-system lock, device side by an event, so
 *    a call's work is ordered after the work of the previous call on the same system,
 *    whatever stream that ran on (calls on different systems run concurrently). Freeing a
 *    system while another thread still uses it is the caller's error.
 *  - Device pointers are caller-owned (e.g. PyTorch tensors); the library never frees
 *    them; they must stay valid until the enqueued work completes. All device work is
 *    enqueued on the caller's stream (femi_stream == cudaStream_t; NULL = legacy default
 *    stream). Calls that return host outputs synchronise that stream before returning.
 *  - Every call returns a femi_status; on failure femi_last_error() returns a thread-local
 *    message. No C++ exception crosses the ABI. There is no CPU fallback: without a usable
 *    sm_100 device the device calls return FEMI_E_CUDA.
 */
#ifndef FEMI_H
#define FEMI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* femi_stream; /* == cudaStream_t */

typedef enum {
    FEMI_OK = 0,
    FEMI_E_ARG = 1,           /* invalid argument (NULL, negative size, bad option)      */
    FEMI_E_DEGENERATE = 2,    /* W < 2 or H < 2: every vertex collinear                  */
    FEMI_E_NO_MASK = 3,       /* no Dirichlet vertex: A_uu singular  */
    FEMI_E_NOT_CONVERGED = 4, /* max_iter reached; outputs hold the last iterate          */
    FEMI_E_NONFINITE = 5,     /* NaN/Inf in inputs or iterates                            */
    FEMI_E_NEG_CURVATURE = 6, /* p.Ap <= 0 inside CG: matrix not SPD                      */
    FEMI_E_SIZE = 7,          /* pix out of range, duplicates, mask/unknown overlap, W or H > 16384 */
    FEMI_E_CUDA = 8,          /* CUDA runtime error (message has the CUDA error string)   */
    FEMI_E_OOM = 9            /* host or device allocation failed                         */
} femi_status;

const char* femi_last_error(void);
const char* femi_version(void);
/* Number of CUDA kernels this library has launched since it was loaded (all threads). */
int64_t femi_kernel_launches(void);

/* Device-side bounds-check failures recorded since the last call, then reset; *first_site (if
 * not NULL) receives the first failing check (file id * 100000 + line). Always 0 unless the
 * library was built with device checks (libfemi_check.so, FEMI_DEVICE_CHECKS): that build,
 * run under the GPU test suite, stands in for compute-sanitizer memcheck on the index paths.
 * Returns -1 if the counters cannot be read. */
int64_t femi_device_check_failures(int64_t* first_site);

typedef struct femi_mesh_s* femi_mesh;
typedef struct femi_system_s* femi_system;

typedef struct {
    int64_t width, height;
    int64_t n_vert, n_unknown, n_mask, n_tri;
    int64_t nnz_uu; /* A_uu entries incl. the diagonal (reading A5) */
    int64_t nnz_uk; /* A_uk entries                                  */
} femi_mesh_info;

/* ---------------------------------------------------------------------------------
 * S0 mesh_build (HOST setup stage, timed separately).
 * "Every mask pixel is a vertex in this mesh, and a subset of the
 * remaining non-mask pixels are chosen as unknowns ... a Delaunay triangulation is
 * constructed from the point set formed by the vertices". Corners missing from both sets
 * are added as unknowns (reading A2). Cocircular ties are broken by the symbolic
 * perturbation of reading A3, so the triangulation is unique and independent of the
 * input order. Triangles are CCW, rotated so the smallest pix comes first, sorted
 * lexicographically by pix triple.
 *   mask_px[m], unknown_px[p]: HOST arrays of distinct pixels, any order, disjoint.
 *   out: receives a new handle (free with femi_mesh_free).
 * Errors: FEMI_E_ARG (NULL), FEMI_E_DEGENERATE (W<2 or H<2), FEMI_E_SIZE (range,
 * duplicates, overlap, W or H > 16384), FEMI_E_NO_MASK (m == 0), FEMI_E_OOM.
 * ------------------------------------------------------------------------------- */
femi_status femi_mesh_build(int32_t W, int32_t H, const int32_t* mask_px, int64_t m,
                            const int32_t* unknown_px, int64_t p, femi_mesh* out);
/* S0 incremental, for densification (every iteration adds b_t mask
 * pixels): the mesh of prev's vertices plus the b new MASK pixels.
 * The new vertices are inserted into prev's triangulation (Bowyer-Watson); the SoS
 * triangulation of reading A3 is unique, so the result -- triangles, canonical numbering,
 * tables -- is identical to femi_mesh_build on the union (unknowns keep their indices,
 * masks are re-ranked). prev is not modified.
 *   new_mask_px[b]: HOST array of distinct pixels that are not vertices of prev, any order.
 *   out: receives a new handle (free with femi_mesh_free).
 * Errors: FEMI_E_ARG (NULL, b < 0), FEMI_E_SIZE (out of range, duplicate, already a vertex),
 * FEMI_E_OOM. */
femi_status femi_mesh_insert(femi_mesh prev, const int32_t* new_mask_px, int64_t b, femi_mesh* out);
femi_status femi_mesh_info_get(femi_mesh mesh, femi_mesh_info* info);
/* Canonical arrays to HOST buffers (any pointer may be NULL to skip it):
 *   vert_px[n_vert], tri_vert[3*n_tri] (canonical vertex indices),
 *   uu_rowptr[n_unknown+1], uu_col[nnz_uu] (unknown indices, ascending, diagonal included),
 *   uk_rowptr[n_unknown+1], uk_col[nnz_uk] (mask indices, ascending). */
femi_status femi_mesh_export(femi_mesh mesh, int32_t* vert_px, int32_t* tri_vert,
                             int32_t* uu_rowptr, int32_t* uu_col,
                             int32_t* uk_rowptr, int32_t* uk_col);
/* Host seconds spent in the last femi_mesh_build of this handle (triangulation, canonical
 * ordering, tables) and the host threads it used. */
femi_status femi_mesh_timing(femi_mesh mesh, double* seconds, int32_t* threads);
void femi_mesh_free(femi_mesh mesh);

/* ---------------------------------------------------------------------------------
 * S1 assemble (DEVICE). PAPER.md:L229-237 linear FEM: for each triangle (i,j,k) the entry
 * A_ij receives -1/2 cot(angle at k); the diagonal makes every row of the full matrix
 * sum to zero (natural Neumann border, Eq. (3)); Dirichlet elimination of
 * the mask vertices (Eq. (2)) splits the unknown rows into A_uu and A_uk (reading A6 fixes
 * the rounding). Also builds the pixel-ownership flags (reading A7) and the Jacobi scaling
 * used by the solver. Uploads the mesh tables and enqueues the assembly kernels on
 * `stream`; returns after enqueueing (the handle is usable by later calls on any stream
 * ordered after it).
 * Errors: FEMI_E_ARG, FEMI_E_CUDA, FEMI_E_OOM.
 * ------------------------------------------------------------------------------- */
femi_status femi_assemble(femi_mesh mesh, femi_stream stream, femi_system* out);
femi_status femi_system_info_get(femi_system sys, femi_mesh_info* info);
/* Unscaled CSR values (pattern of femi_mesh_export) to HOST buffers uu_val[nnz_uu],
 * uk_val[nnz_uk]; synchronises `stream`. */
femi_status femi_system_export(femi_system sys, double* uu_val, double* uk_val, femi_stream stream);
void femi_system_free(femi_system sys);

/* ---------------------------------------------------------------------------------
 * S2 inpaint_solve_batched (DEVICE). PAPER.md:L236-239: A_uu is SPD given >= 1 mask
 * pixel; "we can use the conjugate gradient method". Solves A_uu x = -A_uk g for B
 * right-hand sides with Jacobi-preconditioned CG (preconditioning changes iterates, not
 * the solution). Stops when the relative residual ||b - A x||_2 / ||b||_2 <= rtol, the
 * residual being confirmed with a fresh SpMV at exit (reading A11).
 *   sys[B]: system handles (distinct meshes -> block-diagonal batch; a repeated handle
 *           shares its matrix).
 *   g[B]: HOST array of DEVICE pointers, g[b] has n_mask values of sys[b].
 *   u_vert[B]: HOST array of DEVICE pointers, u_vert[b] has n_vert values: on return the
 *           unknown entries hold x and the mask entries hold g exactly. With x0 == 2 the
 *           unknown entries are read as the initial guess.
 *   opts: rtol (> 0), max_iter (> 0), precond (must be 1: Jacobi, folded into the matrix at
 *         assembly; plain CG (0) is not offered -- it reaches the same solution in ~6x the
 *         iterations, reading A11 -- and is rejected with FEMI_E_ARG), x0 (0 zeros, 1
 *         midrange(g) = (min g + max g)/2 (reading A11), 2 caller-provided, 3 mask-neighbour
 *         fill: each unknown starts at the value of its most strongly coupled mask neighbour,
 *         unknowns without one at their first filled unknown neighbour's (two hops), the rest
 *         at midrange(g) -- same solution, fewer iterations (reading A11b); systems below
 *         8192 unknowns use midrange instead (the fill's extra launches cost more there); with
 *         a given b (tonal adjoint solves) modes 1 and 3 start from 0), check_every (reserved, must be 0:
 *         convergence is tested on the device every iteration).
 *   iters[B], relres[B]: HOST outputs (iteration count, final true relative residual).
 * Special cases: ||b|| == 0 -> x = 0, 0 iterations; n_unknown == 0 -> no-op; an initial
 * guess that already satisfies rtol exits with 0 iterations and is returned unchanged.
 * Synchronises `stream`. Errors: FEMI_E_ARG, FEMI_E_NOT_CONVERGED (outputs written),
 * FEMI_E_NONFINITE, FEMI_E_NEG_CURVATURE, FEMI_E_CUDA, FEMI_E_OOM.
 * ------------------------------------------------------------------------------- */
typedef struct {
    double rtol;
    int32_t max_iter;
    int32_t precond;
    int32_t x0;
    int32_t check_every;
} femi_cg_opts;

femi_status femi_inpaint_solve_batched(int32_t B, const femi_system* sys, const double* const* g,
                                       double* const* u_vert, const femi_cg_opts* opts,
                                       int32_t* iters, double* relres, femi_stream stream);

/* Which solver the last femi_inpaint_solve_batched (or inner solve) on `sys` ran: a
 * diagnostic for tests and benchmarks; it does not change results beyond rounding order.
 *   FEMI_PATH_RESIDENT     whole CG loop on chip (one thread-block cluster per system)
 *   FEMI_PATH_PERSISTENT   one persistent kernel with global vectors
 *   FEMI_PATH_GRAPH_SELL   CUDA-graph WHILE loop, sliced-ELL SpMV
 *   FEMI_PATH_GRAPH_TMA    CUDA-graph WHILE loop, TMA-streamed jagged-diagonal SpMV
 *   FEMI_PATH_GRAPH_MULTI  shared-matrix multi-right-hand-side graph loop
 * Errors: FEMI_E_ARG (NULL). */
enum { FEMI_PATH_NONE = 0, FEMI_PATH_RESIDENT = 1, FEMI_PATH_PERSISTENT = 2, FEMI_PATH_GRAPH_SELL = 3,
       FEMI_PATH_GRAPH_TMA = 4, FEMI_PATH_GRAPH_MULTI = 5 };
femi_status femi_system_solver_path(femi_system sys, int32_t* path);

/* ---------------------------------------------------------------------------------
 * S3+S4 rasterise_error (DEVICE). PAPER.md:L239-241 "the solution is linearly
 * interpolated within each triangle"; "error map e_i = (u_i - f_i)^2 ...
 * the total L2 error in each triangle". Each pixel belongs to the lowest-index closed
 * triangle containing it (reading A7). A vertex pixel takes its vertex value exactly;
 * otherwise u = u_a + l_b (u_b - u_a) + l_c (u_c - u_a) with exact-integer barycentric
 * numerators (S3).
 *   u_vert[n_vert], f[W*H]: DEVICE inputs.
 *   u_px[W*H], e_px[W*H]: DEVICE outputs, nullable.
 *   tri_err[n_tri]: DEVICE output, nullable: sum of e over the triangle's pixels.
 *   tri_best_px[n_tri]: DEVICE output, nullable: owned non-vertex pixel with the largest
 *           e (ties: lowest pix), -1 if none (reading A8).
 *   sse: DEVICE scalar output (sum of e over all pixels; MSE = sse / (W*H)).
 * Enqueues only (no synchronisation). Errors: FEMI_E_ARG, FEMI_E_CUDA.
 * The _batched form takes B systems and HOST arrays of DEVICE pointers (entries of the
 * optional outputs may be NULL); sse[b] are separate device scalars.
 * ------------------------------------------------------------------------------- */
femi_status femi_rasterise_error(femi_system sys, const double* u_vert, const double* f,
                                 double* u_px, double* e_px, double* tri_err, int32_t* tri_best_px,
                                 double* sse, femi_stream stream);
femi_status femi_rasterise_error_batched(int32_t B, const femi_system* sys, const double* const* u_vert,
                                         const double* const* f, double* const* u_px, double* const* e_px,
                                         double* const* tri_err, int32_t* const* tri_best_px,
                                         double* const* sse, femi_stream stream);

/* ---------------------------------------------------------------------------------
 * S5 densify_step (DEVICE + host result). PAPER.md:L262-268: "We insert a single mask
 * pixel in each triangle, in descending order of the L2 error. The position of the mask
 * pixel within a triangle is chosen to be at the empty location with the largest
 * pointwise error." Rasterises u_vert against f, orders triangles by (tri_err desc, index
 * asc), skips triangles with zero error or no empty pixel, takes the first b, and fills
 * any shortfall with the globally largest-error empty pixels (ties: lowest pix) (readings
 * A8-A10).
 *   f[W*H], u_vert[n_vert]: DEVICE inputs; b >= 0.
 *   new_mask_px[b]: HOST output, ascending pix; *n_added = number written (== b unless
 *           fewer than b empty pixels exist).
 * Synchronises `stream`. Errors: FEMI_E_ARG, FEMI_E_CUDA, FEMI_E_OOM.
 * ------------------------------------------------------------------------------- */
femi_status femi_densify_step(femi_system sys, const double* f, const double* u_vert, int64_t b,
                              int32_t* new_mask_px, int64_t* n_added, femi_stream stream);

/* ---------------------------------------------------------------------------------
 * Colour (C channels on one mesh). PAPER.md:L521-524 "Extending the
 * method to colour images is straightforward": every channel is inpainted on the same mask
 * and mesh (femi_inpaint_solve_batched with the system repeated C times solves all channels
 * with one shared-matrix multi-right-hand-side CG); the error map is the channel sum
 * e = sum_c (u_c - f_c)^2 (SPEC.md:L74, L83 convention), accumulated in channel order.
 *   C in 1..4; u_vert[C], f[C]: HOST arrays of DEVICE pointers (f may be NULL: raster only);
 *   u_px: NULL or HOST array of C DEVICE pointers (entries nullable); e_px, tri_err,
 *   tri_best_px, sse: as femi_rasterise_error, for the channel-summed error.
 * rasterise_error_channels enqueues only; densify_step_channels selects from the summed
 * error exactly as femi_densify_step and synchronises `stream`.
 * Errors: FEMI_E_ARG, FEMI_E_CUDA, FEMI_E_OOM.
 * ------------------------------------------------------------------------------- */
femi_status femi_rasterise_error_channels(femi_system sys, int32_t C, const double* const* u_vert,
                                          const double* const* f, double* const* u_px, double* e_px,
                                          double* tri_err, int32_t* tri_best_px, double* sse,
                                          femi_stream stream);
femi_status femi_densify_step_channels(femi_system sys, int32_t C, const double* const* f,
                                       const double* const* u_vert, int64_t b, int32_t* new_mask_px,
                                       int64_t* n_added, femi_stream stream);

/* ---------------------------------------------------------------------------------
 * S6 tonal_optimise (DEVICE + host report). PAPER.md:L280-316, Eqs. (4)-(5):
 * g* = argmin ||B g - f||^2 solved as B^T B g = B^T f by CG on the normal equations in
 * CGLS form ("nested conjugate gradient solver"), B g = P_k g + P_u A_uu^-1 (-A_uk g)
 * applied matrix-free: each outer iteration runs one forward and one adjoint inner
 * inpainting solve. Starts from g (in), stops when ||B^T(f - B g)|| / ||B^T f|| < outer_rtol
 * or after outer_max iterations; the reported gradient and MSE are recomputed with fresh
 * solves at exit (reading A13).
 *   f[W*H]: DEVICE; g[n_mask]: DEVICE, in = initial values (e.g. f at the mask), out = g*.
 *   report: HOST output. Synchronises `stream`.
 * Errors: FEMI_E_ARG, FEMI_E_NOT_CONVERGED (g written), FEMI_E_NONFINITE, FEMI_E_CUDA,
 * FEMI_E_OOM.
 * ------------------------------------------------------------------------------- */
/* ---------------------------------------------------------------------------------
 * The operator B of the tonal problem and its adjoint (DEVICE; SPEC.md:L339-351 apply /
 * apply_adjoint). PAPER.md:L281-311, Eq. (4): u = B g is the rasterised inpainting from the
 * mask values g, B g = P_k g + P_u A_uu^-1 (-A_uk g); its adjoint is
 * B^T r = P_k^T r - A_uk^T A_uu^-1 (P_u^T r), where P^T r is the adjoint of the raster
 * (each pixel's r spread onto the vertices of its owner triangle with its barycentric
 * weights, reading A7). Each call runs one inner solve with `opts` (x0 = midrange for B,
 * zero for B^T).
 *   femi_apply_B:  g[n_mask] DEVICE in, u_px[W*H] DEVICE out.
 *   femi_apply_BT: r[W*H] DEVICE in, s[n_mask] DEVICE out.
 * Synchronise `stream` (the inner solve reports its status). Errors: FEMI_E_ARG,
 * FEMI_E_NOT_CONVERGED (output written), FEMI_E_NONFINITE, FEMI_E_CUDA, FEMI_E_OOM.
 * ------------------------------------------------------------------------------- */
femi_status femi_apply_B(femi_system sys, const double* g, double* u_px, const femi_cg_opts* opts,
                         femi_stream stream);
femi_status femi_apply_BT(femi_system sys, const double* r, double* s, const femi_cg_opts* opts,
                          femi_stream stream);

typedef struct {
    double outer_rtol;
    int32_t outer_max;
    femi_cg_opts inner;
    int32_t warm_start; /* reserved, must be 0 in this version */
} femi_tonal_opts;

typedef struct {
    int32_t outer_iters;
    int32_t inner_solves;
    int64_t inner_iters;
    double rel_grad;           /* recomputed at exit with fresh solves */
    double rel_grad_recursive; /* the CGLS recursion's value at exit    */
    double mse_before, mse_after;
} femi_tonal_report;

femi_status femi_tonal_optimise(femi_system sys, const double* f, double* g, const femi_tonal_opts* opts,
                                femi_tonal_report* report, femi_stream stream);

/* Colour tonal optimisation ("Extending the method to
 * colour images is straightforward", reading R4): C channels on one mesh are C independent
 * least-squares problems (B acts on each channel; the colour error is the channel sum), each
 * solved exactly as femi_tonal_optimise. They run in lockstep: every inner solve is one batched
 * shared-matrix solve of the active channels, and a converged channel leaves the batch.
 *   C in 1..4; f[C], g[C]: HOST arrays of DEVICE pointers (f_c: W*H; g_c: n_mask, in/out).
 *   reports[C]: HOST, one report per channel. Synchronises `stream`.
 * Errors: as femi_tonal_optimise. */
femi_status femi_tonal_optimise_channels(femi_system sys, int32_t C, const double* const* f, double* const* g,
                                         const femi_tonal_opts* opts, femi_tonal_report* reports, femi_stream stream);

/* ---------------------------------------------------------------------------------
 * L1 tonal optimisation (DEVICE + host report). PAPER.md:L524-526:
 * "we have ... optimised the L1 error instead of the L2 one"; the paper does not give the
 * method. Reading R3: iteratively reweighted least squares -- `irls`
 * reweightings, each setting w_i = 1 / max(|f_i - (B g)_i|, eps) and minimising
 * || W^1/2 (B g - f) ||^2 by the weighted nested CGLS of femi_tonal_optimise, warm-started
 * from the current g (opts as there: outer_rtol bounds the weighted relative gradient).
 *   f[W*H], g[n_mask]: as femi_tonal_optimise; irls >= 0; eps > 0 (0-255 scale; 1 is the
 *   SPEC default).
 *   report: HOST; l1_before / l1_after = mean |f - B g| at entry / exit.
 * Synchronises `stream`. Errors: as femi_tonal_optimise.
 * ------------------------------------------------------------------------------- */
typedef struct {
    int32_t irls_steps;
    int32_t outer_iters;  /* summed over the reweightings */
    int32_t inner_solves;
    int32_t pad;
    int64_t inner_iters;
    double l1_before, l1_after;
    double mse_before, mse_after;
} femi_tonal_l1_report;

femi_status femi_tonal_optimise_l1(femi_system sys, const double* f, double* g, const femi_tonal_opts* opts,
                                   int32_t irls, double eps, femi_tonal_l1_report* report, femi_stream stream);

/* ---------------------------------------------------------------------------------
 * Row-band multi-GPU solve of ONE image ("very large
 * images", L498-502 memory linear in the image size; the iteration is PAPER.md:L236-239's CG).
 * Canonical unknowns are in ascending pixel order, so rank r of R owns the unknowns
 * [row0, row1) = [n_u r / R, n_u (r+1) / R): a band of image rows, its rows of A_uu / A_uk
 * assembled on its own device (reading A6 arithmetic). The band's rows reference HALO unknowns
 * owned by other ranks (ascending canonical id, grouped by owner = peer); by the symmetry of
 * A_uu, rank r's SEND list to peer q is r's rows with a column in q's band, ascending -- the same
 * sequence as q's halo slots owned by r. Jacobi-PCG in single-reduction form on the unscaled
 * A_uu, x^0 = midrange(g) (reading A11): per iteration ONE halo exchange and ONE all-reduce of
 * four doubles. The caller sequences
 *     begin -> [all-reduce dots] -> pack(0) -> [exchange] -> spmv(0) -> [all-reduce dots] ->
 *     { update -> pack(0) -> [exchange] -> spmv(0) -> [all-reduce dots] }*  (status: done?)
 *     -> pack(1) -> [exchange] -> spmv(1) -> [all-reduce dots] -> status (true residual)
 * where [exchange] copies, for every peer p, send[send_off[p]..send_off[p+1]) of this rank to
 * the peer and the peer's send segment for this rank into halo[recv_off[p]..recv_off[p+1]),
 * and [all-reduce dots] sums the four doubles of `dots` over all ranks (NCCL, or a loopback
 * over bands of one process). All arithmetic is in the library's kernels.
 * ------------------------------------------------------------------------------- */
typedef struct femi_band_s* femi_band;
typedef struct {
    int32_t nranks, rank;
    int64_t n_unknown;   /* global unknowns */
    int64_t row0, row1;  /* owned canonical unknowns [row0, row1) */
    int64_t n_halo;      /* halo slots (unknowns of other bands the band's rows reference) */
    int64_t n_send;      /* send slots over all peers */
    int64_t nnz_uu, nnz_uk;  /* entries of the band's rows */
    int32_t n_peers, pad;
} femi_band_info;

/* HOST only (no device): the band plan of `rank` of `nranks`. Errors: FEMI_E_ARG. */
femi_status femi_band_plan(femi_mesh mesh, int32_t nranks, int32_t rank, femi_band_info* info);
/* HOST only: the plan's arrays (each NULL-able; sizes from femi_band_plan): peer[n_peers];
 * recv_off[n_peers+1] (halo slots per peer); send_off[n_peers+1]; halo_id[n_halo] (canonical
 * unknown ids); send_row[n_send] (local rows, i.e. canonical id - row0); rowptr[nloc+1] and
 * col[nnz_uu] of the band's A_uu rows in canonical entry order, columns local: c < nloc is the
 * own row row0 + c, c >= nloc is halo slot c - nloc. */
femi_status femi_band_plan_export(femi_mesh mesh, int32_t nranks, int32_t rank, int32_t* peer, int64_t* recv_off,
                                  int64_t* send_off, int64_t* halo_id, int32_t* send_row, int32_t* rowptr,
                                  int32_t* col);
/* DEVICE: the band object on the current device (plan, band matrix assembled, vectors).
 * Synchronises `stream`. Errors: FEMI_E_ARG, FEMI_E_CUDA, FEMI_E_OOM. */
femi_status femi_band_create(femi_mesh mesh, int32_t nranks, int32_t rank, femi_stream stream, femi_band* out);
femi_status femi_band_info_get(femi_band band, femi_band_info* info);
/* Caller-owned DEVICE communication buffers (they must outlive the band's use): halo[n_halo]
 * (written by the exchange), send[n_send] (written by pack), dots[4] (written by begin / spmv,
 * all-reduced in place by the caller). */
femi_status femi_band_set_buffers(femi_band band, double* halo, double* send, double* dots);
/* DEVICE, enqueued: x^0, b = -A_uk g and r^0 of the band's rows; dots = (0, 0, 0, ||b_band||^2).
 * g: DEVICE, all n_mask mask values (every rank holds g). rtol > 0: ||b - A x|| <= rtol ||b||. */
femi_status femi_band_begin(femi_band band, const double* g, double rtol, femi_stream stream);
/* DEVICE, enqueued: send = which ? x : u at the send rows. */
femi_status femi_band_pack(femi_band band, int32_t which, femi_stream stream);
/* DEVICE, enqueued (halo filled): which 0: w = A u, dots = (r.u, w.u, r.r, 0) of the band;
 * which 1: r = b - A x (true residual, unscaled rows), dots = (0, 0, ||r_band||^2, 0). */
femi_status femi_band_spmv(femi_band band, int32_t which, femi_stream stream);
/* DEVICE, enqueued (dots all-reduced): one CG update, or none once ||r||^2 <= rtol^2 ||b||^2
 * (the all-reduced ||b||^2 of begin is captured by the first spmv after it). */
femi_status femi_band_update(femi_band band, femi_stream stream);
/* After a true-residual spmv(1) that missed rtol: restart the recurrence from r = b - A x.
 * Synchronises `stream`. */
femi_status femi_band_restart(femi_band band, femi_stream stream);
/* HOST outputs, synchronises `stream`: converged flag, CG iterations so far, dots4 = the first
 * three doubles of the dots buffer and the all-reduced ||b||^2 (captured by the first spmv). */
femi_status femi_band_status(femi_band band, femi_stream stream, int32_t* done, int32_t* iters, double* dots4);
/* DEVICE, enqueued: the band's solution x (unknowns row0..row1-1, canonical) into u_local. */
femi_status femi_band_result(femi_band band, double* u_local, femi_stream stream);
void femi_band_free(femi_band band);

/* DEVICE: the raster / error tables of rank `rank`'s share of the triangles -- the canonical range
 * [t0, t1) = [T r / R, T (r+1) / R) -- over the image rows [y0, y0 + rows) its triangles touch
 * (PAPER.md:L239-241, L262-265). Pixel ownership (reading A7) is per triangle, so the shares
 * partition the pixels exactly as the whole mesh does. The result is a RASTER-ONLY femi_system:
 * femi_rasterise_error(_batched / _channels) take it with a GLOBAL u_vert (n_vert, canonical; the
 * triangles keep their global vertex ids) and band-local images f, u_px, e_px of rows x W
 * starting at row y0 (each rank writes only the pixels its triangles own); tri_err / best are
 * per band triangle (t - t0), best as a band-local pixel index (global = best + y0 W); sse is
 * the band's share (all-reduce for the image's). Solve, densify and tonal calls reject it
 * (FEMI_E_ARG). info (HOST, nullable) = {t0, t1, y0, rows}. Synchronises `stream`. */
typedef struct {
    int64_t t0, t1, y0, rows;
} femi_band_raster_info;
femi_status femi_band_raster_system(femi_mesh mesh, int32_t nranks, int32_t rank, femi_stream stream,
                                    femi_system* out, femi_band_raster_info* info);

#ifdef __cplusplus
}
#endif
#endif /* FEMI_H */
