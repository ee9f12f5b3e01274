// device.cuh -- device-side types and helpers of libfemi (sm_100a). Internal.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "femi_internal.h"

namespace femi {

// One triangle as the rasteriser reads it: 32 bytes, one aligned load per lane group.
struct __align__(16) TriRec {
    int32_t v[3];    // canonical vertex indices; v[0] has the smallest pix
    uint32_t flags;  // bit k: owns the edge opposite v[k]; bit 3+k: owns the vertex v[k] (reading A7)
    int16_t x[3], y[3];
    int32_t pad;
};
static_assert(sizeof(TriRec) == 32, "TriRec must be 32 bytes");

// Per-RHS solver state, device resident; scalars of one CG recursion.
struct CgState {
    double rr;     // r^.r^ (scaled residual)
    double rru;    // ||r||^2 unscaled (r = r^ / s)
    double pq;     // p.q
    double alpha, beta;
    double bn2;    // ||b||^2 unscaled
    double tol2;   // (rtol ||b||)^2
    double rtol;
    double res2;   // true ||b - A x||^2 at exit
    unsigned long long kmin, kmax;  // order-preserving keys of min(g), max(g)
    int32_t iters, active, status, max_iter;
    uint32_t cnt[4];  // last-block counters (one per reduction site)
    int32_t need_rho;  // graph mode: the next SpMV computes the unscaled residual norm (else it is skipped)
    int32_t x_pend;    // graph mode: the last k_gu deferred its x += alpha_pend p (k_finalize applies it)
    double alpha_pend; // graph mode: alpha of the previous k_gu
};


}  // namespace femi

// Device system handle (S1 output).
struct femi_system_s {
    int32_t W = 0, H = 0;
    int64_t n_u = 0, m = 0, nv = 0, T = 0, nnz_uu = 0, nnz_uk = 0;
    // mesh tables
    int32_t* vpix = nullptr;
    femi::TriRec* tri = nullptr;
    int32_t* vt_ptr = nullptr;
    int32_t* vt_idx = nullptr;
    int32_t* uu_rowptr = nullptr;
    int32_t* uu_col = nullptr;
    int32_t* uu_opp = nullptr;
    double* uu_val = nullptr;
    int32_t* uk_rowptr = nullptr;
    int32_t* uk_col = nullptr;
    int32_t* uk_opp = nullptr;
    double* uk_val = nullptr;
    int32_t* ku_rowptr = nullptr;
    int32_t* ku_src = nullptr;
    int32_t* ku_row = nullptr;
    // scaled (Jacobi) solver matrix: off-diagonal part only, unit diagonal implied
    int32_t* o_rowptr = nullptr;
    int32_t* o_col = nullptr;
    double* o_val = nullptr;
    double* s = nullptr;
    // Sliced ELL (SELL-32-sigma) copy of the scaled off-diagonal matrix for the solver:
    // windows of kSellSigma rows, rows sorted by length inside a window, slices of 32 rows
    // stored column-major (entry k of lane l of slice s at sell_base[s] + 32k + l).
    int32_t nwin = 0, nslices = 0;
    int32_t* win_slice = nullptr;  // nwin+1: first slice of each window
    int32_t* sell_perm = nullptr;  // 32*nslices: natural row of each slice lane, -1 = padding
    int32_t* sell_len = nullptr;   // nslices: entries per lane
    int32_t* sell_base = nullptr;  // nslices: first entry
    std::vector<int32_t> sell_base_h;  // host copy (sizes the on-chip resident solver)
    int32_t* sell_cbase = nullptr; // nslices: first row of the slice's window (int16 column base)
    double* sell_val = nullptr;
    int16_t* sell_c16 = nullptr;   // column - window_row0 (when the bandwidth allows)
    int32_t* sell_c32 = nullptr;   // absolute column otherwise
    int64_t sell_nnz = 0;
    int32_t* sell_src_tmp = nullptr;  // assembly-time map SELL entry -> o_val index
    // pixel ownership (reading A7), resolved once per mesh: triangle-major pixel lists
    // tp_ptr[T+1] / tp_pix[N] (ascending pix per triangle; pix | cls << 30, cls 1..3 = vertex pixel)
    int32_t* tp_ptr = nullptr;
    uint32_t* tp_pix = nullptr;
    // raster windows (raster.cu): per 16-triangle group g, windows tp_wptr[g] .. tp_wptr[g+1] of
    // <= 128 consecutive group-list entries spanning < 128 rows; a 32-byte record each
    int32_t* tp_wptr = nullptr;
    void* tp_win = nullptr;
    int64_t tp_nwin = 0;
    // Tiled jagged-diagonal copy of the scaled off-diagonal matrix for the TMA-streamed SpMV of
    // large systems (graph mode): tiles of kJdsRows internal rows; per tile a contiguous
    // entry block [jds_eb[t], jds_eb[t+1]) (a multiple of 8 entries), inside it slice w (32
    // rows) stores diagonal k = the k-th off-diagonal of every lane whose row has > k of them,
    // lanes ascending; columns as int16 offsets from the tile's first row (int32 for a tile
    // with a neighbour farther than 32767 rows, e.g. long image-border edges). jds_meta: per tile
    // jds_meta_bytes = uint8 row lengths[kJdsRows] | uint16 diagonal offsets[kJdsRows/32][jds_kmax]
    // (rows of a slice are in descending length order, so diagonal k of slice w is the lanes
    // 0 .. cnt_k-1 at doff[w][k] + lane).
    int32_t jds_ntile = 0, jds_maxe = 0, jds_kmax = 0, jds_meta_bytes = 0;
    size_t jds_block_bytes = 0;  // jds_val | jds_col | jds_meta are one allocation of this size
    int32_t* jds_eb = nullptr;
    int32_t* jds_cb = nullptr;   // per tile: byte offset of its columns (int32 if 4 bytes per entry)
    uint8_t* jds_meta = nullptr;
    double* jds_val = nullptr;
    uint8_t* jds_col = nullptr;
    int32_t* jds_src_tmp = nullptr;
    int64_t jds_nnz = 0;
    // A_uk and A_uu (unscaled) rows in the internal solver order (coalesced row access for the
    // right-hand side and the true residual); columns canonical; values gathered after assembly
    int32_t *ukI_rowptr = nullptr, *ukI_col = nullptr, *uuI_rowptr = nullptr, *uuI_col = nullptr;
    double *ukI_val = nullptr, *uuI_val = nullptr;
    int32_t *ukI_src_tmp = nullptr, *uuI_src_tmp = nullptr;
    int32_t* sell_inv = nullptr;      // n_u: internal solver row -> canonical unknown index
    double* s_int = nullptr;          // D^-1/2 in internal order
    double* q_int = nullptr;          // D^1/2 = 1/s_int (unscaled residual monitor: r = r^ q)
    // cached single-RHS scratch (x, r, q, b, p0, p1, state, items, chunks, partials)
    void* scratch = nullptr;
    void* scratch_m[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // multi-RHS graph caches (NR = 2..4)
    size_t scratch_bytes = 0;
    int32_t last_path = 0;  // FEMI_PATH_* of the last solve (femi_system_solver_path)
    void* rz_cache = nullptr;  // whole-solve resident kernel: halo codes / lists / send lists (pcg.cu)
    // calls on one system from several threads / streams are serialised (abi.cu SysGuard): the
    // host side by this mutex, the device side by an event recorded after each call's work
    std::mutex mu;
    cudaEvent_t ev = nullptr;
    cudaStream_t ev_stream = nullptr;
    // device memory of the system comes from the stream-ordered pool (cudaMallocAsync on the
    // assembling stream; the pool keeps freed memory, so a densification step's assemble and
    // the previous system's release cost no cudaMalloc / cudaFree device synchronisation)
    cudaStream_t ast = nullptr;
    bool raster_only = false;         // femi_band_raster_system: raster tables of a triangle range only
    std::vector<void*> allocs;        // pooled large arrays
    std::vector<void*> arena_chunks;  // pooled arena chunks (small arrays carved from them)
    char* arena_cur = nullptr;  // next free byte of the current arena chunk
    size_t arena_left = 0;
};

namespace femi {

// error helpers
femi_status cuda_fail(cudaError_t e, const char* what);
#define FEMI_CUDA(call)                                              \
    do {                                                             \
        cudaError_t _e = (call);                                     \
        if (_e != cudaSuccess) return femi::cuda_fail(_e, #call);   \
    } while (0)

// kernel-launch accounting (femi_kernel_launches)
void count_launches(int64_t n);

}  // namespace femi

// Device-side bounds checks, compiled in only with -DFEMI_DEVICE_CHECKS (the checked build
// libfemi_check.so; tests select it with FEMI_LIB). compute-sanitizer is closed on the GPU
// pool, so the checked build run under the GPU test suite stands in for memcheck on the
// index paths: a failed check counts in a per-translation-unit device counter and records its
// site (file id * 100000 + line); the kernel carries on. femi_device_check_failures() reads
// and resets the counters of every translation unit (FEMI_DCHECK_READER).
#ifdef FEMI_DEVICE_CHECKS
namespace {
__device__ unsigned long long g_dcheck[2];
}
#define FEMI_DCHECK(cond, file_id)                                                           \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            if (atomicAdd(&g_dcheck[0], 1ull) == 0ull) g_dcheck[1] = (file_id) * 100000ull + __LINE__; \
        }                                                                                    \
    } while (0)
#define FEMI_DCHECK_READER(name)                                                             \
    namespace femi {                                                                         \
    int64_t name(int64_t* site) {                                                            \
        unsigned long long h[2] = {0ull, 0ull};                                              \
        if (cudaMemcpyFromSymbol(h, g_dcheck, sizeof(h)) != cudaSuccess) return -1;          \
        const unsigned long long z[2] = {0ull, 0ull};                                        \
        cudaMemcpyToSymbol(g_dcheck, z, sizeof(z));                                          \
        if (h[0] && site && *site == 0) *site = (int64_t)h[1];                               \
        return (int64_t)h[0];                                                                \
    }                                                                                        \
    }
#else
#define FEMI_DCHECK(cond, file_id) \
    do {                           \
    } while (0)
#define FEMI_DCHECK_READER(name) \
    namespace femi {             \
    int64_t name(int64_t*) { return 0; } \
    }
#endif

namespace femi {
int64_t dcheck_abi(int64_t*);
int64_t dcheck_assemble(int64_t*);
int64_t dcheck_pcg(int64_t*);
int64_t dcheck_raster(int64_t*);
int64_t dcheck_select(int64_t*);
int64_t dcheck_tonal(int64_t*);
int64_t dcheck_band(int64_t*);

constexpr int kSellSigma = 64;   // rows per SELL window (length-sorting scope)
constexpr int kBand = 32;        // image band height (pixels) of the internal solver order
constexpr int kBandJds = 64;     // the same for graph-mode systems (JDS tiles, in-tile gathers from smem)
femi_status launch_sell_values(femi_system_s* S, const int32_t* d_src, cudaStream_t st);
constexpr int64_t kGraphNnz = 600000;  // nnz(A_uu) above which one system solves in graph mode
constexpr int kJdsRows = 512;          // rows per TMA tile of the jagged-diagonal layout
constexpr int kJdsMaxK = 24;           // longest row (off-diagonals) the JDS layout takes

// launchers (defined in the .cu files)
femi_status launch_tri_records(femi_system_s* S, const int32_t* d_tri, const uint32_t* d_flags, cudaStream_t st);
femi_status launch_assemble_values(femi_system_s* S, cudaStream_t st);
// S1 solver layouts on the device (assemble.cu): SELL slices + internal-order A_uu / A_uk rows
// from the internal order d_pi; sets S->sell_*, S->sell_base_h, S->ukI_*, S->uuI_*
femi_status sell_layout_device(femi_system_s* S, int64_t n, const int32_t* d_pi, cudaStream_t st,
                               const std::function<femi_status(void**, size_t)>& alloc_dev, int32_t* n_slices,
                               int64_t* n_entries, bool* fits16);
femi_status launch_raster(int B, femi_system_s* const* S, const double* const* u_vert, const double* const* f,
                          double* const* u_px, double* const* e_px, double* const* tri_err,
                          int32_t* const* best, double* const* sse, cudaStream_t st);
femi_status launch_raster_channels(femi_system_s* S, int nc, const double* const* u_vert, const double* const* f,
                                   double* const* u_px, double* e_px, double* tri_err, int32_t* best, double* sse,
                                   cudaStream_t st);  // colour: e = sum over channels
femi_status launch_adjoint_raster(femi_system_s* S, const double* r, double* tri_w, cudaStream_t st);
femi_status build_owner_tables(femi_system_s* S, cudaStream_t st);
void pcg_cache_free(femi_system_s* S);  // graph-mode workspace + instantiated graphs
// Device-side statistics of asynchronous solves (tonal loops): CG iterations and solves summed,
// the first non-OK status kept (a solve whose true residual misses rtol: FEMI_E_NOT_CONVERGED)
struct DevStats {
    unsigned long long iters;
    int32_t solves, status;
};
// ds == nullptr: the ABI behaviour (host outputs, host-side restart loop, synchronised stream).
// ds != nullptr: asynchronous -- nothing is read back, one restart round runs on the device gated
// by the true residual, and the outcome accumulates in *ds (stream-ordered).
femi_status pcg_solve(int B, femi_system_s* const* S, const double* const* g, const double* const* bin,
                      double* const* u_vert, const femi_cg_opts& o, int32_t* iters, double* relres,
                      cudaStream_t st, int64_t* total_iters, DevStats* ds = nullptr);
femi_status densify_select(femi_system_s* S, int nc, const double* const* f, const double* const* u_vert, int64_t b,
                           int32_t* new_px, int64_t* n_added, cudaStream_t st);
femi_status tonal_cgls(femi_system_s* S, const double* f, double* g, const femi_tonal_opts& o,
                       femi_tonal_report* rep, cudaStream_t st, const double* sw = nullptr);
// u_px = B g (mode 0) or s = B^T r (mode 1) with inner solves at opts (tonal.cu)
femi_status tonal_apply(femi_system_s* S, int mode, const double* in, double* out, const femi_cg_opts& o,
                        cudaStream_t st);
femi_status tonal_cgls_channels(femi_system_s* S, int C, const double* const* f, double* const* g,
                                const femi_tonal_opts& o, femi_tonal_report* rep, cudaStream_t st);
femi_status tonal_irls(femi_system_s* S, const double* f, double* g, const femi_tonal_opts& o, int irls, double eps,
                       femi_tonal_l1_report* rep, cudaStream_t st);

// device helpers
// release/acquire at gpu scope: the last-arriver pattern needs only these, not the
// sequentially consistent fence (__threadfence = MEMBAR.SC.GPU, several microseconds under load)
__device__ __forceinline__ unsigned atom_add_release_gpu(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum (fixed tree): every thread returns the total.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh /* >= NT/32 */) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) t += sh[w];
    return t;
}

}  // namespace femi
