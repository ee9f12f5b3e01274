// pcg.cu -- S2: batched Jacobi-preconditioned CG for A_uu x = -A_uk g.
//
// B200 design. The Jacobi preconditioner is folded into the matrix at assembly
// (A^ = D^-1/2 A D^-1/2, unit diagonal, only the off-diagonal part stored), so CG runs on
// A^ x^ = b^ (x = D^-1/2 x^, b^ = D^-1/2 b). One solve =
//   k_pro1         min/max of g, the fill's first hop, b = -A_uk g (or the given b), internal order
//   k_x0_fill2 x2  the fill's second hop (x0 mode 3, reading A11b)
//   k_pro2         x^0 and r0 = s (b - A x0) (unscaled rows)
//   k_cg           ONE persistent launch running the whole CG loop on device
//   k_finalize     x = D^-1/2 x^ scattered to canonical order (u_vert)
//   k_true_res     ||b - A x|| with the unscaled matrix (reading A11); a failed check
//                  relaunches k_cg from the current iterate
// k_cg runs the single-reduction form of CG (Chronopoulos-Gear). Per iteration
//   U: p = r + beta p ; s = w + beta s ; x += alpha p ; r -= alpha s      (own rows)
//   -- group barrier (r published) --
//   S: w = A^ r (gathers r) ; partial (r.r, w.r, ||D^1/2 r||^2)
//   -- group barrier fused with the reduction -- every CTA sums the partials in the same
//   fixed order, so alpha/beta/convergence are bit-identical in all CTAs (deterministic).
// The SpMV reads the matrix in sliced-ELL form (SELL-32-sigma): every warp load of values
// / int16 window-relative columns is one coalesced 32-lane access; two slices per warp
// keep two independent load chains in flight. Each batch item owns a group of CTAs and
// each CTA a contiguous range of rows; p and s (and x when it fits) stay in shared memory
// for the whole solve. Group barriers: __syncthreads (1 CTA), the hardware cluster
// barrier (a cluster of <= 16 CTAs: C1-C4), or a flag-array barrier over a cooperative
// grid (one huge system: C5).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "device.cuh"
#include "tma.cuh"

namespace femi {
namespace {

__device__ __forceinline__ unsigned long long dkey(double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

// All solver vectors (b, x, r, w, p, s) live in the INTERNAL row order (see abi.cu:
// 2-D blocked numbering, length-sorted inside kSellSigma windows); inv maps an internal
// row to its canonical unknown index for the input/output vectors (g, u_vert).
// Graph mode, lean tail: the CG recurrence scalars of the loop, double-buffered by iteration
// parity (k_gur of body slot k reads ls[k & 1] and writes ls[(k + 1) & 1], so no CTA reads a
// slot another CTA of the same launch writes). The final values go to the item's CgState.
struct LoopState {
    double alpha;  // alpha of the update this state's k_gur performed
    double rr;     // gamma = r^.r^ of that update's residual
    int32_t iters, active, started, need_rho;
    int32_t status;
};

struct RItem {
    const int32_t* inv;   // internal row -> canonical unknown
    const int32_t* len;   // per 32-row slice
    const int32_t* base;  // per slice: first SELL entry
    const double* val;
    const int16_t* c16;   // column - window base (internal numbering)
    const int32_t* c32;
    const double* s;     // D^-1/2 (internal order)
    const double* q;     // D^1/2 (internal order): unscaled residual r = r^ q (monitor)
    const int32_t* urp;  // unscaled A_uu (diagonal included), internal rows, canonical columns
    const int32_t* uci;
    const double* uav;
    const int32_t* krp;  // A_uk, internal rows, canonical (mask) columns
    const int32_t* kci;
    const double* kav;
    const double* g;    // mask values or NULL (b given)
    const double* bin;  // given b (canonical order) or NULL
    double* u_vert;
    double* b;  // unscaled right-hand side
    double* x;  // x^ (initial guess gathers; the iterate when it does not fit in smem)
    double* r;  // r^ (published every iteration)
    double* w;  // A^ r^
    double* p;  // used when the CTA's rows do not fit shared memory
    double* sv;
    const double* jval;   // graph mode: tiled jagged-diagonal matrix (device.cuh), TMA-streamed
    const uint8_t* jcol;
    const uint8_t* jmeta;
    const int32_t* jeb;
    const int32_t* jcb;
    int32_t ntile, jmaxe, jkmax, jmbytes;
    double dmin;         // min_i diag(A_uu)_i: ||r||^2 >= dmin ||r^||^2 (skips the monitor far from rtol)
    const int32_t* jpart;  // [gt_blocks + 1] first tile of each k_gt CTA
    double* part;  // [ncta][4] partial sums / barrier slots
    double* red;   // [reduction blocks] partials of the ordinary kernels
    CgState* st;
    LoopState* ls;  // graph mode (lean tail): ls[2]
    // whole-solve resident kernel (k_cgs): per SELL entry the 16-bit index into the CTA's
    // extended vector (own rows | halo), per CTA the halo (canonical-internal rows it reads from
    // peers, ascending) and the send list (src row | peer << 12 | peer's halo slot << 16), both at
    // the CTA's first entry offset; rzn[0..16) halo counts, rzn[16..32) send counts
    uint16_t* rzc;
    int32_t* rzh;
    int32_t* rzs;
    int32_t* rzn;
    int32_t rzhmax, rzpad;
    int32_t n, m, cta0, ncta, nwin, x0mode;
    double rtol;  // graph mode reads the options from the item (the graph is reused)
    int32_t max_iter, pad2;
};

// per-system tables of the whole-solve resident kernel for one cluster size (k_rz_halo / k_rz_send)
struct RzCache {
    int C = 0;
    void* block = nullptr;  // code | halo | send | counts
    uint16_t* code = nullptr;
    int32_t* halo = nullptr;
    int32_t* snd = nullptr;
    int32_t* cnt = nullptr;  // [32] (device)
    int32_t cnt_h[32] = {};  // host copy: halo counts [0, 16), send counts [16, 32)
    int32_t hmax = 0;
};

constexpr int RNT = 512;  // threads per CTA of the persistent solver (block/cluster modes)
constexpr int SIG = kSellSigma;
constexpr int KNT = 256;  // threads per CTA of the ordinary kernels
constexpr int KGRID = 296;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// FEMI_LOOP_PROF: per iteration, earliest CTA start / latest CTA end of k_gu and k_gt (globaltimer)
constexpr int kLoopProfMax = 4096;
__device__ int g_loop_prof;
__device__ int g_kbench;
__device__ int g_l2pol;  // L2 policy of the matrix stream: 0 evict_first, 1 evict_last, 2 evict_normal (FEMI_L2POL)
// the matrix stream's bulk copies: with an L2 cache hint, or none (g_l2pol 3: the kernel's
// persisting access-policy window decides)
__device__ __forceinline__ void mat_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    if (g_l2pol == 3)
        bulk_g2s(dst, src, bytes, bar);
    else
        bulk_g2s_hint(dst, src, bytes, bar, pol);
}
__device__ __forceinline__ uint64_t matrix_policy() {
    return g_l2pol == 1 ? policy_evict_last() : (g_l2pol == 2 ? policy_evict_normal() : policy_evict_first());
}  // FEMI_PCG_KBENCH: k_gur skips the advance and updates with alpha = beta = 0
__device__ int g_pdl_pre = 6;
__device__ int g_smem_gather = 1;  // k_gt: in-tile neighbours from the staged r slice (FEMI_SMEM_GATHER=0: all from L1/L2)  // k_gt: stages streamed before grid_dep_wait (FEMI_PDL_PRE, <= JNS)
__device__ unsigned long long g_loop_ts[4 * kLoopProfMax];
__device__ unsigned long long g_loop_ts2[4 * kLoopProfMax];
constexpr int kCtaProfIt = 60;  // FEMI_LOOP_PROF: per-CTA start / consumer end of this iteration's k_gt
__device__ unsigned long long g_cta_prof[2 * 1024];  // k_gt: max start, min/max consumer end
__device__ unsigned long long g_tail_ts[4 * kLoopProfMax];   // cg_tail stamps (see cg_tail)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void loop_stamp(int kern, int iter, unsigned long long t0) {
    if (iter < 0 || iter >= kLoopProfMax) return;
    atomicMin(&g_loop_ts[4 * iter + 2 * kern], t0);
    atomicMax(&g_loop_ts[4 * iter + 2 * kern + 1], gtime());
}

// ------------------------------------------------------------------ ordinary kernels
__global__ void k_reset(int B, CgState* st, double rtol, int max_iter) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    CgState s = {};
    s.rtol = rtol;
    s.max_iter = max_iter;
    s.kmin = ~0ull;
    s.kmax = 0ull;
    st[b] = s;
}

// x0 mode 3, the mask-neighbour fill (reading A11b): the initial guess of an unknown is the value
// of its most strongly coupled mask neighbour (the most negative A_uk entry of its row, ties ->
// lowest mask index); an unknown without one takes the value of its first filled unknown
// neighbour (ascending canonical column), over up to two hops; what is left takes midrange(g).
// k_pro1 takes the first hop, k_x0_fill2 (u_vert -> w, w -> u_vert) the second, k_pro2 the
// midrange leftovers. The guess is written to u_vert (canonical), then the solve proceeds as
// with a caller's x0 (mode 2): same solution (reading A11), ~15 % fewer iterations on the C5 recipe. A constant g
// fills every unknown with that constant exactly (A16 still holds).
__global__ void k_x0_fill2(const RItem* __restrict__ items, int to_w) {
    const RItem& it = items[blockIdx.y];
    if (it.x0mode != 3) return;
    const double* __restrict__ src = to_w ? it.u_vert : it.w;
    double* __restrict__ dst = to_w ? it.w : it.u_vert;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < it.n; i += gridDim.x * blockDim.x) {
        const int nat = it.inv[i];
        double v = src[nat];
        if (isnan(v))
            for (int e = it.urp[i]; e < it.urp[i + 1]; ++e) {
                const double c = src[it.uci[e]];
                if (!isnan(c)) {
                    v = c;
                    break;
                }
            }
        dst[nat] = v;
    }
}
// Graph-mode epilogue fusion: k_finalize + k_copy_g (the mask entries of u_vert are g exactly)
__global__ void k_finalize_g(const RItem* __restrict__ items) {
    const RItem& it = items[blockIdx.y];
    const CgState* S = it.st;
    const double x0v = (it.x0mode == 1) ? 0.5 * (dkey_inv(S->kmin) + dkey_inv(S->kmax)) : 0.0;
    const int nmax = max(it.n, it.g ? it.m : 0);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nmax; i += gridDim.x * blockDim.x) {
        if (it.g && i < it.m) it.u_vert[it.n + i] = it.g[i];
        if (i >= it.n) continue;
        const int nat = it.inv[i];
        if (S->iters == 0 && it.x0mode >= 2 && S->bn2 != 0.0) continue;  // the guess in u_vert stays
        double xi;
        if (S->bn2 == 0.0) {
            xi = 0.0;
        } else if (S->iters == 0) {
            xi = x0v;
        } else {
            double xh = it.x[i];
            if (S->x_pend) {
                xh = fma(S->alpha_pend, it.p[i], xh);
                it.x[i] = xh;
            }
            xi = it.s[i] * xh;
        }
        it.u_vert[nat] = xi;
    }
}

// asynchronous solves: does any item need the restart round (the recursion converged but the
// true residual misses rtol)? Same rule as the host loop of pcg_solve.
__global__ void k_restart_flag(int B, const RItem* __restrict__ items, int* gate) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    int again = 0;
    for (int b = 0; b < B; ++b) {
        const CgState* S = items[b].st;
        again |= items[b].n > 0 && S->status == FEMI_OK && S->iters > 0 && S->iters < S->max_iter && S->bn2 > 0.0 &&
                 !(S->res2 <= S->tol2);
    }
    *gate = again;
}
// the same for the graph path: sets the IF condition of the restart graph
__global__ void k_restart_cond(const RItem* __restrict__ items, cudaGraphConditionalHandle h) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const CgState* S = items[0].st;
    const int again = S->status == FEMI_OK && S->iters > 0 && S->iters < S->max_iter && S->bn2 > 0.0 &&
                      !(S->res2 <= S->tol2);
    cudaGraphSetConditional(h, again ? 1u : 0u);
}
__global__ void k_stats(int B, const RItem* __restrict__ items, DevStats* ds) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int b = 0; b < B; ++b) {
        const CgState* S = items[b].st;
        if (items[b].n == 0) continue;
        ds->iters += (unsigned long long)S->iters;
        ds->solves += 1;
        int st = S->status;
        if (st == FEMI_OK && S->bn2 > 0.0 && !(S->res2 <= S->tol2)) st = FEMI_E_NOT_CONVERGED;
        if (st != FEMI_OK && ds->status == FEMI_OK) ds->status = st;
    }
}

// Deterministic grid reduction helper: per-block partial, the last block sums in order.
template <int NQ>
__device__ __forceinline__ bool grid_partial(double (&v)[NQ], double* red, unsigned* cnt, double* shm) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = warp_sum_d(v[q]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NQ; ++q) shm[NQ * wid + q] = v[q];
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) {
        for (int q = 0; q < NQ; ++q) {
            double t = 0.0;
            for (int w = 0; w < KNT / 32; ++w) t += shm[NQ * w + q];
            red[NQ * blockIdx.x + q] = t;
        }
        __threadfence();
        last = atomicAdd(cnt, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    // all threads of the last block: strided partial sums, then the fixed block tree
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double t = 0.0;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += KNT) t += __ldcg(red + NQ * b + q);
        v[q] = warp_sum_d(t);
    }
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NQ; ++q) shm[NQ * wid + q] = v[q];
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q < NQ; ++q) {
            double t = 0.0;
            for (int w = 0; w < KNT / 32; ++w) t += shm[NQ * w + q];
            v[q] = t;
        }
        *cnt = 0;
    }
    return true;
}

// ---- fused prologue (every solve path): k_pro1 -> [k_x0_fill2 x 2] -> k_pro2 replaces
// k_minmax -> k_x0_fill1 -> k_rhs -> [fill2 x 2] -> k_x0_fill_end -> k_init_x -> k_zero_ps ->
// k_init_r: the A_uk rows are read once for the fill candidates and b, the A_uu rows once for
// x^0 and r^0 = s (b - A x0), the true-residual form with the unscaled matrix (reading A11).

// In-order walk of one CSR row, four entries per step: the column / value loads and the
// gathers of a step are independent (memory-level parallelism for the latency-bound walk),
// f(a, col, src[col]) is applied in entry order, so sums keep the sequential rounding.
template <class F>
__device__ __forceinline__ void row_walk4(int e0, int e1, const int* __restrict__ ci, const double* __restrict__ va,
                                          const double* __restrict__ src, F&& f) {
    for (int e = e0; e < e1; e += 4) {
        int c[4];
        double a[4], x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool ok = e + q < e1;
            c[q] = ok ? ci[e + q] : -1;
            a[q] = ok ? va[e + q] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = c[q] >= 0 ? src[c[q]] : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (e + q < e1) f(a[q], c[q], x[q]);
    }
}

// the same walk with the gathers through L2 (ld.global.cg): data another CTA of the launch wrote
template <class F>
__device__ __forceinline__ void row_walk4cg(int e0, int e1, const int* __restrict__ ci, const double* __restrict__ va,
                                            const double* src, F&& f) {
    for (int e = e0; e < e1; e += 4) {
        int c[4];
        double a[4], x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool ok = e + q < e1;
            c[q] = ok ? ci[e + q] : -1;
            a[q] = ok ? va[e + q] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = c[q] >= 0 ? __ldcg(src + c[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (e + q < e1) f(a[q], c[q], x[q]);
    }
}

// In-order walks of up to RP CSR rows at once (the rows of one lane, k_cgs): per step the column
// and value loads of every row, then their gathers, then f(j, a, col, src[col]) in entry order per
// row -- the rows' dependent load chains overlap instead of running one after another, and each
// row's sums keep the sequential rounding. CG: gathers through L2 (data other CTAs wrote).
template <int RP, bool CG, class F>
__device__ __forceinline__ void walk_rows(const bool (&ok)[RP], const int (&row)[RP], const int* __restrict__ rp,
                                          const int* __restrict__ ci, const double* __restrict__ va,
                                          const double* src, F&& f) {
    constexpr int W = RP <= 2 ? 4 : 2;
    int e[RP], e1[RP];
    int len = 0;
#pragma unroll
    for (int j = 0; j < RP; ++j) {
        e[j] = ok[j] ? rp[row[j]] : 0;
        e1[j] = ok[j] ? rp[row[j] + 1] : 0;
        len = max(len, e1[j] - e[j]);
    }
    for (int s = 0; s < len; s += W) {
        int c[RP][W];
        double a[RP][W], x[RP][W];
#pragma unroll
        for (int j = 0; j < RP; ++j)
#pragma unroll
            for (int q = 0; q < W; ++q) {
                const bool in = e[j] + s + q < e1[j];
                c[j][q] = in ? ci[e[j] + s + q] : -1;
                a[j][q] = in ? va[e[j] + s + q] : 0.0;
            }
#pragma unroll
        for (int j = 0; j < RP; ++j)
#pragma unroll
            for (int q = 0; q < W; ++q)
                x[j][q] = c[j][q] >= 0 ? (CG ? __ldcg(src + c[j][q]) : src[c[j][q]]) : 0.0;
#pragma unroll
        for (int j = 0; j < RP; ++j)
#pragma unroll
            for (int q = 0; q < W; ++q)
                if (c[j][q] >= 0) f(j, a[j][q], c[j][q], x[j][q]);
    }
}

// pass 1: min/max of g (x0 modes 1, 3), the fill's first hop (mode 3: the value of the most
// strongly coupled mask neighbour, the most negative A_uk entry, ties -> first), b = -A_uk g
// (ascending mask index, reading A6 order) or the given b, r^0 for modes 0 and 1 with a
// given b (x0 = 0: r0 = b), ||b||^2 -> state
__global__ void __launch_bounds__(KNT) k_pro1(const RItem* __restrict__ items, unsigned* cnt) {
    __shared__ double shm[4 * (KNT / 32)];
    __shared__ unsigned long long slo[KNT / 32], shi[KNT / 32];
    const RItem& it = items[blockIdx.y];
    const int mode = it.x0mode;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if ((mode == 1 || mode == 3) && it.g != nullptr) {
        unsigned long long lo = ~0ull, hi = 0ull;
        for (int k = blockIdx.x * KNT + threadIdx.x; k < it.m; k += gridDim.x * KNT) {
            const unsigned long long key = dkey(it.g[k]);
            lo = min(lo, key);
            hi = max(hi, key);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            slo[wid] = lo;
            shi[wid] = hi;
        }
        __syncthreads();
        if (wid == 0) {
            lo = lane < KNT / 32 ? slo[lane] : ~0ull;
            hi = lane < KNT / 32 ? shi[lane] : 0ull;
            for (int o = 16; o > 0; o >>= 1) {
                lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
                hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            }
            if (lane == 0 && hi != 0ull) {
                atomicMin(&it.st->kmin, lo);
                atomicMax(&it.st->kmax, hi);
            }
        }
    }
    double v[1] = {0.0};
    for (int i = blockIdx.x * KNT + threadIdx.x; i < it.n; i += gridDim.x * KNT) {
        double bi;
        if (it.bin) {
            bi = it.bin[it.inv[i]];
            if (mode < 2) it.r[i] = it.s[i] * bi;
        } else {
            double acc = 0.0, best = 0.0;
            double fv = __longlong_as_double(0x7ff8000000000000ll);  // NaN: not filled yet
            row_walk4(it.krp[i], it.krp[i + 1], it.kci, it.kav, it.g, [&](double a, int k, double gk) {
                FEMI_DCHECK(k >= 0 && k < it.m, 3);
                acc = fma(a, gk, acc);
                if (a < best) {
                    best = a;
                    fv = gk;
                }
            });
            bi = -acc;
            if (mode == 0) it.r[i] = it.s[i] * bi;
            if (mode == 3) it.u_vert[it.inv[i]] = fv;
        }
        it.b[i] = bi;
        v[0] += bi * bi;
    }
    if (grid_partial<1>(v, it.red, cnt + blockIdx.y, shm) && threadIdx.x == 0) {
        it.st->bn2 = v[0];
        it.st->tol2 = it.st->rtol * it.st->rtol * v[0];
    }
}

// pass 2 (after the fill's second hop): x^0 = x0 / s (mode 3: what the fill did not reach
// takes midrange(g)), p = s = 0, the lean-tail loop state, and r^0 = s r0:
//   mode 1 (x0 = c 1, no given b): r0 = -A_uk (g - c 1) (zero row sums: A_uu 1 = -A_uk 1);
//   modes 2, 3: r0 = b - A_uu x0 over the unscaled rows (neighbours' x0 read from u_vert,
//   with the same midrange substitution their own rows make).
__global__ void __launch_bounds__(KNT) k_pro2(const RItem* __restrict__ items) {
    const RItem& it = items[blockIdx.y];
    const CgState* S = it.st;
    const int mode = it.x0mode;
    if (it.ls && blockIdx.x == 0 && threadIdx.x == 0) {
        LoopState l = {};
        l.iters = S->iters;
        l.active = 1;
        it.ls[0] = l;
    }
    const double x0v = (mode == 1 || mode == 3) ? 0.5 * (dkey_inv(S->kmin) + dkey_inv(S->kmax)) : 0.0;
    for (int i = blockIdx.x * KNT + threadIdx.x; i < it.n; i += gridDim.x * KNT) {
        double x0 = x0v;
        if (mode >= 2) {
            const int nat = it.inv[i];
            x0 = it.u_vert[nat];
            if (mode == 3 && isnan(x0)) {
                x0 = x0v;
                it.u_vert[nat] = x0;
            }
        }
        const double si = it.s[i];
        it.x[i] = x0 / si;
        if (it.p) it.p[i] = 0.0;
        if (it.sv) it.sv[i] = 0.0;
        if (mode == 1 && !it.bin) {
            double accr = 0.0;
            row_walk4(it.krp[i], it.krp[i + 1], it.kci, it.kav, it.g,
                      [&](double a, int, double gk) { accr = fma(a, gk - x0v, accr); });
            it.r[i] = si * -accr;
        } else if (mode >= 2) {
            double ax = 0.0;
            row_walk4(it.urp[i], it.urp[i + 1], it.uci, it.uav, it.u_vert, [&](double a, int c, double u) {
                FEMI_DCHECK(c >= 0 && c < it.n, 3);
                if (mode == 3 && isnan(u)) u = x0v;
                ax = fma(a, u, ax);
            });
            it.r[i] = si * (it.b[i] - ax);
        }
    }
}

// x = D^-1/2 x^ into u_vert (canonical), or x0 untouched after a 0-iteration exit, 0 if b == 0
__global__ void k_finalize(const RItem* __restrict__ items, const int* gate = nullptr) {
    if (gate && !*gate) return;  // asynchronous restart round not needed
    const RItem& it = items[blockIdx.y];
    const CgState* S = it.st;
    const double x0v = (it.x0mode == 1) ? 0.5 * (dkey_inv(S->kmin) + dkey_inv(S->kmax)) : 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < it.n; i += gridDim.x * blockDim.x) {
        const int nat = it.inv[i];
        if (S->iters == 0 && it.x0mode >= 2 && S->bn2 != 0.0) continue;  // the guess in u_vert stays
        double xi;
        if (S->bn2 == 0.0) {
            xi = 0.0;
        } else if (S->iters == 0) {
            xi = x0v;
        } else {
            double xh = it.x[i];
            if (S->x_pend) {  // the deferred half of k_gu's paired x update (graph mode)
                xh = fma(S->alpha_pend, it.p[i], xh);
                it.x[i] = xh;
            }
            xi = it.s[i] * xh;
        }
        it.u_vert[nat] = xi;
    }
}

// true residual with the unscaled matrix (canonical rows); keeps s_i * r_true in r
__global__ void __launch_bounds__(KNT) k_true_res(const RItem* __restrict__ items, unsigned* cnt,
                                                 const int* gate = nullptr) {
    if (gate && !*gate) return;
    __shared__ double shm[4 * (KNT / 32)];
    const RItem& it = items[blockIdx.y];
    double v[1] = {0.0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < it.n; i += gridDim.x * blockDim.x) {
        double ax = 0.0;
        row_walk4(it.urp[i], it.urp[i + 1], it.uci, it.uav, it.u_vert, [&](double a, int c, double u) {
            FEMI_DCHECK(c >= 0 && c < it.n, 3);
            ax = fma(a, u, ax);
        });
        const double ri = it.b[i] - ax;
        it.r[i] = it.s[i] * ri;
        v[0] += ri * ri;
    }
    if (grid_partial<1>(v, it.red, cnt + blockIdx.y, shm) && threadIdx.x == 0) {
        it.st->res2 = v[0];
        it.st->x_pend = 0;  // k_finalize has applied it
    }
}

__global__ void k_copy_g(const RItem* __restrict__ items) {
    const RItem& it = items[blockIdx.y];
    if (!it.g) return;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < it.m; k += gridDim.x * blockDim.x)
        it.u_vert[it.n + k] = it.g[k];
}

// ------------------------------------------------------------------ group barriers
// MODE 2 (cooperative grid): flag-array barrier. Every CTA owns a 32-byte slot
// {partial x, y, z, epoch} in it.part. Arrival = (optional partials) + gpu-scope fence +
// epoch store into the CTA's own slot -- no serialized atomics on a shared counter.
// Waiting = each thread polls one slot until its epoch reaches the barrier's epoch, then
// an acquire fence. Data published at epoch e is overwritten only at epoch e+2
// (reductions and plain barriers alternate), i.e. after every CTA has passed the plain
// barrier e+1 that follows its reads.
__device__ __forceinline__ void flag_arrive(const RItem& it, int rank, unsigned long long epoch, const double4* t) {
    __syncthreads();
    if (threadIdx.x == 0) {
        double* P = it.part + 4 * rank;
        if (t) {
            P[0] = t->x;
            P[1] = t->y;
            P[2] = t->z;
        }
        __threadfence();
        *(volatile unsigned long long*)(P + 3) = epoch;
    }
}

__device__ __forceinline__ void flag_wait(const RItem& it, unsigned long long epoch) {
    for (int k = threadIdx.x; k < it.ncta; k += blockDim.x) {
        volatile unsigned long long* E = (volatile unsigned long long*)(it.part + 4 * k + 3);
        while (*E < epoch) {
        }
    }
    __threadfence();
    __syncthreads();
}

template <int MODE>
__device__ __forceinline__ void group_sync(const RItem& it, int rank, unsigned long long& epoch) {
    if constexpr (MODE == 0) {
        __syncthreads();
    } else if constexpr (MODE == 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
        ++epoch;
        flag_arrive(it, rank, epoch, nullptr);
        flag_wait(it, epoch);
    }
}

// optional phase timers (FEMI_PCG_TIMERS=1): rank-0 thread-0 %globaltimer deltas, ns
__device__ unsigned long long g_pcg_timers[16];
__device__ int g_pcg_timers_on;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// block sum of 3 values (fixed tree; result valid in every thread)
template <int NWARP>
__device__ __forceinline__ double4 block_sum3(double4 v, double* sh /* [NWARP][4] */) {
    v.x = warp_sum_d(v.x);
    v.y = warp_sum_d(v.y);
    v.z = warp_sum_d(v.z);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) {
        sh[4 * wid] = v.x;
        sh[4 * wid + 1] = v.y;
        sh[4 * wid + 2] = v.z;
    }
    __syncthreads();
    double4 t = make_double4(0.0, 0.0, 0.0, 0.0);
#pragma unroll
    for (int w = 0; w < NWARP; ++w) {
        t.x += sh[4 * w];
        t.y += sh[4 * w + 1];
        t.z += sh[4 * w + 2];
    }
    return t;
}

// publish this CTA's partials, barrier, and sum all partials of the group in a fixed order
template <int MODE, int NT>
__device__ __forceinline__ double4 group_reduce(const RItem& it, int rank, double4 loc, double* sh,
                                                unsigned long long& epoch) {
    double4 t = block_sum3<NT / 32>(loc, sh);
    if constexpr (MODE == 0) return t;
    if constexpr (MODE == 2) {
        ++epoch;
        flag_arrive(it, rank, epoch, &t);
        flag_wait(it, epoch);
    } else {
        if (threadIdx.x == 0) {
            double* P = it.part + 4 * rank;
            P[0] = t.x;
            P[1] = t.y;
            P[2] = t.z;
        }
        group_sync<MODE>(it, rank, epoch);
    }
    double4 a = make_double4(0.0, 0.0, 0.0, 0.0);
    for (int k = threadIdx.x; k < it.ncta; k += NT) {
        const double* P = it.part + 4 * k;
        a.x += __ldcg(P);
        a.y += __ldcg(P + 1);
        a.z += __ldcg(P + 2);
    }
    return block_sum3<NT / 32>(a, sh);
}

// w = r + A^_off r over the CTA's slices; partial (r.r, w.r, ||r/s||^2). Two slices per warp.
template <int NWARP>
__device__ __forceinline__ double4 spmv_w(const RItem& it, int S0, int S1, const int2* __restrict__ meta) {
    double4 loc = make_double4(0.0, 0.0, 0.0, 0.0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* __restrict__ val = it.val;
    const int16_t* __restrict__ c16 = it.c16;
    const int32_t* __restrict__ c32 = it.c32;
    const double* __restrict__ r = it.r;
    for (int sa = S0 + 2 * warp; sa < S1; sa += 2 * NWARP) {
        const bool hb = sa + 1 < S1;
        int row[2], len[2], base[2], cb[2];
        double xi[2], si[2], acc[2] = {0.0, 0.0};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int s = sa + h;
            const bool ok = h == 0 || hb;
            const int2 md = ok ? meta[s - S0] : make_int2(0, 0);
            row[h] = (ok && 32 * s + lane < it.n) ? 32 * s + lane : -1;  // internal numbering
            len[h] = md.x;
            base[h] = md.y + lane;
            cb[h] = (32 * s / SIG) * SIG;
            const int rr = row[h] >= 0 ? row[h] : 32 * sa;
            xi[h] = r[rr];
            si[h] = it.q[rr];
        }
        const int L = max(len[0], len[1]);
        for (int k0 = 0; k0 < L; k0 += 4) {
            double v[8];
            int c[8];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int e = base[h] + 32 * (k0 + q);
                    if (k0 + q < len[h]) {
                        v[4 * h + q] = val[e];
                        c[4 * h + q] = c16 ? cb[h] + (int)c16[e] : c32[e];
                    } else {
                        v[4 * h + q] = 0.0;
                        c[4 * h + q] = 32 * sa;
                    }
                }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double gv = r[c[q]];
                if (q < 4) acc[0] = fma(v[q], gv, acc[0]);
                else acc[1] = fma(v[q], gv, acc[1]);
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (row[h] < 0) continue;
            const double y = xi[h] + acc[h];
            it.w[row[h]] = y;
            const double ru = xi[h] * si[h];
            loc.x += xi[h] * xi[h];
            loc.y += y * xi[h];
            loc.z += ru * ru;
        }
    }
    return loc;
}

// ------------------------------------------------------------------ the CG loop
template <int MODE, int NT, int MINB, int NV>
__global__ void __launch_bounds__(NT, MINB)
    k_cg(const RItem* __restrict__ items, int nitems, int vrows, int nvec_unused, int mrows) {
    constexpr int nvec = NV;  // vectors resident in shared memory (p, s[, x]); compile-time
    extern __shared__ double smem[];  // meta[mrows/32] (int2) | p[vrows] | s[vrows] | x[vrows]
    constexpr int NWARP = NT / 32;
    constexpr int RNT = NT;
    __shared__ double sh[4 * NWARP];
    int item = 0, rank = 0;
    if constexpr (MODE == 1) {
        unsigned cr, cid;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
        asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
        item = (int)cid;
        rank = (int)cr;
    } else if constexpr (MODE == 0) {
        item = blockIdx.x;
    } else {
        for (int k = 0; k < nitems; ++k)
            if ((int)blockIdx.x >= items[k].cta0) item = k;
        rank = blockIdx.x - items[item].cta0;
    }
    // the item descriptor lives in shared memory: its ~25 pointers are re-read from there
    // instead of pinning registers (the 64-register cap of the 2-CTA/SM grid mode)
    __shared__ RItem its;
    if (threadIdx.x == 0) its = items[item];
    __syncthreads();
    const RItem& it = its;
    CgState* S = it.st;
    const int W0 = (int)((long long)it.nwin * rank / it.ncta);
    const int W1 = (int)((long long)it.nwin * (rank + 1) / it.ncta);
    const int R0 = min(it.n, W0 * SIG), R1 = min(it.n, W1 * SIG);
    const int S0 = R0 / 32, S1 = (R1 + 31) / 32;
    int2* meta = (int2*)smem;
    double* vbase = smem + (mrows / 32 + 1);
    double* P = nvec >= 2 ? vbase : it.p + R0;
    double* SV = nvec >= 2 ? vbase + vrows : it.sv + R0;
    double* X = nvec >= 3 ? vbase + 2 * vrows : it.x + R0;
    const int tid = threadIdx.x;
    for (int s = S0 + tid; s < S1; s += RNT) meta[s - S0] = make_int2(it.len[s], it.base[s]);
    for (int i = R0 + tid; i < R1; i += RNT) {
        P[i - R0] = 0.0;
        SV[i - R0] = 0.0;
        if (nvec >= 3) X[i - R0] = it.x[i];
    }
    __syncthreads();
    const double tol2 = S->tol2, bn2 = S->bn2;
    const int max_iter = S->max_iter;
    int iters = S->iters, status = FEMI_OK;
    unsigned long long epoch = 0;
    double4 tot = group_reduce<MODE, NT>(it, rank, spmv_w<NWARP>(it, S0, S1, meta), sh, epoch);
    double gam = tot.x, del = tot.y, rho = tot.z;
    double alpha = 0.0, beta = 0.0;
    bool run = bn2 > 0.0 && rho > tol2 && isfinite(rho) && iters < max_iter;
    if (!isfinite(gam) || !isfinite(bn2)) {
        status = FEMI_E_NONFINITE;
        run = false;
    }
    if (run) {
        if (!(del > 0.0)) {
            status = FEMI_E_NEG_CURVATURE;
            run = false;
        } else {
            alpha = gam / del;
        }
    }
    const bool tmr = g_pcg_timers_on && rank == 0 && tid == 0;
    unsigned long long tl = tmr ? gtimer() : 0ull;
    auto mark = [&](int k) {
        if (tmr) {
            const unsigned long long t = gtimer();
            g_pcg_timers[k] += t - tl;
            tl = t;
        }
    };
    constexpr int UB = 6;  // rows per thread with loads in flight in the update phase
    while (run) {
        // U: p = r + beta p ; s = w + beta s ; x += alpha p ; r -= alpha s
        for (int b0 = R0 + tid; b0 < R1; b0 += UB * RNT) {
            double rv[UB], wv[UB];
#pragma unroll
            for (int q = 0; q < UB; ++q) {
                const int i = b0 + q * RNT;
                if (i < R1) {
                    rv[q] = it.r[i];
                    wv[q] = it.w[i];
                }
            }
#pragma unroll
            for (int q = 0; q < UB; ++q) {
                const int i = b0 + q * RNT;
                if (i < R1) {
                    const int l = i - R0;
                    const double pi = fma(beta, P[l], rv[q]);
                    const double si = fma(beta, SV[l], wv[q]);
                    P[l] = pi;
                    SV[l] = si;
                    X[l] = fma(alpha, pi, X[l]);
                    it.r[i] = fma(-alpha, si, rv[q]);
                }
            }
        }
        ++iters;
        mark(0);
        group_sync<MODE>(it, rank, epoch);  // r published
        mark(1);
        const double4 lsp = spmv_w<NWARP>(it, S0, S1, meta);
        mark(2);
        tot = group_reduce<MODE, NT>(it, rank, lsp, sh, epoch);
        mark(3);
        const double gam2 = tot.x, del2 = tot.y, rho2 = tot.z;
        if (!isfinite(gam2) || !isfinite(del2)) {
            status = FEMI_E_NONFINITE;
            break;
        }
        if (rho2 <= tol2) break;
        if (iters >= max_iter) {
            status = FEMI_E_NOT_CONVERGED;
            break;
        }
        beta = gam2 / gam;
        const double den = del2 - beta * gam2 / alpha;  // = p.A^p of the next direction
        if (!(den > 0.0)) {
            status = FEMI_E_NEG_CURVATURE;
            break;
        }
        alpha = gam2 / den;
        gam = gam2;
    }
    if (nvec >= 3)
        for (int i = R0 + tid; i < R1; i += RNT) it.x[i] = X[i - R0];
    if (rank == 0 && tid == 0) {
        S->iters = iters;
        S->status = status;
    }
}

// ------------------------------------------------------------------ on-chip resident CG
// Small and medium systems (C1-C4, C2's 32 meshes): the whole CG loop in one launch with NO
// global-memory traffic per iteration. One cluster of C <= 16 CTAs per system (C = 1: a
// single CTA); CTA k owns rows [R0, R1) (whole 64-row windows). At entry the CTA copies its
// SELL slices into shared memory, with every column pre-resolved to (owner CTA, local row);
// each warp owns fixed slices, so a lane keeps x, p, s, w (and q) of its <= RPL rows in
// registers; only r is published, in the owner's shared memory, and neighbours read it
// there -- locally or through distributed shared memory (DSMEM) across the cluster. Per
// iteration: U in registers, r -> smem, cluster barrier, SpMV from smem/DSMEM, partial dots
// written into every CTA's slot array (DSMEM), cluster barrier, fixed-order sums (identical
// scalars in every CTA: deterministic).
constexpr int RZT = 512;           // threads per CTA
constexpr int RZW = RZT / 32;      // warps
constexpr int RPL = 6;             // rows per lane (slices per warp) kept in registers

template <bool CL>
__device__ __forceinline__ void rz_sync() {
    if constexpr (CL)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    else
        __syncthreads();
}

template <bool CL>
__global__ void __launch_bounds__(RZT, 1) k_cgr(const RItem* __restrict__ items, const int* gate) {
    if (gate && !*gate) return;  // asynchronous restart round not needed (uniform over the cluster)
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) unsigned char rzm[];
    __shared__ RItem its;
    __shared__ double part_s[16][4];  // partial dots of every CTA of the cluster (DSMEM-written)
    __shared__ double sh[4 * RZW];
    __shared__ double bc[4];
    int item = blockIdx.x, rank = 0;
    if constexpr (CL) {
        unsigned cr, cid;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
        asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
        item = (int)cid;
        rank = (int)cr;
    }
    if (threadIdx.x == 0) its = items[item];
    __syncthreads();
    const RItem& it = its;
    CgState* S = it.st;
    const int C = it.ncta;
    const int n = it.n, nwin = it.nwin;
    auto row0 = [&](int k) { return min(n, (int)((long long)nwin * k / C) * SIG); };
    const int R0 = row0(rank), R1 = row0(rank + 1);
    const int S0 = R0 / 32, S1 = (R1 + 31) / 32, nsl = S1 - S0;
    const int e0 = nsl > 0 ? it.base[S0] : 0;
    const int ne = nsl > 0 ? (S1 < (n + 31) / 32 ? it.base[S1] : it.base[S1 - 1] + 32 * it.len[S1 - 1]) - e0 : 0;
    // shared memory: r | q (one slot per slice lane) | values | (owner << 16 | local row) codes | len | base
    double* r_s = (double*)rzm;
    double* q_s = r_s + 32 * nsl;
    double* val_s = q_s + 32 * nsl;
    int* code_s = (int*)(val_s + ne);
    int* len_s = code_s + ne;
    int* base_s = len_s + nsl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // ---- load the CTA's matrix slices, resolving every column to (owner CTA, local row)
    for (int sl = warp; sl < nsl; sl += RZW) {
        const int sg = S0 + sl, L = it.len[sg], b = it.base[sg] - e0, cb = (32 * sg / SIG) * SIG;
        if (lane == 0) {
            len_s[sl] = L;
            base_s[sl] = b;
        }
        for (int k = 0; k < L; ++k) {
            const int e = b + 32 * k + lane;
            const int ge = e + e0;
            const int c = it.c16 ? cb + (int)it.c16[ge] : it.c32[ge];
            const int w = c / SIG;
            int o = (int)(((long long)w * C) / nwin);  // owner CTA of window w: row0(o) <= c < row0(o + 1)
            while (o + 1 < C && row0(o + 1) <= c) ++o;
            while (o > 0 && row0(o) > c) --o;
            FEMI_DCHECK(c >= 0 && c < n && o >= 0 && o < C && c >= row0(o) && c < row0(o + 1), 3);
            val_s[e] = it.val[ge];
            code_s[e] = (o << 16) | (c - row0(o));
        }
    }
    // ---- registers: this lane's rows (slice warp + RZW j)
    double x[RPL], p[RPL], sv[RPL], w[RPL], r[RPL];
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
        const int sl = warp + RZW * j;
        const int row = 32 * (S0 + sl) + lane;
        const bool ok = sl < nsl && row < R1;
        x[j] = ok ? it.x[row] : 0.0;
        r[j] = ok ? it.r[row] : 0.0;
        p[j] = sv[j] = w[j] = 0.0;
        if (sl < nsl) {
            r_s[32 * sl + lane] = r[j];
            q_s[32 * sl + lane] = ok ? it.q[row] : 0.0;
        }
    }
    rz_sync<CL>();
    cg::cluster_group cluster = cg::this_cluster();
    auto spmv = [&](double4& loc) {
        loc = make_double4(0.0, 0.0, 0.0, 0.0);
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
            const int sl = warp + RZW * j;
            if (sl >= nsl) break;  // warp-uniform
            const int L = len_s[sl], b = base_s[sl] + lane;
            double acc = 0.0;
            for (int k0 = 0; k0 < L; k0 += 4) {
                double vv[4], gv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    vv[u] = 0.0;
                    gv[u] = 0.0;
                    if (k0 + u < L) {
                        const int e = b + 32 * (k0 + u);
                        vv[u] = val_s[e];
                        const int cd = code_s[e];
                        const int o = cd >> 16, lr = cd & 0xffff;
                        // local row lr of CTA o sits in slot lr of its r_s (rows start on a slice)
                        if (!CL || o == rank) gv[u] = r_s[lr];
                        else gv[u] = cluster.map_shared_rank(r_s, o)[lr];
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) acc = fma(vv[u], gv[u], acc);
            }
            const int row = 32 * (S0 + sl) + lane;
            if (row < R1) {
                w[j] = r[j] + acc;
                const double ru = r[j] * q_s[32 * sl + lane];
                loc.x += r[j] * r[j];
                loc.y += w[j] * r[j];
                loc.z += ru * ru;
            }
        }
    };
    // cluster-wide fixed-order sum of the three dots
    auto reduce = [&](double4 loc) -> double4 {
        loc.x = warp_sum_d(loc.x);
        loc.y = warp_sum_d(loc.y);
        loc.z = warp_sum_d(loc.z);
        if (lane == 0) {
            sh[4 * warp] = loc.x;
            sh[4 * warp + 1] = loc.y;
            sh[4 * warp + 2] = loc.z;
        }
        __syncthreads();
        if (tid < C) {  // thread k writes this CTA's partial into CTA k's slot array
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int wv = 0; wv < RZW; ++wv) {
                t0 += sh[4 * wv];
                t1 += sh[4 * wv + 1];
                t2 += sh[4 * wv + 2];
            }
            double* dst = CL ? cluster.map_shared_rank(&part_s[0][0], tid) : &part_s[0][0];
            dst[4 * rank] = t0;
            dst[4 * rank + 1] = t1;
            dst[4 * rank + 2] = t2;
        }
        rz_sync<CL>();
        if (tid == 0) {
            double a0 = 0.0, a1 = 0.0, a2 = 0.0;
            for (int k = 0; k < C; ++k) {
                a0 += part_s[k][0];
                a1 += part_s[k][1];
                a2 += part_s[k][2];
            }
            bc[0] = a0;
            bc[1] = a1;
            bc[2] = a2;
        }
        __syncthreads();
        return make_double4(bc[0], bc[1], bc[2], 0.0);
    };
    const double tol2 = S->tol2, bn2 = S->bn2;
    const int max_iter = S->max_iter;
    int iters = S->iters, status = FEMI_OK;
    double4 loc;
    spmv(loc);
    double4 tot = reduce(loc);
    double gam = tot.x, del = tot.y, rho = tot.z;
    double alpha = 0.0, beta = 0.0;
    bool run = bn2 > 0.0 && rho > tol2 && isfinite(rho) && iters < max_iter;
    if (!isfinite(gam) || !isfinite(bn2)) {
        status = FEMI_E_NONFINITE;
        run = false;
    }
    if (run) {
        if (!(del > 0.0)) {
            status = FEMI_E_NEG_CURVATURE;
            run = false;
        } else {
            alpha = gam / del;
        }
    }
    const bool tmr = g_pcg_timers_on && item == 0 && rank == 0 && tid == 0;
    unsigned long long tl = tmr ? gtimer() : 0ull;
    auto mark = [&](int k) {
        if (tmr) {
            const unsigned long long t = gtimer();
            g_pcg_timers[k] += t - tl;
            tl = t;
        }
    };
    while (run) {
        // U (registers) and r published in shared memory
#pragma unroll
        for (int j = 0; j < RPL; ++j) {
            const int sl = warp + RZW * j;
            if (sl >= nsl) break;
            p[j] = fma(beta, p[j], r[j]);
            sv[j] = fma(beta, sv[j], w[j]);
            x[j] = fma(alpha, p[j], x[j]);
            r[j] = fma(-alpha, sv[j], r[j]);
            r_s[32 * sl + lane] = r[j];
        }
        ++iters;
        mark(0);
        rz_sync<CL>();  // r published (cluster-wide)
        mark(1);
        spmv(loc);
        mark(2);
        tot = reduce(loc);  // its cluster barrier also orders the next U's r writes after all reads
        mark(3);
        const double gam2 = tot.x, del2 = tot.y, rho2 = tot.z;
        if (!isfinite(gam2) || !isfinite(del2)) {
            status = FEMI_E_NONFINITE;
            break;
        }
        if (rho2 <= tol2) break;
        if (iters >= max_iter) {
            status = FEMI_E_NOT_CONVERGED;
            break;
        }
        beta = gam2 / gam;
        const double den = del2 - beta * gam2 / alpha;
        if (!(den > 0.0)) {
            status = FEMI_E_NEG_CURVATURE;
            break;
        }
        alpha = gam2 / den;
        gam = gam2;
    }
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
        const int sl = warp + RZW * j;
        const int row = 32 * (S0 + sl) + lane;
        if (sl < nsl && row < R1) it.x[row] = x[j];
    }
    if (rank == 0 && tid == 0) {
        S->iters = iters;
        S->status = status;
    }
    rz_sync<CL>();  // no CTA leaves while others may still read its shared memory
}

// ---- halo tables of the whole-solve resident kernel (built once per system and cluster size).
// CTA k of a C-CTA cluster owns the internal rows [R0, R1) (whole windows); the columns of its
// entries outside that range form its HALO (ascending, deduplicated through a bitmap of all n
// rows); an entry's code is its index into the CTA's extended vector: own row - R0, or
// HB + halo slot with HB = 32 x the largest slice count of the cluster. Because the pattern is
// symmetric, a row c of CTA o is in CTA k's halo iff c has a neighbour in k; CTA o's send list
// holds (c - R0_o, k, slot) for every such pair (found by binary search in k's sorted halo), at
// most one per remote entry of o, so it fits in o's entry range.
__device__ __forceinline__ int rz_row0(int n, int nwin, int C, int k) { return min(n, (nwin * k / C) * SIG); }

__global__ void __launch_bounds__(512) k_rz_halo(const RItem* __restrict__ items, int C) {
    extern __shared__ unsigned int bm[];  // [nw] bitmap of halo rows | [nw] exclusive prefix popcounts
    const RItem& it = items[blockIdx.x / C];
    if (!it.rzc) return;  // the item's tables exist
    const int k = blockIdx.x % C, n = it.n, nwin = it.nwin;
    const int R0 = rz_row0(n, nwin, C, k), R1 = rz_row0(n, nwin, C, k + 1);
    const int S0 = R0 / 32, S1 = (R1 + 31) / 32, nsl = S1 - S0;
    const int e0 = nsl > 0 ? it.base[S0] : 0;
    int nslm = 0;
    for (int q = 0; q < C; ++q) nslm = max(nslm, (rz_row0(n, nwin, C, q + 1) + 31) / 32 - rz_row0(n, nwin, C, q) / 32);
    const int HB = 32 * nslm;
    const int nw = (n + 31) / 32;
    unsigned int* pre = bm + nw;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int w = tid; w < nw; w += 512) bm[w] = 0u;
    __syncthreads();
    auto col = [&](int sg, int ge) {
        const int cb = (32 * sg / SIG) * SIG;
        return it.c16 ? cb + (int)it.c16[ge] : it.c32[ge];
    };
    for (int sl = warp; sl < nsl; sl += 16) {
        const int sg = S0 + sl, L = it.len[sg], b = it.base[sg];
        for (int q = 0; q < L; ++q) {
            const int c = col(sg, b + 32 * q + lane);
            FEMI_DCHECK(c >= 0 && c < n, 3);
            if (c < R0 || c >= R1) atomicOr(&bm[c >> 5], 1u << (c & 31));
        }
    }
    __syncthreads();
    // exclusive scan of the popcounts: thread t owns words [t ch, (t + 1) ch)
    const int ch = (nw + 511) / 512;
    int loc = 0;
    for (int w = tid * ch; w < min(nw, (tid + 1) * ch); ++w) loc += __popc(bm[w]);
    int inc = loc;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    __shared__ int wsum[16];
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int wo = 0;
    for (int q = 0; q < warp; ++q) wo += wsum[q];
    int run = wo + inc - loc;
    for (int w = tid * ch; w < min(nw, (tid + 1) * ch); ++w) {
        pre[w] = run;
        run += __popc(bm[w]);
    }
    __syncthreads();
    int tot = 0;
    for (int q = 0; q < 16; ++q) tot += wsum[q];
    for (int sl = warp; sl < nsl; sl += 16) {
        const int sg = S0 + sl, L = it.len[sg], b = it.base[sg];
        for (int q = 0; q < L; ++q) {
            const int ge = b + 32 * q + lane;
            const int c = col(sg, ge);
            int code;
            if (c >= R0 && c < R1) code = c - R0;
            else code = HB + (int)pre[c >> 5] + __popc(bm[c >> 5] & ((1u << (c & 31)) - 1u));
            FEMI_DCHECK(code >= 0 && code < 65536, 3);
            it.rzc[ge] = (uint16_t)code;
        }
    }
    for (int w = tid; w < nw; w += 512) {
        unsigned int bits = bm[w];
        int sidx = (int)pre[w];
        while (bits) {
            const int bit = __ffs(bits) - 1;
            bits &= bits - 1u;
            it.rzh[e0 + sidx++] = 32 * w + bit;
        }
    }
    if (tid == 0) it.rzn[k] = tot;
}

__global__ void __launch_bounds__(512) k_rz_send(const RItem* __restrict__ items, int C) {
    const RItem& it = items[blockIdx.x / C];
    if (!it.rzc) return;
    const int o = blockIdx.x % C, n = it.n, nwin = it.nwin;
    const int R0 = rz_row0(n, nwin, C, o), R1 = rz_row0(n, nwin, C, o + 1);
    const int S0 = R0 / 32, nsl = (R1 + 31) / 32 - S0;
    const int e0 = nsl > 0 ? it.base[S0] : 0;
    int off = 0;
    for (int k = 0; k < C; ++k) {
        if (k == o || nsl == 0) continue;
        const int R0k = rz_row0(n, nwin, C, k), R1k = rz_row0(n, nwin, C, k + 1);
        if (R1k <= R0k) continue;
        const int* H = it.rzh + it.base[R0k / 32];
        const int hc = it.rzn[k];
        int lo = 0, hi = hc;  // first slot >= R0
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (H[mid] < R0) lo = mid + 1;
            else hi = mid;
        }
        const int a = lo;
        hi = hc;  // first slot >= R1
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (H[mid] < R1) lo = mid + 1;
            else hi = mid;
        }
        for (int h = a + threadIdx.x; h < lo; h += 512)
            it.rzs[e0 + off + (h - a)] = (H[h] - R0) | (k << 12) | (h << 16);
        off += lo - a;
    }
    if (threadIdx.x == 0) it.rzn[16 + o] = off;
}

// Whole-solve resident kernel (k_cgs, the default for systems that fit; FEMI_CG_PIPE=0 selects
// k_cgr + the separate prologue/epilogue kernels). ONE cluster launch per solve does what the
// sequence k_reset, k_pro1, k_x0_fill2 x2, k_pro2, k_cgr, k_finalize, k_true_res, (restart
// rounds), k_copy_g did -- the same arithmetic, rows walked in the same entry order -- so a
// small or medium solve costs one launch instead of ~14 (the fixed cost dominated C1-C4).
//   prologue: min/max of g (x0 modes 1, 3), b = -A_uk g (or the given b), the mask-neighbour
//     fill (reading A11b: first hop from A_uk, two hops over A_uu through u_vert / w), x^0 and
//     r^0 = s b - A^ x^0 (modes 2, 3; = s (b - A x0) with the solver's matrix in shared memory),
//     -s A_uk (g - c1) (mode 1), s b (mode 0); the rows of a lane are walked together;
//   CG: pipelined single-reduction recurrence (Ghysels & Vanroose; Jacobi folded into A^ as
//     everywhere here). With w = A^ r, s = A^ p, z = A^ s, per iteration
//       gamma = r.r, delta = w.r, rho = ||D^1/2 r^||^2 (partials of r_i, w_i)  |  n = A^ w_i
//       beta = gamma/gamma_prev, alpha = gamma/(delta - beta gamma/alpha_prev) (first: gamma/delta)
//       z = n + beta z ; s = w + beta s ; p = r + beta p ; x += alpha p ; r -= alpha s ; w -= alpha z
//     In exact arithmetic these are k_cgr's iterates; ONE cluster barrier per iteration carries
//     both w_i (shared-memory buffer of parity i & 1; the own rows written by their lanes, the
//     halo entries pushed into the peers' buffers by DSMEM stores from per-CTA send lists) and
//     the CTA's three partial dots (per warp, then per CTA in a fixed warp order, then written
//     into every CTA's slot array of parity i & 1); every warp then sums the C slots in a fixed
//     order (xor butterfly: the same bits in every lane, warp and CTA, so alpha / beta / the
//     stopping decision agree everywhere) and multiplies from its own shared memory only. A
//     buffer of parity k is rewritten two barriers later, after every CTA has passed the barrier
//     in between, i.e. after every read of it. Slices are dealt to warps in snake order (rows
//     are length-sorted inside 64-row windows);
//   epilogue: x = s x^ into u_vert, the true residual ||b - A x|| with the unscaled rows (reading
//     A11) and, when it misses rtol, up to 8 restarts of the recurrence from r = s (b - A x)
//     inside the same launch; the mask entries of u_vert = g; the CgState for the host.
// Global data written here and read by other CTAs of the cluster (u_vert, w as the fill's
// temporary) is ordered by the cluster barrier (release / acquire at cluster scope) and read
// with ld.global.cg.
template <bool CL, int RP>
__global__ void __launch_bounds__(RZT, 1) k_cgs(const RItem* __restrict__ items, double rtol, int max_iter) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) unsigned char rzm[];
    __shared__ RItem its;
    __shared__ unsigned long long kmm[16 * RZW][2];  // per-warp min / max keys of g
    __shared__ double wsum3[2][RZW][3];              // per-warp partial dots [parity][warp]
    __shared__ double cpart[2][16][3];               // CG loop: per-CTA partial dots [parity][cta], DSMEM-written
    int item = blockIdx.x, rank = 0;
    if constexpr (CL) {
        unsigned cr, cid;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
        asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
        item = (int)cid;
        rank = (int)cr;
    }
    // every CTA of the cluster must be running before its shared memory is addressed: arrive
    // now, wait just before the first DSMEM store (the slice loading runs in between)
    if constexpr (CL) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    const unsigned long long t_k0 = g_pcg_timers_on ? gtimer() : 0ull;
    if (threadIdx.x == 0) its = items[item];
    __syncthreads();
    const RItem& it = its;
    CgState* S = it.st;
    const int C = it.ncta;
    const int n = it.n, nwin = it.nwin, m = it.m, mode = it.x0mode;
    auto row0 = [&](int k) { return min(n, (nwin * k / C) * SIG); };
    const int R0 = row0(rank), R1 = row0(rank + 1);
    const int S0 = R0 / 32, S1 = (R1 + 31) / 32, nsl = S1 - S0;
    const int e0 = nsl > 0 ? it.base[S0] : 0;
    const int ne = nsl > 0 ? (S1 < (n + 31) / 32 ? it.base[S1] : it.base[S1 - 1] + 32 * it.len[S1 - 1]) - e0 : 0;
    // shared memory: extended vector (own rows | halo) x2 (parity) | q | values | codes | len |
    // base | send list. The layout of the vectors is the same in every CTA of the cluster (own
    // part 32 x the largest slice count HB, then the largest halo), since peers write halo
    // entries into it through DSMEM.
    int nslm = 0;
    for (int k = 0; k < C; ++k) nslm = max(nslm, (row0(k + 1) + 31) / 32 - row0(k) / 32);
    const int HB = 32 * nslm, WS = HB + it.rzhmax;
    double* wb0 = (double*)rzm;
    double* wb1 = wb0 + WS;
    double* q_s = wb1 + WS;
    double* val_s = q_s + 32 * nsl;
    uint16_t* code_s = (uint16_t*)(val_s + ne);  // index into the extended vector
    int* len_s = (int*)(code_s + ((ne + 1) & ~1));
    int* base_s = len_s + nsl;
    uint32_t* snd_s = (uint32_t*)(base_s + nsl);
    const int nsnd = it.rzn ? it.rzn[16 + rank] : 0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    cg::cluster_group cluster = cg::this_cluster();
    for (int sl = tid; sl < nsl; sl += RZT) {
        len_s[sl] = it.len[S0 + sl];
        base_s[sl] = it.base[S0 + sl] - e0;
    }
    {  // the CTA's entries are one contiguous range: a flat copy, sixteen loads in flight per thread
        const double* __restrict__ gv = it.val + e0;
        const uint16_t* __restrict__ gc = it.rzc + e0;
        constexpr int CU = 16;  // loads in flight per thread (registers are free before the prologue)
        for (int i0 = 0; i0 < ne; i0 += CU * RZT) {
            double v[CU];
            uint16_t c[CU];
#pragma unroll
            for (int u = 0; u < CU; ++u) {
                const int i = i0 + u * RZT + tid;
                v[u] = i < ne ? gv[i] : 0.0;
                c[u] = i < ne ? gc[i] : (uint16_t)0;
            }
#pragma unroll
            for (int u = 0; u < CU; ++u) {
                const int i = i0 + u * RZT + tid;
                if (i < ne) {
                    val_s[i] = v[u];
                    code_s[i] = c[u];
                }
            }
        }
    }
    for (int i = tid; i < nsnd; i += RZT) snd_s[i] = (uint32_t)it.rzs[e0 + i];
    __syncthreads();  // the CTA's slice metadata, entries and send list are in place
    // FEMI_PCG_TIMERS: rank-0 thread-0 %globaltimer deltas -- per iteration [0..3], per launch
    // [4] setup (from the kernel's start), [5] pass 1 + ||b||, [6] fill + pass 2, [7] epilogue
    const bool tmr = g_pcg_timers_on && item == 0 && rank == 0 && tid == 0;
    unsigned long long tl = tmr ? t_k0 : 0ull;
    auto mark = [&](int k) {
        if (tmr) {
            const unsigned long long t = gtimer();
            g_pcg_timers[k] += t - tl;
            tl = t;
        }
    };
    mark(4);
    unsigned long long tsub = tl;  // finer split of the prologue: slots 8.. (from the previous sub-mark)
    auto smark = [&](int k) {
        if (tmr) {
            const unsigned long long t = gtimer();
            g_pcg_timers[k] += t - tsub;
            tsub = t;
        }
    };
    // slot j of this warp = slice 16 j + warp (even j) or 16 j + 15 - warp (odd j): inside a
    // 64-row window the rows are sorted by length, so even slices hold the longer rows; the
    // snake order gives every warp as many long as short slices (the iteration waits for the
    // slowest warp of the cluster). Slot j + 1's slices all follow slot j's, so the first
    // slot past nsl ends every warp's loop.
    auto slot = [&](int j) { return RZW * j + ((j & 1) ? RZW - 1 - warp : warp); };
    // publish this lane's values of a vector into buffer buf (own part), then push the halo
    // entries peers read into their copies of buf (DSMEM stores; the caller's cluster barrier
    // makes them visible)
    auto publish = [&](double* buf, const double (&v)[RP]) {
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            const int sl = slot(j);
            if (sl >= nsl) break;
            buf[32 * sl + lane] = v[j];
        }
        if (CL && C > 1) {
            __syncthreads();
            // warps 1.. push the halo entries; warp 0 goes on to the CTA's partial sums
            if (warp > 0)
            for (int i = tid - 32; i < nsnd; i += RZT - 32) {
                const uint32_t e = snd_s[i];
                double* dst = cluster.map_shared_rank(buf, (int)((e >> 12) & 15u));
                dst[HB + (int)(e >> 16)] = buf[e & 0xfffu];
            }
        }
    };
    // this lane's rows: one per slot
    auto row_of = [&](int j) { return 32 * (S0 + slot(j)) + lane; };
    auto row_ok = [&](int j) { return slot(j) < nsl && row_of(j) < R1; };
    // cluster-wide fixed-order sum of three per-warp values (every warp gets the same bits)
    int par = 0;
    auto csum3 = [&](double l0, double l1, double l2, double& t0, double& t1, double& t2) {
        l0 = warp_sum_d(l0);
        l1 = warp_sum_d(l1);
        l2 = warp_sum_d(l2);
        if (lane == 0) {
            wsum3[par][warp][0] = l0;
            wsum3[par][warp][1] = l1;
            wsum3[par][warp][2] = l2;
        }
        __syncthreads();
        if (warp == 0) {  // the CTA's sums (fixed warp order) into every CTA's slot array
            double c0 = lane < RZW ? wsum3[par][lane][0] : 0.0;
            double c1 = lane < RZW ? wsum3[par][lane][1] : 0.0;
            double c2 = lane < RZW ? wsum3[par][lane][2] : 0.0;
            c0 = warp_sum_d(c0);
            c1 = warp_sum_d(c1);
            c2 = warp_sum_d(c2);
            if (lane < C) {
                double* dst = CL ? cluster.map_shared_rank(&cpart[par][0][0], lane) : &cpart[par][0][0];
                dst[3 * rank] = c0;
                dst[3 * rank + 1] = c1;
                dst[3 * rank + 2] = c2;
            }
        }
        rz_sync<CL>();
        t0 = warp_sum_d(lane < C ? cpart[par][lane][0] : 0.0);
        t1 = warp_sum_d(lane < C ? cpart[par][lane][1] : 0.0);
        t2 = warp_sum_d(lane < C ? cpart[par][lane][2] : 0.0);
        par ^= 1;
    };
    // ---------------- prologue
    const bool want_mm = (mode == 1 || mode == 3) && it.g != nullptr;
    if (want_mm) {  // min / max keys of g over a strided share, per warp -> every CTA's slots
        unsigned long long lo = ~0ull, hi = 0ull;
        for (int k = rank * RZT + tid; k < m; k += C * RZT) {
            const unsigned long long key = dkey(it.g[k]);
            lo = min(lo, key);
            hi = max(hi, key);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane < C) {
            unsigned long long* dst = CL ? cluster.map_shared_rank(&kmm[0][0], lane) : &kmm[0][0];
            dst[2 * (rank * RZW + warp)] = lo;
            dst[2 * (rank * RZW + warp) + 1] = hi;
        }
    }
    // pass 1: b = -A_uk g (ascending mask index), the fill's first hop
    bool okr[RP];
    int rowr[RP];
#pragma unroll
    for (int j = 0; j < RP; ++j) {
        okr[j] = row_ok(j);
        rowr[j] = okr[j] ? row_of(j) : 0;
    }
    double l_bn = 0.0;
    {
        double bv[RP];
        if (it.bin) {
#pragma unroll
            for (int j = 0; j < RP; ++j) bv[j] = okr[j] ? it.bin[it.inv[rowr[j]]] : 0.0;
        } else {
            double acc[RP], best[RP], fv[RP];
#pragma unroll
            for (int j = 0; j < RP; ++j) {
                acc[j] = 0.0;
                best[j] = 0.0;
                fv[j] = __longlong_as_double(0x7ff8000000000000ll);  // NaN: not filled yet
            }
            walk_rows<RP, false>(okr, rowr, it.krp, it.kci, it.kav, it.g, [&](int j, double a, int k, double gk) {
                FEMI_DCHECK(k >= 0 && k < it.m, 3);
                acc[j] = fma(a, gk, acc[j]);
                if (a < best[j]) {
                    best[j] = a;
                    fv[j] = gk;
                }
            });
#pragma unroll
            for (int j = 0; j < RP; ++j) {
                bv[j] = -acc[j];
                if (mode == 3 && okr[j]) it.u_vert[it.inv[rowr[j]]] = fv[j];
            }
        }
#pragma unroll
        for (int j = 0; j < RP; ++j)
            if (okr[j]) {
                it.b[rowr[j]] = bv[j];
                l_bn += bv[j] * bv[j];
            }
    }
    smark(8);
    double bn2, d1, d2;
    csum3(l_bn, 0.0, 0.0, bn2, d1, d2);  // also publishes the min / max slots and the first hop
    const double tol2 = rtol * rtol * bn2;
    smark(9);
    mark(5);
    unsigned long long kmin = ~0ull, kmax = 0ull;
    if (want_mm) {
        for (int k = lane; k < C * RZW; k += 32) {
            kmin = min(kmin, kmm[k][0]);
            kmax = max(kmax, kmm[k][1]);
        }
        for (int o = 16; o > 0; o >>= 1) {
            kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
            kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
        }
    }
    const double x0v = want_mm && kmax != 0ull ? 0.5 * (dkey_inv(kmin) + dkey_inv(kmax)) : 0.0;
    if (mode == 3) {  // the fill's second hop: u_vert -> w, barrier, w -> u_vert, barrier
        for (int pass = 0; pass < 2; ++pass) {
            const double* src = pass == 0 ? it.u_vert : it.w;
            double* dst = pass == 0 ? it.w : it.u_vert;
            double v[RP];
            bool need[RP];
            int nat[RP];
#pragma unroll
            for (int j = 0; j < RP; ++j) {
                nat[j] = okr[j] ? it.inv[rowr[j]] : 0;
                v[j] = okr[j] ? __ldcg(src + nat[j]) : 0.0;
                need[j] = okr[j] && isnan(v[j]);
            }
            // the first non-NaN neighbour in ascending column order (rows that need one)
            walk_rows<RP, true>(need, rowr, it.urp, it.uci, it.uav, src, [&](int j, double, int, double c) {
                if (isnan(v[j]) && !isnan(c)) v[j] = c;
            });
#pragma unroll
            for (int j = 0; j < RP; ++j)
                if (okr[j]) dst[nat[j]] = v[j];
            smark(10 + 2 * pass);
            rz_sync<CL>();
            smark(11 + 2 * pass);
        }
    }
    // ---------------- SpMV from a published buffer: out_j = in_j + sum_k a_jk buf[col_jk]
    int Ls[RP], bs[RP];
#pragma unroll
    for (int j = 0; j < RP; ++j) {
        const int sl = slot(j);
        Ls[j] = sl < nsl ? len_s[sl] : 0;
        bs[j] = sl < nsl ? base_s[sl] + lane : 0;
    }
    auto spmv = [&](const double* buf, double (&out)[RP], const double (&in)[RP]) {
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            if (slot(j) >= nsl) break;  // warp-uniform
            const int L = Ls[j], b = bs[j];
            double acc = 0.0;
            for (int k0 = 0; k0 < L; k0 += 4) {
                double vv[4], gv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    vv[u] = 0.0;
                    gv[u] = 0.0;
                    if (k0 + u < L) {
                        const int e = b + 32 * (k0 + u);
                        vv[u] = val_s[e];
                        gv[u] = buf[code_s[e]];
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) acc = fma(vv[u], gv[u], acc);
            }
            out[j] = in[j] + acc;
        }
    };
#pragma unroll
    for (int j = 0; j < RP; ++j)
        if (slot(j) < nsl) q_s[32 * slot(j) + lane] = row_ok(j) ? it.q[row_of(j)] : 0.0;
    // pass 2: x^0 = x0 / s and r^0 = s (b - A x0) = s b - A^ x^0 (A = D^1/2 A^ D^1/2, s = D^-1/2):
    // the product with the solver's own matrix in shared memory -- x^0 published like any CG
    // vector -- instead of a second walk over the unscaled rows in global memory (any r^0
    // consistent with x^0 starts the recurrence; the exit check uses the unscaled rows, A11).
    // A row the fill did not reach takes midrange(g), also in u_vert (only its owner reads it).
    double x[RP], r[RP], w[RP], p[RP], sv[RP], z[RP];
    {
        double acc[RP];
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            x[j] = r[j] = w[j] = p[j] = sv[j] = z[j] = 0.0;
            acc[j] = 0.0;
            if (!okr[j]) continue;
            const int i = rowr[j];
            double x0 = mode == 1 || mode == 3 ? x0v : 0.0;
            if (mode >= 2) {
                const int nat = it.inv[i];
                x0 = __ldcg(it.u_vert + nat);
                if (mode == 3 && isnan(x0)) {
                    x0 = x0v;
                    it.u_vert[nat] = x0;
                }
            }
            x[j] = x0 / it.s[i];
        }
        if (mode == 1 && !it.bin) {  // r0 = -A_uk (g - c 1) (zero row sums)
            walk_rows<RP, false>(okr, rowr, it.krp, it.kci, it.kav, it.g,
                                 [&](int j, double a, int, double gk) { acc[j] = fma(a, gk - x0v, acc[j]); });
        } else if (mode >= 2) {
            publish(par ? wb1 : wb0, x);
            rz_sync<CL>();
            spmv(par ? wb1 : wb0, acc, x);  // A^ x^0
            par ^= 1;  // the buffer is rewritten two barriers later
        }
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            if (!okr[j]) continue;
            const int i = rowr[j];
            const double si = it.s[i];
            if (mode == 0 || (mode == 1 && it.bin)) r[j] = si * __ldcg(it.b + i);
            else if (mode == 1) r[j] = si * -acc[j];
            else r[j] = fma(si, __ldcg(it.b + i), -acc[j]);
        }
    }
    smark(14);
    smark(15);
    mark(6);
    int iters = 0, status = FEMI_OK, restarts = 0;
    double res2 = 0.0;
    bool first_round = true;
    for (;;) {  // CG rounds: the first, then restarts from the true residual
        double* wb_r = par ? wb1 : wb0;  // r^0 of the round in the buffer of the current parity
        publish(wb_r, r);
        rz_sync<CL>();  // r^0 published
        spmv(wb_r, w, r);  // w^0 = A^ r^0
        par ^= 1;          // the buffer of r^0 is rewritten two barriers later
        const int iters0 = iters;
        double alpha = 0.0, gam = 0.0, rgam = 0.0, ralpha = 0.0;
        for (;;) {
            double* wbp = par ? wb1 : wb0;
            // partial dots of (r_i, w_i): per warp into shared memory, summed per CTA (fixed warp
            // order) by warp 0 after the block barrier inside publish, which then writes the
            // CTA's three values into every CTA's slot array; one cluster barrier; every warp
            // sums the C slots (xor butterfly: the same bits everywhere)
            double l0 = 0.0, l1 = 0.0, l2 = 0.0;
#pragma unroll
            for (int j = 0; j < RP; ++j) {
                const int sl = slot(j);
                if (sl >= nsl) break;
                if (row_of(j) < R1) {
                    const double ru = r[j] * q_s[32 * sl + lane];
                    l0 += r[j] * r[j];
                    l1 += w[j] * r[j];
                    l2 += ru * ru;
                }
            }
            l0 = warp_sum_d(l0);
            l1 = warp_sum_d(l1);
            l2 = warp_sum_d(l2);
            if (lane == 0) {
                wsum3[par][warp][0] = l0;
                wsum3[par][warp][1] = l1;
                wsum3[par][warp][2] = l2;
            }
            double gam2, del2, rho2;
            const int pp = par;
            if constexpr (!CL) {  // one CTA: ONE block barrier, every warp sums the warp slots itself
                publish(wbp, w);
                mark(0);
                __syncthreads();
                gam2 = warp_sum_d(lane < RZW ? wsum3[par][lane][0] : 0.0);
                del2 = warp_sum_d(lane < RZW ? wsum3[par][lane][1] : 0.0);
                rho2 = warp_sum_d(lane < RZW ? wsum3[par][lane][2] : 0.0);
            } else {
            publish(wbp, w);
            if (warp == 0) {
                double c0 = lane < RZW ? wsum3[par][lane][0] : 0.0;
                double c1 = lane < RZW ? wsum3[par][lane][1] : 0.0;
                double c2 = lane < RZW ? wsum3[par][lane][2] : 0.0;
                c0 = warp_sum_d(c0);
                c1 = warp_sum_d(c1);
                c2 = warp_sum_d(c2);
                if (lane < C) {
                    double* dst = CL ? cluster.map_shared_rank(&cpart[par][0][0], lane) : &cpart[par][0][0];
                    dst[3 * rank] = c0;
                    dst[3 * rank + 1] = c1;
                    dst[3 * rank + 2] = c2;
                }
            }
            mark(0);
            rz_sync<CL>();
            {
                double a0 = lane < C ? cpart[par][lane][0] : 0.0;
                double a1 = lane < C ? cpart[par][lane][1] : 0.0;
                double a2 = lane < C ? cpart[par][lane][2] : 0.0;
                gam2 = warp_sum_d(a0);
                del2 = warp_sum_d(a1);
                rho2 = warp_sum_d(a2);
            }
            }
            par ^= 1;
            mark(1);
            double nv[RP];
#pragma unroll
            for (int j = 0; j < RP; ++j) nv[j] = 0.0;
            spmv(pp ? wb1 : wb0, nv, w);  // n = A^ w_i
            mark(2);
            if (!isfinite(gam2) || !isfinite(del2) || !isfinite(bn2)) {
                status = FEMI_E_NONFINITE;
                break;
            }
            if (!(bn2 > 0.0) || rho2 <= tol2) break;
            if (iters >= max_iter) {
                if (iters > iters0) status = FEMI_E_NOT_CONVERGED;
                break;
            }
            double beta = 0.0;
            if (iters == iters0) {
                if (!(del2 > 0.0)) {
                    status = FEMI_E_NEG_CURVATURE;
                    break;
                }
                alpha = gam2 / del2;
            } else {  // 1/gamma_prev and 1/alpha_prev were formed off the critical path
                beta = gam2 * rgam;
                const double den = del2 - beta * gam2 * ralpha;
                if (!(den > 0.0)) {
                    status = FEMI_E_NEG_CURVATURE;
                    break;
                }
                alpha = gam2 / den;
            }
            gam = gam2;
#pragma unroll
            for (int j = 0; j < RP; ++j) {
                if (slot(j) >= nsl) break;
                z[j] = fma(beta, z[j], nv[j]);
                sv[j] = fma(beta, sv[j], w[j]);
                p[j] = fma(beta, p[j], r[j]);
                x[j] = fma(alpha, p[j], x[j]);
                r[j] = fma(-alpha, sv[j], r[j]);
                w[j] = fma(-alpha, z[j], w[j]);
            }
            rgam = 1.0 / gam;  // (their latency hides in the next publish and barrier wait)
            ralpha = 1.0 / alpha;
            ++iters;
            mark(3);
        }
        first_round = false;
        const unsigned long long t_ep = tmr ? gtimer() : 0ull;
        // x = s x^ into u_vert (a 0-iteration exit keeps the guess: modes 2, 3 leave u_vert, mode
        // 1 writes the midrange exactly, b = 0 gives x = 0), then the true residual
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            if (!row_ok(j)) continue;
            const int i = row_of(j);
            if (iters == 0 && mode >= 2 && bn2 != 0.0) continue;
            double xi;
            if (bn2 == 0.0) xi = 0.0;
            else if (iters == 0) xi = mode == 1 || mode == 3 ? x0v : 0.0;
            else xi = it.s[i] * x[j];
            it.u_vert[it.inv[i]] = xi;
        }
        rz_sync<CL>();
        double l_res = 0.0;
        {
            double ax[RP];
#pragma unroll
            for (int j = 0; j < RP; ++j) ax[j] = 0.0;
            walk_rows<RP, true>(okr, rowr, it.urp, it.uci, it.uav, it.u_vert, [&](int j, double a, int c, double u) {
                FEMI_DCHECK(c >= 0 && c < it.n, 3);
                ax[j] = fma(a, u, ax[j]);
            });
#pragma unroll
            for (int j = 0; j < RP; ++j) {
                if (!okr[j]) continue;
                const int i = rowr[j];
                const double ri = __ldcg(it.b + i) - ax[j];
                r[j] = it.s[i] * ri;  // the restart's r^0
                l_res += ri * ri;
            }
        }
        csum3(l_res, 0.0, 0.0, res2, d1, d2);
        if (tmr) {
            const unsigned long long t = gtimer();
            g_pcg_timers[7] += t - t_ep;
            tl = t;
        }
        const bool again = status == FEMI_OK && iters > 0 && iters < max_iter && bn2 > 0.0 && !(res2 <= tol2);
        if (!again || restarts >= 8) break;
        ++restarts;
#pragma unroll
        for (int j = 0; j < RP; ++j) p[j] = sv[j] = z[j] = 0.0;
    }
    if (it.g)
        for (int k = rank * RZT + tid; k < m; k += C * RZT) it.u_vert[n + k] = it.g[k];
    if (rank == 0 && tid == 0) {
        S->iters = iters;
        S->status = status;
        S->bn2 = bn2;
        S->tol2 = tol2;
        S->res2 = res2;
        S->kmin = want_mm ? kmin : ~0ull;
        S->kmax = want_mm ? kmax : 0ull;
        S->x_pend = 0;
        S->rtol = rtol;
        S->max_iter = max_iter;
    }
    rz_sync<CL>();  // no CTA leaves while others may still read its shared memory
}

// ------------------------------------------------------------------ graph mode
// Large single systems (C5): the CG loop is a device-driven WHILE node of a CUDA graph whose
// body is two lean, full-occupancy kernels -- k_gu (update, element-wise) and k_gs (SELL
// SpMV + dots; its last block turns the partials into alpha/beta/convergence in a fixed
// order and sets the loop condition). Lean kernels run 64 warps/SM, i.e. 2-3x the memory-
// level parallelism of the persistent kernel, which is what the latency-bound SpMV needs.
constexpr int GNT = 256;

__global__ void k_reset_items(int B, const RItem* __restrict__ items) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    CgState s = {};
    s.rtol = items[b].rtol;
    s.max_iter = items[b].max_iter;
    s.kmin = ~0ull;
    s.kmax = 0ull;
    *items[b].st = s;
}

// p = s = 0 (start and restart of the recurrence)
__global__ void k_zero_ps(const RItem* __restrict__ items) {
    const RItem& it = items[blockIdx.y];
    if (it.ls && blockIdx.x == 0 && threadIdx.x == 0) {  // (re)start of the lean-tail recurrence
        LoopState l = {};
        l.iters = it.st->iters;  // a restart continues the count
        l.active = 1;
        it.ls[0] = l;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < it.n; i += gridDim.x * blockDim.x) {
        it.p[i] = 0.0;
        it.sv[i] = 0.0;
    }
}

// U: p = r + beta p ; s = w + beta s ; x += alpha p ; r -= alpha s
// x is only needed at exit, so it moves every other iteration: an even iteration defers its
// alpha_i p_i, the odd one after it applies x += alpha_{i-1} p_{i-1} + alpha_i p_i (both p's are
// in registers there), k_finalize applies a deferred term left at exit. Saves the x read and
// write of every other iteration (2 of the 9 vector streams).
__global__ void __launch_bounds__(GNT) k_gu(const RItem* __restrict__ items) {
    grid_dep_wait();  // behind the previous SpMV through a programmatic edge (graph body)
    const RItem& it = items[blockIdx.y];
    const CgState* S = it.st;
    if (!S->active) return;
    const unsigned long long tprof = g_loop_prof ? gtime() : 0ull;
    const double alpha = S->alpha, beta = S->beta;
    if ((S->iters & 1) == 0) {
        double* __restrict__ r = it.r;
        const double* __restrict__ w = it.w;
        double* __restrict__ p = it.p;
        double* __restrict__ sv = it.sv;
        const int n = it.n, stride = gridDim.x * blockDim.x;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 2 * stride) {
            const int j = i + stride;
            const bool hj = j < n;
            const double ri = r[i], wi = w[i], pi0 = p[i], si0 = sv[i];
            double rj = 0.0, wj = 0.0, pj0 = 0.0, sj0 = 0.0;
            if (hj) {
                rj = r[j];
                wj = w[j];
                pj0 = p[j];
                sj0 = sv[j];
            }
            const double si = fma(beta, si0, wi);
            p[i] = fma(beta, pi0, ri);
            sv[i] = si;
            r[i] = fma(-alpha, si, ri);
            if (hj) {
                const double sj = fma(beta, sj0, wj);
                p[j] = fma(beta, pj0, rj);
                sv[j] = sj;
                r[j] = fma(-alpha, sj, rj);
            }
        }
        if (g_loop_prof) {
            __syncthreads();
            if (threadIdx.x == 0) loop_stamp(0, S->iters, tprof);
        }
        return;
    }
    const double ap = S->alpha_pend;
    double* __restrict__ r = it.r;
    const double* __restrict__ w = it.w;
    double* __restrict__ p = it.p;
    double* __restrict__ sv = it.sv;
    double* __restrict__ x = it.x;
    const int n = it.n, stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 2 * stride) {
        const int j = i + stride;
        const bool hj = j < n;
        const double ri = r[i], wi = w[i], pi0 = p[i], si0 = sv[i], xi = x[i];
        double rj = 0.0, wj = 0.0, pj0 = 0.0, sj0 = 0.0, xj = 0.0;
        if (hj) {
            rj = r[j];
            wj = w[j];
            pj0 = p[j];
            sj0 = sv[j];
            xj = x[j];
        }
        const double pi = fma(beta, pi0, ri), si = fma(beta, si0, wi);
        p[i] = pi;
        sv[i] = si;
        x[i] = fma(alpha, pi, fma(ap, pi0, xi));
        r[i] = fma(-alpha, si, ri);
        if (hj) {
            const double pj = fma(beta, pj0, rj), sj = fma(beta, sj0, wj);
            p[j] = pj;
            sv[j] = sj;
            x[j] = fma(alpha, pj, fma(ap, pj0, xj));
            r[j] = fma(-alpha, sj, rj);
        }
    }
    if (g_loop_prof) {
        __syncthreads();
        if (threadIdx.x == 0) loop_stamp(0, S->iters, tprof);
    }
}

// One CG recurrence step from the summed dots (gam2 = r^.r^, del2 = w.r^, rho2 = ||D^1/2 r^||^2):
// FIRST starts the recurrence; otherwise counts the iteration, tests convergence on rho2 (when it
// was computed), and advances alpha, beta. Returns whether the recurrence continues; also sets
// need_rho for the next SpMV (||r||^2 >= dmin ||r^||^2, two orders of slack).
template <bool FIRST>
__device__ __forceinline__ int cg_advance(CgState* S, bool act, double gam2, double del2, double rho2, double dmin,
                                          double s_bn2, double s_tol2, double s_rr, double s_alpha, int s_iters,
                                          int s_max, int s_need) {
    int active = 0;
    if (!act) return 0;
    if (FIRST) {
        const bool fin = isfinite(gam2) && isfinite(s_bn2);
        active = (s_bn2 > 0.0 && rho2 > s_tol2 && fin && s_iters < s_max) ? 1 : 0;
        if (!fin) S->status = FEMI_E_NONFINITE;
        if (active && !(del2 > 0.0)) {
            S->status = FEMI_E_NEG_CURVATURE;
            active = 0;
        }
        if (active) {
            S->alpha = gam2 / del2;
            S->beta = 0.0;
            S->rr = gam2;
        }
    } else {
        const int it1 = s_iters + 1;
        S->iters = it1;
        if (!isfinite(gam2) || !isfinite(del2)) {
            S->status = FEMI_E_NONFINITE;
        } else if (s_need && rho2 <= s_tol2) {
            // converged (rho2 is only computed when dmin gam2 was within 100x of tol2)
        } else if (it1 >= s_max) {
            S->status = FEMI_E_NOT_CONVERGED;
        } else {
            const double beta = gam2 / s_rr;
            const double den = del2 - beta * gam2 / s_alpha;
            if (!(den > 0.0)) {
                S->status = FEMI_E_NEG_CURVATURE;
            } else {
                S->beta = beta;
                S->alpha = gam2 / den;
                S->rr = gam2;
                active = 1;
            }
        }
    }
    S->active = active;
    S->need_rho = (gam2 * dmin <= 100.0 * s_tol2) ? 1 : 0;
    return active;
}

// Block partials -> part[item][block]; the last block of the item sums them in block order
// (deterministic), advances the CG recurrence scalars (FIRST: starts it) and, once every item
// has reported, sets the WHILE condition (any item still active -> 1).
template <bool FIRST, int NT = GNT>
__device__ __forceinline__ void cg_tail(double (&v)[3], bool act, CgState* S, int B, double* __restrict__ part,
                                        unsigned* __restrict__ gcnt, cudaGraphConditionalHandle h, int prof_it = -1,
                                        double dmin = 0.0) {
    const bool tp = prof_it >= 0 && prof_it < kLoopProfMax && g_loop_prof;
    // the recurrence state the last CTA needs, loaded up front (off the tail's critical path);
    // it only changes in the last CTA of the previous launch
    double s_bn2 = 0.0, s_tol2 = 0.0, s_rr = 0.0, s_alpha = 0.0;
    int s_iters = 0, s_max = 0, s_need = 1;
    if (threadIdx.x == 0) {
        s_need = FIRST ? 1 : S->need_rho;
        s_bn2 = S->bn2;
        s_tol2 = S->tol2;
        s_rr = S->rr;
        s_alpha = S->alpha;
        s_iters = S->iters;
        s_max = S->max_iter;
    }
    __shared__ double shm[4 * (NT / 32)];
    __shared__ int last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 3; ++q) v[q] = warp_sum_d(v[q]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 3; ++q) shm[4 * wid + q] = v[q];
    __syncthreads();
    double* P = part + 4 * (size_t)gridDim.x * blockIdx.y;
    // the arrival is made by the first thread of the LAST warp: in k_gt that is the producer
    // warp, which issued no global stores, so its release fence does not wait for the
    // consumers' in-flight w stores (only P has to be visible to the last CTA; w is ordered
    // by the kernel boundary)
    constexpr int AT = NT - 32;
    if (threadIdx.x == AT) {
        for (int q = 0; q < 3; ++q) {
            double t = 0.0;
            for (int w = 0; w < NT / 32; ++w) t += shm[4 * w + q];
            P[4 * blockIdx.x + q] = t;
        }
        last = atom_add_release_gpu(&S->cnt[0], 1u) == gridDim.x - 1;
        if (tp) atomicMax(&g_tail_ts[4 * prof_it], gtime());  // A: CTA arrived
    }
    __syncthreads();
    if (!last) return;
    fence_acq_rel_gpu();
    double tot[3] = {0.0, 0.0, 0.0};
    for (unsigned b = threadIdx.x; b < gridDim.x; b += NT)
#pragma unroll
        for (int q = 0; q < 3; ++q) tot[q] += __ldcg(P + 4 * b + q);
#pragma unroll
    for (int q = 0; q < 3; ++q) tot[q] = warp_sum_d(tot[q]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 3; ++q) shm[4 * wid + q] = tot[q];
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (tp) g_tail_ts[4 * prof_it + 1] = gtime();  // B: last CTA has the partials
    double gam2 = 0.0, del2 = 0.0, rho2 = 0.0;
    for (int w = 0; w < NT / 32; ++w) {
        gam2 += shm[4 * w];
        del2 += shm[4 * w + 1];
        rho2 += shm[4 * w + 2];
    }
    S->cnt[0] = 0;
    if (!FIRST && act) {  // the k_gu before this SpMV: deferred its x term (even) or not
        S->x_pend = (s_iters & 1) == 0 ? 1 : 0;
        S->alpha_pend = s_alpha;
    }
    const int active = cg_advance<FIRST>(S, act, gam2, del2, rho2, dmin, s_bn2, s_tol2, s_rr, s_alpha, s_iters, s_max,
                                         s_need);
    if (tp) g_tail_ts[4 * prof_it + 2] = gtime();  // C: scalars done
    // all items reported? -> loop condition (one item: set it directly)
    if (B == 1) {
        if (h) cudaGraphSetConditional(h, active ? 1u : 0u);
    } else {
    if (active) atom_add_release_gpu(gcnt + 1, 1u);
    if (atom_add_release_gpu(gcnt, 1u) == (unsigned)B - 1) {
        fence_acq_rel_gpu();
        const unsigned any = atomicExch(gcnt + 1, 0u);
        gcnt[0] = 0;
        if (h) cudaGraphSetConditional(h, any ? 1u : 0u);  // h == 0: standalone launch (kbench)
    }
    }
    if (tp) g_tail_ts[4 * prof_it + 3] = gtime();  // D: condition set
}

// The CTA's three partial dots in fixed warp order -> P[0..2]
template <int NT>
__device__ __forceinline__ void cta_partials(double (&v)[3], double* P) {
    __shared__ double shp[3 * (NT / 32)];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 3; ++q) v[q] = warp_sum_d(v[q]);
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 3; ++q) shp[3 * wid + q] = v[q];
    __syncthreads();
    if (threadIdx.x < 3) {
        double t = 0.0;
        for (int w = 0; w < NT / 32; ++w) t += shp[3 * w + threadIdx.x];
        P[threadIdx.x] = t;
    }
}

// Graph mode, lean tail: ONE kernel per iteration does the reduction AND the update. Every CTA
// sums the previous SpMV's per-CTA partials in the same fixed order (bit-identical scalars in
// all CTAs), advances the CG recurrence (cg_advance's rules) from ls[par] and applies the
// update p = r + beta p ; s = w + beta s ; r -= alpha s ; x every other iteration (as k_gu).
// Block 0 publishes the new scalars in ls[par ^ 1]; on termination it writes the final state
// (iteration count, status, the deferred x term) to the item's CgState and ends the WHILE loop.
// Compared with the last-CTA tail of cg_tail, nothing serialises behind an atomic counter.
constexpr int GRT = 256;
constexpr int64_t kFillMinRows = 0;  // reading A11b: systems below this size start at midrange (FEMI_FILL_MIN)
__global__ void __launch_bounds__(GRT) k_gur(const RItem* __restrict__ items, const double* __restrict__ part,
                                            int nparts, int par, cudaGraphConditionalHandle h) {
    __shared__ double red[3 * (GRT / 32)];
    __shared__ double sc[4];  // alpha, beta, alpha_pend
    __shared__ int si[2];     // active, iters
    grid_dep_wait();  // behind the SpMV through a programmatic edge (graph body)
    const RItem& it = items[0];
    const LoopState L = it.ls[par];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (!L.active && !g_kbench) {  // finished earlier in this launch: keep the next slot inactive
        if (blockIdx.x == 0 && threadIdx.x == 0) it.ls[par ^ 1].active = 0;
        return;
    }
    const unsigned long long tprof = g_loop_prof ? gtime() : 0ull;
    double v[3] = {0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < nparts; b += GRT)
#pragma unroll
        for (int q = 0; q < 3; ++q) v[q] += __ldcg(part + 4 * b + q);
#pragma unroll
    for (int q = 0; q < 3; ++q) v[q] = warp_sum_d(v[q]);
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 3; ++q) red[3 * wid + q] = v[q];
    __syncthreads();
    if (threadIdx.x == 0) {
        double gam2 = 0.0, del2 = 0.0, rho2 = 0.0;
        for (int w = 0; w < GRT / 32; ++w) {
            gam2 += red[3 * w];
            del2 += red[3 * w + 1];
            rho2 += red[3 * w + 2];
        }
        const CgState* S = it.st;
        const double tol2 = S->tol2, bn2 = S->bn2;
        LoopState N = L;
        N.started = 1;
        int active = 0;
        int status = L.status;
        double alpha = 0.0, beta = 0.0;
        int iters = L.iters;
        if (!L.started) {  // the first SpMV: start the recurrence (cg_advance<true>)
            const bool fin = isfinite(gam2) && isfinite(bn2);
            active = (bn2 > 0.0 && rho2 > tol2 && fin && L.iters < S->max_iter) ? 1 : 0;
            if (!fin) status = FEMI_E_NONFINITE;
            if (active && !(del2 > 0.0)) {
                status = FEMI_E_NEG_CURVATURE;
                active = 0;
            }
            if (active) {
                alpha = gam2 / del2;
                beta = 0.0;
            }
        } else {  // cg_advance<false>: count the iteration, test convergence, next alpha / beta
            iters = L.iters + 1;
            if (!isfinite(gam2) || !isfinite(del2)) {
                status = FEMI_E_NONFINITE;
            } else if (L.need_rho && rho2 <= tol2) {
                // converged
            } else if (iters >= S->max_iter) {
                status = FEMI_E_NOT_CONVERGED;
            } else {
                beta = gam2 / L.rr;
                const double den = del2 - beta * gam2 / L.alpha;
                if (!(den > 0.0)) {
                    status = FEMI_E_NEG_CURVATURE;
                } else {
                    alpha = gam2 / den;
                    active = 1;
                }
            }
        }
        // the previous update deferred its x term when its iteration label was even
        const bool deferred = L.started && (L.iters & 1) == 0;
        N.alpha = alpha;
        N.rr = gam2;
        N.iters = iters;
        N.active = active;
        N.status = status;
        N.need_rho = (gam2 * it.dmin <= 100.0 * tol2) ? 1 : 0;
        sc[0] = alpha;
        sc[1] = beta;
        sc[2] = (deferred && L.started) ? L.alpha : 0.0;
        si[0] = active;
        si[1] = iters;
        if (blockIdx.x == 0 && !g_kbench) {
            it.ls[par ^ 1] = N;
            if (!active) {  // final state for k_finalize / k_true_res / the host
                CgState* Sw = it.st;
                Sw->iters = iters;
                Sw->status = status;
                Sw->active = 0;
                Sw->x_pend = deferred ? 1 : 0;
                Sw->alpha_pend = L.alpha;
                Sw->rr = gam2;
                if (h) cudaGraphSetConditional(h, 0u);
            }
        }
    }
    __syncthreads();
    if (g_kbench) {  // profiling aid: the full update traffic with a no-op update
        if (threadIdx.x == 0) {
            sc[0] = sc[1] = sc[2] = 0.0;
            si[0] = 1;
        }
        __syncthreads();
    }
    if (!si[0]) return;
    const double alpha = sc[0], beta = sc[1], ap = sc[2];
    double* __restrict__ r = it.r;
    const double* __restrict__ w = it.w;
    double* __restrict__ p = it.p;
    double* __restrict__ sv = it.sv;
    const int n = it.n, stride = gridDim.x * blockDim.x;
    if ((si[1] & 1) == 0) {  // even label: x's term deferred to the next update (or k_finalize)
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 2 * stride) {
            const int j = i + stride;
            const bool hj = j < n;
            const double ri = r[i], wi = w[i], pi0 = p[i], si0 = sv[i];
            double rj = 0.0, wj = 0.0, pj0 = 0.0, sj0 = 0.0;
            if (hj) {
                rj = r[j];
                wj = w[j];
                pj0 = p[j];
                sj0 = sv[j];
            }
            const double si = fma(beta, si0, wi);
            p[i] = fma(beta, pi0, ri);
            sv[i] = si;
            r[i] = fma(-alpha, si, ri);
            if (hj) {
                const double sj = fma(beta, sj0, wj);
                p[j] = fma(beta, pj0, rj);
                sv[j] = sj;
                r[j] = fma(-alpha, sj, rj);
            }
        }
    } else {
        double* __restrict__ x = it.x;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 2 * stride) {
            const int j = i + stride;
            const bool hj = j < n;
            const double ri = r[i], wi = w[i], pi0 = p[i], si0 = sv[i], xi = x[i];
            double rj = 0.0, wj = 0.0, pj0 = 0.0, sj0 = 0.0, xj = 0.0;
            if (hj) {
                rj = r[j];
                wj = w[j];
                pj0 = p[j];
                sj0 = sv[j];
                xj = x[j];
            }
            const double pi = fma(beta, pi0, ri), si = fma(beta, si0, wi);
            p[i] = pi;
            sv[i] = si;
            x[i] = fma(alpha, pi, fma(ap, pi0, xi));
            r[i] = fma(-alpha, si, ri);
            if (hj) {
                const double pj = fma(beta, pj0, rj), sj = fma(beta, sj0, wj);
                p[j] = pj;
                sv[j] = sj;
                x[j] = fma(alpha, pj, fma(ap, pj0, xj));
                r[j] = fma(-alpha, sj, rj);
            }
        }
    }
    if (g_loop_prof) {
        __syncthreads();
        if (threadIdx.x == 0) loop_stamp(0, si[1], tprof);
    }
}

// S: w = r + A^_off r (SELL, two slices per warp) and the dots; the last block updates the
// recurrence scalars and (FIRST: starts it) and sets the WHILE condition when every item has
// reported (any item still active -> 1).
template <bool FIRST>
__global__ void __launch_bounds__(GNT, 4) k_gs(const RItem* __restrict__ items, int B, double* __restrict__ part,
                                           unsigned* __restrict__ gcnt, cudaGraphConditionalHandle h) {
    const RItem& it = items[blockIdx.y];
    CgState* S = it.st;
    const bool act = FIRST || S->active;
    double v[3] = {0.0, 0.0, 0.0};
    if (act) {
        const int lane = threadIdx.x & 31;
        const int nsl = (it.n + 31) / 32;
        const int gw = (blockIdx.x * GNT + threadIdx.x) >> 5, nw = (gridDim.x * GNT) >> 5;
        const double* __restrict__ r = it.r;
        double* __restrict__ wout = it.w;
        for (int sa = 2 * gw; sa < nsl; sa += 2 * nw) {
            const bool hb = sa + 1 < nsl;
            int row[2], len[2], base[2], cb[2];
            double xi[2], si[2], acc[2] = {0.0, 0.0};
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const int s = sa + hh;
                const bool ok = hh == 0 || hb;
                row[hh] = (ok && 32 * s + lane < it.n) ? 32 * s + lane : -1;
                len[hh] = ok ? it.len[s] : 0;
                base[hh] = ok ? it.base[s] + lane : 0;
                cb[hh] = (32 * s / SIG) * SIG;
                const int rr = row[hh] >= 0 ? row[hh] : 32 * sa;
                xi[hh] = r[rr];
                si[hh] = it.q[rr];
            }
            const int L = max(len[0], len[1]);
            for (int k0 = 0; k0 < L; k0 += 4) {
                double vv[8];
                int c[8];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int e = base[hh] + 32 * (k0 + q);
                        if (k0 + q < len[hh]) {
                            vv[4 * hh + q] = it.val[e];
                            c[4 * hh + q] = it.c16 ? cb[hh] + (int)it.c16[e] : it.c32[e];
                        } else {
                            vv[4 * hh + q] = 0.0;
                            c[4 * hh + q] = 32 * sa;
                        }
                    }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const double gv = r[c[q]];
                    if (q < 4) acc[0] = fma(vv[q], gv, acc[0]);
                    else acc[1] = fma(vv[q], gv, acc[1]);
                }
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                if (row[hh] < 0) continue;
                const double y = xi[hh] + acc[hh];
                wout[row[hh]] = y;
                const double ru = xi[hh] * si[hh];
                v[0] += xi[hh] * xi[hh];
                v[1] += y * xi[hh];
                v[2] += ru * ru;
            }
        }
    }
    cg_tail<FIRST>(v, act, S, B, part, gcnt, h);
}

// S of the graph-mode body for large systems: w = r + A^_off r and the dots, with the matrix
// and the own-row vectors STREAMED by TMA. One CTA per SM owns a contiguous range of
// kJdsRows-row tiles; its producer warp (one elected lane) issues per tile five bulk copies
// (values, int16 columns, row lengths + diagonal offsets, r, q) into a JNS-stage shared-memory ring
// guarded by full/empty mbarriers; JCW consumer warps take one 32-row slice each, read the
// jagged diagonals of their slice from shared memory (rows in descending length: diagonal k is
// lanes 0 .. cnt_k-1 at doff[k] + lane) and gather the neighbours' r: from the tile's own r
// slice in shared memory when the neighbour is in the tile (about 3/4 of the gathers with the
// 64-pixel bands of graph-mode systems), else through L1/L2 -- the gathers' 32-byte sectors
// were the largest share of the loop's L2 traffic.
// Bytes per iteration: 10 B per stored nonzero (no ELL padding) + 1.06 B/row of metadata +
// r, s read + w written; the async stream keeps ~JNS tiles of loads in flight per SM.
constexpr int JCW = kJdsRows / 32;  // consumer warps = slices per tile
constexpr int JNT = 32 * (JCW + 1);
constexpr int JNS = 6;
constexpr int JNS_M = 4;  // ring stages of the multi-RHS SpMV (larger stages: NR r slices)
constexpr int kUnroll = 8;  // CG iterations per WHILE body (graph mode; measured: x4 2.9 us, x8 2.2 us of WHILE gap per iteration)

struct JStage {
    double* val;
    uint8_t* col;
    uint8_t* meta;
    double* r;
    double* s;
};

template <bool FIRST, bool LEAN, int NS = JNS>
__global__ void __launch_bounds__(JNT, 1) k_gt(const RItem* __restrict__ items, int B, double* __restrict__ part,
                                            unsigned* __restrict__ gcnt, cudaGraphConditionalHandle h, int lsi) {
    extern __shared__ __align__(128) unsigned char jsm[];
    unsigned long long t_start = 0;
    if (g_loop_prof && threadIdx.x == 0) t_start = gtime();
    __shared__ __align__(8) uint64_t full[NS], empty[NS];
    __shared__ int2 tile_e[NS], tile_c[NS];  // entry / column-byte range of the tile in each stage
    const RItem& it = items[0];
    CgState* S = it.st;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tb = it.jpart[blockIdx.x], te = it.jpart[blockIdx.x + 1];  // this CTA's tiles
    const int maxe = it.jmaxe, kmax = it.jkmax, mb = it.jmbytes;
    const size_t stage_bytes = ((size_t)maxe * 12 + mb + 16 * kJdsRows + 127) & ~(size_t)127;
    auto stage = [&](int k) {  // r | q | values | columns | lengths + diagonal offsets
        unsigned char* b = jsm + (size_t)k * stage_bytes;
        JStage q;
        q.r = (double*)b;
        q.s = q.r + kJdsRows;
        q.val = q.s + kJdsRows;
        q.col = (uint8_t*)(q.val + maxe);
        q.meta = q.col + 4 * (size_t)maxe;
        return q;
    };
    if (threadIdx.x == 0) {
        for (int k = 0; k < NS; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], JCW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    // The matrix does not depend on the previous kernel: behind a programmatic edge (graph
    // body) this CTA is resident while k_gu still runs, and the producer already streams the
    // values, columns and metadata of its first NS tiles (expect_tx without an arrival keeps
    // each stage's phase open); r and q follow once the update kernel has completed.
    // no prefetch for the no-op tail of the unrolled body: active only goes 1 -> 0 inside one
    // graph launch, so a 0 read before the dependency wait is final (a stale 1 only prefetches)
    const bool live = FIRST || (LEAN ? *(volatile const int*)&it.ls[lsi].active : *(volatile const int*)&S->active);
    const int npre = live ? min(g_pdl_pre, te - tb) : 0;
    const uint64_t pol = matrix_policy();  // evict-first by default: keep the CG vectors L2-resident
    if (warp == JCW && lane == 0) {
        for (int i = 0; i < npre; ++i) {
            const int t = tb + i;
            const int e0 = it.jeb[t], e1 = it.jeb[t + 1], c0 = it.jcb[t], c1 = it.jcb[t + 1];
            const JStage q = stage(i);
            tile_e[i] = make_int2(e0, e1 - e0);
            tile_c[i] = make_int2(c0, c1 - c0);
            mbar_expect_tx(&full[i], (uint32_t)(e1 - e0) * 8u + (uint32_t)(c1 - c0) + (uint32_t)mb);
            bulk_g2s(q.meta, it.jmeta + (size_t)t * mb, (uint32_t)mb, &full[i]);
            if (e1 > e0) {
                mat_g2s(q.val, it.jval + e0, 8u * (e1 - e0), &full[i], pol);
                mat_g2s(q.col, it.jcol + c0, (uint32_t)(c1 - c0), &full[i], pol);
            }
        }
    }
    grid_dep_wait();
    const bool act = FIRST || (LEAN ? it.ls[lsi].active : S->active);
    // else the q stream and the residual monitor are skipped
    const bool nrho = FIRST || (LEAN ? it.ls[lsi].need_rho : S->need_rho);
    double v[3] = {0.0, 0.0, 0.0};
    if (!act && warp == JCW && lane == 0) {
        // nothing to compute: close the prefetched stages and let their copies land before exit
        for (int i = 0; i < npre; ++i) {
            mbar_arrive(&full[i]);
            mbar_wait(&full[i], 0);
        }
    }
    if (act) {
        if (warp == JCW) {
            // ---- producer: one elected lane streams the CTA's tiles into the ring
            if (lane == 0) {
                for (int i = 0; i < npre; ++i) {  // the prefetched stages: r (and q) only
                    const JStage q = stage(i);
                    const int t = tb + i;
                    mbar_arrive_expect_tx(&full[i], (nrho ? 16u : 8u) * kJdsRows);
                    bulk_g2s(q.r, it.r + (size_t)t * kJdsRows, 8 * kJdsRows, &full[i]);
                    if (nrho) bulk_g2s(q.s, it.q + (size_t)t * kJdsRows, 8 * kJdsRows, &full[i]);
                }
                int e0 = tb + npre < te ? it.jeb[tb + npre] : 0, c0 = tb + npre < te ? it.jcb[tb + npre] : 0;
                for (int t = tb + npre, i = npre; t < te; ++t, ++i) {
                    const int k = i % NS;
                    const int e1 = it.jeb[t + 1], c1 = it.jcb[t + 1];  // loaded before the wait
                    if (i >= NS) mbar_wait(&empty[k], ((i / NS) - 1) & 1);
                    const JStage q = stage(k);
                    const int ne = e1 - e0, nc = c1 - c0;
                    tile_e[k] = make_int2(e0, ne);
                    tile_c[k] = make_int2(c0, nc);
                    mbar_arrive_expect_tx(&full[k], (uint32_t)ne * 8u + (uint32_t)nc + (uint32_t)mb +
                                                        (nrho ? 16u : 8u) * kJdsRows);
                    bulk_g2s(q.r, it.r + (size_t)t * kJdsRows, 8 * kJdsRows, &full[k]);
                    if (nrho) bulk_g2s(q.s, it.q + (size_t)t * kJdsRows, 8 * kJdsRows, &full[k]);
                    bulk_g2s(q.meta, it.jmeta + (size_t)t * mb, (uint32_t)mb, &full[k]);
                    if (ne) {
                        mat_g2s(q.val, it.jval + e0, 8u * ne, &full[k], pol);
                        mat_g2s(q.col, it.jcol + c0, (uint32_t)nc, &full[k], pol);
                    }
                    e0 = e1;
                    c0 = c1;
                }
            }
        } else {
            // ---- consumers: warp = slice of the tile, lane = row (rows in descending length)
            const double* __restrict__ rg = it.r;
            double* __restrict__ wout = it.w;
            const int rl = 32 * warp + lane;
            for (int t = tb, i = 0; t < te; ++t, ++i) {
                const int k = i % NS;
                mbar_wait(&full[k], (i / NS) & 1);
                const JStage q = stage(k);
                const int row = t * kJdsRows + rl;
                const int len = q.meta[rl];
                const uint16_t* doff = (const uint16_t*)(q.meta + kJdsRows) + warp * kmax;
                const double xi = q.r[rl], qi = nrho ? q.s[rl] : 0.0;
                const int L = __shfl_sync(0xffffffffu, len, 0);  // lane 0 holds the longest row
                const bool wide = tile_c[k].y > 2 * tile_e[k].y;  // int32 columns in this tile
                const int16_t* c16 = (const int16_t*)q.col;
                const int32_t* c32 = (const int32_t*)q.col;
                const double* rt = rg + (int64_t)t * kJdsRows;
                const unsigned tile_lim = g_smem_gather ? (unsigned)kJdsRows : 0u;
                double acc = 0.0;
                for (int k0 = 0; k0 < L; k0 += 8) {
                    double vv[8], gv[8];
                    int c[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const bool a = k0 + u < len;
                        const int idx = (k0 + u < L ? doff[k0 + u] : 0) + lane;
                        vv[u] = a ? q.val[idx] : 0.0;
                        c[u] = a ? (wide ? c32[idx] : (int)c16[idx]) : rl;
                        FEMI_DCHECK(!a || idx < tile_e[k].y, 3);
                        FEMI_DCHECK((unsigned)c[u] < (unsigned)kJdsRows ||
                                        ((int64_t)t * kJdsRows + c[u] >= 0 &&
                                         (int64_t)t * kJdsRows + c[u] < (int64_t)it.ntile * kJdsRows),
                                    3);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)  // neighbours' r: this tile's slice from shared memory, else L1/L2
                        gv[u] = (unsigned)c[u] < tile_lim ? q.r[c[u]] : rt[c[u]];
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc = fma(vv[u], gv[u], acc);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[k]);
                if (row < it.n) {
                    const double y = xi + acc;
                    wout[row] = y;
                    const double ru = xi * qi;
                    v[0] += xi * xi;
                    v[1] += y * xi;
                    v[2] += ru * ru;
                }
            }
        }
    }
    const int it_prof = LEAN ? (FIRST ? 0 : it.ls[lsi].iters) : S->iters;
    if (g_loop_prof && act && it_prof < kLoopProfMax) {
        __syncthreads();  // profiling only: every warp of the CTA is done
        if (threadIdx.x == 0) {
            const unsigned long long t = gtime();
            if (it_prof == kCtaProfIt && blockIdx.x < 1024) {
                g_cta_prof[2 * blockIdx.x] = t_start;
                g_cta_prof[2 * blockIdx.x + 1] = t;
            }
            atomicMax(&g_loop_ts2[4 * it_prof], t_start);
            atomicMin(&g_loop_ts2[4 * it_prof + 1], t);
            atomicMax(&g_loop_ts2[4 * it_prof + 2], t);
        }
    }
    if constexpr (LEAN) {
        // lean tail: this CTA's partial dots (fixed warp order) to its slot; the next k_gur
        // sums the slots and advances the recurrence in every CTA
        if (act) cta_partials<JNT>(v, part + 4 * (size_t)blockIdx.x);
    } else {
        cg_tail<FIRST, JNT>(v, act, S, B, part, gcnt, h, (act && !FIRST) ? it_prof : -1, it.dmin);
    }
    if (g_loop_prof && act && !FIRST && threadIdx.x == 0) {
        if (it_prof < kLoopProfMax) atomicMax(&g_loop_ts2[4 * it_prof + 3], gtime());
        loop_stamp(1, it_prof, t_start);
    }
}

// ------------------------------------------------------------------ shared-matrix multi-RHS
// NR <= 4 right-hand sides on ONE large system (colour channels): one CG
// recurrence per RHS (own scalars, own convergence), but every iteration streams the matrix
// ONCE for all of them -- the TMA tile carries the NR r slices next to the shared values /
// columns / q, and each consumer lane gathers the NR neighbour values per nonzero. Per
// iteration 12 nnz + 4 (n+1) + 80 NR n algorithmic bytes instead of NR (12 nnz + ...).
template <int NR>
__global__ void __launch_bounds__(GNT) k_gum(const RItem* __restrict__ items) {
    // per RHS the same update as k_gu, x included in every other iteration only (its own
    // iteration count decides: even defers alpha_i p_i, odd applies both terms)
    double al[NR], be[NR], ap[NR];
    bool on[NR], lazy[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c) {
        const CgState* S = items[c].st;
        on[c] = S->active;
        al[c] = S->alpha;
        be[c] = S->beta;
        ap[c] = S->alpha_pend;
        lazy[c] = (S->iters & 1) == 0;
    }
    const int n = items[0].n, stride = gridDim.x * blockDim.x;
#pragma unroll
    for (int c = 0; c < NR; ++c) {
        if (!on[c]) continue;  // converged RHS keep x and r
        const RItem& it = items[c];
        double* __restrict__ r = it.r;
        const double* __restrict__ w = it.w;
        double* __restrict__ p = it.p;
        double* __restrict__ sv = it.sv;
        double* __restrict__ x = it.x;
        if (lazy[c]) {
            for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
                const double ri = r[i], wi = w[i], pi0 = p[i], si0 = sv[i];
                const double si = fma(be[c], si0, wi);
                p[i] = fma(be[c], pi0, ri);
                sv[i] = si;
                r[i] = fma(-al[c], si, ri);
            }
        } else {
            for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
                const double ri = r[i], wi = w[i], pi0 = p[i], si0 = sv[i], xi = x[i];
                const double pi = fma(be[c], pi0, ri), si = fma(be[c], si0, wi);
                p[i] = pi;
                sv[i] = si;
                x[i] = fma(al[c], pi, fma(ap[c], pi0, xi));
                r[i] = fma(-al[c], si, ri);
            }
        }
    }
}

// last-CTA reduction of NR x 3 dots (fixed order) and the NR recurrence steps
template <bool FIRST, int NR>
__device__ __forceinline__ void cg_tail_m(double (&v)[NR][3], const bool (&act)[NR], const RItem* __restrict__ items,
                                          double* __restrict__ part, cudaGraphConditionalHandle h, double dmin) {
    constexpr int NQ = 3 * NR;
    __shared__ double shm[NQ * (JNT / 32)];
    __shared__ int last;
    __shared__ int anyact[NR];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    CgState* S0 = items[0].st;
#pragma unroll
    for (int c = 0; c < NR; ++c)
#pragma unroll
        for (int q = 0; q < 3; ++q) v[c][q] = warp_sum_d(v[c][q]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int c = 0; c < NR; ++c)
#pragma unroll
            for (int q = 0; q < 3; ++q) shm[NQ * wid + 3 * c + q] = v[c][q];
    __syncthreads();
    constexpr int AT = JNT - 32;
    if (threadIdx.x == AT) {
        for (int k = 0; k < NQ; ++k) {
            double t = 0.0;
            for (int w = 0; w < JNT / 32; ++w) t += shm[NQ * w + k];
            part[NQ * blockIdx.x + k] = t;
        }
        last = atom_add_release_gpu(&S0->cnt[0], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    fence_acq_rel_gpu();
    double tot[NQ];
#pragma unroll
    for (int k = 0; k < NQ; ++k) tot[k] = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += JNT)
#pragma unroll
        for (int k = 0; k < NQ; ++k) tot[k] += __ldcg(part + NQ * b + k);
#pragma unroll
    for (int k = 0; k < NQ; ++k) tot[k] = warp_sum_d(tot[k]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NQ; ++k) shm[NQ * wid + k] = tot[k];
    __syncthreads();
    if (threadIdx.x < NR) {  // thread c advances RHS c
        const int c = threadIdx.x;
        CgState* S = items[c].st;
        double d[3] = {0.0, 0.0, 0.0};
        for (int w = 0; w < JNT / 32; ++w)
            for (int q = 0; q < 3; ++q) d[q] += shm[NQ * w + 3 * c + q];
        const int need = FIRST ? 1 : S->need_rho;
        if (!FIRST && act[c]) {  // the k_gum before this SpMV deferred its x term (even) or not
            S->x_pend = (S->iters & 1) == 0 ? 1 : 0;
            S->alpha_pend = S->alpha;
        }
        anyact[c] = cg_advance<FIRST>(S, act[c], d[0], d[1], d[2], dmin, S->bn2, S->tol2, S->rr, S->alpha, S->iters,
                                      S->max_iter, need);
    }
    __syncwarp();
    if (threadIdx.x == 0) {
        S0->cnt[0] = 0;
        int any = 0;
        for (int c = 0; c < NR; ++c) any |= anyact[c];
        if (h) cudaGraphSetConditional(h, any ? 1u : 0u);
    }
}

template <int NR, bool FIRST>
__global__ void __launch_bounds__(JNT, 1) k_gtm(const RItem* __restrict__ items, double* __restrict__ part,
                                             cudaGraphConditionalHandle h) {
    extern __shared__ __align__(128) unsigned char jsm[];
    __shared__ __align__(8) uint64_t full[JNS_M], empty[JNS_M];
    __shared__ int2 tile_e[JNS_M], tile_c[JNS_M];
    const RItem& it = items[0];  // the shared matrix and q
    bool act[NR];
    bool anyon = false, nrho = FIRST;
#pragma unroll
    for (int c = 0; c < NR; ++c) {
        act[c] = FIRST || items[c].st->active;
        anyon |= act[c];
        nrho |= (bool)items[c].st->need_rho;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tb = it.jpart[blockIdx.x], te = it.jpart[blockIdx.x + 1];
    const int maxe = it.jmaxe, kmax = it.jkmax, mb = it.jmbytes;
    const size_t stage_bytes = ((size_t)maxe * 12 + mb + 8 * (NR + 1) * kJdsRows + 127) & ~(size_t)127;
    // stage: r_0 .. r_{NR-1} | q | values | columns | lengths + diagonal offsets
    auto sbase = [&](int k) { return jsm + (size_t)k * stage_bytes; };
    if (threadIdx.x == 0) {
        for (int k = 0; k < JNS_M; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], JCW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    double v[NR][3];
#pragma unroll
    for (int c = 0; c < NR; ++c) v[c][0] = v[c][1] = v[c][2] = 0.0;
    if (anyon) {
        if (warp == JCW) {
            if (lane == 0) {
                int e0 = tb < te ? it.jeb[tb] : 0, c0 = tb < te ? it.jcb[tb] : 0;
                const uint64_t pol = matrix_policy();
                for (int t = tb, i = 0; t < te; ++t, ++i) {
                    const int k = i % JNS_M;
                    const int e1 = it.jeb[t + 1], c1 = it.jcb[t + 1];
                    if (i >= JNS_M) mbar_wait(&empty[k], ((i / JNS_M) - 1) & 1);
                    unsigned char* b = sbase(k);
                    double* qs = (double*)b + NR * kJdsRows;
                    double* vs = qs + kJdsRows;
                    uint8_t* cs = (uint8_t*)(vs + maxe);
                    uint8_t* ms = cs + 4 * (size_t)maxe;
                    const int ne = e1 - e0, nc = c1 - c0;
                    tile_e[k] = make_int2(e0, ne);
                    tile_c[k] = make_int2(c0, nc);
                    mbar_arrive_expect_tx(&full[k], (uint32_t)ne * 8u + (uint32_t)nc + (uint32_t)mb +
                                                        (NR + (nrho ? 1u : 0u)) * 8u * kJdsRows);
#pragma unroll
                    for (int c = 0; c < NR; ++c)
                        bulk_g2s((double*)b + c * kJdsRows, items[c].r + (size_t)t * kJdsRows, 8 * kJdsRows, &full[k]);
                    if (nrho) bulk_g2s(qs, it.q + (size_t)t * kJdsRows, 8 * kJdsRows, &full[k]);
                    bulk_g2s(ms, it.jmeta + (size_t)t * mb, (uint32_t)mb, &full[k]);
                    if (ne) {
                        bulk_g2s_hint(vs, it.jval + e0, 8u * ne, &full[k], pol);
                        bulk_g2s_hint(cs, it.jcol + c0, (uint32_t)nc, &full[k], pol);
                    }
                    e0 = e1;
                    c0 = c1;
                }
            }
        } else {
            const int rl = 32 * warp + lane;
            const double* rg[NR];
            double* wo[NR];
#pragma unroll
            for (int c = 0; c < NR; ++c) {
                rg[c] = items[c].r;
                wo[c] = items[c].w;
            }
            for (int t = tb, i = 0; t < te; ++t, ++i) {
                const int k = i % JNS_M;
                mbar_wait(&full[k], (i / JNS_M) & 1);
                unsigned char* b = sbase(k);
                const double* rs = (const double*)b;
                const double* qs = rs + NR * kJdsRows;
                const double* vs = qs + kJdsRows;
                const uint8_t* cs = (const uint8_t*)(vs + maxe);
                const uint8_t* ms = cs + 4 * (size_t)maxe;
                const int row = t * kJdsRows + rl;
                const int len = ms[rl];
                const uint16_t* doff = (const uint16_t*)(ms + kJdsRows) + warp * kmax;
                const int L = __shfl_sync(0xffffffffu, len, 0);
                const bool wide = tile_c[k].y > 2 * tile_e[k].y;
                const int16_t* c16 = (const int16_t*)cs;
                const int32_t* c32 = (const int32_t*)cs;
                const size_t t0 = (size_t)t * kJdsRows;
                double acc[NR];
#pragma unroll
                for (int c = 0; c < NR; ++c) acc[c] = 0.0;
                for (int k0 = 0; k0 < L; k0 += 4) {
                    double vv[4];
                    int cc[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const bool a = k0 + u < len;
                        const int idx = (k0 + u < L ? doff[k0 + u] : 0) + lane;
                        vv[u] = a ? vs[idx] : 0.0;
                        cc[u] = a ? (wide ? c32[idx] : (int)c16[idx]) : rl;
                    }
                    double gv[NR][4];
#pragma unroll
                    for (int c = 0; c < NR; ++c)
#pragma unroll
                        for (int u = 0; u < 4; ++u)  // in-tile neighbours from the staged r slices
                            gv[c][u] = (unsigned)cc[u] < (unsigned)kJdsRows ? rs[c * kJdsRows + cc[u]]
                                                                            : rg[c][t0 + cc[u]];
#pragma unroll
                    for (int c = 0; c < NR; ++c)
#pragma unroll
                        for (int u = 0; u < 4; ++u) acc[c] = fma(vv[u], gv[c][u], acc[c]);
                }
                const double qi = nrho ? qs[rl] : 0.0;
                double xi[NR];
#pragma unroll
                for (int c = 0; c < NR; ++c) xi[c] = rs[c * kJdsRows + rl];
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[k]);
                if (row < it.n) {
#pragma unroll
                    for (int c = 0; c < NR; ++c) {
                        const double y = xi[c] + acc[c];
                        wo[c][row] = y;
                        const double ru = xi[c] * qi;
                        v[c][0] += xi[c] * xi[c];
                        v[c][1] += y * xi[c];
                        v[c][2] += ru * ru;
                    }
                }
            }
        }
    }
    cg_tail_m<FIRST, NR>(v, act, items, part, h, it.dmin);
}

// min over i of q_i^2 = diag(A_uu)_i (order-preserving bits of positive doubles)
__global__ void k_qmin(int64_t n, const double* __restrict__ q, unsigned long long* __restrict__ out) {
    unsigned long long m = ~0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = min(m, (unsigned long long)__double_as_longlong(q[i] * q[i]));
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMin(out, m);
}

struct GraphCache {
    void* ws = nullptr;
    RItem* d_items = nullptr;
    CgState* d_state = nullptr;
    unsigned* d_cnt = nullptr;  // [0,1]: init/true-res counters; [2,3]: loop condition counters
    double* d_part = nullptr;
    cudaGraphExec_t main = nullptr, restart = nullptr;
    cudaGraphExec_t restart_if = nullptr;  // asynchronous solves: the restart round gated on the device
    RItem item{};
    RItem item_dev{};  // what d_items holds (skip the upload when unchanged)
    bool item_dev_valid = false;
    int gs_blocks = 0, gx = 0, gt_blocks = 0;
    unsigned gt_smem = 0;  // > 0: the SpMV is the TMA-streamed k_gt (JDS layout); else SELL k_gs
    int gt_ns = JNS;       // ring stages of k_gt (FEMI_JNS=8: the deeper ring when it fits)
    const void* mat_base = nullptr;  // the SpMV's matrix stream (one allocation) and its size
    size_t mat_bytes = 0;
    size_t persist_bytes = 0;        // > 0: k_gt nodes carry a persisting L2 access-policy window
};

struct Workspace {
    void* base = nullptr;
    cudaStream_t st = nullptr;
    ~Workspace() {
        if (base) cudaFreeAsync(base, st);
    }
};

int g_l2pol_host = 0;
int g_smem_optin = -1;
int g_occ_grid = -1;
int g_nsm = 0;
bool g_timers = false;
int g_nvec_max = 3;
int g_shape = 1;

}  // namespace

namespace {

femi_status add_kernel(cudaGraph_t gr, cudaGraphNode_t* dep, void* fn, dim3 grid, dim3 block, void** args,
                       cudaGraphNode_t* out, unsigned smem = 0) {
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeKernel;
    p.kernel.func = fn;
    p.kernel.gridDim = grid;
    p.kernel.blockDim = block;
    p.kernel.sharedMemBytes = smem;
    p.kernel.kernelParams = args;
    FEMI_CUDA(cudaGraphAddNode(out, gr, dep, dep ? 1 : 0, &p));
    return FEMI_OK;
}

// the same behind a programmatic edge: the node may launch once every block of `dep` has
// started (it must grid_dep_wait() before touching dep's results). FEMI_NO_PDL=1 turns the
// edges into ordinary ones.
femi_status add_kernel_pdl(cudaGraph_t gr, cudaGraphNode_t* dep, void* fn, dim3 grid, dim3 block, void** args,
                           cudaGraphNode_t* out, unsigned smem = 0) {
    static const bool off = std::getenv("FEMI_NO_PDL") != nullptr;
    if (!dep || off) return add_kernel(gr, dep, fn, grid, block, args, out, smem);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeKernel;
    p.kernel.func = fn;
    p.kernel.gridDim = grid;
    p.kernel.blockDim = block;
    p.kernel.sharedMemBytes = smem;
    p.kernel.kernelParams = args;
    cudaGraphEdgeData e = {};
    e.from_port = cudaGraphKernelNodePortLaunchCompletion;
    e.type = cudaGraphDependencyTypeProgrammatic;
    FEMI_CUDA(cudaGraphAddNode_v2(out, gr, dep, &e, 1, &p));
    return FEMI_OK;
}

// main:    reset -> minmax -> rhs -> init_x -> zero_ps -> init_r -> SpMV<FIRST> ->
//          WHILE{ kUnroll x (k_gu -> SpMV) } -> finalize -> true_res -> copy_g
// restart: zero_ps -> SpMV<FIRST> -> WHILE{...} -> finalize -> true_res -> copy_g
// (SpMV = k_gt on the JDS tiles, or k_gs on the SELL slices when the JDS layout is absent)
femi_status build_graph(GraphCache& C, bool restart, cudaGraphExec_t* out, bool gated = false) {
    cudaGraph_t top;
    FEMI_CUDA(cudaGraphCreate(&top, 0));
    cudaGraph_t gr = top;
    if (gated) {  // [k_restart_cond] -> IF (true residual misses rtol) { the restart graph's nodes }
        cudaGraphConditionalHandle hif;
        FEMI_CUDA(cudaGraphConditionalHandleCreate(&hif, top, 0u, cudaGraphCondAssignDefault));
        RItem* di0 = C.d_items;
        void* a_rc[2] = {&di0, &hif};
        cudaGraphNode_t nc, nif;
        const femi_status fs = add_kernel(top, nullptr, (void*)k_restart_cond, dim3(1), dim3(32), a_rc, &nc);
        if (fs != FEMI_OK) return fs;
        cudaGraphNodeParams ip = {};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = hif;
        ip.conditional.type = cudaGraphCondTypeIf;
        ip.conditional.size = 1;
        FEMI_CUDA(cudaGraphAddNode(&nif, top, &nc, 1, &ip));
        gr = ip.conditional.phGraph_out[0];
    }
    const bool tma = C.gt_smem > 0;  // TMA SpMV: lean tail (k_gur ends the loop); SELL: cg_tail does
    cudaGraphConditionalHandle h;
    FEMI_CUDA(cudaGraphConditionalHandleCreate(&h, top, tma ? 1u : 0u, cudaGraphCondAssignDefault));
    RItem* di = C.d_items;
    int one = 1;
    double* part = C.d_part;
    unsigned* cnt0 = C.d_cnt;
    unsigned* cnt1 = C.d_cnt + 1;
    unsigned* gcnt = C.d_cnt + 2;
    void* a_items[1] = {&di};
    void* a_reset[2] = {&one, &di};
    void* a_cnt0[2] = {&di, &cnt0};
    void* a_gs[5] = {&di, &one, &part, &gcnt, &h};
    int lsi0 = 0;
    void* a_gt0[6] = {&di, &one, &part, &gcnt, &h, &lsi0};
    const dim3 gk(C.gx, 1), bk(KNT);
    cudaGraphNode_t prev = nullptr, nd;
    cudaGraphNode_t* dep = nullptr;
    auto chain = [&](void* fn, dim3 gg, dim3 bb, void** args, unsigned smem = 0) -> femi_status {
        femi_status s = add_kernel(gr, dep, fn, gg, bb, args, &nd, smem);
        prev = nd;
        dep = &prev;
        return s;
    };
    void* spmv_first = tma ? (C.gt_ns == 8 ? (void*)k_gt<true, true, 8> : (void*)k_gt<true, true>) : (void*)k_gs<true>;
    void* spmv = tma ? (C.gt_ns == 8 ? (void*)k_gt<false, true, 8> : (void*)k_gt<false, true>) : (void*)k_gs<false>;
    const dim3 gsp(tma ? C.gt_blocks : C.gs_blocks), bsp(tma ? JNT : GNT);
    const unsigned ssp = tma ? C.gt_smem : 0;
    femi_status s = FEMI_OK;
    if (!restart) {
        if ((s = chain((void*)k_reset_items, dim3(1), dim3(32), a_reset))) return s;
        int tw1 = 1, tw0 = 0;
        void* a_f1[2] = {&di, &tw1};
        void* a_f0[2] = {&di, &tw0};
        if ((s = chain((void*)k_pro1, gk, bk, a_cnt0))) return s;  // minmax + fill hop 1 + b
        if ((s = chain((void*)k_x0_fill2, gk, bk, a_f1))) return s;
        if ((s = chain((void*)k_x0_fill2, gk, bk, a_f0))) return s;
        if ((s = chain((void*)k_pro2, gk, bk, a_items))) return s;  // fill end + x^0 + p = s = 0 + r^0
    } else {
        if ((s = chain((void*)k_zero_ps, gk, bk, a_items))) return s;
    }
    if ((s = chain(spmv_first, gsp, bsp, tma ? a_gt0 : a_gs, ssp))) return s;
    // FEMI_L2POL=3: the matrix stream (46 MB at C5) persists in L2 across iterations through an
    // access-policy window on the SpMV nodes; the vectors share the rest of the 126 MB
    auto persist = [&](cudaGraphNode_t node) -> femi_status {
        if (!tma || C.persist_bytes == 0) return FEMI_OK;
        cudaKernelNodeAttrValue v = {};
        v.accessPolicyWindow.base_ptr = const_cast<void*>(C.mat_base);
        v.accessPolicyWindow.num_bytes = C.mat_bytes;
        v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)C.persist_bytes / (double)C.mat_bytes);
        v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        FEMI_CUDA(cudaGraphKernelNodeSetAttribute(node, cudaKernelNodeAttributeAccessPolicyWindow, &v));
        return FEMI_OK;
    };
    if ((s = persist(nd))) return s;
    {
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        FEMI_CUDA(cudaGraphAddNode(&nd, gr, dep, 1, &cp));
        prev = nd;
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        // kUnroll iterations per body: the WHILE re-evaluation costs several us; kernels after
        // convergence return at once (S->active == 0)
        cudaGraphNode_t bprev = nullptr, u, sn;
        // 4 CTAs per SM: measured best at C5 (1184: 3.94 ms, 888: 3.92, 740: 3.97, 592: 3.88,
        // 444: 4.04 per solve) -- with PDL the next k_gt CTA shares the SM with k_gu's CTAs
        int gu_ctas = std::min(C.gx * 2, 4 * 148);
        if (const char* e = std::getenv("FEMI_GU_CTAS")) gu_ctas = std::max(1, std::atoi(e));
        const dim3 gu(gu_ctas);
        // inside the body, k_gu -> k_gt -> k_gu ... are programmatic edges (k_gt streams its
        // first matrix tiles while k_gu runs; each waits in grid_dep_wait for its inputs)
        for (int k = 0; k < kUnroll; ++k) {
            if (tma) {
                // lean tail: k_gur (reduce the SpMV partials + update, body slot parity k & 1)
                // -> k_gt (reads the scalars k_gur published in ls[(k + 1) & 1])
                int par = k & 1, lsi = (k + 1) & 1, np = C.gt_blocks;
                void* a_gur[5] = {&di, &part, &np, &par, &h};
                void* a_gt[6] = {&di, &one, &part, &gcnt, &h, &lsi};
                if ((s = add_kernel_pdl(body, bprev ? &bprev : nullptr, (void*)k_gur, gu, dim3(GRT), a_gur, &u)))
                    return s;
                if ((s = add_kernel_pdl(body, &u, spmv, gsp, bsp, a_gt, &sn, ssp))) return s;
                if ((s = persist(sn))) return s;
            } else {
                if ((s = add_kernel(body, bprev ? &bprev : nullptr, (void*)k_gu, gu, dim3(GNT), a_items, &u)))
                    return s;
                if ((s = add_kernel(body, &u, spmv, gsp, bsp, a_gs, &sn, ssp))) return s;
            }
            bprev = sn;
        }
    }
    const int* nogate = nullptr;
    void* a_tres[3] = {&di, &cnt1, &nogate};
    if ((s = chain((void*)k_finalize_g, gk, bk, a_items))) return s;  // x -> u_vert and the mask entries
    if ((s = chain((void*)k_true_res, gk, bk, a_tres))) return s;
    FEMI_CUDA(cudaGraphInstantiate(out, top, 0));
    FEMI_CUDA(cudaGraphDestroy(top));
    return FEMI_OK;
}


// profiling aid (FEMI_PCG_KBENCH): an empty kernel, to measure the fixed launch cost of the
// k_gt configuration (148 x 544 threads, with and without its dynamic shared memory)
__global__ void k_probe(int* p) {
    extern __shared__ unsigned char probe_sm[];
    if (p && threadIdx.x == 0 && blockIdx.x == 0) *p = (int)probe_sm[0];
}

// FEMI_LOOP_PROF=1: per-iteration timeline of the graph loop from %globaltimer stamps
femi_status loop_prof_begin(cudaStream_t st) {
    std::vector<unsigned long long> init(4 * kLoopProfMax);
    for (int k = 0; k < kLoopProfMax; ++k) {
        init[4 * k] = init[4 * k + 2] = ~0ull;
        init[4 * k + 1] = init[4 * k + 3] = 0ull;
    }
    FEMI_CUDA(cudaMemcpyToSymbolAsync(g_loop_ts, init.data(), sizeof(unsigned long long) * init.size(), 0,
                                      cudaMemcpyHostToDevice, st));
    for (int k = 0; k < kLoopProfMax; ++k) {
        init[4 * k] = 0ull;
        init[4 * k + 1] = ~0ull;
        init[4 * k + 2] = init[4 * k + 3] = 0ull;
    }
    FEMI_CUDA(cudaMemcpyToSymbolAsync(g_loop_ts2, init.data(), sizeof(unsigned long long) * init.size(), 0,
                                      cudaMemcpyHostToDevice, st));
    const int on = 1;
    FEMI_CUDA(cudaMemcpyToSymbolAsync(g_loop_prof, &on, sizeof(int), 0, cudaMemcpyHostToDevice, st));
    return FEMI_OK;
}

femi_status loop_prof_end(cudaStream_t st) {
    const int off = 0;
    std::vector<unsigned long long> ts(4 * kLoopProfMax), t2(4 * kLoopProfMax), t3(4 * kLoopProfMax);
    FEMI_CUDA(cudaMemcpyToSymbolAsync(g_loop_prof, &off, sizeof(int), 0, cudaMemcpyHostToDevice, st));
    FEMI_CUDA(cudaMemcpyFromSymbolAsync(ts.data(), g_loop_ts, sizeof(unsigned long long) * ts.size(), 0,
                                        cudaMemcpyDeviceToHost, st));
    FEMI_CUDA(cudaMemcpyFromSymbolAsync(t2.data(), g_loop_ts2, sizeof(unsigned long long) * t2.size(), 0,
                                        cudaMemcpyDeviceToHost, st));
    FEMI_CUDA(cudaMemcpyFromSymbolAsync(t3.data(), g_tail_ts, sizeof(unsigned long long) * t3.size(), 0,
                                        cudaMemcpyDeviceToHost, st));
    std::vector<unsigned long long> cp(2 * 1024);
    FEMI_CUDA(cudaMemcpyFromSymbolAsync(cp.data(), g_cta_prof, sizeof(unsigned long long) * cp.size(), 0,
                                        cudaMemcpyDeviceToHost, st));
    FEMI_CUDA(cudaStreamSynchronize(st));
    if (std::getenv("FEMI_CTA_PROF")) {
        unsigned long long t0 = ~0ull;
        for (int b = 0; b < 1024; ++b)
            if (cp[2 * b]) t0 = std::min(t0, cp[2 * b]);
        std::fprintf(stderr, "[femi cta] iteration %d: cta start_us end_us\n", kCtaProfIt);
        for (int b = 0; b < 1024; ++b)
            if (cp[2 * b])
                std::fprintf(stderr, "[femi cta] %d %.3f %.3f\n", b, (cp[2 * b] - t0) / 1e3, (cp[2 * b + 1] - t0) / 1e3);
    }
    double su = 0, sg = 0, g1 = 0, g2 = 0, c0 = 0, c1 = 0, c2 = 0, tA = 0, tB = 0;
    int cnt = 0, ctail = 0;  // ctail: iterations with last-CTA tail stamps (not the lean tail)
    for (int k = 1; k + 1 < kLoopProfMax; ++k) {
        const unsigned long long* a = &ts[4 * k];
        const unsigned long long* nx = &ts[4 * (k + 1)];
        if (a[1] == 0 || a[3] == 0 || nx[1] == 0) break;
        su += (double)(a[1] - a[0]);
        sg += (double)(a[3] - a[2]);
        g1 += (double)a[2] - (double)a[1];
        g2 += (double)nx[0] - (double)a[3];
        c0 += (double)t2[4 * k + 1] - (double)a[2];
        c1 += (double)t2[4 * k + 2] - (double)a[2];
        c2 += (double)t2[4 * k + 3] - (double)a[2];
        if (t3[4 * k] && t3[4 * k + 1]) {
            tA += (double)t3[4 * k] - (double)a[2];
            tB += (double)t3[4 * k + 1] - (double)a[2];
            ++ctail;
        }
        ++cnt;
    }
    if (cnt) {
        std::fprintf(stderr,
                     "[femi loop] %d iterations: k_gu span %.2f us, gap %.2f, SpMV span %.2f us, gap %.2f -> %.2f "
                     "us/iteration | SpMV from first CTA start: first CTA done +%.2f, last CTA done +%.2f",
                     cnt, su / cnt / 1e3, g1 / cnt / 1e3, sg / cnt / 1e3, g2 / cnt / 1e3,
                     (su + sg + g1 + g2) / cnt / 1e3, c0 / cnt / 1e3, c1 / cnt / 1e3);
        if (ctail)  // last-CTA tail only (the lean tail has no arrival counter)
            std::fprintf(stderr, ", last CTA arrival +%.2f, partials summed +%.2f", tA / ctail / 1e3,
                         tB / ctail / 1e3);
        std::fprintf(stderr, ", last CTA out +%.2f\n", c2 / cnt / 1e3);
    }
    return FEMI_OK;
}

// Tiles -> k_gt CTAs: contiguous ranges of equal tile counts. (Measured at C5 with
// FEMI_CTA_PROF: the CTA times correlate 0.8 with the entry counts, yet a split weighted by
// cost(tile) = a + stored entries was slower for every a tried -- +0.02 to +0.19 ms per solve:
// the spread follows the image region, not the entry count -- so it was removed.)
femi_status tile_split(const femi_system_s* S, int nblocks, std::vector<int32_t>& jpart) {
    const int nt = S->jds_ntile;
    jpart.assign(nblocks + 1, 0);
    for (int b = 0; b <= nblocks; ++b) jpart[b] = (int)((int64_t)nt * b / nblocks);
    return FEMI_OK;
}

femi_status graph_solve(femi_system_s* S, const double* g, const double* bin, double* u_vert,
                        const femi_cg_opts& o, int32_t* iters, double* relres, cudaStream_t st,
                        int64_t* total_iters, DevStats* ds = nullptr) {
    static int pre_set_dev = -1;  // __device__ switches live per device
    int cur_dev = 0;
    FEMI_CUDA(cudaGetDevice(&cur_dev));
    if (pre_set_dev != cur_dev) {
        if (const char* e = std::getenv("FEMI_PDL_PRE")) {
            const int v = std::max(0, std::min(JNS, std::atoi(e)));
            FEMI_CUDA(cudaMemcpyToSymbol(g_pdl_pre, &v, sizeof(int)));
        }
        if (const char* e = std::getenv("FEMI_L2POL")) {
            const int v = std::atoi(e);
            FEMI_CUDA(cudaMemcpyToSymbol(g_l2pol, &v, sizeof(int)));
            g_l2pol_host = v;
        }
        if (const char* e = std::getenv("FEMI_SMEM_GATHER")) {
            const int v = std::atoi(e) ? 1 : 0;
            FEMI_CUDA(cudaMemcpyToSymbol(g_smem_gather, &v, sizeof(int)));
        }
        pre_set_dev = cur_dev;
    }
    GraphCache* C = (GraphCache*)S->scratch;
    const int64_t n = S->n_u;
    if (!C) {
        C = new GraphCache();
        const int nsl = (int)((n + 31) / 32);
        // one row per thread for the prologue/epilogue kernels (memory-level parallelism)
        C->gx = (int)std::max<int64_t>(1, std::min<int64_t>((n + KNT - 1) / KNT, 148 * 16));
        C->gs_blocks = (int)std::max<int64_t>(1, std::min<int64_t>((nsl + 2 * (GNT / 32) - 1) / (2 * (GNT / 32)),
                                                                   148 * 8));
        auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
        const size_t vb = al(sizeof(double) * std::max<int64_t>(n + 1, (int64_t)S->jds_ntile * kJdsRows));
        std::vector<int32_t> jpart;
        if (S->jds_ntile > 0 && std::getenv("FEMI_PCG_NOTMA") == nullptr) {
            const size_t stage_bytes =
                ((size_t)S->jds_maxe * 12 + S->jds_meta_bytes + 16 * kJdsRows + 127) & ~(size_t)127;
            int dev = 0, nsm = 0, optin = 0;
            FEMI_CUDA(cudaGetDevice(&dev));
            FEMI_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
            FEMI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
            if (JNS * stage_bytes + 4096 <= (size_t)optin) {
                C->gt_smem = (unsigned)(JNS * stage_bytes);
                if (const char* e = std::getenv("FEMI_JNS"))
                    if (std::atoi(e) == 8 && 8 * stage_bytes + 4096 <= (size_t)optin) {
                        C->gt_ns = 8;
                        C->gt_smem = (unsigned)(8 * stage_bytes);
                        for (const void* fn : {(const void*)k_gt<false, true, 8>, (const void*)k_gt<true, true, 8>})
                            FEMI_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           (int)C->gt_smem));
                    }
                if (std::getenv("FEMI_DEBUG"))
                    std::fprintf(stderr, "[femi] k_gt stage %zu B x %d stages (optin %d)\n", stage_bytes, C->gt_ns, optin);
                C->gt_blocks = std::max(1, std::min(nsm, S->jds_ntile));
                for (const void* fn : {(const void*)k_gt<false, true>, (const void*)k_gt<true, true>,
                                       (const void*)k_gt<false, false>})
                    FEMI_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)(JNS * stage_bytes)));
                femi_status ts = tile_split(S, C->gt_blocks, jpart);
                if (ts != FEMI_OK) return ts;
            }
        }
        const int pb = std::max(C->gs_blocks, C->gt_blocks);
        const size_t bytes = al(sizeof(int32_t) * (jpart.size() + 1)) + al(sizeof(RItem)) + al(sizeof(CgState)) +
                             al(sizeof(LoopState) * 2) +
                             al(sizeof(unsigned) * 4) + al(sizeof(double) * 8 * pb) + al(sizeof(double) * C->gx) +
                             6 * vb;
        FEMI_CUDA(cudaMalloc(&C->ws, bytes));
        char* cur = (char*)C->ws;
        auto take = [&](size_t x) {
            char* p = cur;
            cur += al(x);
            return p;
        };
        C->d_items = (RItem*)take(sizeof(RItem));
        int32_t* d_jpart = (int32_t*)take(sizeof(int32_t) * (jpart.size() + 1));
        if (!jpart.empty())
            FEMI_CUDA(cudaMemcpy(d_jpart, jpart.data(), sizeof(int32_t) * jpart.size(), cudaMemcpyHostToDevice));
        C->d_state = (CgState*)take(sizeof(CgState));
        LoopState* d_ls = (LoopState*)take(sizeof(LoopState) * 2);
        C->d_cnt = (unsigned*)take(sizeof(unsigned) * 4);
        C->d_part = (double*)take(sizeof(double) * 8 * pb);
        RItem& it = C->item;
        it.red = (double*)take(sizeof(double) * C->gx);
        it.b = (double*)take(vb);
        it.x = (double*)take(vb);
        it.r = (double*)take(vb);
        it.w = (double*)take(vb);
        it.p = (double*)take(vb);
        it.sv = (double*)take(vb);
        C->mat_base = S->jds_val;
        C->mat_bytes = S->jds_block_bytes;
        if (g_l2pol_host == 3 && C->gt_smem > 0 && C->mat_bytes > 0) {
            int dev = 0, maxp = 0, maxw = 0;
            FEMI_CUDA(cudaGetDevice(&dev));
            FEMI_CUDA(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
            FEMI_CUDA(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev));
            C->mat_bytes = std::min(C->mat_bytes, (size_t)maxw);
            C->persist_bytes = std::min(C->mat_bytes, (size_t)maxp);
            FEMI_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, C->persist_bytes));
            if (std::getenv("FEMI_DEBUG"))
                std::fprintf(stderr, "[femi] L2 persisting window %zu B of %zu (max persisting %d, max window %d)\n",
                             C->persist_bytes, C->mat_bytes, maxp, maxw);
        }
        it.jval = S->jds_val;
        it.jcol = S->jds_col;
        it.jmeta = S->jds_meta;
        it.jeb = S->jds_eb;
        it.jcb = S->jds_cb;
        it.ntile = S->jds_ntile;
        it.jmaxe = S->jds_maxe;
        it.jkmax = S->jds_kmax;
        it.jmbytes = S->jds_meta_bytes;
        it.jpart = d_jpart;
        it.dmin = 0.0;
        if (n > 0) {  // dmin = min_i diag(A_uu)_i, for skipping the residual monitor far from rtol
            unsigned long long* d_m = nullptr;
            unsigned long long h_m = ~0ull;
            FEMI_CUDA(cudaMallocAsync(&d_m, sizeof(unsigned long long), st));
            FEMI_CUDA(cudaMemcpyAsync(d_m, &h_m, sizeof(h_m), cudaMemcpyHostToDevice, st));
            k_qmin<<<296, 256, 0, st>>>(n, S->q_int, d_m);
            FEMI_CUDA(cudaMemcpyAsync(&h_m, d_m, sizeof(h_m), cudaMemcpyDeviceToHost, st));
            FEMI_CUDA(cudaFreeAsync(d_m, st));
            FEMI_CUDA(cudaStreamSynchronize(st));
            double dm;
            std::memcpy(&dm, &h_m, sizeof(dm));
            if (std::isfinite(dm) && dm > 0.0) it.dmin = dm * (1.0 - 1e-12);
        }
        it.inv = S->sell_inv;
        it.len = S->sell_len;
        it.base = S->sell_base;
        it.val = S->sell_val;
        it.c16 = S->sell_c16;
        it.c32 = S->sell_c32;
        it.s = S->s_int;
        it.q = S->q_int;
        it.urp = S->uuI_rowptr;
        it.uci = S->uuI_col;
        it.uav = S->uuI_val;
        it.krp = S->ukI_rowptr;
        it.kci = S->ukI_col;
        it.kav = S->ukI_val;
        it.part = nullptr;
        it.st = C->d_state;
        it.ls = C->gt_smem > 0 ? d_ls : nullptr;
        it.n = (int32_t)n;
        it.m = (int32_t)S->m;
        it.cta0 = 0;
        it.ncta = 1;
        it.nwin = S->nwin;
        FEMI_CUDA(cudaMemsetAsync(C->d_cnt, 0, sizeof(unsigned) * 4, st));
        femi_status s = build_graph(*C, false, &C->main);
        if (s == FEMI_OK) s = build_graph(*C, true, &C->restart);
        if (s != FEMI_OK) {  // publish the cache only once both graphs are instantiated
            if (C->main) cudaGraphExecDestroy(C->main);
            if (C->restart) cudaGraphExecDestroy(C->restart);
            cudaFree(C->ws);
            delete C;
            return s;
        }
        S->scratch = C;
    }
    S->last_path = C->gt_smem > 0 ? FEMI_PATH_GRAPH_TMA : FEMI_PATH_GRAPH_SELL;
    RItem it = C->item;
    it.g = g;
    it.bin = bin;
    it.u_vert = u_vert;
    it.x0mode = (g == nullptr && (o.x0 == 1 || o.x0 == 3)) ? 0 : o.x0;
    it.rtol = o.rtol;
    it.max_iter = o.max_iter;
    // the device copy of the item is rewritten only when the arguments changed (repeated solves of
    // one system -- the bench steps, a tonal loop's same-kind solves -- skip the copy)
    if (!C->item_dev_valid || std::memcmp(&C->item_dev, &it, sizeof(RItem)) != 0) {
        FEMI_CUDA(cudaMemcpyAsync(C->d_items, &it, sizeof(RItem), cudaMemcpyHostToDevice, st));
        C->item_dev = it;
        C->item_dev_valid = true;
    }
    static const bool loop_prof = std::getenv("FEMI_LOOP_PROF") != nullptr;
    if (loop_prof && !ds) {
        const femi_status ps = loop_prof_begin(st);
        if (ps != FEMI_OK) return ps;
    }
    FEMI_CUDA(cudaGraphLaunch(C->main, st));
    count_launches(10);
    if (ds) {  // asynchronous: the restart round gated on the device, statistics on the device
        if (!C->restart_if) {
            const femi_status bs = build_graph(*C, true, &C->restart_if, true);
            if (bs != FEMI_OK) return bs;
        }
        FEMI_CUDA(cudaGraphLaunch(C->restart_if, st));
        k_stats<<<1, 32, 0, st>>>(1, C->d_items, ds);
        count_launches(2 + 2 * (int64_t)kUnroll);
        FEMI_CUDA(cudaGetLastError());
        return FEMI_OK;
    }
    if (loop_prof) {
        const femi_status ps = loop_prof_end(st);
        if (ps != FEMI_OK) return ps;
        if (std::getenv("FEMI_CTA_PROF") && S->jds_ntile > 0) {  // entries per k_gt CTA (static split)
            std::vector<int32_t> eb(S->jds_ntile + 1), jp;
            FEMI_CUDA(cudaMemcpy(eb.data(), S->jds_eb, sizeof(int32_t) * eb.size(), cudaMemcpyDeviceToHost));
            const femi_status ts = tile_split(S, C->gt_blocks, jp);
            if (ts != FEMI_OK) return ts;
            for (int b = 0; b < C->gt_blocks; ++b)
                std::fprintf(stderr, "[femi ctaw] %d %d %d\n", b, jp[b + 1] - jp[b], eb[jp[b + 1]] - eb[jp[b]]);
        }
    }
    CgState hs;
    for (int restarts = 0;; ++restarts) {
        FEMI_CUDA(cudaMemcpyAsync(&hs, C->d_state, sizeof(CgState), cudaMemcpyDeviceToHost, st));
        FEMI_CUDA(cudaStreamSynchronize(st));
        const bool fail = hs.bn2 > 0.0 && !(hs.res2 <= hs.tol2);
        if (!(hs.status == FEMI_OK && hs.iters > 0 && hs.iters < hs.max_iter && fail) || restarts >= 8) break;
        FEMI_CUDA(cudaGraphLaunch(C->restart, st));  // from the current iterate (r = s * r_true)
        count_launches(6);
    }
    // the body runs whole unrolled groups: kernels after convergence exit at once but still launch
    count_launches(2 * (int64_t)((hs.iters + kUnroll - 1) / kUnroll) * kUnroll);
    if (std::getenv("FEMI_PROLOGUE_BENCH") && C->gt_smem > 0) {
        // profiling aid: the solve graph's prologue / epilogue kernels launched one by one on the
        // converged state (event times, median of 5) -- the graph itself cannot be split by ncu
        cudaEvent_t e0, e1;
        FEMI_CUDA(cudaEventCreate(&e0));
        FEMI_CUDA(cudaEventCreate(&e1));
        const dim3 gk(C->gx, 1), bk(KNT);
        RItem* di = C->d_items;
        unsigned* c0 = C->d_cnt;
        unsigned* c1 = C->d_cnt + 1;
        auto tm = [&](const char* name, auto launch) -> femi_status {
            std::vector<float> v;
            for (int k = 0; k < 7; ++k) {
                FEMI_CUDA(cudaEventRecord(e0, st));
                launch();
                FEMI_CUDA(cudaEventRecord(e1, st));
                FEMI_CUDA(cudaEventSynchronize(e1));
                float x = 0.f;
                FEMI_CUDA(cudaEventElapsedTime(&x, e0, e1));
                if (k >= 2) v.push_back(x);
            }
            std::sort(v.begin(), v.end());
            std::fprintf(stderr, "[femi prologue] %-14s %8.2f us\n", name, 1e3 * v[v.size() / 2]);
            return FEMI_OK;
        };
        tm("pro1", [&] { k_pro1<<<gk, bk, 0, st>>>(di, c0); });
        tm("x0_fill2", [&] { k_x0_fill2<<<gk, bk, 0, st>>>(di, 1); });
        tm("pro2", [&] { k_pro2<<<gk, bk, 0, st>>>(di); });
        tm("finalize_g", [&] { k_finalize_g<<<gk, bk, 0, st>>>(di); });
        tm("true_res", [&] { k_true_res<<<gk, bk, 0, st>>>(di, c1, nullptr); });
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        FEMI_CUDA(cudaMemcpyAsync(C->d_state, &hs, sizeof(CgState), cudaMemcpyHostToDevice, st));
        FEMI_CUDA(cudaStreamSynchronize(st));
    }
    if (std::getenv("FEMI_PCG_KBENCH") && C->gt_smem > 0 && C->item.ls) {
        // profiling aid: the loop body's kernels launched standalone on the converged state
        // (alpha = beta = 0 keeps the iterate), so ncu can capture them -- kernel nodes of a
        // graph with conditional nodes cannot be profiled one by one. Event times to stderr.
        CgState a = hs;
        a.active = 1;
        a.alpha = a.beta = a.alpha_pend = 0.0;
        a.x_pend = 0;
        unsigned* gcnt = C->d_cnt + 2;
        cudaEvent_t e0, e1, e2;
        FEMI_CUDA(cudaEventCreate(&e0));
        FEMI_CUDA(cudaEventCreate(&e1));
        FEMI_CUDA(cudaEventCreate(&e2));
        float tu = 0.f, tg = 0.f;
        const int reps = 12;
        const int on = 1, off = 0;
        FEMI_CUDA(cudaMemcpyToSymbolAsync(g_kbench, &on, sizeof(int), 0, cudaMemcpyHostToDevice, st));
        LoopState lsb = {};
        lsb.active = 1;
        lsb.started = 1;
        // FEMI_KBENCH_FLUSH=1: write a 256 MB buffer before each rep (cold L2, like a loop whose
        // matrix stream misses L2); FEMI_KBENCH_NOGU=1: k_gt alone, back to back
        const bool kflush = std::getenv("FEMI_KBENCH_FLUSH") != nullptr;
        const bool knogu = std::getenv("FEMI_KBENCH_NOGU") != nullptr;
        void* flush_buf = nullptr;
        if (kflush) FEMI_CUDA(cudaMalloc(&flush_buf, 256u << 20));
        for (int k = 0; k < reps; ++k) {
            if (kflush) FEMI_CUDA(cudaMemsetAsync(flush_buf, k & 0xff, 256u << 20, st));
            FEMI_CUDA(cudaMemcpyAsync(C->d_state, &a, sizeof(CgState), cudaMemcpyHostToDevice, st));
            FEMI_CUDA(cudaMemcpyAsync(C->item.ls, &lsb, sizeof(LoopState), cudaMemcpyHostToDevice, st));
            FEMI_CUDA(cudaMemcpyAsync(C->item.ls + 1, &lsb, sizeof(LoopState), cudaMemcpyHostToDevice, st));
            FEMI_CUDA(cudaEventRecord(e0, st));
            if (!knogu)
                k_gur<<<dim3(std::min(C->gx * 2, 4 * 148)), GRT, 0, st>>>(C->d_items, C->d_part, C->gt_blocks, 0,
                                                                            (cudaGraphConditionalHandle)0);
            FEMI_CUDA(cudaEventRecord(e1, st));
            k_gt<false, true><<<dim3(C->gt_blocks), JNT, C->gt_smem, st>>>(C->d_items, 1, C->d_part, gcnt,
                                                                            (cudaGraphConditionalHandle)0, 1);
            FEMI_CUDA(cudaEventRecord(e2, st));
            FEMI_CUDA(cudaEventSynchronize(e2));
            float x = 0.f, y = 0.f;
            FEMI_CUDA(cudaEventElapsedTime(&x, e0, e1));
            FEMI_CUDA(cudaEventElapsedTime(&y, e1, e2));
            if (k >= 2) {
                tu += x;
                tg += y;
            }
        }
        FEMI_CUDA(cudaMemcpyToSymbolAsync(g_kbench, &off, sizeof(int), 0, cudaMemcpyHostToDevice, st));
        if (flush_buf) FEMI_CUDA(cudaFree(flush_buf));
        std::fprintf(stderr, "[femi kbench] standalone k_gur %.2f us, k_gt %.2f us\n", 1e3 * tu / (reps - 2),
                     1e3 * tg / (reps - 2));
        {
            FEMI_CUDA(cudaFuncSetAttribute((const void*)k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)C->gt_smem));
            float tp[2] = {0.f, 0.f};
            for (int m = 0; m < 2; ++m)
                for (int k = 0; k < reps; ++k) {
                    FEMI_CUDA(cudaEventRecord(e1, st));
                    k_probe<<<dim3(C->gt_blocks), JNT, m ? C->gt_smem : 0, st>>>(nullptr);
                    FEMI_CUDA(cudaEventRecord(e2, st));
                    FEMI_CUDA(cudaEventSynchronize(e2));
                    float y = 0.f;
                    FEMI_CUDA(cudaEventElapsedTime(&y, e1, e2));
                    if (k >= 2) tp[m] += y;
                }
            std::fprintf(stderr, "[femi kbench] empty kernel %d x %d: %.2f us (no smem), %.2f us (%u B dynamic smem)\n",
                         C->gt_blocks, JNT, 1e3 * tp[0] / (reps - 2), 1e3 * tp[1] / (reps - 2), C->gt_smem);
        }
        FEMI_CUDA(cudaMemcpyAsync(C->d_state, &hs, sizeof(CgState), cudaMemcpyHostToDevice, st));
        FEMI_CUDA(cudaStreamSynchronize(st));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaEventDestroy(e2);
        count_launches(2 * reps);
    }
    const double rel = hs.bn2 > 0.0 ? std::sqrt(hs.res2 / hs.bn2) : 0.0;
    if (iters) *iters = hs.iters;
    if (relres) *relres = rel;
    if (total_iters) *total_iters = hs.iters;
    femi_status sb = (femi_status)hs.status;
    if (sb == FEMI_OK && !(rel <= o.rtol)) sb = FEMI_E_NOT_CONVERGED;
    if (sb != FEMI_OK) set_error("inpaint_solve: CG did not converge (status " + std::to_string((int)sb) + ")");
    return sb;
}

}  // namespace

namespace {

struct GraphCacheM {
    void* ws = nullptr;
    RItem* d_items = nullptr;
    CgState* d_state = nullptr;
    unsigned* d_cnt = nullptr;
    double* d_part = nullptr;
    cudaGraphExec_t main = nullptr, restart = nullptr;
    std::vector<RItem> items;
    int nr = 0, gx = 0, gt_blocks = 0;
    unsigned smem = 0;
};

femi_status build_graph_m(GraphCacheM& C, bool restart, cudaGraphExec_t* out) {
    cudaGraph_t gr;
    FEMI_CUDA(cudaGraphCreate(&gr, 0));
    cudaGraphConditionalHandle h;
    FEMI_CUDA(cudaGraphConditionalHandleCreate(&h, gr, 0, cudaGraphCondAssignDefault));
    RItem* di = C.d_items;
    int nr = C.nr;
    double* part = C.d_part;
    unsigned* cnt0 = C.d_cnt;
    unsigned* cnt1 = C.d_cnt + nr;
    void* a_items[1] = {&di};
    void* a_reset[2] = {&nr, &di};
    void* a_cnt0[2] = {&di, &cnt0};
    void* a_t[3] = {&di, &part, &h};
    const dim3 gk(C.gx, nr), bk(KNT);
    cudaGraphNode_t prev = nullptr, nd;
    cudaGraphNode_t* dep = nullptr;
    auto chain = [&](void* fn, dim3 gg, dim3 bb, void** args, unsigned smem = 0) -> femi_status {
        femi_status s = add_kernel(gr, dep, fn, gg, bb, args, &nd, smem);
        prev = nd;
        dep = &prev;
        return s;
    };
    void *f_first, *f_body, *f_up;
    switch (nr) {
        case 2: f_first = (void*)k_gtm<2, true>; f_body = (void*)k_gtm<2, false>; f_up = (void*)k_gum<2>; break;
        case 3: f_first = (void*)k_gtm<3, true>; f_body = (void*)k_gtm<3, false>; f_up = (void*)k_gum<3>; break;
        default: f_first = (void*)k_gtm<4, true>; f_body = (void*)k_gtm<4, false>; f_up = (void*)k_gum<4>; break;
    }
    femi_status s = FEMI_OK;
    if (!restart) {
        if ((s = chain((void*)k_reset_items, dim3(1), dim3(32), a_reset))) return s;
        int tw1 = 1, tw0 = 0;
        void* a_f1[2] = {&di, &tw1};
        void* a_f0[2] = {&di, &tw0};
        if ((s = chain((void*)k_pro1, gk, bk, a_cnt0))) return s;
        if ((s = chain((void*)k_x0_fill2, gk, bk, a_f1))) return s;
        if ((s = chain((void*)k_x0_fill2, gk, bk, a_f0))) return s;
        if ((s = chain((void*)k_pro2, gk, bk, a_items))) return s;
    } else {
        if ((s = chain((void*)k_zero_ps, gk, bk, a_items))) return s;
    }
    if ((s = chain(f_first, dim3(C.gt_blocks), dim3(JNT), a_t, C.smem))) return s;
    {
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        FEMI_CUDA(cudaGraphAddNode(&nd, gr, dep, 1, &cp));
        prev = nd;
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        cudaGraphNode_t bprev = nullptr, u, sn;
        for (int k = 0; k < kUnroll; ++k) {
            if ((s = add_kernel(body, bprev ? &bprev : nullptr, f_up, dim3(std::min(C.gx * 2, 1184)), dim3(GNT),
                                a_items, &u)))
                return s;
            if ((s = add_kernel(body, &u, f_body, dim3(C.gt_blocks), dim3(JNT), a_t, &sn, C.smem))) return s;
            bprev = sn;
        }
    }
    const int* nogate = nullptr;
    void* a_fin[2] = {&di, &nogate};
    void* a_tres[3] = {&di, &cnt1, &nogate};
    if ((s = chain((void*)k_finalize, gk, bk, a_fin))) return s;
    if ((s = chain((void*)k_true_res, gk, bk, a_tres))) return s;
    if ((s = chain((void*)k_copy_g, dim3(296, nr), dim3(256), a_items))) return s;
    FEMI_CUDA(cudaGraphInstantiate(out, gr, 0));
    FEMI_CUDA(cudaGraphDestroy(gr));
    return FEMI_OK;
}

// NR right-hand sides on one large system with the JDS layout; returns FEMI_E_ARG when the
// shared-memory ring does not fit (the caller falls back to one RHS at a time)
femi_status graph_solve_multi(femi_system_s* S, int nr, const double* const* g, const double* const* bin,
                              double* const* u_vert, const femi_cg_opts& o, int32_t* iters, double* relres,
                              cudaStream_t st, int64_t* total_iters) {
    GraphCacheM* C = (GraphCacheM*)S->scratch_m[nr];
    const int64_t n = S->n_u;
    if (!C) {
        const size_t stage_bytes =
            ((size_t)S->jds_maxe * 12 + S->jds_meta_bytes + 8 * (nr + 1) * kJdsRows + 127) & ~(size_t)127;
        int dev = 0, nsm = 0, optin = 0;
        FEMI_CUDA(cudaGetDevice(&dev));
        FEMI_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        FEMI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        if (JNS_M * stage_bytes + 4096 > (size_t)optin) return FEMI_E_ARG;
        C = new GraphCacheM();
        C->nr = nr;
        C->smem = (unsigned)(JNS_M * stage_bytes);
        C->gt_blocks = std::max(1, std::min(nsm, S->jds_ntile));
        C->gx = (int)std::max<int64_t>(1, std::min<int64_t>((n + KNT - 1) / KNT, 148 * 16));
        const void* fns[6] = {(const void*)k_gtm<2, true>, (const void*)k_gtm<2, false>, (const void*)k_gtm<3, true>,
                              (const void*)k_gtm<3, false>, (const void*)k_gtm<4, true>, (const void*)k_gtm<4, false>};
        for (const void* fn : fns)
            FEMI_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C->smem));
        std::vector<int32_t> jpart;
        femi_status ts = tile_split(S, C->gt_blocks, jpart);
        if (ts != FEMI_OK) return ts;
        auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
        const size_t vb = al(sizeof(double) * std::max<int64_t>(n + 1, (int64_t)S->jds_ntile * kJdsRows));
        const size_t bytes = al(sizeof(int32_t) * jpart.size()) + al(sizeof(RItem) * nr) + al(sizeof(CgState) * nr) +
                             al(sizeof(unsigned) * 2 * nr) + al(sizeof(double) * 3 * nr * C->gt_blocks) +
                             nr * (al(sizeof(double) * C->gx) + 6 * vb);
        FEMI_CUDA(cudaMalloc(&C->ws, bytes));
        char* cur = (char*)C->ws;
        auto take = [&](size_t x) {
            char* p = cur;
            cur += al(x);
            return p;
        };
        C->d_items = (RItem*)take(sizeof(RItem) * nr);
        int32_t* d_jpart = (int32_t*)take(sizeof(int32_t) * jpart.size());
        FEMI_CUDA(cudaMemcpy(d_jpart, jpart.data(), sizeof(int32_t) * jpart.size(), cudaMemcpyHostToDevice));
        C->d_state = (CgState*)take(sizeof(CgState) * nr);
        C->d_cnt = (unsigned*)take(sizeof(unsigned) * 2 * nr);
        C->d_part = (double*)take(sizeof(double) * 3 * nr * C->gt_blocks);
        FEMI_CUDA(cudaMemset(C->d_cnt, 0, sizeof(unsigned) * 2 * nr));
        double dmin = 0.0;
        {
            unsigned long long* d_m = nullptr;
            unsigned long long h_m = ~0ull;
            FEMI_CUDA(cudaMallocAsync(&d_m, sizeof(unsigned long long), st));
            FEMI_CUDA(cudaMemcpyAsync(d_m, &h_m, sizeof(h_m), cudaMemcpyHostToDevice, st));
            k_qmin<<<296, 256, 0, st>>>(n, S->q_int, d_m);
            FEMI_CUDA(cudaMemcpyAsync(&h_m, d_m, sizeof(h_m), cudaMemcpyDeviceToHost, st));
            FEMI_CUDA(cudaFreeAsync(d_m, st));
            FEMI_CUDA(cudaStreamSynchronize(st));
            double dm;
            std::memcpy(&dm, &h_m, sizeof(dm));
            if (std::isfinite(dm) && dm > 0.0) dmin = dm * (1.0 - 1e-12);
        }
        C->items.resize(nr);
        for (int c = 0; c < nr; ++c) {
            RItem& it = C->items[c];
            it = RItem{};
            it.red = (double*)take(sizeof(double) * C->gx);
            it.b = (double*)take(vb);
            it.x = (double*)take(vb);
            it.r = (double*)take(vb);
            it.w = (double*)take(vb);
            it.p = (double*)take(vb);
            it.sv = (double*)take(vb);
            it.jval = S->jds_val;
            it.jcol = S->jds_col;
            it.jmeta = S->jds_meta;
            it.jeb = S->jds_eb;
            it.jcb = S->jds_cb;
            it.ntile = S->jds_ntile;
            it.jmaxe = S->jds_maxe;
            it.jkmax = S->jds_kmax;
            it.jmbytes = S->jds_meta_bytes;
            it.jpart = d_jpart;
            it.dmin = dmin;
            it.inv = S->sell_inv;
            it.len = S->sell_len;
            it.base = S->sell_base;
            it.val = S->sell_val;
            it.c16 = S->sell_c16;
            it.c32 = S->sell_c32;
            it.s = S->s_int;
            it.q = S->q_int;
            it.urp = S->uuI_rowptr;
            it.uci = S->uuI_col;
            it.uav = S->uuI_val;
            it.krp = S->ukI_rowptr;
            it.kci = S->ukI_col;
            it.kav = S->ukI_val;
            it.st = C->d_state + c;
            it.n = (int32_t)n;
            it.m = (int32_t)S->m;
            it.cta0 = 0;
            it.ncta = 1;
            it.nwin = S->nwin;
        }
        femi_status s = build_graph_m(*C, false, &C->main);
        if (s == FEMI_OK) s = build_graph_m(*C, true, &C->restart);
        if (s != FEMI_OK) {  // publish the cache only once both graphs are instantiated
            if (C->main) cudaGraphExecDestroy(C->main);
            if (C->restart) cudaGraphExecDestroy(C->restart);
            cudaFree(C->ws);
            delete C;
            return s;
        }
        S->scratch_m[nr] = C;
    }
    std::vector<RItem> its = C->items;
    for (int c = 0; c < nr; ++c) {
        its[c].g = g ? g[c] : nullptr;
        its[c].bin = bin ? bin[c] : nullptr;
        its[c].u_vert = u_vert[c];
        its[c].x0mode = (its[c].g == nullptr && (o.x0 == 1 || o.x0 == 3)) ? 0 : o.x0;
        its[c].rtol = o.rtol;
        its[c].max_iter = o.max_iter;
    }
    FEMI_CUDA(cudaMemcpyAsync(C->d_items, its.data(), sizeof(RItem) * nr, cudaMemcpyHostToDevice, st));
    FEMI_CUDA(cudaGraphLaunch(C->main, st));
    count_launches(10);
    std::vector<CgState> hs(nr);
    for (int restarts = 0;; ++restarts) {
        FEMI_CUDA(cudaMemcpyAsync(hs.data(), C->d_state, sizeof(CgState) * nr, cudaMemcpyDeviceToHost, st));
        FEMI_CUDA(cudaStreamSynchronize(st));
        bool again = false;
        for (int c = 0; c < nr; ++c) {
            const CgState& h = hs[c];
            again |= h.status == FEMI_OK && h.iters > 0 && h.iters < h.max_iter && h.bn2 > 0.0 && !(h.res2 <= h.tol2);
        }
        if (!again || restarts >= 8) break;
        FEMI_CUDA(cudaGraphLaunch(C->restart, st));
        count_launches(6);
    }
    femi_status ret = FEMI_OK;
    int64_t tot = 0, itmax = 0;
    for (int c = 0; c < nr; ++c) {
        const CgState& h = hs[c];
        const double rel = h.bn2 > 0.0 ? std::sqrt(h.res2 / h.bn2) : 0.0;
        if (iters) iters[c] = h.iters;
        if (relres) relres[c] = rel;
        tot += h.iters;
        itmax = std::max<int64_t>(itmax, h.iters);
        femi_status sb = (femi_status)h.status;
        if (sb == FEMI_OK && !(rel <= o.rtol)) sb = FEMI_E_NOT_CONVERGED;
        if (sb != FEMI_OK && ret == FEMI_OK) ret = sb;
    }
    count_launches(2 * ((itmax + kUnroll - 1) / kUnroll) * kUnroll);
    if (total_iters) *total_iters = tot;
    if (ret != FEMI_OK) set_error("inpaint_solve: CG did not converge (status " + std::to_string((int)ret) + ")");
    return ret;
}

}  // namespace

void pcg_cache_free(femi_system_s* S) {
    if (S->rz_cache) {
        RzCache* Z = (RzCache*)S->rz_cache;
        if (Z->block) cudaFreeAsync(Z->block, nullptr);
        delete Z;
        S->rz_cache = nullptr;
    }
    for (int k = 0; k < 5; ++k) {
        GraphCacheM* M = (GraphCacheM*)S->scratch_m[k];
        if (!M) continue;
        if (M->main) cudaGraphExecDestroy(M->main);
        if (M->restart) cudaGraphExecDestroy(M->restart);
        if (M->ws) cudaFree(M->ws);
        delete M;
        S->scratch_m[k] = nullptr;
    }
    GraphCache* C = (GraphCache*)S->scratch;
    if (!C) return;
    if (C->main) cudaGraphExecDestroy(C->main);
    if (C->restart) cudaGraphExecDestroy(C->restart);
    if (C->restart_if) cudaGraphExecDestroy(C->restart_if);
    if (C->ws) cudaFree(C->ws);
    delete C;
    S->scratch = nullptr;
}

// per-item outputs of a synchronous solve from the final CgStates
static femi_status solve_outcome(int B, femi_system_s* const* S, const std::vector<CgState>& hs, const femi_cg_opts& o,
                                 int32_t* iters, double* relres, int64_t* total_iters) {
    femi_status ret = FEMI_OK;
    int64_t tot = 0;
    for (int b = 0; b < B; ++b) {
        const CgState& s = hs[b];
        double rel = s.bn2 > 0.0 ? std::sqrt(s.res2 / s.bn2) : 0.0;
        if (S[b]->n_u == 0) rel = 0.0;
        if (iters) iters[b] = S[b]->n_u == 0 ? 0 : s.iters;
        if (relres) relres[b] = rel;
        tot += S[b]->n_u == 0 ? 0 : s.iters;
        femi_status sb = S[b]->n_u == 0 ? FEMI_OK : (femi_status)s.status;
        if (sb == FEMI_OK && !(rel <= o.rtol)) sb = FEMI_E_NOT_CONVERGED;
        if (sb != FEMI_OK && ret == FEMI_OK) ret = sb;
    }
    if (total_iters) *total_iters = tot;
    if (ret != FEMI_OK) set_error("inpaint_solve: CG did not converge (status " + std::to_string((int)ret) + ")");
    return ret;
}

femi_status pcg_solve(int B, femi_system_s* const* S, const double* const* g, const double* const* bin,
                      double* const* u_vert, const femi_cg_opts& o_in, int32_t* iters, double* relres,
                      cudaStream_t st, int64_t* total_iters, DevStats* ds) {
    // FEMI_SOLVE_HOSTPROF=1: host-side time stamps of the whole-solve path (diagnostic)
    static const bool hprof = std::getenv("FEMI_SOLVE_HOSTPROF") != nullptr;
    const auto h0 = std::chrono::steady_clock::now();
    auto hstamp = [&](const char* what) {
        if (hprof)
            std::fprintf(stderr, "[femi solve host] %-12s %7.2f us\n", what,
                         1e6 * std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count());
    };
    // reading A11b: with the separate prologue kernels the fill cost four extra launches, more
    // than it saved below 8192 unknowns (C2 5.76K -> 5.18K Mpx/s); inside the whole-solve
    // resident kernel it costs two cluster barriers, and it pays at every size (C2 50.4 -> 42.2
    // mean iterations, 7.34K -> 7.80K Mpx/s), so the threshold is 0 (FEMI_FILL_MIN=k restores it)
    femi_cg_opts o = o_in;
    {
        int64_t nfill = 0;
        for (int b = 0; b < B; ++b) nfill = std::max(nfill, S[b]->n_u);
        static const int64_t fill_min = std::getenv("FEMI_FILL_MIN") ? std::atoll(std::getenv("FEMI_FILL_MIN"))
                                                                     : kFillMinRows;
        if (o.x0 == 3 && nfill < fill_min) o.x0 = 1;
    }
    {
        static int graph_mode = -1;  // FEMI_PCG_MODE=persistent forces the persistent kernel
        if (graph_mode < 0) {
            const char* pm = std::getenv("FEMI_PCG_MODE");
            graph_mode = (pm && std::string(pm) == "persistent") ? 0 : 1;
        }
        if (graph_mode && B == 1 && S[0]->nnz_uu > 600000 && S[0]->n_u > 0)
            return graph_solve(S[0], g ? g[0] : nullptr, bin ? bin[0] : nullptr, u_vert[0], o, iters, relres, st,
                               total_iters, ds);
        // a repeated large system (colour channels): shared-matrix multi-RHS, <= 4 per pass
        bool shared = graph_mode && B > 1 && S[0]->nnz_uu > 600000 && S[0]->n_u > 0 && S[0]->jds_ntile > 0 &&
                      std::getenv("FEMI_NO_MULTI") == nullptr;
        for (int b = 1; b < B && shared; ++b) shared = S[b] == S[0];
        if (shared) {
            bool used_multi = false;
            femi_status ret = FEMI_OK;
            int64_t tot = 0;
            for (int b0 = 0; b0 < B;) {
                const int nr = std::min(4, B - b0);
                int64_t t1 = 0;
                femi_status sb;
                if (nr == 1)
                    sb = graph_solve(S[0], g ? g[b0] : nullptr, bin ? bin[b0] : nullptr, u_vert[b0], o,
                                     iters ? iters + b0 : nullptr, relres ? relres + b0 : nullptr, st, &t1);
                else
                    sb = graph_solve_multi(S[0], nr, g ? g + b0 : nullptr, bin ? bin + b0 : nullptr, u_vert + b0, o,
                                           iters ? iters + b0 : nullptr, relres ? relres + b0 : nullptr, st, &t1);
                used_multi |= nr > 1 && sb != FEMI_E_ARG;
                if (sb == FEMI_E_ARG && nr > 1) {  // ring does not fit: one RHS at a time
                    for (int c = 0; c < nr; ++c) {
                        int64_t t2 = 0;
                        const femi_status s2 =
                            graph_solve(S[0], g ? g[b0 + c] : nullptr, bin ? bin[b0 + c] : nullptr, u_vert[b0 + c], o,
                                        iters ? iters + b0 + c : nullptr, relres ? relres + b0 + c : nullptr, st, &t2);
                        t1 += t2;
                        if (s2 != FEMI_OK && ret == FEMI_OK) ret = s2;
                    }
                } else if (sb != FEMI_OK && ret == FEMI_OK) {
                    ret = sb;
                }
                tot += t1;
                b0 += nr;
            }
            if (total_iters) *total_iters = tot;
            if (used_multi) S[0]->last_path = FEMI_PATH_GRAPH_MULTI;
            return ret;
        }
    }
    // kernel table: [mode 0/1/2][nvec 0/2/3]; grid mode: 768 threads x 1 CTA/SM (shape 1,
    // measured best) or 512 x 2 (shape 0); FEMI_CG_SHAPE selects for experiments
    static void* const fn_block[3] = {(void*)k_cg<0, RNT, 1, 0>, (void*)k_cg<0, RNT, 1, 2>, (void*)k_cg<0, RNT, 1, 3>};
    static void* const fn_clus[3] = {(void*)k_cg<1, RNT, 1, 0>, (void*)k_cg<1, RNT, 1, 2>, (void*)k_cg<1, RNT, 1, 3>};
    static void* const fn_grid[2][3] = {
        {(void*)k_cg<2, 512, 2, 0>, (void*)k_cg<2, 512, 2, 2>, (void*)k_cg<2, 512, 2, 3>},
        {(void*)k_cg<2, 768, 1, 0>, (void*)k_cg<2, 768, 1, 2>, (void*)k_cg<2, 768, 1, 3>}};
    static const int grid_nt[2] = {512, 768};
    static const int grid_per_sm[2] = {2, 1};
    auto nv_idx = [](int nv) { return nv == 0 ? 0 : (nv == 2 ? 1 : 2); };
    static int attr_dev = -1;  // function attributes are per device: redo them on a device change
    int cur_dev = 0;
    FEMI_CUDA(cudaGetDevice(&cur_dev));
    if (attr_dev != cur_dev) {
        attr_dev = cur_dev;
        const int dev = cur_dev;
        FEMI_CUDA(cudaDeviceGetAttribute(&g_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        FEMI_CUDA(cudaDeviceGetAttribute(&g_nsm, cudaDevAttrMultiProcessorCount, dev));
        for (int k = 0; k < 3; ++k) {
            FEMI_CUDA(cudaFuncSetAttribute(fn_block[k], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           g_smem_optin - 2048));
            FEMI_CUDA(cudaFuncSetAttribute(fn_clus[k], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           g_smem_optin - 2048));
            FEMI_CUDA(cudaFuncSetAttribute(fn_clus[k], cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            for (int s = 0; s < 2; ++s)
                FEMI_CUDA(cudaFuncSetAttribute(fn_grid[s][k], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               g_smem_optin / grid_per_sm[s] - 2048));
        }
        const char* tm = std::getenv("FEMI_PCG_TIMERS");
        g_timers = tm && tm[0] == '1';
        const char* nv = std::getenv("FEMI_PCG_NVEC");  // experiments: max vectors kept in smem
        if (nv) g_nvec_max = std::atoi(nv);
        const char* sp = std::getenv("FEMI_CG_SHAPE");
        if (sp) g_shape = std::max(0, std::min(1, std::atoi(sp)));
        int per_sm = 0;
        FEMI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn_grid[g_shape][0], grid_nt[g_shape],
                                                                g_smem_optin / grid_per_sm[g_shape] - 2048));
        g_occ_grid = std::max(1, per_sm) * g_nsm;
    }
    // ---- launch shape: one huge system -> cooperative grid; otherwise one cluster per item
    int64_t nmax = 0, nnz_max = 0;
    for (int b = 0; b < B; ++b) {
        nmax = std::max(nmax, S[b]->n_u);
        nnz_max = std::max(nnz_max, S[b]->nnz_uu);
    }
    int mode, ncta_item = 1;
    // on-chip resident solver (k_cgr): the smallest cluster (1..16 CTAs) whose CTAs hold their
    // matrix slices and r in shared memory and their rows in registers (<= RPL slices per warp)
    size_t rz_smem = 0;
    int rz_C = 0, rz_rp = RPL;
    static const bool rz_off = std::getenv("FEMI_NO_RESIDENT") != nullptr;
    // whole-solve pipelined resident kernel k_cgs (default) or k_cgr + prologue/epilogue kernels (FEMI_CG_PIPE=0)
    static const bool rz_pipe = !(std::getenv("FEMI_CG_PIPE") && std::getenv("FEMI_CG_PIPE")[0] == '0');
    const size_t rz_static = rz_pipe ? 16 * 16 * RZW + sizeof(double) * (6 * RZW + 2 * 16 * 3) + 2048 : 0;
    if (!rz_off && !(B == 1 && S[0]->nnz_uu > 600000)) {
        const size_t rz_budget = (size_t)g_smem_optin - 4096;
        // cluster size: enough CTAs to fill the GPU (B C <= #SMs) while every warp keeps at least
        // one slice -- the per-iteration critical path is a warp's slice sequence -- and at
        // least the smallest size whose CTAs fit in shared memory
        int64_t nsl_max = 0;
        for (int b = 0; b < B; ++b) nsl_max = std::max<int64_t>(nsl_max, S[b]->nslices);
        int c_fill = 1, c_use = 1;
        while (c_fill * 2 <= 16 && (int64_t)B * c_fill * 2 <= g_nsm) c_fill *= 2;
        while (c_use < 16 && (int64_t)c_use * RZW < nsl_max) c_use *= 2;
        const int c_pref = std::min(c_fill, c_use);
        for (int C = 1; C <= 16 && !rz_C; C <<= 1) {
            if (C < c_pref) continue;
            bool ok = true;
            size_t need = 0;
            int64_t nsl_cta = 0;
            for (int b = 0; b < B && ok; ++b) {
                const femi_system_s* sy = S[b];
                if (sy->n_u == 0) continue;
                if ((int)sy->sell_base_h.size() != sy->nslices + 1) {
                    ok = false;
                    break;
                }
                for (int k = 0; k < C && ok; ++k) {
                    const int64_t r0 = std::min<int64_t>(sy->n_u, (int64_t)sy->nwin * k / C * SIG);
                    const int64_t r1 = std::min<int64_t>(sy->n_u, (int64_t)sy->nwin * (k + 1) / C * SIG);
                    const int64_t s0 = r0 / 32, s1 = (r1 + 31) / 32, nsl = s1 - s0;
                    if (nsl > (int64_t)RZW * RPL || r1 - r0 > 65535) ok = false;
                    nsl_cta = std::max(nsl_cta, nsl);
                    const int64_t ne = nsl > 0 ? sy->sell_base_h[s1] - sy->sell_base_h[s0] : 0;
                    need = std::max(need, (size_t)(16 * 32 * nsl + 12 * ne + 8 * nsl + 64));
                }
            }
            if (ok && need <= rz_budget) {
                rz_C = C;
                rz_smem = need;
                rz_rp = (int)((nsl_cta + RZW - 1) / RZW);
            }
        }
    }
    if (rz_C > 0) {
        mode = 3;
        ncta_item = rz_C;
    } else if (B == 1 && S[0]->nnz_uu > 600000) {
        mode = 2;
        ncta_item = std::max(1, std::min(g_occ_grid, S[0]->nwin));
    } else {
        ncta_item = (int)std::min<int64_t>(16, std::max<int64_t>(1, (nnz_max + 23999) / 24000));
        int c = 1;
        while (c < ncta_item) c <<= 1;
        ncta_item = std::min(c, 16);
        mode = ncta_item == 1 ? 0 : 1;
    }
    const int grid = B * ncta_item;
    for (int b = 0; b < B; ++b) S[b]->last_path = mode == 3 ? FEMI_PATH_RESIDENT : FEMI_PATH_PERSISTENT;
    // rows of the largest CTA; shared memory: slice metadata, then as many of p, s, x as fit
    int64_t vrows = 0;
    for (int b = 0; b < B; ++b) {
        const int nw = S[b]->nwin;
        for (int k = 0; k < ncta_item; ++k) {
            const int64_t w0 = (int64_t)nw * k / ncta_item, w1 = (int64_t)nw * (k + 1) / ncta_item;
            vrows = std::max(vrows, std::min(S[b]->n_u, w1 * SIG) - std::min(S[b]->n_u, w0 * SIG));
        }
    }
    const int mrows = (int)(vrows + 32);
    const size_t meta_bytes = sizeof(double) * (mrows / 32 + 1);
    const size_t budget = (size_t)(mode == 2 ? g_smem_optin / grid_per_sm[g_shape] - 2048 : g_smem_optin - 2048);
    int nvec = g_nvec_max;
    while (nvec >= 2 && meta_bytes + sizeof(double) * (nvec * (size_t)vrows) > budget) --nvec;
    if (nvec < 2) nvec = 0;
    const size_t smem_bytes = meta_bytes + sizeof(double) * ((size_t)nvec * vrows);

    hstamp("shape");
    // ---- workspace
    std::vector<RItem> items(B);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t total = al(sizeof(RItem) * B) + al(sizeof(CgState) * B) + al(sizeof(unsigned) * 2 * B);
    for (int b = 0; b < B; ++b)
        total += al(sizeof(double) * (S[b]->n_u + 1)) * (nvec == 0 ? 6 : 4) + al(sizeof(double) * 4 * ncta_item) +
                 al(sizeof(double) * KGRID);
    Workspace ws;
    ws.st = st;
    FEMI_CUDA(cudaMallocAsync(&ws.base, total, st));
    char* cur = (char*)ws.base;
    auto take = [&](size_t x) {
        char* p = cur;
        cur += al(x);
        return p;
    };
    RItem* d_items = (RItem*)take(sizeof(RItem) * B);
    CgState* d_state = (CgState*)take(sizeof(CgState) * B);
    unsigned* d_cnt = (unsigned*)take(sizeof(unsigned) * 2 * B);
    // barrier/partial slots of all items in one contiguous block (zeroed before each k_cg)
    const size_t part_bytes = sizeof(double) * 4 * (size_t)ncta_item * B;
    char* part_lo = take(part_bytes);
    for (int b = 0; b < B; ++b) {
        femi_system_s* s = S[b];
        RItem& it = items[b];
        const size_t vb = sizeof(double) * (s->n_u + 1);
        it.inv = s->sell_inv;
        it.len = s->sell_len;
        it.base = s->sell_base;
        it.val = s->sell_val;
        it.c16 = s->sell_c16;
        it.c32 = s->sell_c32;
        it.s = s->s_int;
        it.q = s->q_int;
        it.urp = s->uuI_rowptr;
        it.uci = s->uuI_col;
        it.uav = s->uuI_val;
        it.krp = s->ukI_rowptr;
        it.kci = s->ukI_col;
        it.kav = s->ukI_val;
        it.g = g ? g[b] : nullptr;
        it.bin = bin ? bin[b] : nullptr;
        it.u_vert = u_vert[b];
        it.b = (double*)take(vb);
        it.x = (double*)take(vb);
        it.r = (double*)take(vb);
        it.w = (double*)take(vb);
        it.p = nvec == 0 ? (double*)take(vb) : nullptr;
        it.sv = nvec == 0 ? (double*)take(vb) : nullptr;
        it.part = (double*)(part_lo + sizeof(double) * 4 * (size_t)ncta_item * b);
        it.red = (double*)take(sizeof(double) * KGRID);
        it.st = d_state + b;
        it.n = (int32_t)s->n_u;
        it.m = (int32_t)s->m;
        it.cta0 = b * ncta_item;
        it.ncta = ncta_item;
        it.nwin = s->nwin;
        it.x0mode = (it.g == nullptr && (o.x0 == 1 || o.x0 == 3)) ? 0 : o.x0;
    }
    // whole-solve resident kernel: halo tables per system (built on first use for this cluster
    // size), then the shared-memory size of the largest CTA; too large -> the k_cgr path
    bool use_cgs = mode == 3 && rz_pipe;
    if (use_cgs) {
        const int C = ncta_item;
        std::vector<RItem> bitems(items);
        bool build = false;
        for (int b = 0; b < B; ++b) {
            femi_system_s* sy = S[b];
            RzCache* Z = (RzCache*)sy->rz_cache;
            bitems[b].rzc = nullptr;
            if (sy->n_u == 0) continue;
            if (Z && Z->C == C) continue;
            if (!Z) {
                Z = new RzCache();
                sy->rz_cache = Z;
            }
            if (Z->block) FEMI_CUDA(cudaFreeAsync(Z->block, st));
            const size_t ne = (size_t)std::max<int64_t>(1, sy->sell_nnz);
            const size_t bytes = ((2 * ne + 15) & ~(size_t)15) + 8 * ne + 128;
            FEMI_CUDA(cudaMallocAsync(&Z->block, bytes, st));  // the stream-ordered pool
            Z->C = C;
            Z->code = (uint16_t*)Z->block;
            Z->halo = (int32_t*)((char*)Z->block + ((2 * ne + 15) & ~(size_t)15));
            Z->snd = Z->halo + ne;
            Z->cnt = Z->snd + ne;
            bitems[b].rzc = Z->code;
            bitems[b].rzh = Z->halo;
            bitems[b].rzs = Z->snd;
            bitems[b].rzn = Z->cnt;
            build = true;
        }
        if (build) {
            RItem* d_bi = nullptr;
            FEMI_CUDA(cudaMallocAsync(&d_bi, sizeof(RItem) * B, st));
            FEMI_CUDA(cudaMemcpyAsync(d_bi, bitems.data(), sizeof(RItem) * B, cudaMemcpyHostToDevice, st));
            static int halo_attr_dev = -1;
            if (halo_attr_dev != cur_dev) {
                FEMI_CUDA(cudaFuncSetAttribute((void*)k_rz_halo, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               g_smem_optin - 4096));
                halo_attr_dev = cur_dev;
            }
            const size_t hsm = sizeof(unsigned) * 2 * (size_t)((nmax + 31) / 32);
            k_rz_halo<<<B * C, 512, hsm, st>>>(d_bi, C);
            k_rz_send<<<B * C, 512, 0, st>>>(d_bi, C);
            count_launches(2);
            FEMI_CUDA(cudaGetLastError());
            for (int b = 0; b < B; ++b)
                if (bitems[b].rzc) {
                    RzCache* Z = (RzCache*)S[b]->rz_cache;
                    FEMI_CUDA(cudaMemcpyAsync(Z->cnt_h, Z->cnt, sizeof(Z->cnt_h), cudaMemcpyDeviceToHost, st));
                }
            FEMI_CUDA(cudaFreeAsync(d_bi, st));
            FEMI_CUDA(cudaStreamSynchronize(st));
            for (int b = 0; b < B; ++b)
                if (bitems[b].rzc) {
                    RzCache* Z = (RzCache*)S[b]->rz_cache;
                    Z->hmax = 0;
                    for (int k = 0; k < C; ++k) Z->hmax = std::max(Z->hmax, Z->cnt_h[k]);
                }
        }
        const size_t budget = (size_t)g_smem_optin - 4096 - rz_static;
        size_t need = 0;
        for (int b = 0; b < B && use_cgs; ++b) {
            femi_system_s* sy = S[b];
            if (sy->n_u == 0) continue;
            const RzCache* Z = (const RzCache*)sy->rz_cache;
            int64_t nslm = 0;
            for (int k = 0; k < C; ++k) {
                const int64_t r0 = std::min<int64_t>(sy->n_u, (int64_t)sy->nwin * k / C * SIG);
                const int64_t r1 = std::min<int64_t>(sy->n_u, (int64_t)sy->nwin * (k + 1) / C * SIG);
                nslm = std::max(nslm, (r1 + 31) / 32 - r0 / 32);
            }
            for (int k = 0; k < C; ++k) {
                const int64_t r0 = std::min<int64_t>(sy->n_u, (int64_t)sy->nwin * k / C * SIG);
                const int64_t r1 = std::min<int64_t>(sy->n_u, (int64_t)sy->nwin * (k + 1) / C * SIG);
                const int64_t s0 = r0 / 32, s1 = (r1 + 31) / 32, nsl = s1 - s0;
                const int64_t ne = nsl > 0 ? sy->sell_base_h[s1] - sy->sell_base_h[s0] : 0;
                need = std::max(need, (size_t)(16 * (32 * nslm + Z->hmax) + 8 * 32 * nsl + 10 * ne + 8 * nsl +
                                               4 * Z->cnt_h[16 + k] + 64));
            }
            items[b].rzc = Z->code;
            items[b].rzh = Z->halo;
            items[b].rzs = Z->snd;
            items[b].rzn = Z->cnt;
            items[b].rzhmax = Z->hmax;
        }
        if (need > budget) use_cgs = false;
        else rz_smem = need;
    }
    FEMI_CUDA(cudaMemcpyAsync(d_items, items.data(), sizeof(RItem) * B, cudaMemcpyHostToDevice, st));
    hstamp("items_up");
    FEMI_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned) * 2 * B, st));

    // ---- whole-solve resident kernel: one cluster launch per item does everything
    if (use_cgs) {
        static int cgs_attr_dev = -1;
        if (cgs_attr_dev != cur_dev) {
            const int pmax = g_smem_optin - 4096 - (int)rz_static;
            for (void* fp : {(void*)k_cgs<false, 2>, (void*)k_cgs<false, 4>, (void*)k_cgs<false, 6>,
                             (void*)k_cgs<true, 2>, (void*)k_cgs<true, 4>, (void*)k_cgs<true, 6>})
                FEMI_CUDA(cudaFuncSetAttribute(fp, cudaFuncAttributeMaxDynamicSharedMemorySize, pmax));
            for (void* fp : {(void*)k_cgs<true, 2>, (void*)k_cgs<true, 4>, (void*)k_cgs<true, 6>})
                FEMI_CUDA(cudaFuncSetAttribute(fp, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cgs_attr_dev = cur_dev;
        }
        if (g_timers) {
            unsigned long long z[16] = {};
            int on = 1;
            FEMI_CUDA(cudaMemcpyToSymbolAsync(g_pcg_timers, z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
            FEMI_CUDA(cudaMemcpyToSymbolAsync(g_pcg_timers_on, &on, sizeof(int), 0, cudaMemcpyHostToDevice, st));
        }
        void* fp_cl[3] = {(void*)k_cgs<true, 2>, (void*)k_cgs<true, 4>, (void*)k_cgs<true, 6>};
        void* fp_1[3] = {(void*)k_cgs<false, 2>, (void*)k_cgs<false, 4>, (void*)k_cgs<false, 6>};
        const int rpi = rz_rp <= 2 ? 0 : (rz_rp <= 4 ? 1 : 2);  // rows per lane the CTAs need
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(RZT);
        cfg.dynamicSmemBytes = rz_smem;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 0;
        if (ncta_item > 1) {
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = ncta_item;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.numAttrs = 1;
        }
        const RItem* di = d_items;
        double rt = o.rtol;
        int mi = o.max_iter;
        void* args[3] = {(void*)&di, (void*)&rt, (void*)&mi};
        hstamp("pre_launch");
        const cudaError_t e = cudaLaunchKernelExC(&cfg, ncta_item > 1 ? fp_cl[rpi] : fp_1[rpi], args);
        if (e != cudaSuccess) return cuda_fail(e, "k_cgs launch");
        hstamp("launched");
        count_launches(1);
        if (ds) {
            k_stats<<<1, 32, 0, st>>>(B, d_items, ds);
            count_launches(1);
            FEMI_CUDA(cudaGetLastError());
            return FEMI_OK;  // the workspace is released stream-ordered (Workspace)
        }
        std::vector<CgState> hs(B);
        FEMI_CUDA(cudaMemcpyAsync(hs.data(), d_state, sizeof(CgState) * B, cudaMemcpyDeviceToHost, st));
        FEMI_CUDA(cudaStreamSynchronize(st));
        hstamp("synced");
        if (g_timers) {
            unsigned long long t[16];
            FEMI_CUDA(cudaMemcpyFromSymbol(t, g_pcg_timers, sizeof(t)));
            const double it_n = std::max(1, hs[0].iters);
            std::fprintf(stderr,
                         "[femi pcg timers] k_cgs ctas %d iters %d | per iter us: publish %.2f barrier+sums %.2f spmv "
                         "%.2f update %.2f | per launch us: setup %.2f pass1 %.2f fill+pass2 %.2f epilogue %.2f\n",
                         grid, hs[0].iters, t[0] / it_n / 1e3, t[1] / it_n / 1e3, t[2] / it_n / 1e3, t[3] / it_n / 1e3,
                         t[4] / 1e3, t[5] / 1e3, t[6] / 1e3, t[7] / 1e3);
            std::fprintf(stderr,
                         "[femi pcg timers] k_cgs prologue us: pass1 walk %.2f | csum %.2f | hop1 %.2f bar %.2f | hop2 "
                         "%.2f bar %.2f | pass2 %.2f | fixup+q %.2f\n",
                         t[8] / 1e3, t[9] / 1e3, t[10] / 1e3, t[11] / 1e3, t[12] / 1e3, t[13] / 1e3, t[14] / 1e3,
                         t[15] / 1e3);
        }
        return solve_outcome(B, S, hs, o, iters, relres, total_iters);
    }

    // ---- setup launches
    const unsigned gy = (unsigned)B;
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nmax + KNT - 1) / KNT, KGRID / B));
    k_reset<<<(B + 127) / 128, 128, 0, st>>>(B, d_state, o.rtol, o.max_iter);
    count_launches(1);
    if (nmax > 0) {  // min/max of g, b, x^0 (the mask-neighbour fill of reading A11b for x0 = 3), r^0
        k_pro1<<<dim3(gx, gy), KNT, 0, st>>>(d_items, d_cnt);
        if (o.x0 == 3) {
            k_x0_fill2<<<dim3(gx, gy), KNT, 0, st>>>(d_items, 1);
            k_x0_fill2<<<dim3(gx, gy), KNT, 0, st>>>(d_items, 0);
            count_launches(2);
        }
        k_pro2<<<dim3(gx, gy), KNT, 0, st>>>(d_items);
        count_launches(2);
    }
    FEMI_CUDA(cudaGetLastError());
    std::vector<CgState> hs(B);
    int restarts = 0;
    // asynchronous mode (ds): rounds 0 and 1 are enqueued back to back, round 1 gated on the
    // device by the true residual of round 0 (k_restart_flag); nothing is read back
    const bool async = ds != nullptr && mode == 3;
    int* d_gate = nullptr;
    if (async) FEMI_CUDA(cudaMallocAsync(&d_gate, sizeof(int), st));
    for (int round = 0;; ++round) {
        if (async && round == 1) {
            k_restart_flag<<<1, 32, 0, st>>>(B, d_items, d_gate);
            count_launches(1);
        }
        if (nmax > 0) {
            FEMI_CUDA(cudaMemsetAsync(part_lo, 0, part_bytes, st));  // barrier slots at epoch 0
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(mode == 2 ? grid_nt[g_shape] : RNT);
            cfg.dynamicSmemBytes = smem_bytes;
            cfg.stream = st;
            cfg.attrs = attr;
            cfg.numAttrs = 0;
            const int vr = (int)vrows;
            if (g_timers) {
                unsigned long long z[16] = {};
                int on = 1;
                FEMI_CUDA(cudaMemcpyToSymbolAsync(g_pcg_timers, z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
                FEMI_CUDA(cudaMemcpyToSymbolAsync(g_pcg_timers_on, &on, sizeof(int), 0, cudaMemcpyHostToDevice, st));
            }
            const RItem* di = d_items;
            int bb = B;
            void* args[5] = {(void*)&di, (void*)&bb, (void*)&vr, (void*)&nvec, (void*)&mrows};
            void* fn;
            if (mode == 3) {
                static int rz_attr_dev = -1;
                if (rz_attr_dev != cur_dev) {
                    FEMI_CUDA(cudaFuncSetAttribute((void*)k_cgr<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   g_smem_optin - 4096));
                    FEMI_CUDA(cudaFuncSetAttribute((void*)k_cgr<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   g_smem_optin - 4096));
                    FEMI_CUDA(cudaFuncSetAttribute((void*)k_cgr<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                    rz_attr_dev = cur_dev;
                }
                cfg.blockDim = dim3(RZT);
                cfg.dynamicSmemBytes = rz_smem;
                const int* gate = round == 0 ? nullptr : d_gate;  // the async restart round is gated
                void* args1[2] = {(void*)&di, (void*)&gate};
                if (ncta_item > 1) {
                    attr[0].id = cudaLaunchAttributeClusterDimension;
                    attr[0].val.clusterDim.x = ncta_item;
                    attr[0].val.clusterDim.y = 1;
                    attr[0].val.clusterDim.z = 1;
                    cfg.numAttrs = 1;
                }
                const cudaError_t e3 = cudaLaunchKernelExC(&cfg, ncta_item > 1 ? (void*)k_cgr<true> : (void*)k_cgr<false>,
                                                           args1);
                if (e3 != cudaSuccess) return cuda_fail(e3, "k_cgr launch");
                k_finalize<<<dim3(gx, gy), KNT, 0, st>>>(d_items, gate);
                k_true_res<<<dim3(gx, gy), KNT, 0, st>>>(d_items, d_cnt + B, gate);
                count_launches(3);
                FEMI_CUDA(cudaGetLastError());
            } else {
            if (mode == 2) {
                attr[0].id = cudaLaunchAttributeCooperative;
                attr[0].val.cooperative = 1;
                cfg.numAttrs = 1;
                fn = fn_grid[g_shape][nv_idx(nvec)];
            } else if (mode == 1) {
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = ncta_item;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.numAttrs = 1;
                fn = fn_clus[nv_idx(nvec)];
            } else {
                fn = fn_block[nv_idx(nvec)];
            }
            const cudaError_t e = cudaLaunchKernelExC(&cfg, fn, args);
            if (e != cudaSuccess) return cuda_fail(e, "k_cg launch");
            k_finalize<<<dim3(gx, gy), KNT, 0, st>>>(d_items);
            k_true_res<<<dim3(gx, gy), KNT, 0, st>>>(d_items, d_cnt + B);
            count_launches(3);
            FEMI_CUDA(cudaGetLastError());
            }
        }
        if (async) {
            if (round == 1) break;
            continue;
        }
        FEMI_CUDA(cudaMemcpyAsync(hs.data(), d_state, sizeof(CgState) * B, cudaMemcpyDeviceToHost, st));
        FEMI_CUDA(cudaStreamSynchronize(st));
        if (g_timers && nmax > 0) {
            unsigned long long t[16];
            FEMI_CUDA(cudaMemcpyFromSymbol(t, g_pcg_timers, sizeof(t)));
            const double it_n = std::max(1, hs[0].iters);
            std::fprintf(stderr,
                         "[femi pcg timers] mode %d ctas %d nvec %d iters %d | per iter us: U %.2f sync %.2f spmv "
                         "%.2f reduce %.2f\n",
                         mode, grid, nvec, hs[0].iters, t[0] / it_n / 1e3, t[1] / it_n / 1e3, t[2] / it_n / 1e3,
                         t[3] / it_n / 1e3);
        }
        // restart the items whose true residual misses rtol (recursion drift), from the current iterate
        bool again = false;
        for (int b = 0; b < B; ++b) {
            const CgState& s = hs[b];
            const bool fail = s.bn2 > 0.0 && !(s.res2 <= s.tol2);
            again |= S[b]->n_u > 0 && s.status == FEMI_OK && s.iters > 0 && s.iters < s.max_iter && fail;
        }
        if (!again || restarts >= 8) break;
        ++restarts;
        // k_true_res left r = s * r_true and x^ is current: the CG loop restarts from there.
        // Items that already passed run zero iterations (rho <= tol2 at entry).
    }
    {
        int64_t mmax = 1;
        for (int b = 0; b < B; ++b) mmax = std::max(mmax, S[b]->m);
        k_copy_g<<<dim3((unsigned)std::min<int64_t>((mmax + 255) / 256, 296), gy), 256, 0, st>>>(d_items);
        count_launches(1);
        FEMI_CUDA(cudaGetLastError());
        if (async) {
            k_stats<<<1, 32, 0, st>>>(B, d_items, ds);
            count_launches(1);
            FEMI_CUDA(cudaFreeAsync(d_gate, st));
            FEMI_CUDA(cudaGetLastError());
            return FEMI_OK;  // the workspace is released stream-ordered (Workspace)
        }
        // the header promises a synchronised stream: u_vert's mask entries are written when we return
        FEMI_CUDA(cudaStreamSynchronize(st));
    }
    if (ds) {  // asynchronous caller on a synchronous path (persistent kernel): same statistics
        k_stats<<<1, 32, 0, st>>>(B, d_items, ds);
        count_launches(1);
    }
    return solve_outcome(B, S, hs, o, iters, relres, total_iters);
}

}  // namespace femi

FEMI_DCHECK_READER(dcheck_pcg)
