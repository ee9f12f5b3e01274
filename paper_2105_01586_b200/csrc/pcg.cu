// pcg.cu -- S2: batched Jacobi-preconditioned CG for A_uu x = -A_uk g.
//
// The Jacobi preconditioner is folded into the matrix at assembly (A^ = D^-1/2 A D^-1/2,
// unit diagonal, only the off-diagonal CSR is stored), so CG runs on A^ x^ = b^ with
// x = D^-1/2 x^, b^ = D^-1/2 b. Per iteration two kernels, both over row chunks of all
// active batch items (block-diagonal batching: one chunk table spans every system):
//   K1  p_new = r + beta p_old (computed on the fly for every column it touches, so no
//       separate update pass), q = A^ p_new via a CSR-stream SpMV (coalesced val/col
//       loads into shared memory, one row per thread), partial dot(p_new, q);
//       the last CTA of an item turns the partials into alpha.
//   K2  x += alpha p_new, r -= alpha q, partial dot(r,r) and ||D^1/2 r||^2 (the unscaled
//       residual used by the stopping rule); the last CTA computes beta, the iteration
//       count and the convergence flag.
// All reductions are per-CTA partials summed in a fixed order by the item's last CTA
// (deterministic). Vector traffic per iteration: K1 reads r,p_old and writes p_new,q;
// K2 reads x,p_new,r,q,s and writes x,r (11 streams of 8 B per row, SURVEY §8(d) S=11).
// The stopping rule uses the true unscaled relative residual ||b - A x|| / ||b||,
// confirmed at exit with the unscaled matrix; a failed confirmation restarts CG from the
// current iterate (reading A11).
#include <algorithm>
#include <cmath>

#include "device.cuh"

namespace femi {
namespace {

constexpr int NT = kRowsPerChunk;  // threads per CTA == max rows per chunk

__device__ __forceinline__ unsigned long long dkey(double v) {
    unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

// Last-CTA election for a per-item reduction: returns true in every thread of the last CTA.
__device__ __forceinline__ bool last_cta(uint32_t* counter, uint32_t total, int* sh_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        uint32_t prev = atomicAdd(counter, 1u);
        *sh_flag = (prev == total - 1);
    }
    __syncthreads();
    if (*sh_flag) __threadfence();
    return *sh_flag != 0;
}

__global__ void k_reset(int B, SolveItem* items, CgState* st, double rtol, int max_iter) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    CgState s = {};
    s.rtol = rtol;
    s.max_iter = max_iter;
    s.kmin = ~0ull;
    s.kmax = 0ull;
    s.active = 1;
    st[b] = s;
}

__global__ void k_minmax(int B, const SolveItem* __restrict__ items, CgState* st) {
    for (int b = 0; b < B; ++b) {
        const SolveItem& it = items[b];
        if (it.x0mode != 1 || it.g == nullptr) continue;
        unsigned long long lo = ~0ull, hi = 0ull;
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < it.m; k += gridDim.x * blockDim.x) {
            unsigned long long key = dkey(it.g[k]);
            lo = min(lo, key);
            hi = max(hi, key);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if ((threadIdx.x & 31) == 0 && hi != 0ull) {
            atomicMin(&st[b].kmin, lo);
            atomicMax(&st[b].kmax, hi);
        }
    }
}

// b = -A_uk g (or the given b); x^0; ||b||^2
__global__ void __launch_bounds__(NT) k_rhs(const SolveItem* __restrict__ items, CgState* __restrict__ st,
                                            const Chunk* __restrict__ chunks, double* __restrict__ part) {
    __shared__ double red[NT / 32];
    __shared__ int flag;
    const Chunk c = chunks[blockIdx.x];
    const SolveItem& it = items[c.item];
    CgState* S = st + c.item;
    const int i = c.row0 + threadIdx.x;
    double loc = 0.0;
    if (i < c.row1) {
        double bi;
        if (it.bin) {
            bi = it.bin[i];
        } else {
            double acc = 0.0;
            for (int e = it.krp[i]; e < it.krp[i + 1]; ++e) acc = acc + it.kav[e] * it.g[it.kci[e]];
            bi = -acc;
        }
        it.b[i] = bi;
        loc = bi * bi;
        const double si = it.s[i];
        double x0;
        if (it.x0mode == 1) x0 = 0.5 * (dkey_inv(S->kmin) + dkey_inv(S->kmax));
        else if (it.x0mode == 2) x0 = it.u_vert[i];
        else x0 = 0.0;
        it.x[i] = x0 / si;
    }
    double tot = block_sum<NT>(loc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
    if (last_cta(&S->cnt[0], it.nchunks, &flag)) {
        double s = 0.0;
        for (int k = threadIdx.x; k < it.nchunks; k += NT) s += __ldcg(&part[it.chunk0 + k]);
        s = block_sum<NT>(s, red);
        if (threadIdx.x == 0) {
            S->bn2 = s;
            S->tol2 = S->rtol * S->rtol * s;
            S->cnt[0] = 0;
        }
    }
}

// r^ = b^ - A^ x^ ; p_old = 0 ; rr, rru. keep_iters: restart after a failed confirmation.
__global__ void __launch_bounds__(NT) k_init_res(const SolveItem* __restrict__ items, CgState* __restrict__ st,
                                                 const Chunk* __restrict__ chunks, double2* __restrict__ part,
                                                 int restart) {
    __shared__ double red[NT / 32];
    __shared__ int flag;
    const Chunk c = chunks[blockIdx.x];
    const SolveItem& it = items[c.item];
    CgState* S = st + c.item;
    if (restart && !S->active) return;
    const int i = c.row0 + threadIdx.x;
    double l1 = 0.0, l2 = 0.0;
    if (i < c.row1) {
        const double si = it.s[i];
        if (restart) it.x[i] = it.u_vert[i] / si;
        double ax = 0.0;
        for (int e = it.orp[i]; e < it.orp[i + 1]; ++e) {
            const int j = it.oci[e];
            const double xj = restart ? it.u_vert[j] / it.s[j] : it.x[j];
            ax = fma(it.oav[e], xj, ax);
        }
        const double xi = restart ? it.u_vert[i] / si : it.x[i];
        const double ri = si * it.b[i] - (xi + ax);
        it.r[i] = ri;
        it.p[0][i] = 0.0;
        it.p[1][i] = 0.0;
        l1 = ri * ri;
        const double ru = ri / si;
        l2 = ru * ru;
    }
    double t1 = block_sum<NT>(l1, red);
    double t2 = block_sum<NT>(l2, red);
    if (threadIdx.x == 0) part[blockIdx.x] = make_double2(t1, t2);
    if (last_cta(&S->cnt[1], it.nchunks, &flag)) {
        double s1 = 0.0, s2 = 0.0;
        for (int k = threadIdx.x; k < it.nchunks; k += NT) {
            double2 v = __ldcg(&part[it.chunk0 + k]);
            s1 += v.x;
            s2 += v.y;
        }
        s1 = block_sum<NT>(s1, red);
        s2 = block_sum<NT>(s2, red);
        if (threadIdx.x == 0) {
            S->rr = s1;
            S->rru = s2;
            S->beta = 0.0;
            if (!restart) S->iters = 0;
            S->cnt[1] = 0;
            if (!isfinite(s1) || !isfinite(S->bn2)) {
                S->active = 0;
                S->status = FEMI_E_NONFINITE;
            } else {
                S->active = (S->bn2 > 0.0 && s2 > S->tol2) ? 1 : 0;
            }
        }
    }
}

// K1: p_new = r + beta p_old ; q = A^ p_new ; partial p_new.q ; alpha
__global__ void __launch_bounds__(NT) k_spmv_dot(const SolveItem* __restrict__ items, CgState* __restrict__ st,
                                                 const Chunk* __restrict__ chunks, double* __restrict__ part) {
    __shared__ double prod[kChunkNnzCap];
    __shared__ double red[NT / 32];
    __shared__ int flag;
    const Chunk c = chunks[blockIdx.x];
    CgState* S = st + c.item;
    if (!S->active) return;
    const SolveItem& it = items[c.item];
    const double beta = S->beta;
    const int par = S->iters & 1;
    const double* __restrict__ po = it.p[par];
    double* __restrict__ pn = it.p[par ^ 1];
    const double* __restrict__ r = it.r;
    const int32_t* __restrict__ orp = it.orp;
    const int32_t* __restrict__ oci = it.oci;
    const double* __restrict__ oav = it.oav;
    const int e0 = orp[c.row0], e1 = orp[c.row1];
    const bool staged = (e1 - e0) <= kChunkNnzCap;
    if (staged)
        for (int e = e0 + threadIdx.x; e < e1; e += NT) {
            const int j = oci[e];
            prod[e - e0] = oav[e] * fma(beta, po[j], r[j]);
        }
    __syncthreads();
    double loc = 0.0;
    const int i = c.row0 + threadIdx.x;
    if (i < c.row1) {
        const double pi = fma(beta, po[i], r[i]);
        double acc = pi;  // unit diagonal
        const int a = orp[i], b = orp[i + 1];
        if (staged) {
            for (int e = a; e < b; ++e) acc += prod[e - e0];
        } else {
            for (int e = a; e < b; ++e) {
                const int j = oci[e];
                acc += oav[e] * fma(beta, po[j], r[j]);
            }
        }
        pn[i] = pi;
        it.q[i] = acc;
        loc = pi * acc;
    }
    double tot = block_sum<NT>(loc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
    if (last_cta(&S->cnt[2], it.nchunks, &flag)) {
        double s = 0.0;
        for (int k = threadIdx.x; k < it.nchunks; k += NT) s += __ldcg(&part[it.chunk0 + k]);
        s = block_sum<NT>(s, red);
        if (threadIdx.x == 0) {
            S->pq = s;
            S->cnt[2] = 0;
            if (!(s > 0.0)) {
                S->active = 0;
                S->status = isfinite(s) ? FEMI_E_NEG_CURVATURE : FEMI_E_NONFINITE;
            } else {
                S->alpha = S->rr / s;
            }
        }
    }
}

// K2: x += alpha p_new ; r -= alpha q ; rr ; rru ; beta ; convergence
__global__ void __launch_bounds__(NT) k_update(const SolveItem* __restrict__ items, CgState* __restrict__ st,
                                               const Chunk* __restrict__ chunks, double2* __restrict__ part) {
    __shared__ double red[NT / 32];
    __shared__ int flag;
    const Chunk c = chunks[blockIdx.x];
    CgState* S = st + c.item;
    if (!S->active) return;
    const SolveItem& it = items[c.item];
    const double alpha = S->alpha;
    const double* __restrict__ pn = it.p[(S->iters & 1) ^ 1];
    const int i = c.row0 + threadIdx.x;
    double l1 = 0.0, l2 = 0.0;
    if (i < c.row1) {
        it.x[i] = fma(alpha, pn[i], it.x[i]);
        const double ri = fma(-alpha, it.q[i], it.r[i]);
        it.r[i] = ri;
        l1 = ri * ri;
        const double ru = ri / it.s[i];
        l2 = ru * ru;
    }
    double t1 = block_sum<NT>(l1, red);
    double t2 = block_sum<NT>(l2, red);
    if (threadIdx.x == 0) part[blockIdx.x] = make_double2(t1, t2);
    if (last_cta(&S->cnt[3], it.nchunks, &flag)) {
        double s1 = 0.0, s2 = 0.0;
        for (int k = threadIdx.x; k < it.nchunks; k += NT) {
            double2 v = __ldcg(&part[it.chunk0 + k]);
            s1 += v.x;
            s2 += v.y;
        }
        s1 = block_sum<NT>(s1, red);
        s2 = block_sum<NT>(s2, red);
        if (threadIdx.x == 0) {
            S->cnt[3] = 0;
            S->iters += 1;
            S->beta = s1 / S->rr;
            S->rr = s1;
            S->rru = s2;
            if (!isfinite(s1)) {
                S->active = 0;
                S->status = FEMI_E_NONFINITE;
            } else if (s2 <= S->tol2) {
                S->active = 0;
            } else if (S->iters >= S->max_iter) {
                S->active = 0;
                S->status = FEMI_E_NOT_CONVERGED;
            }
        }
    }
}

// x = D^-1/2 x^ into u_vert (or x0 untouched after a 0-iteration exit, 0 when b == 0),
// then the true residual ||b - A x||^2 with the unscaled matrix.
__global__ void __launch_bounds__(NT) k_finalize(const SolveItem* __restrict__ items, CgState* __restrict__ st,
                                                 const Chunk* __restrict__ chunks) {
    const Chunk c = chunks[blockIdx.x];
    const SolveItem& it = items[c.item];
    CgState* S = st + c.item;
    const int i = c.row0 + threadIdx.x;
    if (i >= c.row1) return;
    double xi;
    if (S->bn2 == 0.0) xi = 0.0;
    else if (S->iters == 0) {
        if (it.x0mode == 2) return;  // caller's initial guess stays as it is
        xi = (it.x0mode == 1) ? 0.5 * (dkey_inv(S->kmin) + dkey_inv(S->kmax)) : 0.0;
    } else {
        xi = it.s[i] * it.x[i];
    }
    it.u_vert[i] = xi;
}

__global__ void __launch_bounds__(NT) k_true_res(const SolveItem* __restrict__ items, CgState* __restrict__ st,
                                                 const Chunk* __restrict__ chunks, double* __restrict__ part) {
    __shared__ double red[NT / 32];
    __shared__ int flag;
    const Chunk c = chunks[blockIdx.x];
    const SolveItem& it = items[c.item];
    CgState* S = st + c.item;
    const int i = c.row0 + threadIdx.x;
    double loc = 0.0;
    if (i < c.row1) {
        double ax = 0.0;
        for (int e = it.urp[i]; e < it.urp[i + 1]; ++e) ax = fma(it.uav[e], it.u_vert[it.uci[e]], ax);
        const double ri = it.b[i] - ax;
        loc = ri * ri;
    }
    double tot = block_sum<NT>(loc, red);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
    if (last_cta(&S->cnt[0], it.nchunks, &flag)) {
        double s = 0.0;
        for (int k = threadIdx.x; k < it.nchunks; k += NT) s += __ldcg(&part[it.chunk0 + k]);
        s = block_sum<NT>(s, red);
        if (threadIdx.x == 0) {
            S->res2 = s;
            S->cnt[0] = 0;
        }
    }
}

__global__ void k_copy_g(int B, const SolveItem* __restrict__ items) {
    const SolveItem& it = items[blockIdx.y];
    if (!it.g) return;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < it.m; k += gridDim.x * blockDim.x)
        it.u_vert[it.n + k] = it.g[k];
}

struct Workspace {
    void* base = nullptr;
    cudaStream_t st = nullptr;
    ~Workspace() {
        if (base) cudaFreeAsync(base, st);
    }
};

}  // namespace

femi_status pcg_solve(int B, femi_system_s* const* S, const double* const* g, const double* const* bin,
                      double* const* u_vert, const femi_cg_opts& o, int32_t* iters, double* relres,
                      cudaStream_t st, int64_t* total_iters) {
    // ---- plan: items, chunk table, scratch layout
    std::vector<SolveItem> items(B);
    std::vector<Chunk> chunks;
    int64_t vec_doubles = 0;
    for (int b = 0; b < B; ++b) vec_doubles += 6 * (S[b]->n_u + 1);
    int32_t total_chunks = 0;
    for (int b = 0; b < B; ++b) total_chunks += (int32_t)S[b]->chunks_h.size();
    const size_t bytes_vec = sizeof(double) * (size_t)vec_doubles;
    const size_t bytes_items = sizeof(SolveItem) * B;
    const size_t bytes_state = sizeof(CgState) * B;
    const size_t bytes_chunks = (B == 1) ? 0 : sizeof(Chunk) * (size_t)total_chunks;
    const size_t bytes_part = sizeof(double2) * (size_t)std::max(total_chunks, 1);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t total = al(bytes_vec) + al(bytes_items) + al(bytes_state) + al(bytes_chunks) + al(bytes_part);
    Workspace ws;
    ws.st = st;
    FEMI_CUDA(cudaMallocAsync(&ws.base, total, st));
    char* cur = (char*)ws.base;
    double* vec = (double*)cur;
    cur += al(bytes_vec);
    SolveItem* d_items = (SolveItem*)cur;
    cur += al(bytes_items);
    CgState* d_state = (CgState*)cur;
    cur += al(bytes_state);
    Chunk* d_chunks = (Chunk*)cur;
    cur += al(bytes_chunks);
    double* d_part = (double*)cur;

    int32_t c0 = 0;
    for (int b = 0; b < B; ++b) {
        femi_system_s* s = S[b];
        SolveItem& it = items[b];
        const int64_t n = s->n_u;
        it.orp = s->o_rowptr;
        it.oci = s->o_col;
        it.oav = s->o_val;
        it.s = s->s;
        it.urp = s->uu_rowptr;
        it.uci = s->uu_col;
        it.uav = s->uu_val;
        it.krp = s->uk_rowptr;
        it.kci = s->uk_col;
        it.kav = s->uk_val;
        it.g = g ? g[b] : nullptr;
        it.bin = bin ? bin[b] : nullptr;
        it.u_vert = u_vert[b];
        it.x = vec;
        it.r = vec + (n + 1);
        it.q = vec + 2 * (n + 1);
        it.b = vec + 3 * (n + 1);
        it.p[0] = vec + 4 * (n + 1);
        it.p[1] = vec + 5 * (n + 1);
        vec += 6 * (n + 1);
        it.n = (int32_t)n;
        it.m = (int32_t)s->m;
        it.chunk0 = c0;
        it.nchunks = (int32_t)s->chunks_h.size();
        it.x0mode = (it.g == nullptr && o.x0 == 1) ? 0 : o.x0;
        if (B > 1)
            for (const Chunk& ch : s->chunks_h) chunks.push_back({b, ch.row0, ch.row1, ch.local});
        c0 += it.nchunks;
    }
    if (B == 1) d_chunks = S[0]->chunks_d;
    FEMI_CUDA(cudaMemcpyAsync(d_items, items.data(), bytes_items, cudaMemcpyHostToDevice, st));
    if (B > 1) FEMI_CUDA(cudaMemcpyAsync(d_chunks, chunks.data(), bytes_chunks, cudaMemcpyHostToDevice, st));

    // ---- init
    k_reset<<<(B + 127) / 128, 128, 0, st>>>(B, d_items, d_state, o.rtol, o.max_iter); count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    if (o.x0 == 1) {
        int64_t mmax = 0;
        for (int b = 0; b < B; ++b) mmax = std::max(mmax, S[b]->m);
        int gb = (int)std::max<int64_t>(1, std::min<int64_t>((mmax + 255) / 256, 296));
        k_minmax<<<gb, 256, 0, st>>>(B, d_items, d_state); count_launches(1);
        FEMI_CUDA(cudaGetLastError());
    }
    if (total_chunks > 0) {
        k_rhs<<<total_chunks, NT, 0, st>>>(d_items, d_state, d_chunks, d_part); count_launches(1);
        FEMI_CUDA(cudaGetLastError());
        k_init_res<<<total_chunks, NT, 0, st>>>(d_items, d_state, d_chunks, (double2*)d_part, 0); count_launches(1);
        FEMI_CUDA(cudaGetLastError());
    }
    {
        int64_t mmax = 1;
        for (int b = 0; b < B; ++b) mmax = std::max(mmax, S[b]->m);
        dim3 gg((unsigned)std::min<int64_t>((mmax + 255) / 256, 64), B);
        k_copy_g<<<gg, 256, 0, st>>>(B, d_items); count_launches(1);
        FEMI_CUDA(cudaGetLastError());
    }

    std::vector<CgState> hs(B);
    const int check = o.check_every > 0 ? o.check_every : 8;
    int restarts = 0;
    for (;;) {
        // ---- iterate until every item is inactive (poll every `check` iterations)
        bool any = total_chunks > 0;
        while (any) {
            for (int k = 0; k < check; ++k) {
                k_spmv_dot<<<total_chunks, NT, 0, st>>>(d_items, d_state, d_chunks, d_part); count_launches(1);
                k_update<<<total_chunks, NT, 0, st>>>(d_items, d_state, d_chunks, (double2*)d_part); count_launches(1);
            }
            FEMI_CUDA(cudaGetLastError());
            FEMI_CUDA(cudaMemcpyAsync(hs.data(), d_state, bytes_state, cudaMemcpyDeviceToHost, st));
            FEMI_CUDA(cudaStreamSynchronize(st));
            any = false;
            for (int b = 0; b < B; ++b) any |= hs[b].active != 0;
        }
        if (total_chunks > 0) {
            k_finalize<<<total_chunks, NT, 0, st>>>(d_items, d_state, d_chunks); count_launches(1);
            k_true_res<<<total_chunks, NT, 0, st>>>(d_items, d_state, d_chunks, d_part); count_launches(1);
            FEMI_CUDA(cudaGetLastError());
        }
        FEMI_CUDA(cudaMemcpyAsync(hs.data(), d_state, bytes_state, cudaMemcpyDeviceToHost, st));
        FEMI_CUDA(cudaStreamSynchronize(st));
        // confirmation of the true residual; restart the items that fail it
        bool again = false;
        for (int b = 0; b < B; ++b) {
            const CgState& s = hs[b];
            double rel = s.bn2 > 0.0 ? std::sqrt(s.res2 / s.bn2) : 0.0;
            if (s.status == FEMI_OK && s.iters > 0 && s.iters < s.max_iter && !(rel <= o.rtol) && restarts < 8)
                again = true;
        }
        if (!again) break;
        ++restarts;
        // reactivate the failing items and rebuild r from the current x
        for (int b = 0; b < B; ++b) {
            const CgState& s = hs[b];
            double rel = s.bn2 > 0.0 ? std::sqrt(s.res2 / s.bn2) : 0.0;
            int act = (s.status == FEMI_OK && s.iters > 0 && s.iters < s.max_iter && !(rel <= o.rtol)) ? 1 : 0;
            FEMI_CUDA(cudaMemcpyAsync(&d_state[b].active, &act, sizeof(int), cudaMemcpyHostToDevice, st));
        }
        k_init_res<<<total_chunks, NT, 0, st>>>(d_items, d_state, d_chunks, (double2*)d_part, 1); count_launches(1);
        FEMI_CUDA(cudaGetLastError());
    }
    femi_status ret = FEMI_OK;
    int64_t tot = 0;
    for (int b = 0; b < B; ++b) {
        const CgState& s = hs[b];
        if (iters) iters[b] = s.iters;
        double rel = s.bn2 > 0.0 ? std::sqrt(s.res2 / s.bn2) : 0.0;
        if (S[b]->n_u == 0) rel = 0.0;
        if (relres) relres[b] = rel;
        tot += s.iters;
        femi_status sb = (femi_status)s.status;
        if (sb == FEMI_OK && !(rel <= o.rtol)) sb = FEMI_E_NOT_CONVERGED;
        if (sb != FEMI_OK && ret == FEMI_OK) ret = sb;
    }
    if (total_iters) *total_iters = tot;
    if (ret != FEMI_OK) set_error("inpaint_solve: CG did not converge (status " + std::to_string((int)ret) + ")");
    return ret;
}

}  // namespace femi
