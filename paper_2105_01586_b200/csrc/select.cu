// select.cu -- S5 densify_step selection (readings A8-A10).
//
// "insert a single mask pixel in each triangle, in descending order of the L2 error ...
// at the empty location with the largest pointwise error": the triangles are ranked by
// (tri_err desc, index asc) -- a top-b selection, not a full sort. Keys are the fp64 bit
// patterns (order-preserving for non-negative values); an 8-pass MSB radix select finds
// the b-th key K, then one pass emits every key > K and the lowest-index ties == K via a
// block-ordered prefix count (deterministic, no sort). The optional shortfall fill runs
// the same selection over the empty pixels' e-values. Output pixels go to the host,
// which returns them ascending.
#include <algorithm>
#include <cstdlib>

#include "device.cuh"

namespace femi {
namespace {

constexpr int ST = 256;
constexpr int64_t kSelBlockMax = 1 << 20;  // T up to which the one-block selection is used

struct SelState {
    unsigned long long prefix, mask;
    long long remaining;  // how many still to take at or below the current prefix
    long long count_gt;   // keys strictly above the final threshold
    long long eligible;   // keys > 0
    unsigned int hist[256];
};

__global__ void k_tri_keys(int64_t T, const double* __restrict__ tri_err, const int32_t* __restrict__ best,
                           unsigned long long* __restrict__ key, SelState* ss) {
    long long cnt = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
        const double e = tri_err[t];
        const bool ok = e > 0.0 && best[t] >= 0;
        const unsigned long long k = ok ? (unsigned long long)__double_as_longlong(e) : 0ull;
        key[t] = k;
        cnt += ok;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd((unsigned long long*)&ss->eligible, (unsigned long long)cnt);
}

// empty pixels: e >= 0 -> key = bits(e) + 1; vertices / already selected -> 0
__global__ void k_px_keys(int64_t N, const double* __restrict__ e_px, const uint8_t* __restrict__ taken,
                          unsigned long long* __restrict__ key, SelState* ss) {
    long long cnt = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
        const bool ok = !taken[p];
        key[p] = ok ? (unsigned long long)__double_as_longlong(e_px[p]) + 1ull : 0ull;
        cnt += ok;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd((unsigned long long*)&ss->eligible, (unsigned long long)cnt);
}

__global__ void k_hist(int64_t n, const unsigned long long* __restrict__ key, SelState* ss, int shift) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long prefix = ss->prefix, mask = ss->mask;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = key[i];
        if (k != 0ull && (k & mask) == prefix) atomicAdd(&h[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&ss->hist[threadIdx.x], h[threadIdx.x]);
}

__global__ void k_pick(SelState* ss, int shift) {
    // one warp: find digit D (descending) where the cumulative count reaches `remaining`
    if (threadIdx.x != 0) return;
    long long cum = 0;
    int D = 0;
    for (int d = 255; d >= 0; --d) {
        const long long c = ss->hist[d];
        if (cum + c >= ss->remaining) {
            D = d;
            break;
        }
        cum += c;
    }
    ss->count_gt += cum;
    ss->remaining -= cum;
    ss->prefix |= (unsigned long long)D << shift;
    ss->mask |= 255ull << shift;
    for (int d = 0; d < 256; ++d) ss->hist[d] = 0;
}

// emit keys > K (any order) and the first `need` ties (ascending index, block-ordered)
__global__ void k_tie_count(int64_t n, int64_t per, const unsigned long long* __restrict__ key, const SelState* ss,
                            long long* __restrict__ bcount) {
    __shared__ long long red[ST / 32];
    const unsigned long long K = ss->prefix;
    const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
    long long c = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += ST) c += (key[i] == K);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < ST / 32; ++w) t += red[w];
        bcount[blockIdx.x] = t;
    }
}

__global__ void k_scan_small(int nb, long long* bcount) {  // exclusive scan, one thread (nb is small)
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    long long run = 0;
    for (int b = 0; b < nb; ++b) {
        long long c = bcount[b];
        bcount[b] = run;
        run += c;
    }
}

__global__ void k_emit(int64_t n, int64_t per, const unsigned long long* __restrict__ key, const SelState* ss,
                       const long long* __restrict__ boff, const int32_t* __restrict__ map, int32_t* __restrict__ out,
                       unsigned long long* __restrict__ out_count) {
    __shared__ int wsum[ST / 32];
    const unsigned long long K = ss->prefix;
    const long long need = ss->remaining;
    const int64_t lo = blockIdx.x * per, hi = min(n, lo + per);
    long long base = boff[blockIdx.x];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t t0 = lo; t0 < hi; t0 += ST) {
        const int64_t i = t0 + threadIdx.x;
        const unsigned long long k = (i < hi) ? key[i] : 0ull;
        const bool gt = k > K;
        const bool tie = (i < hi) && k == K;
        if (gt) {
            unsigned long long pos = atomicAdd(out_count, 1ull);
            out[pos] = map ? map[i] : (int32_t)i;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, tie);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        int before = 0, tot = 0;
        for (int w = 0; w < ST / 32; ++w) {
            if (w < wid) before += wsum[w];
            tot += wsum[w];
        }
        const long long rank = base + before + __popc(bal & ((1u << lane) - 1u));
        if (tie && rank < need) {
            unsigned long long pos = atomicAdd(out_count, 1ull);
            out[pos] = map ? map[i] : (int32_t)i;
        }
        base += tot;
        __syncthreads();
    }
}

__global__ void k_mark(int64_t n, const int32_t* __restrict__ px, uint8_t* __restrict__ taken) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    {
        FEMI_DCHECK(px[i] >= 0, 5);
        taken[px[i]] = 1;
    }
}

__global__ void k_gather_best(int64_t n, const int32_t* __restrict__ idx, const int32_t* __restrict__ best,
                              int32_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    {
        FEMI_DCHECK(idx[i] >= 0, 5);
        out[i] = best[idx[i]];
    }
}

// The whole triangle selection in ONE block for small T (densification of small and medium
// images, where the multi-kernel radix select is launch-latency bound): keys, eligible count,
// k = min(eligible, b), the same 8-pass MSB radix select and the same emission rule (keys > K,
// then the lowest-index ties == K), each selected triangle mapped to its best pixel. out_count
// receives the number emitted (= k). Same result as the multi-kernel path.
constexpr int SB = 1024;
__global__ void __launch_bounds__(SB) k_select_tri_block(int64_t T, const double* __restrict__ tri_err,
                                                        const int32_t* __restrict__ best, long long b,
                                                        unsigned long long* __restrict__ key, int32_t* __restrict__ out,
                                                        unsigned long long* __restrict__ out_count) {
    __shared__ unsigned int hist[256];
    __shared__ long long s_red[SB / 32];
    __shared__ unsigned long long s_prefix, s_mask;
    __shared__ long long s_remaining, s_k;
    __shared__ unsigned int s_out;
    __shared__ int s_wsum[SB / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // keys and the eligible count
    long long cnt = 0;
    for (int64_t t = tid; t < T; t += SB) {
        const double e = tri_err[t];
        const bool ok = e > 0.0 && best[t] >= 0;
        key[t] = ok ? (unsigned long long)__double_as_longlong(e) : 0ull;
        cnt += ok;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s_red[wid] = cnt;
    __syncthreads();
    if (tid == 0) {
        long long E = 0;
        for (int w = 0; w < SB / 32; ++w) E += s_red[w];
        s_k = E < b ? E : b;
        s_remaining = s_k;
        s_prefix = 0ull;
        s_mask = 0ull;
        s_out = 0u;
    }
    __syncthreads();
    if (s_k == 0) {
        if (tid == 0) *out_count = 0ull;
        return;
    }
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        if (tid < 256) hist[tid] = 0u;
        __syncthreads();
        const unsigned long long prefix = s_prefix, mask = s_mask;
        for (int64_t i = tid; i < T; i += SB) {
            const unsigned long long k = key[i];
            if (k != 0ull && (k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (wid == 0) {  // digit D (descending) where the cumulative count reaches `remaining`
            const long long rem = s_remaining;
            long long c = 0;
            for (int q = 0; q < 8; ++q) c += hist[255 - 8 * lane - q];
            long long incl = c;
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, incl >= rem);
            const int L = __ffs(hit) - 1;  // first lane (highest digits) reaching rem
            if (lane == L) {
                long long cum = incl - c;
                int D = 255 - 8 * lane;
                for (int q = 0; q < 8; ++q) {
                    const int d = 255 - 8 * lane - q;
                    const long long h = hist[d];
                    if (cum + h >= rem) {
                        D = d;
                        break;
                    }
                    cum += h;
                }
                s_remaining = rem - cum;
                s_prefix = prefix | ((unsigned long long)D << shift);
                s_mask = mask | (255ull << shift);
            }
        }
        __syncthreads();
    }
    // emission in index order: keys > K anywhere, ties == K by ascending index
    const unsigned long long K = s_prefix;
    const long long need = s_remaining;
    long long base = 0;
    for (int64_t t0 = 0; t0 < T; t0 += SB) {
        const int64_t i = t0 + tid;
        const unsigned long long k = i < T ? key[i] : 0ull;
        const bool tie = i < T && k == K;
        if (k > K) out[atomicAdd(&s_out, 1u)] = best[i];
        const unsigned bal = __ballot_sync(0xffffffffu, tie);
        if (lane == 0) s_wsum[wid] = __popc(bal);
        __syncthreads();
        int before = 0, tot = 0;
        for (int w = 0; w < SB / 32; ++w) {
            before += w < wid ? s_wsum[w] : 0;
            tot += s_wsum[w];
        }
        if (tie && base + before + __popc(bal & ((1u << lane) - 1u)) < need) out[atomicAdd(&s_out, 1u)] = best[i];
        base += tot;
        __syncthreads();
    }
    if (tid == 0) *out_count = s_out;
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + ST - 1) / ST, 148 * 8)); }

// top-k (key desc, index asc) among keys != 0; writes up to k selected indices (mapped through
// `map` if given) to out; returns the count. Keys must already be in d_key; ss->eligible set.
femi_status select_topk(int64_t n, int64_t k, unsigned long long* d_key, SelState* d_ss, const int32_t* map,
                        int32_t* d_out, unsigned long long* d_cnt, long long* d_bcount, int nb, int64_t per,
                        cudaStream_t st) {
    // remaining = k
    long long kk = k;
    FEMI_CUDA(cudaMemcpyAsync(&d_ss->remaining, &kk, sizeof(long long), cudaMemcpyHostToDevice, st));
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        k_hist<<<grid_for(n), ST, 0, st>>>(n, d_key, d_ss, shift); count_launches(1);
        k_pick<<<1, 32, 0, st>>>(d_ss, shift); count_launches(1);
    }
    k_tie_count<<<nb, ST, 0, st>>>(n, per, d_key, d_ss, d_bcount); count_launches(1);
    k_scan_small<<<1, 32, 0, st>>>(nb, d_bcount); count_launches(1);
    k_emit<<<nb, ST, 0, st>>>(n, per, d_key, d_ss, d_bcount, map, d_out, d_cnt); count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    return FEMI_OK;
}

}  // namespace

femi_status densify_select(femi_system_s* S, int nc, const double* const* f, const double* const* u_vert, int64_t b,
                           int32_t* new_px, int64_t* n_added, cudaStream_t st) {
    *n_added = 0;
    if (b <= 0) return FEMI_OK;
    const int64_t T = S->T, N = (int64_t)S->W * S->H;
    const int64_t nmax = std::max(T, N);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const int nb = (int)std::min<int64_t>(1024, std::max<int64_t>(1, (nmax + ST - 1) / ST));
    size_t bytes = al(sizeof(double) * T) + al(sizeof(int32_t) * T) + al(sizeof(unsigned long long) * nmax) +
                   al(sizeof(SelState)) + al(sizeof(int32_t) * (b + 1)) + al(sizeof(int32_t) * (b + 1)) +
                   al(sizeof(unsigned long long)) + al(sizeof(long long) * nb) + al(sizeof(double));
    void* base = nullptr;
    FEMI_CUDA(cudaMallocAsync(&base, bytes, st));
    char* cur = (char*)base;
    auto take = [&](size_t x) {
        char* p = cur;
        cur += al(x);
        return p;
    };
    double* tri_err = (double*)take(sizeof(double) * T);
    int32_t* best = (int32_t*)take(sizeof(int32_t) * T);
    unsigned long long* key = (unsigned long long*)take(sizeof(unsigned long long) * nmax);
    SelState* ss = (SelState*)take(sizeof(SelState));
    int32_t* sel_idx = (int32_t*)take(sizeof(int32_t) * (b + 1));
    int32_t* sel_px = (int32_t*)take(sizeof(int32_t) * (b + 1));
    unsigned long long* cnt = (unsigned long long*)take(sizeof(unsigned long long));
    long long* bcount = (long long*)take(sizeof(long long) * nb);
    double* sse = (double*)take(sizeof(double));
    femi_status rc = FEMI_OK;
    std::vector<int32_t> result;
    auto fail = [&](femi_status s) {
        cudaFreeAsync(base, st);
        return s;
    };

    // the error map is the channel sum of (u_c - f_c)^2 (one channel: the grey error map)
    rc = launch_raster_channels(S, nc, u_vert, f, nullptr, nullptr, tri_err, best, sse, st);
    if (rc) return fail(rc);

    // ---- triangles: top-b by (tri_err desc, index asc)
    if (T <= kSelBlockMax && std::getenv("FEMI_SEL_MULTI") == nullptr) {
        // small T: one block does keys, count, select and emission; one round trip
        k_select_tri_block<<<1, SB, 0, st>>>(T, tri_err, best, b, key, sel_px, cnt);
        count_launches(1);
        unsigned long long hk = 0;
        if (cudaMemcpyAsync(&hk, cnt, sizeof(hk), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(cuda_fail(cudaGetLastError(), "densify: block select"));
        const int64_t k_tri = (int64_t)hk;
        result.resize(k_tri);
        if (k_tri > 0 &&
            cudaMemcpyAsync(result.data(), sel_px, sizeof(int32_t) * k_tri, cudaMemcpyDeviceToHost, st) != cudaSuccess)
            return fail(cuda_fail(cudaGetLastError(), "densify: copy"));
        if (k_tri == b) {
            if (cudaStreamSynchronize(st) != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "densify: sync"));
            std::sort(result.begin(), result.end());
            std::copy(result.begin(), result.end(), new_px);
            *n_added = (int64_t)result.size();
            cudaFreeAsync(base, st);
            return FEMI_OK;
        }
        // shortfall: fall through to the fill below with the triangle picks already in result
    }
    const bool tri_done = T <= kSelBlockMax && std::getenv("FEMI_SEL_MULTI") == nullptr;
    if (!tri_done && cudaMemsetAsync(ss, 0, sizeof(SelState), st) != cudaSuccess) return fail(FEMI_E_CUDA);
    SelState hs;
    int64_t k_tri = (int64_t)result.size();
    if (!tri_done) {
    if (cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st) != cudaSuccess) return fail(FEMI_E_CUDA);
    k_tri_keys<<<grid_for(T), ST, 0, st>>>(T, tri_err, best, key, ss); count_launches(1);
    if (cudaMemcpyAsync(&hs, ss, sizeof(SelState), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return fail(cuda_fail(cudaGetLastError(), "densify: eligible count"));
    const int64_t E = hs.eligible;
    k_tri = std::min(E, b);
    if (k_tri > 0) {
        const int nbt = (int)std::min<int64_t>(1024, (T + ST - 1) / ST);
        const int64_t per = (T + nbt - 1) / nbt;
        rc = select_topk(T, k_tri, key, ss, nullptr, sel_idx, cnt, bcount, nbt, per, st);
        if (rc) return fail(rc);
        k_gather_best<<<grid_for(k_tri), ST, 0, st>>>(k_tri, sel_idx, best, sel_px); count_launches(1);
        result.resize(k_tri);
        if (cudaMemcpyAsync(result.data(), sel_px, sizeof(int32_t) * k_tri, cudaMemcpyDeviceToHost, st) != cudaSuccess)
            return fail(cuda_fail(cudaGetLastError(), "densify: copy"));
    }
    }
    // ---- shortfall: globally largest-e empty pixels (reading A10)
    const int64_t short_b = b - k_tri;
    if (short_b > 0) {
        double* e_px = nullptr;
        uint8_t* taken = nullptr;
        if (cudaMallocAsync(&e_px, sizeof(double) * N, st) != cudaSuccess ||
            cudaMallocAsync(&taken, N, st) != cudaSuccess)
            return fail(cuda_fail(cudaGetLastError(), "densify: fill scratch"));
        rc = launch_raster_channels(S, nc, u_vert, f, nullptr, e_px, nullptr, nullptr, nullptr, st);
        if (rc) return fail(rc);
        cudaMemsetAsync(taken, 0, N, st);
        k_mark<<<grid_for(S->nv), ST, 0, st>>>(S->nv, S->vpix, taken); count_launches(1);
        if (k_tri > 0) k_mark<<<grid_for(k_tri), ST, 0, st>>>(k_tri, sel_px, taken); count_launches(1);
        cudaMemsetAsync(ss, 0, sizeof(SelState), st);
        cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st);
        k_px_keys<<<grid_for(N), ST, 0, st>>>(N, e_px, taken, key, ss); count_launches(1);
        if (cudaMemcpyAsync(&hs, ss, sizeof(SelState), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(cuda_fail(cudaGetLastError(), "densify: fill count"));
        const int64_t k_px = std::min<int64_t>(hs.eligible, short_b);
        if (k_px > 0) {
            const int nbp = (int)std::min<int64_t>(1024, (N + ST - 1) / ST);
            const int64_t per = (N + nbp - 1) / nbp;
            rc = select_topk(N, k_px, key, ss, nullptr, sel_idx, cnt, bcount, nbp, per, st);
            if (rc) return fail(rc);
            size_t off = result.size();
            result.resize(off + k_px);
            if (cudaMemcpyAsync(result.data() + off, sel_idx, sizeof(int32_t) * k_px, cudaMemcpyDeviceToHost, st) !=
                cudaSuccess)
                return fail(cuda_fail(cudaGetLastError(), "densify: copy fill"));
        }
        cudaFreeAsync(e_px, st);
        cudaFreeAsync(taken, st);
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "densify: sync"));
    std::sort(result.begin(), result.end());
    std::copy(result.begin(), result.end(), new_px);
    *n_added = (int64_t)result.size();
    cudaFreeAsync(base, st);
    return FEMI_OK;
}

}  // namespace femi

FEMI_DCHECK_READER(dcheck_select)
