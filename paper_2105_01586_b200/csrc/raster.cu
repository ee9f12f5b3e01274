// raster.cu -- S3+S4: rasterise the P1 solution and reduce the squared error
// (PAPER.md:L239-241 interpolation; L262-265 "e_i = (u_i - f_i)^2", "total L2 error in
// each triangle"), and the adjoint raster P^T r used by tonal optimisation (S6).
//
// Triangle-parallel with load-balanced expansion (raster_common.cuh): a pixel is
// processed by the triangle that owns it (reading A7: lowest index among the closed
// triangles containing it), decided locally from the edge functions and precomputed
// ownership flags -- no owner map, no atomics. A vertex pixel takes its vertex value
// exactly; otherwise u = u_a + l_b (u_b - u_a) + l_c (u_c - u_a), l = exact integer edge
// function / 2*area (S3). Per-triangle error sums and arg-max (ties: lowest pix) are
// sequential per triangle in pixel order; SSE is a per-CTA partial summed in fixed order
// by the last CTA: deterministic.
#include "raster_common.cuh"

namespace femi {
namespace {

struct RasterItem {
    const TriRec* tri;
    const double* u_vert;
    const double* f;
    double* u_px;
    double* e_px;
    double* tri_err;
    int32_t* best;
    double* sse;
    int64_t T;
    int32_t W;
    int32_t pad;
};

__global__ void __launch_bounds__(RB, 3) k_raster_error(const RasterItem* __restrict__ items, double* __restrict__ part,
                                                        uint32_t* __restrict__ counters) {
    __shared__ TriInfo info[RB];
    __shared__ double tu[RB][3];
    __shared__ int off[RB + 1];
    __shared__ int wsum[RB / 32];
    __shared__ double es[RCAP];
    __shared__ unsigned char cs[RCAP];
    __shared__ double red[RB / 32];
    __shared__ int flag;
    const RasterItem it = items[blockIdx.y];
    const int tid = threadIdx.x;
    const int64_t t0 = (int64_t)blockIdx.x * RB;
    double acc = 0.0, be = -1.0;
    int bp = -1, cnt = 0;
    if (t0 < it.T) {
        cnt = load_tris(it.tri, it.T, t0, info, off, wsum);
        if (tid < cnt) {
            const TriRec& R = it.tri[t0 + tid];
            tu[tid][0] = it.u_vert[R.v[0]];
            tu[tid][1] = it.u_vert[R.v[1]];
            tu[tid][2] = it.u_vert[R.v[2]];
        }
        __syncthreads();
        const int total = off[cnt];
        const bool with_f = it.f != nullptr;
        int j = 0;
        for (int r0 = 0; r0 < total; r0 += RCAP) {
            const int rend = min(total, r0 + RCAP);
            for (int k = r0 + tid; k < rend; k += RB) {
                while (off[j + 1] <= k) ++j;
                const TriInfo& I = info[j];
                const int loc = k - off[j];
                const int ry = loc / I.bw;
                const int py = I.y0 + ry, px = I.x0 + loc - ry * I.bw;
                int w0, w1, w2, kv = 0;
                const int cls = classify(I, px, py, w0, w1, w2, kv);
                cs[k - r0] = (unsigned char)cls;
                if (!cls) continue;
                double u;
                if (cls == 2) {
                    u = tu[j][kv];
                } else {
                    const double D = (double)I.D, ua = tu[j][0];
                    u = ua + (w1 / D) * (tu[j][1] - ua) + (w2 / D) * (tu[j][2] - ua);
                }
                const int64_t pix = (int64_t)py * it.W + px;
                if (it.u_px) it.u_px[pix] = u;
                if (with_f) {
                    const double d = u - it.f[pix];
                    const double e = d * d;
                    es[k - r0] = e;
                    if (it.e_px) it.e_px[pix] = e;
                }
            }
            __syncthreads();
            if (with_f && tid < cnt) {
                const int lo = max(off[tid], r0), hi = min(off[tid + 1], rend);
                for (int k = lo; k < hi; ++k) {
                    const int cls = cs[k - r0];
                    if (!cls) continue;
                    const double e = es[k - r0];
                    acc += e;
                    if (cls == 1 && e > be) {
                        be = e;
                        const TriInfo& I = info[tid];
                        const int loc = k - off[tid];
                        const int ry = loc / I.bw;
                        bp = (I.y0 + ry) * it.W + I.x0 + loc - ry * I.bw;
                    }
                }
            }
            __syncthreads();
        }
        if (with_f && tid < cnt) {
            if (it.tri_err) it.tri_err[t0 + tid] = acc;
            if (it.best) it.best[t0 + tid] = bp;
        }
    }
    if (!it.f || !it.sse) return;
    const double tot = block_sum<RB>(tid < cnt ? acc : 0.0, red);
    double* P = part + (size_t)blockIdx.y * gridDim.x;
    if (tid == 0) P[blockIdx.x] = tot;
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        flag = (atomicAdd(&counters[blockIdx.y], 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (flag) {
        __threadfence();
        double s = 0.0;
        for (int k = tid; k < (int)gridDim.x; k += RB) s += __ldcg(&P[k]);
        s = block_sum<RB>(s, red);
        if (tid == 0) {
            *it.sse = s;
            counters[blockIdx.y] = 0;
        }
    }
}

// P^T r: per triangle, sum over its owned pixels of (l_a, l_b, l_c) r (vertex pixels:
// weight 1 on that vertex) -> tri_w[3t+k]; the vertex gather happens in tonal.cu.
__global__ void __launch_bounds__(RB, 3) k_adjoint_raster(const TriRec* __restrict__ tri, int64_t T, int W,
                                                          const double* __restrict__ r, double* __restrict__ tri_w) {
    __shared__ TriInfo info[RB];
    __shared__ int off[RB + 1];
    __shared__ int wsum[RB / 32];
    __shared__ double rs[RCAP];
    __shared__ unsigned char cs[RCAP];
    const int tid = threadIdx.x;
    const int64_t t0 = (int64_t)blockIdx.x * RB;
    if (t0 >= T) return;
    const int cnt = load_tris(tri, T, t0, info, off, wsum);
    const int total = off[cnt];
    double sa = 0.0, sb = 0.0, sc = 0.0;
    int j = 0;
    for (int r0 = 0; r0 < total; r0 += RCAP) {
        const int rend = min(total, r0 + RCAP);
        for (int k = r0 + tid; k < rend; k += RB) {
            while (off[j + 1] <= k) ++j;
            const TriInfo& I = info[j];
            const int loc = k - off[j];
            const int ry = loc / I.bw;
            const int py = I.y0 + ry, px = I.x0 + loc - ry * I.bw;
            int w0, w1, w2, kv = 0;
            const int cls = classify(I, px, py, w0, w1, w2, kv);
            cs[k - r0] = (unsigned char)(cls == 2 ? 2 + kv : cls);
            if (cls) rs[k - r0] = r[(int64_t)py * W + px];
        }
        __syncthreads();
        if (tid < cnt) {
            const TriInfo& I = info[tid];
            const double D = (double)I.D;
            const int lo = max(off[tid], r0), hi = min(off[tid + 1], rend);
            for (int k = lo; k < hi; ++k) {
                const int c = cs[k - r0];
                if (!c) continue;
                const double rv = rs[k - r0];
                if (c >= 2) {
                    if (c == 2) sa += rv;
                    else if (c == 3) sb += rv;
                    else sc += rv;
                    continue;
                }
                const int loc = k - off[tid];
                const int ry = loc / I.bw;
                const int py = I.y0 + ry, px = I.x0 + loc - ry * I.bw;
                const int w0 = orient_xy(I.bx, I.by, I.cx, I.cy, px, py);
                const int w1 = orient_xy(I.cx, I.cy, I.ax, I.ay, px, py);
                const int w2 = orient_xy(I.ax, I.ay, I.bx, I.by, px, py);
                sa += (w0 / D) * rv;
                sb += (w1 / D) * rv;
                sc += (w2 / D) * rv;
            }
        }
        __syncthreads();
    }
    if (tid < cnt) {
        tri_w[3 * (t0 + tid)] = sa;
        tri_w[3 * (t0 + tid) + 1] = sb;
        tri_w[3 * (t0 + tid) + 2] = sc;
    }
}

}  // namespace

femi_status launch_raster(int B, femi_system_s* const* S, const double* const* u_vert, const double* const* f,
                          double* const* u_px, double* const* e_px, double* const* tri_err, int32_t* const* best,
                          double* const* sse, cudaStream_t st) {
    if (B <= 0) return FEMI_OK;
    std::vector<RasterItem> items(B);
    int64_t Tmax = 0;
    for (int b = 0; b < B; ++b) {
        RasterItem& r = items[b];
        r.tri = S[b]->tri;
        r.u_vert = u_vert[b];
        r.f = f ? f[b] : nullptr;
        r.u_px = u_px ? u_px[b] : nullptr;
        r.e_px = e_px ? e_px[b] : nullptr;
        r.tri_err = tri_err ? tri_err[b] : nullptr;
        r.best = best ? best[b] : nullptr;
        r.sse = sse ? sse[b] : nullptr;
        r.T = S[b]->T;
        r.W = S[b]->W;
        Tmax = std::max(Tmax, r.T);
    }
    const int gx = (int)std::max<int64_t>(1, (Tmax + RB - 1) / RB);
    const size_t bytes_items = sizeof(RasterItem) * B;
    const size_t bytes_part = sizeof(double) * (size_t)gx * B;
    const size_t bytes_cnt = sizeof(uint32_t) * B;
    void* base = nullptr;
    FEMI_CUDA(cudaMallocAsync(&base, bytes_items + bytes_part + bytes_cnt + 64, st));
    char* cur = (char*)base;
    RasterItem* d_items = (RasterItem*)cur;
    double* d_part = (double*)(cur + ((bytes_items + 15) & ~(size_t)15));
    uint32_t* d_cnt = (uint32_t*)((char*)d_part + bytes_part);
    FEMI_CUDA(cudaMemcpyAsync(d_items, items.data(), bytes_items, cudaMemcpyHostToDevice, st));
    FEMI_CUDA(cudaMemsetAsync(d_cnt, 0, bytes_cnt, st));
    dim3 grid(gx, B);
    k_raster_error<<<grid, RB, 0, st>>>(d_items, d_part, d_cnt);
    count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    FEMI_CUDA(cudaFreeAsync(base, st));
    return FEMI_OK;
}

femi_status launch_adjoint_raster(femi_system_s* S, const double* r, double* tri_w, cudaStream_t st) {
    if (S->T == 0) return FEMI_OK;
    const int gx = (int)((S->T + RB - 1) / RB);
    k_adjoint_raster<<<gx, RB, 0, st>>>(S->tri, S->T, S->W, r, tri_w);
    count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    return FEMI_OK;
}

}  // namespace femi
