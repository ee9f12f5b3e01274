// raster.cu -- S3+S4: rasterise the P1 solution and reduce the squared error
// (PAPER.md:L239-241 interpolation; L262-265 "e_i = (u_i - f_i)^2", "total L2 error in
// each triangle"), and the adjoint raster P^T r used by tonal optimisation (S6).
//
// Triangle-parallel with warp-cooperative expansion (raster_common.cuh): a pixel is
// processed by the triangle that owns it (reading A7: lowest index among the closed
// triangles containing it), decided locally from the edge functions and precomputed
// ownership flags -- no owner map, no atomics. A vertex pixel takes its vertex value
// exactly; otherwise u = u_a + l_b (u_b - u_a) + l_c (u_c - u_a), l = exact integer edge
// function / 2*area (S3). Per-triangle error sums and arg-max (ties: lowest pix) are
// segmented warp scans in pixel order; SSE is a per-CTA partial summed in fixed order by
// the last CTA: deterministic.
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

__global__ void __launch_bounds__(RT) k_raster_error(const RasterItem* __restrict__ items, double* __restrict__ part,
                                                     uint32_t* __restrict__ counters) {
    __shared__ WTri tris[RWARPS][32];
    __shared__ double tuv[RWARPS][32][3];
    __shared__ double acc_s[RWARPS][32];
    __shared__ double be_s[RWARPS][32];
    __shared__ int bp_s[RWARPS][32];
    __shared__ double red[RWARPS];
    __shared__ int flag;
    const RasterItem it = items[blockIdx.y];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ngroups = (it.T + 31) / 32;
    const int64_t gwarp = (int64_t)blockIdx.x * RWARPS + wid, nwarps = (int64_t)gridDim.x * RWARPS;
    const bool with_f = it.f != nullptr;
    WTri* ws = tris[wid];
    double sse_loc = 0.0;
    for (int64_t g = gwarp; g < ngroups; g += nwarps) {
        const int64_t t0 = g * 32;
        int excl, total;
        TriRec R;
        const int nbox = warp_load_tris(it.tri, it.T, t0, ws, excl, total, R);
        if (nbox) {
            tuv[wid][lane][0] = it.u_vert[R.v[0]];
            tuv[wid][lane][1] = it.u_vert[R.v[1]];
            tuv[wid][lane][2] = it.u_vert[R.v[2]];
        }
        acc_s[wid][lane] = 0.0;
        be_s[wid][lane] = -1.0;
        bp_s[wid][lane] = -1;
        __syncwarp();
        for (int base = 0; base < total; base += 32) {
            const int k = base + lane;
            const int j = warp_find(excl, k, total);
            const int exj = __shfl_sync(0xffffffffu, excl, j & 31);
            double val = 0.0, ce = -1.0;
            int cp = 0x7fffffff;
            if (j < 32) {
                const WTri& I = ws[j];
                const int loc = k - exj;
                const int ry = loc / I.bw;
                const int py = I.y0 + ry, px = I.x0 + loc - ry * I.bw;
                int w0, w1, w2, kv = 0;
                const int cls = classify(I, px, py, w0, w1, w2, kv);
                if (cls) {
                    double u;
                    if (cls == 2) {
                        u = tuv[wid][j][kv];
                    } else {
                        const double D = (double)I.D, ua = tuv[wid][j][0];
                        u = ua + (w1 / D) * (tuv[wid][j][1] - ua) + (w2 / D) * (tuv[wid][j][2] - ua);
                    }
                    const int64_t pix = (int64_t)py * it.W + px;
                    if (it.u_px) it.u_px[pix] = u;
                    if (with_f) {
                        const double d = u - it.f[pix];
                        const double e = d * d;
                        if (it.e_px) it.e_px[pix] = e;
                        val = e;
                        if (cls == 1) {
                            ce = e;
                            cp = (int)pix;
                        }
                    }
                }
            }
            if (!with_f) continue;
            // segmented inclusive scan over runs of equal j: sum and (e desc, pix asc) arg-max
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double vo = __shfl_up_sync(0xffffffffu, val, o);
                const double eo = __shfl_up_sync(0xffffffffu, ce, o);
                const int po = __shfl_up_sync(0xffffffffu, cp, o);
                const int jo = __shfl_up_sync(0xffffffffu, j, o);
                if (lane >= o && jo == j) {
                    val += vo;
                    if (eo > ce || (eo == ce && po < cp)) {
                        ce = eo;
                        cp = po;
                    }
                }
            }
            const int jn = __shfl_down_sync(0xffffffffu, j, 1);
            if (j < 32 && (lane == 31 || jn != j)) {
                acc_s[wid][j] += val;
                if (ce > be_s[wid][j]) {  // earlier windows hold lower pixels: strict > keeps ties
                    be_s[wid][j] = ce;
                    bp_s[wid][j] = cp;
                }
            }
        }
        __syncwarp();
        if (with_f && nbox) {
            const double a = acc_s[wid][lane];
            if (it.tri_err) it.tri_err[t0 + lane] = a;
            if (it.best) it.best[t0 + lane] = be_s[wid][lane] >= 0.0 ? bp_s[wid][lane] : -1;
            sse_loc += a;
        }
        __syncwarp();
    }
    if (!with_f || !it.sse) return;
    // SSE: fixed-order sums (lanes, warps, CTAs)
    const double tot = block_sum<RT>(sse_loc, red);
    double* P = part + (size_t)blockIdx.y * gridDim.x;
    if (threadIdx.x == 0) P[blockIdx.x] = tot;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        flag = (atomicAdd(&counters[blockIdx.y], 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (flag) {
        __threadfence();
        double s = 0.0;
        for (int k = threadIdx.x; k < (int)gridDim.x; k += RT) s += __ldcg(&P[k]);
        s = block_sum<RT>(s, red);
        if (threadIdx.x == 0) {
            *it.sse = s;
            counters[blockIdx.y] = 0;
        }
    }
}

// P^T r: per triangle, sum over its owned pixels of (l_a, l_b, l_c) r (vertex pixels:
// weight 1 on that vertex) -> tri_w[3t+k]; the vertex gather happens in tonal.cu.
__global__ void __launch_bounds__(RT) k_adjoint_raster(const TriRec* __restrict__ tri, int64_t T, int W,
                                                       const double* __restrict__ r, double* __restrict__ tri_w) {
    __shared__ WTri tris[RWARPS][32];
    __shared__ double acc_s[RWARPS][32][3];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ngroups = (T + 31) / 32;
    const int64_t gwarp = (int64_t)blockIdx.x * RWARPS + wid, nwarps = (int64_t)gridDim.x * RWARPS;
    WTri* ws = tris[wid];
    for (int64_t g = gwarp; g < ngroups; g += nwarps) {
        const int64_t t0 = g * 32;
        int excl, total;
        TriRec R;
        const int nbox = warp_load_tris(tri, T, t0, ws, excl, total, R);
        acc_s[wid][lane][0] = 0.0;
        acc_s[wid][lane][1] = 0.0;
        acc_s[wid][lane][2] = 0.0;
        __syncwarp();
        for (int base = 0; base < total; base += 32) {
            const int k = base + lane;
            const int j = warp_find(excl, k, total);
            const int exj = __shfl_sync(0xffffffffu, excl, j & 31);
            double sa = 0.0, sb = 0.0, sc = 0.0;
            if (j < 32) {
                const WTri& I = ws[j];
                const int loc = k - exj;
                const int ry = loc / I.bw;
                const int py = I.y0 + ry, px = I.x0 + loc - ry * I.bw;
                int w0, w1, w2, kv = 0;
                const int cls = classify(I, px, py, w0, w1, w2, kv);
                if (cls) {
                    const double rv = r[(int64_t)py * W + px];
                    if (cls == 2) {
                        if (kv == 0) sa = rv;
                        else if (kv == 1) sb = rv;
                        else sc = rv;
                    } else {
                        const double D = (double)I.D;
                        sa = (w0 / D) * rv;
                        sb = (w1 / D) * rv;
                        sc = (w2 / D) * rv;
                    }
                }
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double ao = __shfl_up_sync(0xffffffffu, sa, o);
                const double bo = __shfl_up_sync(0xffffffffu, sb, o);
                const double co = __shfl_up_sync(0xffffffffu, sc, o);
                const int jo = __shfl_up_sync(0xffffffffu, j, o);
                if (lane >= o && jo == j) {
                    sa += ao;
                    sb += bo;
                    sc += co;
                }
            }
            const int jn = __shfl_down_sync(0xffffffffu, j, 1);
            if (j < 32 && (lane == 31 || jn != j)) {
                acc_s[wid][j][0] += sa;
                acc_s[wid][j][1] += sb;
                acc_s[wid][j][2] += sc;
            }
        }
        __syncwarp();
        if (nbox) {
            tri_w[3 * (t0 + lane)] = acc_s[wid][lane][0];
            tri_w[3 * (t0 + lane) + 1] = acc_s[wid][lane][1];
            tri_w[3 * (t0 + lane) + 2] = acc_s[wid][lane][2];
        }
        __syncwarp();
    }
}

int raster_grid(int64_t T, int B) {
    const int64_t groups = (T + 31) / 32;
    const int64_t want = (groups + RWARPS - 1) / RWARPS;
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)148 * 8 / std::max(1, B) + 1));
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
    const int gx = raster_grid(Tmax, B);
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
    k_raster_error<<<grid, RT, 0, st>>>(d_items, d_part, d_cnt);
    count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    FEMI_CUDA(cudaFreeAsync(base, st));
    return FEMI_OK;
}

femi_status launch_adjoint_raster(femi_system_s* S, const double* r, double* tri_w, cudaStream_t st) {
    if (S->T == 0) return FEMI_OK;
    k_adjoint_raster<<<raster_grid(S->T, 1), RT, 0, st>>>(S->tri, S->T, S->W, r, tri_w);
    count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    return FEMI_OK;
}

}  // namespace femi
