// raster.cu -- S3+S4: rasterise the P1 solution and reduce the squared error
// (PAPER.md:L239-241 interpolation; L262-265 "e_i = (u_i - f_i)^2", "total L2 error in
// each triangle").
//
// Triangle-parallel, one warp per triangle (grid-stride over the canonical triangle
// order, which is spatially coherent, so neighbouring warps touch neighbouring image
// rows and the f / u / e lines are shared through L2). Lanes sweep the triangle's
// bounding box; a pixel is processed by the triangle that owns it (reading A7: lowest
// index among the closed triangles containing it), decided locally from the edge
// functions and the precomputed ownership flags -- no owner map, no atomics:
//   interior           -> owned
//   on the edge opp. k -> owned iff flag bit k   (this triangle has the lower index)
//   at vertex k        -> owned iff flag bit 3+k (this is the vertex's lowest triangle)
// Per-triangle error sums and arg-max (ties: lowest pix) are warp reductions in a fixed
// order, SSE is a per-CTA partial summed in fixed order by the last CTA: deterministic.
#include "device.cuh"

namespace femi {
namespace {

constexpr int RT = 256;  // threads per CTA (8 warps)

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

__device__ __forceinline__ int orient_i(int ax, int ay, int bx, int by, int px, int py) {
    return (bx - ax) * (py - ay) - (by - ay) * (px - ax);
}

__global__ void __launch_bounds__(RT) k_raster_error(const RasterItem* __restrict__ items, double* __restrict__ part,
                                                     uint32_t* __restrict__ counters) {
    __shared__ double red[RT / 32];
    __shared__ int flag;
    const RasterItem it = items[blockIdx.y];
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * RT + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * RT) >> 5;
    double sse_loc = 0.0;
    for (int64_t t = warp; t < it.T; t += nwarps) {
        const TriRec R = it.tri[t];
        const int ax = R.x[0], ay = R.y[0], bx = R.x[1], by = R.y[1], cx = R.x[2], cy = R.y[2];
        const double ua = it.u_vert[R.v[0]], ub = it.u_vert[R.v[1]], uc = it.u_vert[R.v[2]];
        const int x0 = min(ax, min(bx, cx)), x1 = max(ax, max(bx, cx));
        const int y0 = min(ay, min(by, cy)), y1 = max(ay, max(by, cy));
        const int bw = x1 - x0 + 1;
        const int nbox = bw * (y1 - y0 + 1);
        const double D = (double)orient_i(ax, ay, bx, by, cx, cy);
        const double dba = ub - ua, dca = uc - ua;
        double acc = 0.0;
        double be = -1.0;
        int bp = 0x7fffffff;
        for (int k = lane; k < nbox; k += 32) {
            const int py = y0 + k / bw, px = x0 + k % bw;
            const int w0 = orient_i(bx, by, cx, cy, px, py);
            const int w1 = orient_i(cx, cy, ax, ay, px, py);
            const int w2 = orient_i(ax, ay, bx, by, px, py);
            if ((w0 | w1 | w2) < 0) continue;  // outside the closed triangle
            const int z = (w0 == 0) + (w1 == 0) + (w2 == 0);
            double u;
            bool vertex = false;
            if (z == 0) {
                u = ua + (w1 / D) * dba + (w2 / D) * dca;
            } else if (z == 1) {
                const int ke = (w0 == 0) ? 0 : ((w1 == 0) ? 1 : 2);
                if (!(R.flags & (1u << ke))) continue;
                u = ua + (w1 / D) * dba + (w2 / D) * dca;
            } else {
                const int kv = (w0 != 0) ? 0 : ((w1 != 0) ? 1 : 2);
                if (!(R.flags & (8u << kv))) continue;
                u = (kv == 0) ? ua : ((kv == 1) ? ub : uc);
                vertex = true;
            }
            const int pix = py * it.W + px;
            if (it.u_px) it.u_px[pix] = u;
            if (it.f) {
                const double d = u - it.f[pix];
                const double e = d * d;
                if (it.e_px) it.e_px[pix] = e;
                acc += e;
                if (!vertex && (e > be || (e == be && pix < bp))) {
                    be = e;
                    bp = pix;
                }
            }
        }
        if (it.f) {
            acc = warp_sum(acc);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double oe = __shfl_xor_sync(0xffffffffu, be, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                if (oe > be || (oe == be && op < bp)) {
                    be = oe;
                    bp = op;
                }
            }
            if (lane == 0) {
                if (it.tri_err) it.tri_err[t] = acc;
                if (it.best) it.best[t] = (be >= 0.0) ? bp : -1;
            }
            sse_loc += acc;  // identical in every lane; lane 0's copy is used below
        }
    }
    if (!it.f || !it.sse) return;
    const double v = (lane == 0) ? sse_loc : 0.0;
    const double tot = block_sum<RT>(v, red);
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
    // grid: enough warps for one triangle per warp up to ~8 resident CTAs per SM per item
    int64_t want = (Tmax + (RT / 32) - 1) / (RT / 32);
    int gx = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)148 * 8 * 4 / std::max(1, B) + 1));
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
    k_raster_error<<<grid, RT, 0, st>>>(d_items, d_part, d_cnt); count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    FEMI_CUDA(cudaFreeAsync(base, st));
    return FEMI_OK;
}

}  // namespace femi
