// raster_common.cuh -- warp-cooperative triangle expansion shared by the forward raster
// (S3+S4) and the adjoint raster (P^T r, tonal S6). Internal.
//
// A warp takes 32 consecutive canonical triangles (one per lane), scans their bounding-box
// sizes with shuffles and walks the flat list of (triangle, bbox pixel) slots 32 at a time:
// lane l handles slot base+l, so lanes touch consecutive pixels of a bbox row (coalesced
// f / u / e traffic) and the work per lane is balanced whatever the triangle sizes. The
// slot's triangle is found by a 5-step shuffle binary search over the exclusive offsets.
// Per-triangle reductions are segmented warp scans (triangles are contiguous runs of
// lanes); the last lane of each run adds the run's result into the triangle's shared
// accumulator -- one writer per triangle per window, windows in pixel order: deterministic.
// No block barrier anywhere.
#pragma once
#include "device.cuh"

namespace femi {

constexpr int RT = 256;           // threads per CTA (8 warps)
constexpr int RWARPS = RT / 32;

struct WTri {
    int x0, y0, bw, D;
    int ax, ay, bx, by, cx, cy;
    uint32_t flags;
    int pad;
};

__device__ __forceinline__ int orient_xy(int ax, int ay, int bx, int by, int px, int py) {
    return (bx - ax) * (py - ay) - (by - ay) * (px - ax);
}

// Classify pixel (px,py) for triangle T: 0 not owned, 1 owned (interior or edge), 2 owned
// vertex pixel (kv = vertex). Ownership = reading A7 via the flags.
__device__ __forceinline__ int classify(const WTri& T, int px, int py, int& w0, int& w1, int& w2, int& kv) {
    w0 = orient_xy(T.bx, T.by, T.cx, T.cy, px, py);
    w1 = orient_xy(T.cx, T.cy, T.ax, T.ay, px, py);
    w2 = orient_xy(T.ax, T.ay, T.bx, T.by, px, py);
    if ((w0 | w1 | w2) < 0) return 0;
    const int z = (w0 == 0) + (w1 == 0) + (w2 == 0);
    if (z == 0) return 1;
    if (z == 1) {
        const int ke = (w0 == 0) ? 0 : ((w1 == 0) ? 1 : 2);
        return (T.flags & (1u << ke)) ? 1 : 0;
    }
    kv = (w0 != 0) ? 0 : ((w1 != 0) ? 1 : 2);
    return (T.flags & (8u << kv)) ? 2 : 0;
}

// Lane loads triangle t0+lane (if < T) into ws[lane]; returns its bbox size (0 if none)
// and sets excl = exclusive offset, total = sum over the warp.
__device__ __forceinline__ int warp_load_tris(const TriRec* __restrict__ tri, int64_t T, int64_t t0, WTri* ws,
                                              int& excl, int& total, TriRec& R) {
    const int lane = threadIdx.x & 31;
    int nbox = 0;
    if (t0 + lane < T) {
        R = tri[t0 + lane];
        WTri I;
        I.ax = R.x[0];
        I.ay = R.y[0];
        I.bx = R.x[1];
        I.by = R.y[1];
        I.cx = R.x[2];
        I.cy = R.y[2];
        I.x0 = min(I.ax, min(I.bx, I.cx));
        I.y0 = min(I.ay, min(I.by, I.cy));
        I.bw = max(I.ax, max(I.bx, I.cx)) - I.x0 + 1;
        nbox = I.bw * (max(I.ay, max(I.by, I.cy)) - I.y0 + 1);
        I.flags = R.flags;
        I.D = orient_xy(I.ax, I.ay, I.bx, I.by, I.cx, I.cy);
        I.pad = 0;
        ws[lane] = I;
    }
    int incl = nbox;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    excl = incl - nbox;
    total = __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
    return nbox;
}

// triangle (lane index) owning slot k: largest j with excl_j <= k; 32 if k >= total
__device__ __forceinline__ int warp_find(int excl, int k, int total) {
    int j = 0;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const int e = __shfl_sync(0xffffffffu, excl, j + s < 32 ? j + s : 31);
        if (j + s < 32 && e <= k) j += s;
    }
    return k < total ? j : 32;
}

}  // namespace femi
