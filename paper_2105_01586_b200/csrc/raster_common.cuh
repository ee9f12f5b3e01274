// raster_common.cuh -- load-balanced triangle expansion shared by the forward raster
// (S3+S4) and the adjoint raster (P^T r, tonal S6). Internal.
//
// A CTA takes RB consecutive canonical triangles, prefix-sums their bounding-box sizes in
// shared memory and walks the flat list of (triangle, bbox pixel) slots with all threads:
// every thread handles slots tid, tid+RB, ... so consecutive lanes touch consecutive
// pixels of a bbox row (coalesced f / u / e traffic) and the work per thread is balanced
// whatever the triangle sizes. Slots are processed in rounds of RCAP so the per-slot
// scratch stays in shared memory; per-triangle reductions then run one thread per
// triangle over its slots in pixel order (deterministic).
#pragma once
#include "device.cuh"

namespace femi {

constexpr int RB = 256;     // triangles per CTA == threads per CTA
constexpr int RCAP = 2048;  // slots per round (static shared memory <= 48 KB)

struct TriInfo {
    int x0, y0, bw, nbox;
    int ax, ay, bx, by, cx, cy;
    uint32_t flags;
    int D;
};

__device__ __forceinline__ int orient_xy(int ax, int ay, int bx, int by, int px, int py) {
    return (bx - ax) * (py - ay) - (by - ay) * (px - ax);
}

// Classify pixel (px,py) for triangle T: returns 0 (not owned), 1 (owned, interior or
// edge), 2 (owned vertex pixel); w[] are the three edge functions (w0 = orient(b,c,p) ...)
// and kv the vertex index for class 2. Ownership = reading A7 via the flags.
__device__ __forceinline__ int classify(const TriInfo& T, int px, int py, int& w0, int& w1, int& w2, int& kv) {
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

// Load the CTA's triangles into shared memory and scan the bbox sizes.
// off[j] = first slot of triangle j (off[cnt] = total). Returns the triangle count.
__device__ __forceinline__ int load_tris(const TriRec* __restrict__ tri, int64_t T, int64_t t0, TriInfo* info,
                                         int* off, int* wsum) {
    const int tid = threadIdx.x;
    const int cnt = (int)min((int64_t)RB, T - t0);
    int nbox = 0;
    if (tid < cnt) {
        const TriRec R = tri[t0 + tid];
        TriInfo I;
        I.ax = R.x[0];
        I.ay = R.y[0];
        I.bx = R.x[1];
        I.by = R.y[1];
        I.cx = R.x[2];
        I.cy = R.y[2];
        I.x0 = min(I.ax, min(I.bx, I.cx));
        I.y0 = min(I.ay, min(I.by, I.cy));
        I.bw = max(I.ax, max(I.bx, I.cx)) - I.x0 + 1;
        const int bh = max(I.ay, max(I.by, I.cy)) - I.y0 + 1;
        I.nbox = I.bw * bh;
        I.flags = R.flags;
        I.D = orient_xy(I.ax, I.ay, I.bx, I.by, I.cx, I.cy);
        info[tid] = I;
        nbox = I.nbox;
    }
    // block exclusive scan of nbox
    const int lane = tid & 31, wid = tid >> 5;
    int v = nbox;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) wsum[wid] = v;
    __syncthreads();
    if (wid == 0) {
        int s = (lane < RB / 32) ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < RB / 32) wsum[lane] = s;  // inclusive warp totals
    }
    __syncthreads();
    const int excl = v - nbox + (wid > 0 ? wsum[wid - 1] : 0);
    off[tid] = excl;
    if (tid == RB - 1) off[RB] = excl + nbox;
    __syncthreads();
    if (cnt < RB && tid == 0) off[cnt] = off[RB];  // tail CTA: close the list after the last triangle
    __syncthreads();
    return cnt;
}

}  // namespace femi
