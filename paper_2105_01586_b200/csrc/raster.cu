// raster.cu -- S3+S4: rasterise the P1 solution and reduce the squared error
// (PAPER.md:L239-241 interpolation; L262-265 "e_i = (u_i - f_i)^2", "total L2 error in
// each triangle"), and the adjoint raster P^T r used by tonal optimisation (S6).
//
// Pixel ownership (reading A7: lowest index among the closed triangles containing a
// pixel) depends only on the mesh, so it is resolved ONCE per mesh at assembly by a
// warp-cooperative triangle expansion (raster_common.cuh) into the triangle-major lists
//   tp_ptr[t]   = first entry of triangle t in tp_pix (CSR, ascending triangle)
//   tp_pix[q]   = cls << 30 | y << 14 | x for the triangle's owned pixels in ascending pix
//                 order (cls 0: interior/edge pixel, 1..3: the pixel of vertex v[cls-1];
//                 W, H <= 16384 so x and y take 14 bits each).
// Every solve then rasterises with ONE triangle-major kernel (k_raster_tri): values, errors,
// per-triangle error sum and arg-max over non-vertex pixels (ties: lowest pix) by segmented
// warp scans in pixel order, SSE = fixed-order sum of the triangle sums. Deterministic.
// The adjoint P^T r is the same traversal with barycentric weights.
#include <cstdlib>

#include "raster_common.cuh"

namespace femi {
namespace {


// ---------------------------------------------------------------- setup (per mesh)

// MODE 0: owned-pixel count per triangle. MODE 1: triangle-major pixel list.
template <int MODE>
__global__ void __launch_bounds__(RT) k_build_owner(const TriRec* __restrict__ tri, int64_t T, int W,
                                                    int32_t* __restrict__ cnt,
                                                    const int32_t* __restrict__ tp_ptr,
                                                    uint32_t* __restrict__ tp_pix) {
    __shared__ WTri tris[RWARPS][32];
    __shared__ int run_s[RWARPS][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ngroups = (T + 31) / 32;
    const int64_t gwarp = (int64_t)blockIdx.x * RWARPS + wid, nwarps = (int64_t)gridDim.x * RWARPS;
    WTri* ws = tris[wid];
    for (int64_t g = gwarp; g < ngroups; g += nwarps) {
        const int64_t t0 = g * 32;
        int excl, total;
        TriRec R;
        const int nbox = warp_load_tris(tri, T, t0, ws, excl, total, R);
        run_s[wid][lane] = 0;
        __syncwarp();
        for (int base = 0; base < total; base += 32) {
            const int k = base + lane;
            const int j = warp_find(excl, k, total);
            const int exj = __shfl_sync(0xffffffffu, excl, j & 31);
            int own = 0, cls = 0, px = 0, py = 0;
            if (j < 32) {
                const WTri& I = ws[j];
                const int loc = k - exj;
                const int ry = loc / I.bw;
                py = I.y0 + ry;
                px = I.x0 + loc - ry * I.bw;
                int w0, w1, w2, kv = 0;
                const int c = classify(I, px, py, w0, w1, w2, kv);
                if (c) {
                    own = 1;
                    cls = c == 2 ? kv + 1 : 0;
                }
            }
            // rank of this owned pixel inside its triangle (slots are in pixel order)
            int rk = own;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int ro = __shfl_up_sync(0xffffffffu, rk, o);
                const int jo = __shfl_up_sync(0xffffffffu, j, o);
                if (lane >= o && jo == j) rk += ro;
            }
            if (MODE == 1 && own) {
                const int q = tp_ptr[t0 + j] + run_s[wid][j] + rk - 1;
                tp_pix[q] = ((uint32_t)cls << 30) | ((uint32_t)py << 14) | (uint32_t)px;
            }
            __syncwarp();
            const int jn = __shfl_down_sync(0xffffffffu, j, 1);
            if (j < 32 && (lane == 31 || jn != j)) run_s[wid][j] += rk;
            __syncwarp();
        }
        if (MODE == 0 && nbox) cnt[t0 + lane] = run_s[wid][lane];
        __syncwarp();
    }
}

// exclusive scan of cnt[0..n) into ptr[0..n] (ptr[n] = total): block sums, then offsets
constexpr int SCB = 1024;
__global__ void k_scan_blocks(int64_t n, const int32_t* __restrict__ cnt, int32_t* __restrict__ bsum) {
    __shared__ int sh[SCB / 32];
    const int64_t i = (int64_t)blockIdx.x * SCB + threadIdx.x;
    int v = i < n ? cnt[i] : 0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < SCB / 32; ++w) s += sh[w];
        bsum[blockIdx.x] = s;
    }
}
__global__ void k_scan_bsum(int nb, int32_t* __restrict__ bsum) {  // one thread; nb ~ T/1024
    if (threadIdx.x || blockIdx.x) return;
    int run = 0;
    for (int b = 0; b < nb; ++b) {
        const int c = bsum[b];
        bsum[b] = run;
        run += c;
    }
    bsum[nb] = run;
}
__global__ void k_scan_apply(int64_t n, const int32_t* __restrict__ cnt, const int32_t* __restrict__ bsum,
                             int32_t* __restrict__ ptr) {
    __shared__ int sh[SCB / 32];
    const int64_t i = (int64_t)blockIdx.x * SCB + threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int v = i < n ? cnt[i] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) sh[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int s = lane < SCB / 32 ? sh[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < SCB / 32) sh[lane] = s;
    }
    __syncthreads();
    const int off = bsum[blockIdx.x] + (wid ? sh[wid - 1] : 0) + incl - v;
    if (i < n) ptr[i] = off;
    if (i == n - 1) ptr[n] = off + v;
}

// ---------------------------------------------------------------- per solve

constexpr int kMaxCh = 4;  // colour channels of one raster item (shared mesh)

struct RasterItem {
    const TriRec* tri;
    const int32_t* tp_ptr;
    const uint32_t* tp_pix;
    const double* u_vert[kMaxCh];  // per channel
    const double* f[kMaxCh];       // per channel; f[0] == nullptr: no error map
    double* u_px[kMaxCh];          // per channel, nullable
    double* e_px;                  // e = sum over channels of (u_c - f_c)^2
    double* tri_err;
    int32_t* best;
    double* sse;
    int64_t T, N;
    int32_t W;
    int32_t pad;
};

// Warp-cooperative traversal of the triangle-major list: lane l of a warp owns triangle
// t0+l; list entries ptr[t0] .. ptr[t0+32] are walked 32 at a time (coalesced), each entry
// tagged with its triangle by a shuffle binary search over the per-triangle offsets.
struct ListWalk {
    int excl, total, ptr0;
};
__device__ __forceinline__ ListWalk list_begin(const int32_t* __restrict__ tp_ptr, int64_t T, int64_t t0, int& cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t t = t0 + lane;
    const int a = t < T ? tp_ptr[t] : 0;
    const int b = t < T ? tp_ptr[t + 1] : 0;
    cnt = b - a;
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    ListWalk lw;
    lw.excl = incl - cnt;
    lw.total = __shfl_sync(0xffffffffu, incl, 31);
    lw.ptr0 = __shfl_sync(0xffffffffu, a, 0);
    return lw;
}

// One triangle as the fused raster keeps it in shared memory (one slot per lane): the two
// exact integer edge functions as planes w = A px + B py + C (S3: w_b = orient(c,a,p),
// w_c = orient(a,b,p)), D = orient(a,b,c) and its correctly rounded reciprocal, u_a and the
// differences u_b - u_a, u_c - u_a.
// 16-byte aligned (size padded to a multiple of 16): the per-entry reads of a slot become
// 128-bit shared loads (half the LDS instructions and wavefronts of 64-bit ones; the 96-byte
// stride keeps consecutive slots on disjoint banks)
template <int NC>
struct __align__(16) RTri {
    int A1, B1, C1, A2, B2, C2, pad0, pad1;
    double D, rD;
    double db[NC], dc[NC], u[NC][3];
};

__device__ __forceinline__ int tp_x(uint32_t v) { return (int)(v & 0x3fffu); }
__device__ __forceinline__ int tp_y(uint32_t v) { return (int)((v >> 14) & 0x3fffu); }

// Correctly rounded w / D for an exact integer w (|w| < 2^53) given rD = RN(1/D): q = RN(w rD)
// is within 1 ulp of w/D, the remainder w - qD is exact under fma, and RN(q + r rD) is RN(w/D)
// (Markstein's theorem) -- the IEEE quotient of __ddiv_rn at three fp64 operations.
__device__ __forceinline__ double div_rn(double w, double D, double rD) {
    const double q = __dmul_rn(w, rD);
    const double r = __fma_rn(-q, D, w);
    return __fma_rn(r, rD, q);
}

constexpr int RCH = 128;  // list entries per warp chunk (4 x 32 lanes)

// S3+S4 in ONE triangle-major pass. A warp takes 32 consecutive triangles (smem, one slot per
// lane) and walks their owned pixels (tp_pix: ascending pix per triangle) in chunks of RCH:
//  phase 1, lane per entry (coalesced list reads, f gathered and u, e written along row
//   segments): u = the vertex value (vertex pixel) or (u_a + l_b (u_b - u_a)) + l_c (u_c - u_a)
//   with l = w / D in IEEE fp64 (S3's barycentric form, one rounding per operation, no
//   contraction), e = (u - f)^2; e is staged in shared memory;
//  phase 2, lane per triangle: the lane walks its triangle's entries of the chunk in pixel
//   order: tri_err += e, best = first strict maximum over non-vertex pixels (ties: lowest
//   pix) -- the oracle's sequential order, so tri_err and best are bit-identical to it.
// SSE = sum of per-group partials in group order (k_sse). Deterministic, no atomics on values.
template <int MINB, int CH, int NC>
__global__ void __launch_bounds__(RT, MINB) k_raster_tri(const RasterItem* __restrict__ items, double* __restrict__ gpart,
                                                   uint32_t* __restrict__ next, int64_t gstride) {
    extern __shared__ __align__(16) unsigned char rsm[];  // RTri<NC> [RWARPS][32] (dynamic: colour > 48 KB)
    __shared__ double e_s[RWARPS][CH];
    __shared__ int p_s[RWARPS][CH];  // pix, or -1 for a vertex pixel (not a candidate)
    const RasterItem& it = items[blockIdx.y];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t T = it.T;
    const int W = it.W;
    const bool hasf = it.f[0] != nullptr;
    double* __restrict__ e_px = it.e_px;
    const uint32_t* __restrict__ tp_pix = it.tp_pix;
    const int64_t ngroups = (T + 31) / 32;
    RTri<NC>* ws = (RTri<NC>*)rsm + 32 * wid;
    double* __restrict__ gp = gpart + gstride * blockIdx.y;
    double* es = e_s[wid];
    int* ps = p_s[wid];
    // groups of 32 triangles are handed out in canonical order by an atomic counter: the warps
    // in flight cover one narrow band of rows, so the f/u/e sectors they share are completed
    // in L2 before eviction (no partial-sector write-backs)
    for (;;) {
        int64_t g = 0;
        if (lane == 0) g = (int64_t)atomicAdd(next + blockIdx.y, 1u);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= ngroups) break;
        const int64_t t0 = g * 32;
        int cnt;
        const ListWalk lw = list_begin(it.tp_ptr, T, t0, cnt);
        if (t0 + lane < T) {
            const TriRec R = it.tri[t0 + lane];
            const int ax = R.x[0], ay = R.y[0], bx = R.x[1], by = R.y[1], cx = R.x[2], cy = R.y[2];
            RTri<NC> I;
            // w_b = orient(c,a,p) = (ax-cx)(py-cy) - (ay-cy)(px-cx)
            I.A1 = cy - ay;
            I.B1 = ax - cx;
            I.C1 = (ay - cy) * cx - (ax - cx) * cy;
            // w_c = orient(a,b,p) = (bx-ax)(py-ay) - (by-ay)(px-ax)
            I.A2 = ay - by;
            I.B2 = bx - ax;
            I.C2 = (by - ay) * ax - (bx - ax) * ay;
            I.D = (double)orient_xy(ax, ay, bx, by, cx, cy);
            I.rD = __drcp_rn(I.D);
#pragma unroll
            for (int ch = 0; ch < NC; ++ch) {
                I.u[ch][0] = it.u_vert[ch][R.v[0]];
                I.u[ch][1] = it.u_vert[ch][R.v[1]];
                I.u[ch][2] = it.u_vert[ch][R.v[2]];
                I.db[ch] = __dsub_rn(I.u[ch][1], I.u[ch][0]);
                I.dc[ch] = __dsub_rn(I.u[ch][2], I.u[ch][0]);
            }
            ws[lane] = I;
        }
        __syncwarp();
        double acc = 0.0, be = -1.0;
        int bp = -1;
        const int my0 = lw.excl, my1 = lw.excl + cnt;
        // list entries of the next 128-entry block are loaded one block ahead (their latency
        // overlaps the current block's f gathers and arithmetic)
        uint32_t vn[RCH / 32];
#pragma unroll
        for (int h = 0; h < RCH / 32; ++h) {
            const int k = 32 * h + lane;
            vn[h] = k < lw.total ? tp_pix[lw.ptr0 + k] : 0u;
        }
        for (int c0 = 0; c0 < lw.total; c0 += CH) {
          // ---- phase 1: lane per entry, 128 entries at a time (loads in flight together)
          for (int c1 = c0; c1 < min(lw.total, c0 + CH); c1 += RCH) {
            uint32_t v[RCH / 32];
            int j[RCH / 32];
            double fv[RCH / 32][NC];
#pragma unroll
            for (int h = 0; h < RCH / 32; ++h) {
                const int k = c1 + 32 * h + lane;
                j[h] = warp_find(lw.excl, k, lw.total);
                v[h] = vn[h];
                const int kn = k + RCH;
                vn[h] = kn < lw.total ? tp_pix[lw.ptr0 + kn] : 0u;
            }
#pragma unroll
            for (int h = 0; h < RCH / 32; ++h)
#pragma unroll
                for (int ch = 0; ch < NC; ++ch)
                    fv[h][ch] = (hasf && j[h] < 32) ? it.f[ch][(int64_t)tp_y(v[h]) * W + tp_x(v[h])] : 0.0;
#pragma unroll
            for (int h = 0; h < RCH / 32; ++h) {
                if (j[h] >= 32) continue;
                const int px = tp_x(v[h]), py = tp_y(v[h]);
                const int pix = py * W + px;
                const uint32_t cls = v[h] >> 30;
                const RTri<NC>& I = ws[j[h]];
                double lb = 0.0, lc = 0.0;
                if (!cls) {
                    // S3 as the paper's barycentric form, IEEE round-to-nearest per operation
                    // and no contraction: l_b = w_b / D, l_c = w_c / D (shared by the channels),
                    // u = (u_a + l_b (u_b - u_a)) + l_c (u_c - u_a)
                    const int w1 = I.A1 * px + I.B1 * py + I.C1;
                    const int w2 = I.A2 * px + I.B2 * py + I.C2;
                    lb = div_rn((double)w1, I.D, I.rD);
                    lc = div_rn((double)w2, I.D, I.rD);
                }
                double e = 0.0;
#pragma unroll
                for (int ch = 0; ch < NC; ++ch) {
                    const double u = cls ? I.u[ch][cls - 1]
                                         : __dadd_rn(__dadd_rn(I.u[ch][0], __dmul_rn(lb, I.db[ch])),
                                                     __dmul_rn(lc, I.dc[ch]));
                    if (it.u_px[ch]) it.u_px[ch][pix] = u;
                    if (hasf) {
                        const double d = __dsub_rn(u, fv[h][ch]);
                        e = ch == 0 ? __dmul_rn(d, d) : __dadd_rn(e, __dmul_rn(d, d));  // channel sum in order
                    }
                }
                if (hasf) {
                    if (e_px) e_px[pix] = e;
                    // vertex pixels (not arg-max candidates) staged with the sign bit set (-e,
                    // -0.0 for e = 0); phase 2 adds |e| -- the same value
                    es[c1 - c0 + 32 * h + lane] = cls ? -e : e;
                    ps[c1 - c0 + 32 * h + lane] = pix;
                }
            }
          }
            __syncwarp();
            // ---- phase 2: lane per triangle, pixel order
            if (hasf) {
                const int lo = max(my0, c0), hi = min(my1, c0 + CH);
                int bk = -1;
                for (int k = lo; k < hi; ++k) {
                    const double es_k = es[k - c0];
                    const double e = fabs(es_k);
                    acc = __dadd_rn(acc, e);
                    if (__double_as_longlong(es_k) >= 0 && e > be) {
                        be = e;
                        bk = k;
                    }
                }
                if (bk >= 0) bp = ps[bk - c0];
            }
            __syncwarp();
        }
        if (t0 + lane < T && hasf) {
            if (it.tri_err) it.tri_err[t0 + lane] = acc;
            if (it.best) it.best[t0 + lane] = bp;
        }
        if (hasf) {  // group partial of the SSE (fixed tree order); summed in group order by k_sse
            const double gs = warp_sum(t0 + lane < T ? acc : 0.0);
            if (lane == 0) gp[g] = gs;
        }
    }
}

// SSE = sum of the per-group partials in group order (two fixed levels: deterministic)
__global__ void __launch_bounds__(RT) k_sse(const RasterItem* __restrict__ items, const double* __restrict__ gpart,
                                           int64_t gstride, double* __restrict__ part, uint32_t* __restrict__ counters) {
    __shared__ double red[RWARPS];
    __shared__ int flag;
    const RasterItem& it = items[blockIdx.y];
    if (!it.sse || !it.f[0]) return;
    const int64_t ng = (it.T + 31) / 32;
    const int64_t a = ng * blockIdx.x / gridDim.x, b = ng * (blockIdx.x + 1) / gridDim.x;
    const double* gp = gpart + gstride * blockIdx.y;
    double s = 0.0;
    for (int64_t k = a + threadIdx.x; k < b; k += RT) s += gp[k];
    s = block_sum<RT>(s, red);
    double* P = part + (size_t)blockIdx.y * gridDim.x;
    if (threadIdx.x == 0) P[blockIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        flag = (atomicAdd(&counters[blockIdx.y], 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (flag) {
        __threadfence();
        double t = 0.0;
        for (int k = threadIdx.x; k < (int)gridDim.x; k += RT) t += __ldcg(&P[k]);
        t = block_sum<RT>(t, red);
        if (threadIdx.x == 0) {
            *it.sse = t;
            counters[blockIdx.y] = 0;
        }
    }
}

// P^T r: per triangle, sum over its owned pixels of (l_a, l_b, l_c) r (vertex pixels:
// weight 1 on that vertex) -> tri_w[3t+k]; the vertex gather happens in tonal.cu.
__global__ void __launch_bounds__(RT) k_tri_adjoint(const TriRec* __restrict__ tri, const int32_t* __restrict__ tp_ptr,
                                                    const uint32_t* __restrict__ tp_pix, int64_t T, int W,
                                                    const double* __restrict__ r, double* __restrict__ tri_w) {
    __shared__ double acc_s[RWARPS][32][3];
    __shared__ WTri tris[RWARPS][32];
    __shared__ double rd_s[RWARPS][32];  // RN(1/D): w / D as a correctly rounded 3-op quotient
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ngroups = (T + 31) / 32;
    const int64_t gwarp = (int64_t)blockIdx.x * RWARPS + wid, nwarps = (int64_t)gridDim.x * RWARPS;
    WTri* ws = tris[wid];
    for (int64_t g = gwarp; g < ngroups; g += nwarps) {
        const int64_t t0 = g * 32;
        int cnt;
        const ListWalk lw = list_begin(tp_ptr, T, t0, cnt);
        if (t0 + lane < T) {
            const TriRec R = tri[t0 + lane];
            WTri I;
            I.ax = R.x[0];
            I.ay = R.y[0];
            I.bx = R.x[1];
            I.by = R.y[1];
            I.cx = R.x[2];
            I.cy = R.y[2];
            I.D = orient_xy(I.ax, I.ay, I.bx, I.by, I.cx, I.cy);
            ws[lane] = I;
            rd_s[wid][lane] = __drcp_rn((double)I.D);
        }
        acc_s[wid][lane][0] = 0.0;
        acc_s[wid][lane][1] = 0.0;
        acc_s[wid][lane][2] = 0.0;
        __syncwarp();
        for (int base = 0; base < lw.total; base += 32) {
            const int k = base + lane;
            const int j = warp_find(lw.excl, k, lw.total);
            double sa = 0.0, sb = 0.0, sc = 0.0;
            if (j < 32) {
                const uint32_t v = tp_pix[lw.ptr0 + k];
                const int px = (int)(v & 0x3fffu), py = (int)((v >> 14) & 0x3fffu);
                const double rv = r[(int64_t)py * W + px];
                const uint32_t cls = v >> 30;
                if (cls) {
                    if (cls == 1) sa = rv;
                    else if (cls == 2) sb = rv;
                    else sc = rv;
                } else {
                    const WTri& I = ws[j];
                    const double D = (double)I.D, rD = rd_s[wid][j];
                    // div_rn == the IEEE quotient (Markstein), so the sums are unchanged
                    sa = div_rn((double)orient_xy(I.bx, I.by, I.cx, I.cy, px, py), D, rD) * rv;
                    sb = div_rn((double)orient_xy(I.cx, I.cy, I.ax, I.ay, px, py), D, rD) * rv;
                    sc = div_rn((double)orient_xy(I.ax, I.ay, I.bx, I.by, px, py), D, rD) * rv;
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
            __syncwarp();
        }
        __syncwarp();
        if (t0 + lane < T) {
            tri_w[3 * (t0 + lane)] = acc_s[wid][lane][0];
            tri_w[3 * (t0 + lane) + 1] = acc_s[wid][lane][1];
            tri_w[3 * (t0 + lane) + 2] = acc_s[wid][lane][2];
        }
        __syncwarp();
    }
}

int warp_grid(int64_t T, int B) {
    const int64_t groups = (T + 31) / 32;
    const int64_t want = (groups + RWARPS - 1) / RWARPS;
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)148 * 8 / std::max(1, B) + 1));
}

}  // namespace

femi_status build_owner_tables(femi_system_s* S, cudaStream_t st) {
    const int64_t T = S->T, N = (int64_t)S->W * S->H;
    if (T == 0) return FEMI_OK;
    const int nb = (int)((T + SCB - 1) / SCB);
    int32_t* cnt = nullptr;
    int32_t* bsum = nullptr;
    FEMI_CUDA(cudaMallocAsync(&cnt, sizeof(int32_t) * T, st));
    FEMI_CUDA(cudaMallocAsync(&bsum, sizeof(int32_t) * (nb + 1), st));
    const int g = warp_grid(T, 1);
    k_build_owner<0><<<g, RT, 0, st>>>(S->tri, T, S->W, cnt, nullptr, nullptr);
    k_scan_blocks<<<nb, SCB, 0, st>>>(T, cnt, bsum);
    k_scan_bsum<<<1, 32, 0, st>>>(nb, bsum);
    k_scan_apply<<<nb, SCB, 0, st>>>(T, cnt, bsum, S->tp_ptr);
    k_build_owner<1><<<g, RT, 0, st>>>(S->tri, T, S->W, nullptr, S->tp_ptr, S->tp_pix);
    count_launches(5);
    FEMI_CUDA(cudaGetLastError());
    FEMI_CUDA(cudaFreeAsync(cnt, st));
    FEMI_CUDA(cudaFreeAsync(bsum, st));
    (void)N;
    return FEMI_OK;
}

namespace {

// items[b] all with the same channel count nc (1..kMaxCh)
femi_status launch_raster_items(std::vector<RasterItem>& items, int nc, cudaStream_t st) {
    const int B = (int)items.size();
    int64_t Tmax = 0;
    for (const RasterItem& r : items) Tmax = std::max(Tmax, r.T);
    if (B == 0 || Tmax == 0) return FEMI_OK;
    static int resident = 0;
    if (resident == 0) {
        int dev = 0, nsm = 0, per = 0;
        FEMI_CUDA(cudaGetDevice(&dev));
        FEMI_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        FEMI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void*)k_raster_tri<4, 256, 1>, RT,
                                                                RWARPS * 32 * sizeof(RTri<1>)));
        resident = std::max(1, per) * nsm;
    }
    // one wave of resident CTAs (colour: 2 CTAs/SM); 32-triangle groups handed out dynamically
    // in canonical order
    const int64_t groups = (Tmax + 31) / 32;
    const int res = nc == 1 ? resident : resident / 2;
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((groups + RWARPS - 1) / RWARPS,
                                                              (int64_t)std::max(1, res / B)));
    constexpr int SSEB = 148;
    const size_t bytes_items = sizeof(RasterItem) * B;
    const size_t bytes_gpart = sizeof(double) * (size_t)groups * B;
    const size_t bytes_part = sizeof(double) * (size_t)SSEB * B;
    const size_t bytes_cnt = sizeof(uint32_t) * 2 * B;
    void* base = nullptr;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    FEMI_CUDA(cudaMallocAsync(&base, al(bytes_items) + al(bytes_gpart) + al(bytes_part) + al(bytes_cnt), st));
    char* cur = (char*)base;
    RasterItem* d_items = (RasterItem*)cur;
    double* d_gpart = (double*)(cur + al(bytes_items));
    double* d_part = (double*)((char*)d_gpart + al(bytes_gpart));
    uint32_t* d_cnt = (uint32_t*)((char*)d_part + al(bytes_part));
    FEMI_CUDA(cudaMemcpyAsync(d_items, items.data(), bytes_items, cudaMemcpyHostToDevice, st));
    FEMI_CUDA(cudaMemsetAsync(d_cnt, 0, bytes_cnt, st));
    const dim3 gr(gx, B);
    static bool attr = false;
    if (!attr) {
        FEMI_CUDA(cudaFuncSetAttribute((const void*)k_raster_tri<2, 128, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(RWARPS * 32 * sizeof(RTri<3>))));
        FEMI_CUDA(cudaFuncSetAttribute((const void*)k_raster_tri<2, 128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(RWARPS * 32 * sizeof(RTri<4>))));
        attr = true;
    }
    switch (nc) {
        case 1:
            k_raster_tri<4, 256, 1><<<gr, RT, RWARPS * 32 * sizeof(RTri<1>), st>>>(d_items, d_gpart, d_cnt, groups);
            break;
        case 2:
            k_raster_tri<2, 128, 2><<<gr, RT, RWARPS * 32 * sizeof(RTri<2>), st>>>(d_items, d_gpart, d_cnt, groups);
            break;
        case 3:
            k_raster_tri<2, 128, 3><<<gr, RT, RWARPS * 32 * sizeof(RTri<3>), st>>>(d_items, d_gpart, d_cnt, groups);
            break;
        default:
            k_raster_tri<2, 128, 4><<<gr, RT, RWARPS * 32 * sizeof(RTri<4>), st>>>(d_items, d_gpart, d_cnt, groups);
            break;
    }
    k_sse<<<dim3(SSEB, B), RT, 0, st>>>(d_items, d_gpart, groups, d_part, d_cnt + B);
    count_launches(2);
    FEMI_CUDA(cudaGetLastError());
    FEMI_CUDA(cudaFreeAsync(base, st));
    return FEMI_OK;
}

RasterItem raster_item(const femi_system_s* S) {
    RasterItem r = {};
    r.tri = S->tri;
    r.tp_ptr = S->tp_ptr;
    r.tp_pix = S->tp_pix;
    r.T = S->T;
    r.N = (int64_t)S->W * S->H;
    r.W = S->W;
    return r;
}

}  // namespace

femi_status launch_raster(int B, femi_system_s* const* S, const double* const* u_vert, const double* const* f,
                          double* const* u_px, double* const* e_px, double* const* tri_err, int32_t* const* best,
                          double* const* sse, cudaStream_t st) {
    if (B <= 0) return FEMI_OK;
    std::vector<RasterItem> items(B);
    for (int b = 0; b < B; ++b) {
        RasterItem& r = items[b];
        r = raster_item(S[b]);
        r.u_vert[0] = u_vert[b];
        r.f[0] = f ? f[b] : nullptr;
        r.u_px[0] = u_px ? u_px[b] : nullptr;
        r.e_px = e_px ? e_px[b] : nullptr;
        r.tri_err = tri_err ? tri_err[b] : nullptr;
        r.best = best ? best[b] : nullptr;
        r.sse = sse ? sse[b] : nullptr;
    }
    return launch_raster_items(items, 1, st);
}

femi_status launch_raster_channels(femi_system_s* S, int nc, const double* const* u_vert, const double* const* f,
                                   double* const* u_px, double* e_px, double* tri_err, int32_t* best, double* sse,
                                   cudaStream_t st) {
    if (nc < 1 || nc > kMaxCh) return FEMI_E_ARG;
    std::vector<RasterItem> items(1);
    RasterItem& r = items[0];
    r = raster_item(S);
    for (int c = 0; c < nc; ++c) {
        r.u_vert[c] = u_vert[c];
        r.f[c] = f ? f[c] : nullptr;
        r.u_px[c] = u_px ? u_px[c] : nullptr;
    }
    r.e_px = e_px;
    r.tri_err = tri_err;
    r.best = best;
    r.sse = sse;
    return launch_raster_items(items, nc, st);
}

femi_status launch_adjoint_raster(femi_system_s* S, const double* r, double* tri_w, cudaStream_t st) {
    if (S->T == 0) return FEMI_OK;
    k_tri_adjoint<<<warp_grid(S->T, 1), RT, 0, st>>>(S->tri, S->tp_ptr, S->tp_pix, S->T, S->W, r, tri_w);
    count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    return FEMI_OK;
}

}  // namespace femi
