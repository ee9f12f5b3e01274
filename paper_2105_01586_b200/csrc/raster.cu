// raster.cu -- S3+S4: rasterise the P1 solution and reduce the squared error
// (PAPER.md:L239-241 interpolation; L262-265 "e_i = (u_i - f_i)^2", "total L2 error in
// each triangle"), and the adjoint raster P^T r used by tonal optimisation (S6).
//
// Pixel ownership (reading A7: lowest index among the closed triangles containing a
// pixel) depends only on the mesh, so it is resolved ONCE per mesh at assembly by a
// warp-cooperative triangle expansion (raster_common.cuh) into triangle-major lists
// (ascending pixels per triangle), which are then merged per group of 16 consecutive
// canonical triangles into the GROUP LIST the per-solve kernels read:
//   tp_ptr[t]   = first entry of triangle t (CSR over triangles; groups are contiguous)
//   tp_pix[q]   = j << 28 | (y - y0) << 14 | x, the group's owned pixels in ascending pixel
//                 order, j = the owner's slot in the group, y0 = the group's top row
//                 (W, H <= 16384: 14 bits each).
// Every solve then rasterises with ONE kernel (k_raster_grp): lanes take consecutive pixels
// of the group's rows (coalesced f / u / e traffic); per-triangle error sums and arg-max over
// non-vertex pixels (ties: lowest pix) are segmented warp reductions over runs of one
// triangle; SSE = fixed-order sum of the group sums. Deterministic. The adjoint P^T r is the
// same traversal with barycentric weights.
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
    const int32_t* wptr;  // windows per group (CSR)
    const void* win;      // WinRec[]
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

// Correctly rounded w / D for an exact integer w (|w| < 2^53) given rD = RN(1/D): q = RN(w rD)
// is within 1 ulp of w/D, the remainder w - qD is exact under fma, and RN(q + r rD) is RN(w/D)
// (Markstein's theorem) -- the IEEE quotient of __ddiv_rn at three fp64 operations.
__device__ __forceinline__ double div_rn(double w, double D, double rD) {
    const double q = __dmul_rn(w, rD);
    const double r = __fma_rn(-q, D, w);
    return __fma_rn(r, rD, q);
}

constexpr int GT = 32;    // triangles per group (5-bit slot; lane j of a warp owns triangle j)
constexpr int RCH = 128;  // entries per raster window (7-bit slot)

// Group list as built by k_group_list (64-bit, setup only): (y << 14 | x) << 5 | j
__device__ __forceinline__ int gk_j(uint64_t v) { return (int)(v & 31u); }
__device__ __forceinline__ int gk_y(uint64_t v) { return (int)(v >> 19); }
__device__ __forceinline__ int gl_x(uint32_t v) { return (int)(v & 0x3fffu); }
// ... and as the raster reads it (one window of <= 128 entries spanning < 64 rows):
// slot << 25 | j << 20 | (y - y_window) << 14 | x; slot = the entry's position in the window's
// triangle-major order (triangle j's entries at start[j] .. start[j+1], in pixel order)
__device__ __forceinline__ int wl_slot(uint32_t v) { return (int)(v >> 25); }
__device__ __forceinline__ int wl_j(uint32_t v) { return (int)((v >> 20) & 31u); }
__device__ __forceinline__ int wl_dy(uint32_t v) { return (int)((v >> 14) & 63u); }
constexpr int kWinRows = 64;  // rows a window may span (6-bit offsets)

struct __align__(16) WinRec {
    int32_t q0;             // first entry (global index into tp_pix)
    int16_t y0;             // the window's top row
    uint8_t n, pad0;        // entries (1..128)
    uint8_t start[GT + 1];  // triangle-major offsets of the group's triangles in the window
    uint8_t pad1[7];
};
static_assert(sizeof(WinRec) == 48, "WinRec is 48 bytes");

// Per mesh, after k_group_list: split each group's list into windows (greedy: a window ends
// after 128 entries or before an entry 64 or more rows below its first one). FILL = 0 counts
// the windows per group; FILL = 1 writes the records and the 32-bit entries. One WARP per group
// (setup only): the window's end is the first entry of a 32-entry ballot round that breaks the
// row rule; per-triangle counts and the entries' triangle-major slots come from __match_any
// rounds in entry order (rank among the round's lanes of the same triangle + a running count
// per triangle), so the slots are the entries' positions in the window's triangle-major order,
// pixel order inside a triangle.
template <int FILL>
__global__ void __launch_bounds__(RT) k_win(const TriRec* __restrict__ tri, int64_t T,
                                            const int32_t* __restrict__ tp_ptr, const uint64_t* __restrict__ gk,
                                            uint32_t* __restrict__ gl, int32_t* __restrict__ wcnt,
                                            const int32_t* __restrict__ wptr, WinRec* __restrict__ win) {
    __shared__ int run_s[RWARPS][GT + 1];
    __shared__ __align__(16) int rec_s[RWARPS][12];  // the 48-byte record being written
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ngroups = (T + GT - 1) / GT;
    const int64_t gwarp = (int64_t)blockIdx.x * RWARPS + wid, nwarps = (int64_t)gridDim.x * RWARPS;
    int* run = run_s[wid];
    for (int64_t g = gwarp; g < ngroups; g += nwarps) {
        const int64_t t0 = g * GT;
        const int nt = (int)min((int64_t)GT, T - t0);
        const int q0 = tp_ptr[t0], q1 = tp_ptr[t0 + nt];
        int nw = 0;
        int64_t w = FILL ? wptr[g] : 0;
        int q = q0;
        while (q < q1) {
            const int ys = gk_y(gk[q]);
            const int lim = min(q1, q + RCH);
            int e = lim;
            for (int base = q + 1; base < lim; base += 32) {
                const int k = base + lane;
                const bool brk = k < lim && gk_y(gk[k]) - ys >= kWinRows;
                const unsigned m = __ballot_sync(0xffffffffu, brk);
                if (m) {
                    e = base + __ffs(m) - 1;
                    break;
                }
            }
            if (FILL) {
                run[lane] = 0;
                if (lane == 0) run[GT] = 0;
                __syncwarp();
                for (int base = q; base < e; base += 32) {  // entries per triangle
                    const int k = base + lane;
                    const bool act = k < e;
                    const unsigned mask = __ballot_sync(0xffffffffu, act);
                    if (act) {
                        const int j = gk_j(gk[k]);
                        const unsigned mm = __match_any_sync(mask, j);
                        if (lane == __ffs(mm) - 1) run[j] += __popc(mm);
                    }
                    __syncwarp();
                }
                const int c = lane < GT ? run[lane] : 0;
                int inc = c;
                for (int o = 1; o < 32; o <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += v;
                }
                const int total = __shfl_sync(0xffffffffu, inc, 31);
                FEMI_DCHECK(total == e - q && total <= RCH && w < wptr[g + 1], 4);
                if (lane < 12) rec_s[wid][lane] = 0;
                __syncwarp();
                WinRec* R = reinterpret_cast<WinRec*>(rec_s[wid]);
                if (lane == 0) {
                    R->q0 = q;
                    R->y0 = (int16_t)ys;
                    R->n = (uint8_t)(e - q);
                    R->start[GT] = (uint8_t)total;
                }
                R->start[lane] = (uint8_t)(inc - c);
                __syncwarp();
                run[lane] = inc - c;  // running slot per triangle
                __syncwarp();
                if (lane < 3) reinterpret_cast<int4*>(win + w)[lane] = reinterpret_cast<const int4*>(rec_s[wid])[lane];
                for (int base = q; base < e; base += 32) {  // slots in entry order
                    const int k = base + lane;
                    const bool act = k < e;
                    const unsigned mask = __ballot_sync(0xffffffffu, act);
                    int slot = 0, j = 0;
                    uint64_t v = 0;
                    unsigned mm = 0;
                    if (act) {
                        v = gk[k];
                        j = gk_j(v);
                        mm = __match_any_sync(mask, j);
                        slot = run[j] + __popc(mm & ((1u << lane) - 1u));
                    }
                    __syncwarp();
                    if (act && lane == __ffs(mm) - 1) run[j] += __popc(mm);
                    __syncwarp();
                    if (act) {
                        const uint32_t dyw = (uint32_t)(gk_y(v) - ys);
                        gl[k] = ((uint32_t)slot << 25) | ((uint32_t)j << 20) | (dyw << 14) |
                                ((uint32_t)(v >> 5) & 0x3fffu);
                    }
                }
                ++w;
            }
            ++nw;
            q = e;
        }
        if (!FILL && lane == 0) wcnt[g] = nw;
        __syncwarp();
    }
}

// The group's triangles as the raster reads them: structure of arrays in shared memory (lanes
// of a warp index different triangles -- one bank-conflict-free access per field): the exact
// integer edge-function planes w = A px + B py + C (S3: w_b = orient(c,a,p), w_c = orient(a,b,p)),
// D = orient(a,b,c) as int and double, RN(1/D), u_a and the differences u_b - u_a, u_c - u_a,
// and the vertex values u_b, u_c (vertex pixels take them exactly).
template <int NC>
struct GTri {
    int AB1[GT], C1[GT], AB2[GT], C2[GT], Di[GT], pad[3][GT];  // AB = A & 0xffff | B << 16
    double rD[GT];
    double ua[NC][GT], db[NC][GT], dc[NC][GT], ub[NC][GT], uc[NC][GT];
};
// |A|, |B| <= 16383 (coordinates < 2^14): the two plane coefficients share one word, so an
// entry reads its triangle with 5 four-byte and 4 eight-byte shared loads (the vertex values
// u_b, u_c only at vertex pixels, a predicated load); D is converted from the exact integer Di
// (measured at C5: shared-load wavefronts 71 M -> 61 M, raster 0.686 -> 0.679 ms)
__device__ __forceinline__ int ab_pack(int a, int b) { return (a & 0xffff) | (int)((unsigned)b << 16); }
__device__ __forceinline__ int ab_lo(int v) { return (int)(v << 16) >> 16; }
__device__ __forceinline__ int ab_hi(int v) { return v >> 16; }

// S3+S4 in ONE pass over the raster windows of each 16-triangle group (groups handed out in
// canonical order by an atomic counter). Per window of <= 128 entries (the group's owned pixels
// in ascending pixel order: row segments of the group's region, so consecutive lanes read f
// and write u, e at consecutive pixels -- coalesced):
//   lane per entry: u = the vertex value (vertex pixel: both barycentric numerators 0 or one
//   of them == D, exact integers) or (u_a + l_b (u_b - u_a)) + l_c (u_c - u_a) with l = w / D
//   in IEEE fp64 (S3's form, one rounding per operation, no contraction); e = (u - f)^2, staged
//   in shared memory at the entry's precomputed triangle-major slot;
//   lane j < 16: walks triangle j's slots start[j] .. start[j+1] (its entries of the window in
//   pixel order): tri_err += e, best = first strict maximum over non-vertex pixels.
// Windows are in pixel order, so every triangle is summed in the oracle's sequential order:
// u_px, e_px, tri_err and best are bit-identical to it. SSE = per-group sums in group order.
template <int MINB, int NC>
__global__ void __launch_bounds__(RT, MINB) k_raster_grp(const RasterItem* __restrict__ items,
                                                         double* __restrict__ gpart, uint32_t* __restrict__ next,
                                                         int64_t gstride) {
    extern __shared__ __align__(16) unsigned char rsm[];  // GTri<NC> [RWARPS]
    __shared__ double e_s[RWARPS][RCH];                   // staged e (sign bit set: vertex pixel)
    __shared__ int p_s[RWARPS][RCH];                      // staged pix
    const RasterItem& it = items[blockIdx.y];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t T = it.T;
    const int W = it.W;
    const bool hasf = it.f[0] != nullptr;
    double* __restrict__ e_px = it.e_px;
    const uint32_t* __restrict__ gl = it.tp_pix;
    const WinRec* __restrict__ win = (const WinRec*)it.win;
    const int64_t ngroups = (T + GT - 1) / GT;
    GTri<NC>& G = ((GTri<NC>*)rsm)[wid];
    double* __restrict__ gp = gpart + gstride * blockIdx.y;
    double* es = e_s[wid];
    int* ps = p_s[wid];
    for (;;) {
        int64_t g = 0;
        if (lane == 0) g = (int64_t)atomicAdd(next + blockIdx.y, 1u);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= ngroups) break;
        const int64_t t0 = g * GT;
        const int nt = (int)min((int64_t)GT, T - t0);
        const int w0 = it.wptr[g], w1 = it.wptr[g + 1];
        if (lane < nt) {
            const TriRec R = it.tri[t0 + lane];
            const int ax = R.x[0], ay = R.y[0], bx = R.x[1], by = R.y[1], cx = R.x[2], cy = R.y[2];
            // w_b = orient(c,a,p) = (ax-cx)(py-cy) - (ay-cy)(px-cx) = A1 px + B1 py + C1
            G.AB1[lane] = ab_pack(cy - ay, ax - cx);
            G.C1[lane] = (ay - cy) * cx - (ax - cx) * cy;
            // w_c = orient(a,b,p) = (bx-ax)(py-ay) - (by-ay)(px-ax) = A2 px + B2 py + C2
            G.AB2[lane] = ab_pack(ay - by, bx - ax);
            G.C2[lane] = (by - ay) * ax - (bx - ax) * ay;
            const int Di = orient_xy(ax, ay, bx, by, cx, cy);
            G.Di[lane] = Di;
            G.rD[lane] = __drcp_rn((double)Di);
#pragma unroll
            for (int ch = 0; ch < NC; ++ch) {
                const double u0 = it.u_vert[ch][R.v[0]], u1 = it.u_vert[ch][R.v[1]], u2 = it.u_vert[ch][R.v[2]];
                G.ua[ch][lane] = u0;
                G.ub[ch][lane] = u1;
                G.uc[ch][lane] = u2;
                G.db[ch][lane] = __dsub_rn(u1, u0);
                G.dc[ch][lane] = __dsub_rn(u2, u0);
            }
        }
        double acc = 0.0, be = -1.0;  // lane j < nt: triangle j's running sum / best e
        int bp = -1;
        __syncwarp();
        // window w's record and entries are loaded one window ahead
        int nq0 = 0, ny0 = 0, nn = 0, ns0 = 0, ns1 = 0;
        uint32_t vn[RCH / 32];
        auto load_win = [&](int w) {
            // the record through the read-only path: {q0, y0, n} in one 8-byte load, two start bytes
            const int2 h0 = __ldg(reinterpret_cast<const int2*>(win + w));
            nq0 = h0.x;
            ny0 = (int)(int16_t)(h0.y & 0xffff);
            nn = (h0.y >> 16) & 0xff;
            if (lane < nt) {
                ns0 = __ldg(&win[w].start[lane]);
                ns1 = __ldg(&win[w].start[lane + 1]);
            }
#pragma unroll
            for (int h = 0; h < RCH / 32; ++h) {
                const int k = 32 * h + lane;
                vn[h] = k < nn ? __ldg(gl + nq0 + k) : 0xffffffffu;
            }
        };
        if (w0 < w1) load_win(w0);
        for (int w = w0; w < w1; ++w) {
            uint32_t v[RCH / 32];
            const int y0 = ny0, s0 = ns0, s1 = ns1;
#pragma unroll
            for (int h = 0; h < RCH / 32; ++h) v[h] = vn[h];
            if (w + 1 < w1) load_win(w + 1);
            double fv[RCH / 32][NC];
#pragma unroll
            for (int h = 0; h < RCH / 32; ++h)
#pragma unroll
                for (int ch = 0; ch < NC; ++ch)
                    fv[h][ch] = (hasf && v[h] != 0xffffffffu)
                                    ? __ldg(it.f[ch] + (int64_t)(y0 + wl_dy(v[h])) * W + gl_x(v[h]))
                                    : 0.0;
#pragma unroll
            for (int h = 0; h < RCH / 32; ++h) {
                if (v[h] == 0xffffffffu) continue;
                const int j = wl_j(v[h]);
                const int px = gl_x(v[h]), py = y0 + wl_dy(v[h]);
                const int pix = py * W + px;
                FEMI_DCHECK(j < nt && px < W && (int64_t)pix < it.N && wl_slot(v[h]) < RCH, 4);
                const int ab1 = G.AB1[j], ab2 = G.AB2[j];
                const int w1v = ab_lo(ab1) * px + ab_hi(ab1) * py + G.C1[j];
                const int w2v = ab_lo(ab2) * px + ab_hi(ab2) * py + G.C2[j];
                const int Di = G.Di[j];
                // vertex pixels: a (w_b = w_c = 0), b (w_b = D, w_c = 0), c (w_b = 0, w_c = D);
                // branch-free: the quotients are formed for every entry, the vertex value selected
                const bool z1 = w1v == 0, z2 = w2v == 0;
                const bool isa = z1 && z2, isb = w1v == Di && z2, isc = z1 && w2v == Di;
                const bool cls = isa || isb || isc;
                const double D = (double)Di, rD = G.rD[j];
                const double lb = div_rn((double)w1v, D, rD);
                const double lc = div_rn((double)w2v, D, rD);
                double e = 0.0;
#pragma unroll
                for (int ch = 0; ch < NC; ++ch) {
                    const double ua = G.ua[ch][j];
                    const double ui = __dadd_rn(__dadd_rn(ua, __dmul_rn(lb, G.db[ch][j])), __dmul_rn(lc, G.dc[ch][j]));
                    double uv = ua;
                    if (isb || isc) uv = *(isb ? &G.ub[ch][j] : &G.uc[ch][j]);  // predicated: vertex pixels only
                    const double u = cls ? uv : ui;
                    if (it.u_px[ch]) __stcs(it.u_px[ch] + pix, u);  // streaming store (written once)
                    if (hasf) {
                        const double d = __dsub_rn(u, fv[h][ch]);
                        e = ch == 0 ? __dmul_rn(d, d) : __dadd_rn(e, __dmul_rn(d, d));  // channel sum in order
                    }
                }
                if (hasf) {
                    if (e_px) __stcs(e_px + pix, e);
                    const int sl = wl_slot(v[h]);
                    es[sl] = cls ? -e : e;  // -0.0 for e = 0: the sign bit is the flag
                    ps[sl] = pix;
                }
            }
            __syncwarp();
            if (hasf && lane < nt) {
                for (int k = s0; k < s1; ++k) {
                    const double x = es[k];
                    const double e = fabs(x);
                    acc = __dadd_rn(acc, e);
                    if (__double_as_longlong(x) >= 0 && e > be) {
                        be = e;
                        bp = ps[k];
                    }
                }
            }
            __syncwarp();
        }
        if (hasf) {
            if (lane < nt) {
                if (it.tri_err) it.tri_err[t0 + lane] = acc;
                if (it.best) it.best[t0 + lane] = bp;
            }
            const double gs = warp_sum(lane < nt ? acc : 0.0);  // group partial of the SSE (fixed order)
            if (lane == 0) gp[g] = gs;
        }
        __syncwarp();
    }
}

// SSE = sum of the per-group partials in group order (two fixed levels: deterministic)
__global__ void __launch_bounds__(RT) k_sse(const RasterItem* __restrict__ items, const double* __restrict__ gpart,
                                           int64_t gstride, double* __restrict__ part, uint32_t* __restrict__ counters) {
    __shared__ double red[RWARPS];
    __shared__ int flag;
    const RasterItem& it = items[blockIdx.y];
    if (!it.sse || !it.f[0]) return;
    const int64_t ng = (it.T + GT - 1) / GT;
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

// P^T r over the raster windows: per triangle, the sum over its owned pixels of
// (l_a, l_b, l_c) r (vertex pixels: weight 1 on that vertex) -> tri_w[3t+k]. Staged at the
// entries' triangle-major slots and summed per triangle in pixel order (deterministic). The
// vertex gather happens in tonal.cu.
__global__ void __launch_bounds__(RT) k_tri_adjoint(const TriRec* __restrict__ tri, const int32_t* __restrict__ wptr,
                                                    const WinRec* __restrict__ win, const uint32_t* __restrict__ gl,
                                                    int64_t T, int W, const double* __restrict__ r,
                                                    double* __restrict__ tri_w) {
    __shared__ int4 tg_s[RWARPS][GT];      // (A1, B1, C1, D) of w_b
    __shared__ int4 tc_s[RWARPS][GT];      // (A2, B2, C2, -)
    __shared__ double rd_s[RWARPS][GT];    // RN(1/D)
    __shared__ double st_s[RWARPS][3][RCH];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ngroups = (T + GT - 1) / GT;
    const int64_t gwarp = (int64_t)blockIdx.x * RWARPS + wid, nwarps = (int64_t)gridDim.x * RWARPS;
    for (int64_t g = gwarp; g < ngroups; g += nwarps) {
        const int64_t t0 = g * GT;
        const int nt = (int)min((int64_t)GT, T - t0);
        if (lane < nt) {
            const TriRec R = tri[t0 + lane];
            const int ax = R.x[0], ay = R.y[0], bx = R.x[1], by = R.y[1], cx = R.x[2], cy = R.y[2];
            const int D = orient_xy(ax, ay, bx, by, cx, cy);
            tg_s[wid][lane] = make_int4(cy - ay, ax - cx, (ay - cy) * cx - (ax - cx) * cy, D);
            tc_s[wid][lane] = make_int4(ay - by, bx - ax, (by - ay) * ax - (bx - ax) * ay, 0);
            rd_s[wid][lane] = __drcp_rn((double)D);
        }
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        __syncwarp();
        for (int w = wptr[g]; w < wptr[g + 1]; ++w) {
            const WinRec& R = win[w];
            const int q0 = R.q0, y0 = R.y0, n = R.n;
            for (int k = lane; k < n; k += 32) {
                const uint32_t v = gl[q0 + k];
                const int j = wl_j(v), sl = wl_slot(v);
                const int px = gl_x(v), py = y0 + wl_dy(v);
                FEMI_DCHECK(j < nt && sl < n && px < W && (int64_t)py * W + px < (int64_t)W * 16384, 4);
                const double rv = r[(int64_t)py * W + px];
                const int4 P1 = tg_s[wid][j], P2 = tc_s[wid][j];
                const int w1 = P1.x * px + P1.y * py + P1.z;  // w_b
                const int w2 = P2.x * px + P2.y * py + P2.z;  // w_c
                const int D = P1.w;
                double sa = 0.0, sb = 0.0, sc = 0.0;
                if (w1 == 0 && w2 == 0) {
                    sa = rv;
                } else if (w1 == D && w2 == 0) {
                    sb = rv;
                } else if (w2 == D && w1 == 0) {
                    sc = rv;
                } else {
                    const double Dd = (double)D, rD = rd_s[wid][j];
                    sa = div_rn((double)(D - w1 - w2), Dd, rD) * rv;  // w_a = D - w_b - w_c exactly
                    sb = div_rn((double)w1, Dd, rD) * rv;
                    sc = div_rn((double)w2, Dd, rD) * rv;
                }
                st_s[wid][0][sl] = sa;
                st_s[wid][1][sl] = sb;
                st_s[wid][2][sl] = sc;
            }
            __syncwarp();
            if (lane < nt)
                for (int k = R.start[lane]; k < R.start[lane + 1]; ++k) {
                    a0 += st_s[wid][0][k];
                    a1 += st_s[wid][1][k];
                    a2 += st_s[wid][2][k];
                }
            __syncwarp();
        }
        if (lane < nt) {
            tri_w[3 * (t0 + lane)] = a0;
            tri_w[3 * (t0 + lane) + 1] = a1;
            tri_w[3 * (t0 + lane) + 2] = a2;
        }
        __syncwarp();
    }
}

// Group list from the triangle-major lists (per mesh): the entries of GT consecutive triangles
// merged into ascending pixel order (rank = number of the group's entries with a smaller pixel,
// one lower_bound per triangle list), tagged with the triangle slot: (y << 14 | x) << 5 | j,
// written to `out` at the same offsets (the group's entries are contiguous).
__global__ void __launch_bounds__(RT) k_group_list(int64_t T, const int32_t* __restrict__ tp_ptr,
                                                   const uint32_t* __restrict__ tp_pix, uint64_t* __restrict__ out) {
    __shared__ int off_s[RWARPS][GT + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t ngroups = (T + GT - 1) / GT;
    const int64_t gwarp = (int64_t)blockIdx.x * RWARPS + wid, nwarps = (int64_t)gridDim.x * RWARPS;
    int* off = off_s[wid];
    for (int64_t g = gwarp; g < ngroups; g += nwarps) {
        const int64_t t0 = g * GT;
        const int nt = (int)min((int64_t)GT, T - t0);
        if (lane < nt) off[lane] = tp_ptr[t0 + lane];  // the group's offsets
        if (lane == 0) off[nt] = tp_ptr[t0 + nt];
        __syncwarp();
        const int q0 = off[0], q1 = off[nt];
        for (int q = q0 + lane; q < q1; q += 32) {
            const uint32_t key = tp_pix[q] & 0x0fffffffu;  // y << 14 | x: pixel order
            int rank = 0, j = 0;
            for (int jj = 0; jj < nt; ++jj) {
                int a = off[jj], b = off[jj + 1];
                if (q >= a && q < b) j = jj;
                while (a < b) {  // lower_bound of key in triangle jj's ascending list
                    const int mid = (a + b) >> 1;
                    if ((tp_pix[mid] & 0x0fffffffu) < key) a = mid + 1;
                    else b = mid;
                }
                rank += a - off[jj];
            }
            FEMI_DCHECK(q0 + rank < q1, 4);
            out[q0 + rank] = ((uint64_t)key << 5) | (uint64_t)j;
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

// Per mesh: the triangle-major lists (owned-pixel counts, scan, ascending-pixel lists), merged
// per group of GT triangles into ascending pixel order, cut into raster windows and encoded
// into S->tp_pix (S->tp_ptr keeps the per-triangle offsets; its values at multiples of GT
// delimit the groups; S->tp_wptr / tp_win index the windows).
femi_status build_owner_tables(femi_system_s* S, cudaStream_t st) {
    const int64_t T = S->T, N = (int64_t)S->W * S->H;
    if (T == 0) return FEMI_OK;
    const int nb = (int)((T + SCB - 1) / SCB);
    int32_t* cnt = nullptr;
    int32_t* bsum = nullptr;
    uint32_t* tmp = nullptr;
    uint64_t* gk = nullptr;
    FEMI_CUDA(cudaMallocAsync(&cnt, sizeof(int32_t) * T, st));
    FEMI_CUDA(cudaMallocAsync(&bsum, sizeof(int32_t) * (nb + 1), st));
    FEMI_CUDA(cudaMallocAsync(&tmp, sizeof(uint32_t) * N, st));
    FEMI_CUDA(cudaMallocAsync(&gk, sizeof(uint64_t) * N, st));
    const int g = warp_grid(T, 1);
    k_build_owner<0><<<g, RT, 0, st>>>(S->tri, T, S->W, cnt, nullptr, nullptr);
    k_scan_blocks<<<nb, SCB, 0, st>>>(T, cnt, bsum);
    k_scan_bsum<<<1, 32, 0, st>>>(nb, bsum);
    k_scan_apply<<<nb, SCB, 0, st>>>(T, cnt, bsum, S->tp_ptr);
    k_build_owner<1><<<g, RT, 0, st>>>(S->tri, T, S->W, nullptr, S->tp_ptr, tmp);
    k_group_list<<<warp_grid(T, 1), RT, 0, st>>>(T, S->tp_ptr, tmp, gk);
    // raster windows: count per group, scan, allocate, fill (entries re-encoded in place)
    const int64_t ngroups = (T + GT - 1) / GT;
    const int nbg = (int)((ngroups + SCB - 1) / SCB);
    FEMI_CUDA(cudaMallocAsync(&S->tp_wptr, sizeof(int32_t) * (ngroups + 1), st));  // freed with the system
    S->allocs.push_back(S->tp_wptr);
    const int gw = warp_grid(T, 1);
    k_win<0><<<gw, RT, 0, st>>>(S->tri, T, S->tp_ptr, gk, nullptr, cnt, nullptr, nullptr);
    k_scan_blocks<<<nbg, SCB, 0, st>>>(ngroups, cnt, bsum);
    k_scan_bsum<<<1, 32, 0, st>>>(nbg, bsum);
    k_scan_apply<<<nbg, SCB, 0, st>>>(ngroups, cnt, bsum, S->tp_wptr);
    int32_t nwin = 0;
    FEMI_CUDA(cudaMemcpyAsync(&nwin, S->tp_wptr + ngroups, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    FEMI_CUDA(cudaStreamSynchronize(st));
    S->tp_nwin = nwin;
    FEMI_CUDA(cudaMallocAsync(&S->tp_win, sizeof(WinRec) * std::max<int64_t>(nwin, 1), st));
    S->allocs.push_back(S->tp_win);
    k_win<1><<<gw, RT, 0, st>>>(S->tri, T, S->tp_ptr, gk, S->tp_pix, nullptr, S->tp_wptr, (WinRec*)S->tp_win);
    count_launches(11);
    FEMI_CUDA(cudaGetLastError());
    FEMI_CUDA(cudaFreeAsync(cnt, st));
    FEMI_CUDA(cudaFreeAsync(bsum, st));
    FEMI_CUDA(cudaFreeAsync(tmp, st));
    FEMI_CUDA(cudaFreeAsync(gk, st));
    return FEMI_OK;
}

namespace {

// items[b] all with the same channel count nc (1..kMaxCh)
femi_status launch_raster_items(std::vector<RasterItem>& items, int nc, cudaStream_t st) {
    const int B = (int)items.size();
    int64_t Tmax = 0;
    for (const RasterItem& r : items) Tmax = std::max(Tmax, r.T);
    if (B == 0 || Tmax == 0) return FEMI_OK;
    static const bool minb5 = [] {
        const char* e = std::getenv("FEMI_RASTER_MINB");
        return e && std::atoi(e) == 5;
    }();
    static int resident = 0, res_dev = -1;  // per device (occupancy and function attributes)
    int cur_dev = 0;
    FEMI_CUDA(cudaGetDevice(&cur_dev));
    if (res_dev != cur_dev) {
        res_dev = cur_dev;
        int dev = cur_dev, nsm = 0, per = 0;
        FEMI_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        FEMI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, minb5 ? (const void*)k_raster_grp<5, 1>
                                                                      : (const void*)k_raster_grp<4, 1>, RT,
                                                                RWARPS * sizeof(GTri<1>)));
        resident = std::max(1, per) * nsm;
    }
    // one wave of resident CTAs (colour: 2 CTAs/SM); 16-triangle groups handed out dynamically
    // in canonical order
    const int64_t groups = (Tmax + GT - 1) / GT;
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
    static int attr_dev = -1;
    if (attr_dev != cur_dev) {  // colour: the per-warp triangle tables exceed the default 48 KB
        FEMI_CUDA(cudaFuncSetAttribute((const void*)k_raster_grp<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(RWARPS * sizeof(GTri<2>))));
        FEMI_CUDA(cudaFuncSetAttribute((const void*)k_raster_grp<2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(RWARPS * sizeof(GTri<3>))));
        FEMI_CUDA(cudaFuncSetAttribute((const void*)k_raster_grp<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(RWARPS * sizeof(GTri<4>))));
        attr_dev = cur_dev;
    }
    switch (nc) {
        case 1:
            if (minb5)  // FEMI_RASTER_MINB=5: 5 CTAs/SM (48 registers)
                k_raster_grp<5, 1><<<gr, RT, RWARPS * sizeof(GTri<1>), st>>>(d_items, d_gpart, d_cnt, groups);
            else
                k_raster_grp<4, 1><<<gr, RT, RWARPS * sizeof(GTri<1>), st>>>(d_items, d_gpart, d_cnt, groups);
            break;
        case 2:
            k_raster_grp<2, 2><<<gr, RT, RWARPS * sizeof(GTri<2>), st>>>(d_items, d_gpart, d_cnt, groups);
            break;
        case 3:
            k_raster_grp<2, 3><<<gr, RT, RWARPS * sizeof(GTri<3>), st>>>(d_items, d_gpart, d_cnt, groups);
            break;
        default:
            k_raster_grp<2, 4><<<gr, RT, RWARPS * sizeof(GTri<4>), st>>>(d_items, d_gpart, d_cnt, groups);
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
    r.wptr = S->tp_wptr;
    r.win = S->tp_win;
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
    k_tri_adjoint<<<warp_grid(S->T, 1), RT, 0, st>>>(S->tri, S->tp_wptr, (const WinRec*)S->tp_win, S->tp_pix, S->T,
                                                      S->W, r, tri_w);
    count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    return FEMI_OK;
}

}  // namespace femi

FEMI_DCHECK_READER(dcheck_raster)
