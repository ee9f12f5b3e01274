// band.cu -- NEXT-4: row-band decomposition of ONE image's solve over several GPUs
// ("very large images", L498-502 linear memory).
//
// Canonical unknowns are numbered in ascending pixel order, so the unknowns [row0, row1) of
// rank r (equal counts, starts[r] = n_u r / R) are a band of image rows. Rank r owns the rows
// [row0, row1) of A_uu and A_uk (values assembled on its device with the same arithmetic as
// assemble.cu, reading A6). Its rows reference unknowns of other bands -- the HALO (sorted by
// canonical index, so grouped by owner); by the symmetry of the pattern, what rank q needs from
// r (r's SEND list to q) is exactly r's rows that have a column in q's band, in ascending order,
// i.e. the same sequence as q's halo slots owned by r.
//
// The solve is Jacobi-preconditioned CG in the single-reduction (Chronopoulos-Gear) form on the
// unscaled A_uu (M = diag A_uu), so an iteration has ONE exchange and ONE all-reduce:
//   update   beta = gamma/gamma_prev, alpha = gamma/(delta - beta gamma/alpha_prev);
//            p = u + beta p; s = w + beta s; x += alpha p; r -= alpha s; u = M^-1 r
//   pack     send[k] = u[send_row[k]]                 -> halo exchange (NCCL / loopback)
//   spmv     w = A u over own + halo columns; partial (r.u, w.u, r.r) per CTA, then a fixed
//            order sum                                  -> all-reduce of 4 doubles
// Every rank computes the same scalars from the same all-reduced dots (deterministic given the
// all-reduce). Convergence: ||r||^2 <= rtol^2 ||b||^2 on the recursion, then the true residual
// ||b - A x|| with the unscaled rows (reading A11) decides; a miss restarts from r = b - A x.
// x^0 = midrange(g) 1 (x0 mode 1): r^0 = -A_uk (g - c 1) by the zero row sums (Eq. (3)).
// The host side (Python, paper_2105_01586_b200/multi.py) only sequences the calls and the
// communication; every arithmetic step is one of these kernels.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "device.cuh"

namespace femi {

// ---------------------------------------------------------------- host plan
struct BandPlan {
    int32_t nranks = 1, rank = 0;
    int64_t n_u = 0, row0 = 0, row1 = 0, nloc = 0;
    std::vector<int64_t> halo;      // global canonical ids of the halo slots (ascending)
    std::vector<int32_t> peer;      // ranks exchanged with (ascending)
    std::vector<int64_t> recv_off;  // per peer: halo slots [recv_off[p], recv_off[p+1])
    std::vector<int64_t> send_off;  // per peer: send slots [send_off[p], send_off[p+1])
    std::vector<int32_t> send_row;  // local rows sent, ascending per peer
    std::vector<int32_t> rp, col;   // A_uu rows of the band: local columns (own < nloc <= halo)
    std::vector<int32_t> gcol, opp; // the same entries: canonical column, opposite vertices
    std::vector<int32_t> krp, kcol, kopp;  // A_uk rows of the band (mask columns)
};

static int64_t band_start(int64_t n_u, int32_t R, int32_t r) { return n_u * r / R; }
static int32_t band_owner(int64_t n_u, int32_t R, int64_t j) {
    // largest r with start(r) <= j
    int32_t lo = 0, hi = R - 1;
    while (lo < hi) {
        const int32_t mid = (lo + hi + 1) / 2;
        if (band_start(n_u, R, mid) <= j) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

static femi_status build_band_plan(const Mesh& M, int32_t R, int32_t r, BandPlan& P) {
    if (R < 1 || r < 0 || r >= R) {
        set_error("band: need 0 <= rank < nranks");
        return FEMI_E_ARG;
    }
    P = BandPlan();
    P.nranks = R;
    P.rank = r;
    P.n_u = M.n_u;
    P.row0 = band_start(M.n_u, R, r);
    P.row1 = band_start(M.n_u, R, r + 1);
    P.nloc = P.row1 - P.row0;
    const int32_t* rp = M.uu_rowptr.data();
    const int32_t* uc = M.uu_col.data();
    // halo: off-band columns of the band's rows (ascending canonical id = grouped by owner)
    std::vector<int64_t> h;
    for (int64_t i = P.row0; i < P.row1; ++i)
        for (int32_t e = rp[i]; e < rp[i + 1]; ++e)
            if (uc[e] < P.row0 || uc[e] >= P.row1) h.push_back(uc[e]);
    std::sort(h.begin(), h.end());
    h.erase(std::unique(h.begin(), h.end()), h.end());
    P.halo = h;
    // peers: owners of halo slots (by the pattern's symmetry also the ranks that read our rows)
    std::vector<int32_t> owner(h.size());
    for (size_t k = 0; k < h.size(); ++k) owner[k] = band_owner(M.n_u, R, h[k]);
    P.recv_off.push_back(0);
    for (size_t k = 0; k < h.size(); ++k) {
        if (k == 0 || owner[k] != owner[k - 1]) {
            if (k > 0) P.recv_off.push_back((int64_t)k);
            P.peer.push_back(owner[k]);
        }
    }
    if (!h.empty()) P.recv_off.push_back((int64_t)h.size());
    // send lists: own rows with a column in the peer's band, ascending
    P.send_off.push_back(0);
    for (int32_t q : P.peer) {
        const int64_t q0 = band_start(M.n_u, R, q), q1 = band_start(M.n_u, R, q + 1);
        for (int64_t i = P.row0; i < P.row1; ++i) {
            bool ref = false;
            for (int32_t e = rp[i]; e < rp[i + 1] && !ref; ++e) ref = uc[e] >= q0 && uc[e] < q1;
            if (ref) P.send_row.push_back((int32_t)(i - P.row0));
        }
        P.send_off.push_back((int64_t)P.send_row.size());
    }
    // local CSR of A_uu (entries in the canonical row order: ascending canonical column)
    P.rp.assign(P.nloc + 1, 0);
    for (int64_t i = P.row0; i < P.row1; ++i) P.rp[i - P.row0 + 1] = P.rp[i - P.row0] + (rp[i + 1] - rp[i]);
    const int64_t nnz = P.rp[P.nloc];
    P.col.resize(nnz);
    P.gcol.resize(nnz);
    P.opp.resize(2 * nnz);
    for (int64_t i = P.row0; i < P.row1; ++i) {
        int64_t o = P.rp[i - P.row0];
        for (int32_t e = rp[i]; e < rp[i + 1]; ++e, ++o) {
            const int32_t j = uc[e];
            P.gcol[o] = j;
            P.opp[2 * o] = M.uu_opp[2 * e];
            P.opp[2 * o + 1] = M.uu_opp[2 * e + 1];
            if (j >= P.row0 && j < P.row1) {
                P.col[o] = (int32_t)(j - P.row0);
            } else {
                const int64_t slot = std::lower_bound(h.begin(), h.end(), (int64_t)j) - h.begin();
                P.col[o] = (int32_t)(P.nloc + slot);
            }
        }
    }
    // A_uk rows of the band
    P.krp.assign(P.nloc + 1, 0);
    for (int64_t i = P.row0; i < P.row1; ++i)
        P.krp[i - P.row0 + 1] = P.krp[i - P.row0] + (M.uk_rowptr[i + 1] - M.uk_rowptr[i]);
    const int64_t nk = P.krp[P.nloc];
    P.kcol.resize(nk);
    P.kopp.resize(2 * nk);
    for (int64_t i = P.row0; i < P.row1; ++i) {
        int64_t o = P.krp[i - P.row0];
        for (int32_t e = M.uk_rowptr[i]; e < M.uk_rowptr[i + 1]; ++e, ++o) {
            P.kcol[o] = M.uk_col[e];
            P.kopp[2 * o] = M.uk_opp[2 * e];
            P.kopp[2 * o + 1] = M.uk_opp[2 * e + 1];
        }
    }
    return FEMI_OK;
}

static void fill_info(const BandPlan& P, femi_band_info* info) {
    std::memset(info, 0, sizeof(*info));
    info->nranks = P.nranks;
    info->rank = P.rank;
    info->n_unknown = P.n_u;
    info->row0 = P.row0;
    info->row1 = P.row1;
    info->n_halo = (int64_t)P.halo.size();
    info->n_send = (int64_t)P.send_row.size();
    info->nnz_uu = (int64_t)P.col.size();
    info->nnz_uk = (int64_t)P.kcol.size();
    info->n_peers = (int32_t)P.peer.size();
}

// ---------------------------------------------------------------- device
namespace {
constexpr int BNT = 256;  // threads per CTA
constexpr int BRED = 296; // CTAs of the reduction kernels (fixed: deterministic partial order)

struct BandState {     // double-buffered by iteration parity
    double gamma, alpha, tol2;
    int32_t done, iters;
};

__device__ __forceinline__ double half_cot_b(int W, int32_t pi, int32_t pj, int32_t po) {
    // the same arithmetic as assemble.cu (reading A6): exact integer dot / |cross|, one division
    long long xi = pi % W, yi = pi / W, xj = pj % W, yj = pj / W, xo = po % W, yo = po / W;
    long long dot = (xi - xo) * (xj - xo) + (yi - yo) * (yj - yo);
    long long cross = (xi - xo) * (yj - yo) - (yi - yo) * (xj - xo);
    if (cross < 0) cross = -cross;
    return -0.5 * ((double)dot / (double)cross);
}

// values of the band's rows: off-diagonals as assemble.cu, the diagonal = -(sum of the A_uu
// off-diagonals by ascending column, then the A_uk entries by ascending column); dinv = 1/diag
__global__ void k_band_assemble(int64_t nloc, int64_t row0, int W, const int32_t* __restrict__ vpix, int64_t n_u,
                                const int32_t* __restrict__ rp, const int32_t* __restrict__ gcol,
                                const int32_t* __restrict__ opp, double* __restrict__ val,
                                const int32_t* __restrict__ krp, const int32_t* __restrict__ kcol,
                                const int32_t* __restrict__ kopp, double* __restrict__ kval,
                                double* __restrict__ dinv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t gi = row0 + i;
        const int32_t pi = vpix[gi];
        double acc = 0.0;
        int32_t dpos = -1;
        for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
            const int32_t j = gcol[e];
            if (j == gi) {
                dpos = e;
                continue;
            }
            const int32_t o1 = opp[2 * e], o2 = opp[2 * e + 1];
            double v = half_cot_b(W, pi, vpix[j], vpix[o1]);
            if (o2 >= 0) v = v + half_cot_b(W, pi, vpix[j], vpix[o2]);
            val[e] = v;
            acc = acc + v;
        }
        for (int32_t e = krp[i]; e < krp[i + 1]; ++e) {
            const int32_t pj = vpix[n_u + kcol[e]];
            const int32_t o1 = kopp[2 * e], o2 = kopp[2 * e + 1];
            double v = half_cot_b(W, pi, pj, vpix[o1]);
            if (o2 >= 0) v = v + half_cot_b(W, pi, pj, vpix[o2]);
            kval[e] = v;
            acc = acc + v;
        }
        FEMI_DCHECK(dpos >= 0, 7);
        val[dpos] = -acc;
        dinv[i] = 1.0 / -acc;
    }
}

// fixed-order reduction of per-CTA partials (NQ values per CTA) into out[0..NQ)
template <int NQ>
__device__ __forceinline__ void cta_partials(double (&v)[NQ], double* part) {
    __shared__ double sh[BNT / 32];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const double t = block_sum<BNT>(v[q], sh);
        if (threadIdx.x == 0) part[NQ * blockIdx.x + q] = t;
    }
}
// save3 (optional): out[3] is copied there before it is overwritten (the all-reduced ||b||^2 of
// begin, captured by the first SpMV)
template <int NQ>
__global__ void k_band_sum(const double* __restrict__ part, int nb, double* __restrict__ out, int nout,
                           double* __restrict__ save3 = nullptr) {
    __shared__ double sh[BNT / 32];
    if (save3 && threadIdx.x == 0) *save3 = out[3];
    __syncthreads();
    for (int q = 0; q < nout; ++q) {
        double t = 0.0;
        for (int b = threadIdx.x; b < nb; b += BNT) t += q < NQ ? part[NQ * b + q] : 0.0;
        t = block_sum<BNT>(t, sh);
        if (threadIdx.x == 0) out[q] = t;
    }
}

// min / max of g (every rank holds all mask values): midrange for x^0
__global__ void k_band_minmax(int64_t m, const double* __restrict__ g, double* __restrict__ part) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t k = blockIdx.x * (int64_t)BNT + threadIdx.x; k < m; k += (int64_t)gridDim.x * BNT) {
        lo = fmin(lo, g[k]);
        hi = fmax(hi, g[k]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ double sl[BNT / 32], shh[BNT / 32];
    if (lane == 0) {
        sl[wid] = lo;
        shh[wid] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 0; w < BNT / 32; ++w) {
            lo = fmin(lo, sl[w]);
            hi = fmax(hi, shh[w]);
        }
        part[2 * blockIdx.x] = lo;
        part[2 * blockIdx.x + 1] = hi;
    }
}

// prologue: c = midrange(g); b = -A_uk g, r = -A_uk (g - c 1) (= b - A_uu c 1), x = c, u = M^-1 r,
// p = s = 0; partial ||b||^2 -> dots[3] (dots[0..2] = 0)
__global__ void k_band_begin(int64_t nloc, const int32_t* __restrict__ krp, const int32_t* __restrict__ kcol,
                             const double* __restrict__ kval, const double* __restrict__ g,
                             const double* __restrict__ mm, int nbm, const double* __restrict__ dinv,
                             double* __restrict__ b, double* __restrict__ x, double* __restrict__ r,
                             double* __restrict__ u, double* __restrict__ p, double* __restrict__ s,
                             double* __restrict__ part) {
    double lo = INFINITY, hi = -INFINITY;
    for (int k = 0; k < nbm; ++k) {
        lo = fmin(lo, mm[2 * k]);
        hi = fmax(hi, mm[2 * k + 1]);
    }
    const double c = 0.5 * (lo + hi);
    double v[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)BNT + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * BNT) {
        double acc = 0.0, accr = 0.0;
        for (int32_t e = krp[i]; e < krp[i + 1]; ++e) {
            const double a = kval[e], gk = g[kcol[e]];
            acc = fma(a, gk, acc);
            accr = fma(a, gk - c, accr);
        }
        const double bi = -acc, ri = -accr;
        b[i] = bi;
        x[i] = c;
        r[i] = ri;
        u[i] = dinv[i] * ri;
        p[i] = 0.0;
        s[i] = 0.0;
        v[0] += bi * bi;
    }
    cta_partials<1>(v, part);
}

__global__ void k_band_pack(int64_t nsend, const int32_t* __restrict__ row, const double* __restrict__ src,
                            double* __restrict__ send) {
    for (int64_t k = blockIdx.x * (int64_t)BNT + threadIdx.x; k < nsend; k += (int64_t)gridDim.x * BNT)
        send[k] = src[row[k]];
}

// WHICH 0: w = A u, partials (r.u, w.u, r.r). WHICH 1: r = b - A x (true residual, unscaled rows),
// partials (0, 0, r.r).
template <int WHICH>
__global__ void k_band_spmv(int64_t nloc, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const double* __restrict__ val, const double* __restrict__ src,
                            const double* __restrict__ halo, const double* __restrict__ b,
                            double* __restrict__ r, const double* __restrict__ u, double* __restrict__ w,
                            double* __restrict__ part) {
    double v[3] = {0.0, 0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)BNT + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * BNT) {
        double ax = 0.0;
        for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
            const int32_t c = col[e];
            ax = fma(val[e], c < nloc ? src[c] : halo[c - nloc], ax);
        }
        if (WHICH == 0) {
            w[i] = ax;
            const double ri = r[i], ui = u[i];
            v[0] += ri * ui;
            v[1] += ax * ui;
            v[2] += ri * ri;
        } else {
            const double ri = b[i] - ax;
            r[i] = ri;
            v[2] += ri * ri;
        }
    }
    cta_partials<3>(v, part);
}

// one CG update from the all-reduced dots (gamma, delta, rho[, ||b||^2 on the first update]);
// state double-buffered by iteration parity k
__global__ void k_band_update(int64_t nloc, int k, double rtol, const double* __restrict__ dots,
                              const double* __restrict__ bb_slot, BandState* __restrict__ st,
                              const double* __restrict__ dinv, double* __restrict__ x, double* __restrict__ r,
                              double* __restrict__ u, double* __restrict__ p, double* __restrict__ s,
                              const double* __restrict__ w) {
    const double gamma = dots[0], delta = dots[1], rho = dots[2];
    const double bb = *bb_slot;
    const double tol2 = rtol * rtol * bb;
    const BandState prev = st[k & 1];
    BandState nx = prev;
    nx.tol2 = tol2;
    bool skip = k > 0 && prev.done;
    double alpha = 0.0, beta = 0.0;
    if (!skip) {
        if (rho <= tol2 || bb == 0.0) {
            nx.done = 1;
            skip = true;
        } else if (k == 0) {
            alpha = gamma / delta;
            nx.done = 0;
        } else {
            beta = gamma / prev.gamma;
            alpha = gamma / (delta - beta * gamma / prev.alpha);
        }
    }
    if (!skip) {
        nx.gamma = gamma;
        nx.alpha = alpha;
        nx.iters = prev.iters + 1;  // continues across restarts (the restart keeps the slot's count)
        for (int64_t i = blockIdx.x * (int64_t)BNT + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * BNT) {
            const double pi = fma(beta, p[i], u[i]);
            const double si = fma(beta, s[i], w[i]);
            p[i] = pi;
            s[i] = si;
            x[i] = fma(alpha, pi, x[i]);
            const double ri = fma(-alpha, si, r[i]);
            r[i] = ri;
            u[i] = dinv[i] * ri;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) st[(k + 1) & 1] = nx;
}

// restart from r (= b - A x after the true-residual SpMV): u = M^-1 r, p = s = 0
__global__ void k_band_restart(int64_t nloc, const double* __restrict__ dinv, const double* __restrict__ r,
                               double* __restrict__ u, double* __restrict__ p, double* __restrict__ s) {
    for (int64_t i = blockIdx.x * (int64_t)BNT + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * BNT) {
        u[i] = dinv[i] * r[i];
        p[i] = 0.0;
        s[i] = 0.0;
    }
}

int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + BNT - 1) / BNT, 148 * 8)); }
}  // namespace
}  // namespace femi

using namespace femi;

struct femi_band_s {
    BandPlan P;
    int32_t W = 0;
    int64_t m = 0;
    // device (library-owned)
    std::vector<void*> allocs;
    int32_t *vpix = nullptr, *rp = nullptr, *col = nullptr, *gcol = nullptr, *opp = nullptr;
    int32_t *krp = nullptr, *kcol = nullptr, *kopp = nullptr, *send_row = nullptr;
    double *val = nullptr, *kval = nullptr, *dinv = nullptr;
    double *b = nullptr, *x = nullptr, *r = nullptr, *u = nullptr, *p = nullptr, *s = nullptr, *w = nullptr;
    double *part = nullptr, *bb = nullptr;
    BandState* st = nullptr;
    // caller-owned communication buffers
    double *halo = nullptr, *send = nullptr, *dots = nullptr;
    // host sequencing
    int k = 0;
    bool bb_pending = false;  // the next SpMV captures the all-reduced ||b||^2 from dots[3]
    double rtol = 1e-10;
};

namespace {
template <class T>
femi_status band_upload(femi_band_s* B, T** dst, const std::vector<T>& src, cudaStream_t st) {
    void* p = nullptr;
    FEMI_CUDA(cudaMallocAsync(&p, sizeof(T) * std::max<size_t>(src.size(), 1), st));
    B->allocs.push_back(p);
    if (!src.empty()) FEMI_CUDA(cudaMemcpyAsync(p, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, st));
    *dst = (T*)p;
    return FEMI_OK;
}
template <class T>
femi_status band_alloc(femi_band_s* B, T** dst, size_t n, cudaStream_t st) {
    void* p = nullptr;
    FEMI_CUDA(cudaMallocAsync(&p, sizeof(T) * std::max<size_t>(n, 1), st));
    B->allocs.push_back(p);
    *dst = (T*)p;
    return FEMI_OK;
}
femi_status need_buffers(const femi_band_s* B, const char* what) {
    if ((B->P.halo.size() && !B->halo) || (B->P.send_row.size() && !B->send) || !B->dots) {
        set_error(std::string(what) + ": communication buffers not set (femi_band_set_buffers)");
        return FEMI_E_ARG;
    }
    return FEMI_OK;
}
}  // namespace

extern "C" {

femi_status femi_band_plan(femi_mesh mesh, int32_t nranks, int32_t rank, femi_band_info* info) {
    if (!mesh || !info) {
        set_error("band_plan: NULL argument");
        return FEMI_E_ARG;
    }
    BandPlan P;
    femi_status s = build_band_plan(mesh->mesh, nranks, rank, P);
    if (s) return s;
    fill_info(P, info);
    return FEMI_OK;
}

femi_status femi_band_plan_export(femi_mesh mesh, int32_t nranks, int32_t rank, int32_t* peer, int64_t* recv_off,
                                  int64_t* send_off, int64_t* halo_id, int32_t* send_row, int32_t* rowptr,
                                  int32_t* col) {
    if (!mesh) {
        set_error("band_plan_export: NULL mesh");
        return FEMI_E_ARG;
    }
    BandPlan P;
    femi_status s = build_band_plan(mesh->mesh, nranks, rank, P);
    if (s) return s;
    if (peer) std::copy(P.peer.begin(), P.peer.end(), peer);
    if (recv_off) std::copy(P.recv_off.begin(), P.recv_off.end(), recv_off);
    if (send_off) std::copy(P.send_off.begin(), P.send_off.end(), send_off);
    if (halo_id) std::copy(P.halo.begin(), P.halo.end(), halo_id);
    if (send_row) std::copy(P.send_row.begin(), P.send_row.end(), send_row);
    if (rowptr) std::copy(P.rp.begin(), P.rp.end(), rowptr);
    if (col) std::copy(P.col.begin(), P.col.end(), col);
    return FEMI_OK;
}

femi_status femi_band_create(femi_mesh mesh, int32_t nranks, int32_t rank, femi_stream stream, femi_band* out) {
    if (!mesh || !out) {
        set_error("band_create: NULL argument");
        return FEMI_E_ARG;
    }
    *out = nullptr;
    cudaStream_t st = (cudaStream_t)stream;
    femi_band_s* B = new (std::nothrow) femi_band_s();
    if (!B) return FEMI_E_OOM;
    const Mesh& M = mesh->mesh;
    femi_status s = build_band_plan(M, nranks, rank, B->P);
    const BandPlan& P = B->P;
    B->W = M.W;
    B->m = M.m;
#define U(x)                         \
    do {                             \
        s = (x);                     \
        if (s != FEMI_OK) goto fail; \
    } while (0)
    if (s) goto fail;
    U(band_upload(B, &B->vpix, M.vpix, st));
    U(band_upload(B, &B->rp, P.rp, st));
    U(band_upload(B, &B->col, P.col, st));
    U(band_upload(B, &B->gcol, P.gcol, st));
    U(band_upload(B, &B->opp, P.opp, st));
    U(band_upload(B, &B->krp, P.krp, st));
    U(band_upload(B, &B->kcol, P.kcol, st));
    U(band_upload(B, &B->kopp, P.kopp, st));
    U(band_upload(B, &B->send_row, P.send_row, st));
    U(band_alloc(B, &B->val, P.col.size(), st));
    U(band_alloc(B, &B->kval, P.kcol.size(), st));
    U(band_alloc(B, &B->dinv, P.nloc, st));
    for (double** v : {&B->b, &B->x, &B->r, &B->u, &B->p, &B->s, &B->w}) U(band_alloc(B, v, P.nloc, st));
    U(band_alloc(B, &B->part, 4 * (size_t)BRED, st));
    U(band_alloc(B, &B->bb, 1, st));
    {
        void* q = nullptr;
        FEMI_CUDA(cudaMallocAsync(&q, 2 * sizeof(BandState), st));
        B->allocs.push_back(q);
        B->st = (BandState*)q;
        FEMI_CUDA(cudaMemsetAsync(q, 0, 2 * sizeof(BandState), st));
    }
    if (P.nloc > 0) {
        k_band_assemble<<<grid_of(P.nloc), BNT, 0, st>>>(P.nloc, P.row0, M.W, B->vpix, M.n_u, B->rp, B->gcol, B->opp,
                                                         B->val, B->krp, B->kcol, B->kopp, B->kval, B->dinv);
        count_launches(1);
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) {
        s = cuda_fail(cudaGetLastError(), "band_create");
        goto fail;
    }
#undef U
    *out = B;
    return FEMI_OK;
fail:
    femi_band_free(B);
    return s;
}

femi_status femi_band_info_get(femi_band band, femi_band_info* info) {
    if (!band || !info) return FEMI_E_ARG;
    fill_info(band->P, info);
    return FEMI_OK;
}

femi_status femi_band_set_buffers(femi_band band, double* halo, double* send, double* dots) {
    if (!band || !dots || (band->P.halo.size() && !halo) || (band->P.send_row.size() && !send)) {
        set_error("band_set_buffers: NULL buffer");
        return FEMI_E_ARG;
    }
    band->halo = halo;
    band->send = send;
    band->dots = dots;
    return FEMI_OK;
}

femi_status femi_band_begin(femi_band B, const double* g, double rtol, femi_stream stream) {
    if (!B || (B->m > 0 && !g) || !(rtol > 0.0)) {
        set_error("band_begin: NULL argument or rtol <= 0");
        return FEMI_E_ARG;
    }
    femi_status s = need_buffers(B, "band_begin");
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nloc = B->P.nloc;
    const int nbm = (int)std::max<int64_t>(1, std::min<int64_t>((B->m + BNT - 1) / BNT, BRED));
    k_band_minmax<<<nbm, BNT, 0, st>>>(B->m, g, B->part + 2 * BRED);
    k_band_begin<<<BRED, BNT, 0, st>>>(nloc, B->krp, B->kcol, B->kval, g, B->part + 2 * BRED, nbm, B->dinv, B->b, B->x,
                                       B->r, B->u, B->p, B->s, B->part);
    // dots = (0, 0, 0, ||b||^2 of the band); a fresh recurrence state (iteration count 0)
    FEMI_CUDA(cudaMemsetAsync(B->dots, 0, 3 * sizeof(double), st));
    FEMI_CUDA(cudaMemsetAsync(B->st, 0, 2 * sizeof(BandState), st));
    k_band_sum<1><<<1, BNT, 0, st>>>(B->part, BRED, B->dots + 3, 1);
    count_launches(3);
    FEMI_CUDA(cudaGetLastError());
    B->k = 0;
    B->bb_pending = true;
    B->rtol = rtol;
    return FEMI_OK;
}

femi_status femi_band_pack(femi_band B, int32_t which, femi_stream stream) {
    if (!B || which < 0 || which > 1) return FEMI_E_ARG;
    femi_status s = need_buffers(B, "band_pack");
    if (s) return s;
    const int64_t ns = (int64_t)B->P.send_row.size();
    if (ns == 0) return FEMI_OK;
    k_band_pack<<<grid_of(ns), BNT, 0, (cudaStream_t)stream>>>(ns, B->send_row, which ? B->x : B->u, B->send);
    count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    return FEMI_OK;
}

femi_status femi_band_spmv(femi_band B, int32_t which, femi_stream stream) {
    if (!B || which < 0 || which > 1) return FEMI_E_ARG;
    femi_status s = need_buffers(B, "band_spmv");
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nloc = B->P.nloc;
    if (which == 0)
        k_band_spmv<0><<<BRED, BNT, 0, st>>>(nloc, B->rp, B->col, B->val, B->u, B->halo, B->b, B->r, B->u, B->w,
                                             B->part);
    else
        k_band_spmv<1><<<BRED, BNT, 0, st>>>(nloc, B->rp, B->col, B->val, B->x, B->halo, B->b, B->r, B->u, B->w,
                                             B->part);
    k_band_sum<3><<<1, BNT, 0, st>>>(B->part, BRED, B->dots, 4, B->bb_pending ? B->bb : nullptr);  // dots[3] = 0
    B->bb_pending = false;
    count_launches(2);
    FEMI_CUDA(cudaGetLastError());
    return FEMI_OK;
}

femi_status femi_band_update(femi_band B, femi_stream stream) {
    if (!B) return FEMI_E_ARG;
    femi_status s = need_buffers(B, "band_update");
    if (s) return s;
    k_band_update<<<grid_of(B->P.nloc), BNT, 0, (cudaStream_t)stream>>>(
        B->P.nloc, B->k, B->rtol, B->dots, B->bb, B->st, B->dinv, B->x, B->r, B->u, B->p, B->s, B->w);
    count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    ++B->k;
    return FEMI_OK;
}

femi_status femi_band_restart(femi_band B, femi_stream stream) {
    if (!B) return FEMI_E_ARG;
    if (B->P.nloc > 0) {
        k_band_restart<<<grid_of(B->P.nloc), BNT, 0, (cudaStream_t)stream>>>(B->P.nloc, B->dinv, B->r, B->u, B->p,
                                                                            B->s);
        count_launches(1);
        FEMI_CUDA(cudaGetLastError());
    }
    // a fresh recurrence: the iteration count continues, the state slot of k = 0 keeps it
    BandState h[2] = {};
    FEMI_CUDA(cudaMemcpyAsync(h, B->st + (B->k & 1), sizeof(BandState), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    FEMI_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    h[0].done = 0;
    FEMI_CUDA(cudaMemcpyAsync(B->st, h, sizeof(BandState), cudaMemcpyHostToDevice, (cudaStream_t)stream));
    B->k = 0;
    return FEMI_OK;
}

femi_status femi_band_status(femi_band B, femi_stream stream, int32_t* done, int32_t* iters, double* dots4) {
    if (!B) return FEMI_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    BandState h = {};
    FEMI_CUDA(cudaMemcpyAsync(&h, B->st + (B->k & 1), sizeof(BandState), cudaMemcpyDeviceToHost, st));
    double d[4] = {0, 0, 0, 0};
    if (dots4 && B->dots) FEMI_CUDA(cudaMemcpyAsync(d, B->dots, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (dots4) FEMI_CUDA(cudaMemcpyAsync(d + 3, B->bb, sizeof(double), cudaMemcpyDeviceToHost, st));
    FEMI_CUDA(cudaStreamSynchronize(st));
    if (done) *done = h.done;
    if (iters) *iters = h.iters;
    if (dots4) std::memcpy(dots4, d, sizeof(d));
    return FEMI_OK;
}

femi_status femi_band_result(femi_band B, double* u_local, femi_stream stream) {
    if (!B || (B->P.nloc > 0 && !u_local)) return FEMI_E_ARG;
    if (B->P.nloc > 0)
        FEMI_CUDA(cudaMemcpyAsync(u_local, B->x, sizeof(double) * B->P.nloc, cudaMemcpyDeviceToDevice,
                                  (cudaStream_t)stream));
    return FEMI_OK;
}

femi_status femi_band_raster_system(femi_mesh mesh, int32_t nranks, int32_t rank, femi_stream stream,
                                    femi_system* out, femi_band_raster_info* info) {
    if (!mesh || !out || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error("band_raster_system: NULL argument or rank outside [0, nranks)");
        return FEMI_E_ARG;
    }
    *out = nullptr;
    const Mesh& M = mesh->mesh;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t T = M.T, t0 = T * rank / nranks, t1 = T * (rank + 1) / nranks;
    int64_t y0 = M.H, y1 = -1;
    for (int64_t q = 3 * t0; q < 3 * t1; ++q) {
        const int64_t y = M.vpix[M.tri[q]] / M.W;
        y0 = std::min(y0, y);
        y1 = std::max(y1, y);
    }
    if (t1 == t0) y0 = y1 = 0;
    femi_band_raster_info bi = {t0, t1, y0, y1 - y0 + 1};
    if (info) *info = bi;
    femi_system_s* S = new (std::nothrow) femi_system_s();
    if (!S) return FEMI_E_OOM;
    S->raster_only = true;
    S->ast = st;
    S->W = M.W;
    S->H = (int32_t)bi.rows;
    S->n_u = M.n_u;
    S->m = M.m;
    S->nv = M.nv;
    S->T = t1 - t0;
    femi_status s = FEMI_OK;
    int32_t* d_tri = nullptr;
    uint32_t* d_flags = nullptr;
    // vertex pixels shifted to the band's first row (meaningful for the band's vertices only);
    // the triangles keep their GLOBAL vertex ids, so the raster reads a global u_vert
    std::vector<int32_t> vsh(M.nv);
    for (int64_t v = 0; v < M.nv; ++v) vsh[v] = (int32_t)(M.vpix[v] - y0 * M.W);
    auto dalloc = [&](void** p, size_t bytes) -> femi_status {
        FEMI_CUDA(cudaMallocAsync(p, std::max<size_t>(bytes, 1), st));
        S->allocs.push_back(*p);
        return FEMI_OK;
    };
#define U(x)                         \
    do {                             \
        s = (x);                     \
        if (s != FEMI_OK) goto fail; \
    } while (0)
    U(dalloc((void**)&S->vpix, sizeof(int32_t) * vsh.size()));
    U(dalloc((void**)&d_tri, sizeof(int32_t) * 3 * (size_t)S->T));
    U(dalloc((void**)&d_flags, sizeof(uint32_t) * (size_t)S->T));
    U(dalloc((void**)&S->tri, sizeof(TriRec) * (size_t)S->T));
    U(dalloc((void**)&S->tp_ptr, sizeof(int32_t) * ((size_t)S->T + 1)));
    U(dalloc((void**)&S->tp_pix, sizeof(uint32_t) * (size_t)M.W * (size_t)S->H));
    FEMI_CUDA(cudaMemcpyAsync(S->vpix, vsh.data(), sizeof(int32_t) * vsh.size(), cudaMemcpyHostToDevice, st));
    if (S->T > 0) {
        FEMI_CUDA(cudaMemcpyAsync(d_tri, M.tri.data() + 3 * t0, sizeof(int32_t) * 3 * S->T, cudaMemcpyHostToDevice,
                                  st));
        FEMI_CUDA(cudaMemcpyAsync(d_flags, M.flags.data() + t0, sizeof(uint32_t) * S->T, cudaMemcpyHostToDevice, st));
    }
    U(launch_tri_records(S, d_tri, d_flags, st));
    U(build_owner_tables(S, st));
    if (cudaStreamSynchronize(st) != cudaSuccess) {
        s = cuda_fail(cudaGetLastError(), "band_raster_system");
        goto fail;
    }
#undef U
    *out = S;
    return FEMI_OK;
fail:
    femi_system_free(S);
    return s;
}

void femi_band_free(femi_band B) {
    if (!B) return;
    for (void* p : B->allocs) cudaFree(p);
    delete B;
}

}  // extern "C"

FEMI_DCHECK_READER(dcheck_band)
