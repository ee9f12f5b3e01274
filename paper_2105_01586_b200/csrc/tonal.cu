// tonal.cu -- S6 tonal optimisation by nested CG (Eqs. (4)-(5)).
//
// g* = argmin ||B g - f||^2 with B g = P_k g + P_u A_uu^-1 (-A_uk g) (the dense B is never
// formed). CG on the normal equations B^T B g = B^T f in CGLS form;
// every outer iteration applies B once (inner inpainting solve + forward raster) and B^T
// once (adjoint raster + inner solve + A_uk^T product), strictly in sequence
// (reading A13). Vectors stay on the device; the host only sees the outer scalars.
//   B^T r = P_k^T r - A_uk^T A_uu^-1 (P_u^T r)
// P^T r is a per-triangle adjoint raster (warp per triangle, the same ownership rule as
// the forward raster) producing three partial sums per triangle, gathered per vertex over
// the vertex->triangle incidence list in ascending triangle order (deterministic).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "device.cuh"

namespace femi {
namespace {

constexpr int TT = 256;

__global__ void k_vertex_gather(int64_t nv, const int32_t* __restrict__ vt_ptr, const int32_t* __restrict__ vt_idx,
                                const double* __restrict__ tri_w, double* __restrict__ w) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int32_t q = vt_ptr[v]; q < vt_ptr[v + 1]; ++q) s += tri_w[vt_idx[q]];
        w[v] = s;
    }
}

// s_k = w_mask[k] - sum_i A_uk[i,k] y_i  (A_uk^T via the transpose index)
__global__ void k_ku(int64_t m, int64_t n_u, const int32_t* __restrict__ krp, const int32_t* __restrict__ src,
                     const int32_t* __restrict__ row, const double* __restrict__ uk_val, const double* __restrict__ w,
                     const double* __restrict__ y, double* __restrict__ s) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
        double acc = w[n_u + k];
        for (int32_t q = krp[k]; q < krp[k + 1]; ++q) {
            FEMI_DCHECK(row[q] >= 0 && row[q] < n_u && src[q] >= 0, 6);
            acc -= uk_val[src[q]] * y[row[q]];
        }
        s[k] = acc;
    }
}

__global__ void k_dot_part(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ part) {
    __shared__ double red[TT / 32];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)TT + threadIdx.x; i < n; i += (int64_t)gridDim.x * TT) s += a[i] * b[i];
    s = block_sum<TT>(s, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_dot_final(int nb, const double* __restrict__ part, double* __restrict__ out) {
    __shared__ double red[TT / 32];
    double s = 0.0;
    for (int k = threadIdx.x; k < nb; k += TT) s += part[k];
    s = block_sum<TT>(s, red);
    if (threadIdx.x == 0) *out = s;
}

// y += sign (num / den) x with the quotient formed on the device (no host round trip); a
// non-positive den leaves y unchanged (the host sees it at its next synchronisation and stops)
__global__ void k_axpy_q(int64_t n, const double* __restrict__ num, const double* __restrict__ den, double sign,
                         const double* __restrict__ x, double* __restrict__ y) {
    const double d = *den;
    if (!(d > 0.0)) return;
    const double alpha = sign * (*num / d);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = fma(alpha, x[i], y[i]);
}
// y = x + (num / den) y with the quotient formed on the device (the same IEEE quotient the host
// formed before): enqueued before the host has seen the new dot, so no host round trip sits
// between an outer iteration's adjoint solve and the next forward solve
__global__ void k_xpby_q(int64_t n, const double* __restrict__ x, const double* __restrict__ num,
                         const double* __restrict__ den, double* __restrict__ y) {
    const double beta = *num / *den;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = fma(beta, y[i], x[i]);
}
__global__ void k_xpby(int64_t n, const double* __restrict__ x, double beta, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = fma(beta, y[i], x[i]);
}
__global__ void k_sub(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a[i] - b[i];
}
// out = a x (the IRLS sqrt weights applied to a pixel vector; out may alias x)
__global__ void k_mul(int64_t n, const double* __restrict__ a, const double* x, double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a[i] * x[i];
}
// out = a (a x) (the weighted right-hand side W f, as the oracle rounds it)
__global__ void k_mul_aax(int64_t n, const double* __restrict__ a, const double* __restrict__ x, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a[i] * (a[i] * x[i]);
}
// out = (a a) x (the weighted gradient at exit)
__global__ void k_mul_a2x(int64_t n, const double* __restrict__ a, const double* __restrict__ x, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (a[i] * a[i]) * x[i];
}
// IRLS: sqrt weights 1/sqrt(max(|f - u|, eps)) and the partial sums of |f - u| (L1 error)
__global__ void k_irls_weights(int64_t n, const double* __restrict__ f, const double* __restrict__ u, double eps,
                               double* __restrict__ sw, double* __restrict__ part) {
    __shared__ double red[TT / 32];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)TT + threadIdx.x; i < n; i += (int64_t)gridDim.x * TT) {
        const double a = fabs(f[i] - u[i]);
        s += a;
        if (sw) sw[i] = 1.0 / sqrt(a > eps ? a : eps);
    }
    s = block_sum<TT>(s, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + TT - 1) / TT, 148 * 8)); }

struct Tonal {
    femi_system_s* S;
    cudaStream_t st;
    femi_cg_opts inner;
    double* uv;     // nv
    double* yv;     // nv
    double* w;      // nv
    double* tri_w;  // 3T
    double* part;   // dot partials
    double* dres;   // dot result
    DevStats* ds = nullptr;  // non-null: asynchronous inner solves (tonal_cgls), statistics on the device
    int64_t solves = 0, iters = 0;
    femi_status status = FEMI_OK;
    double t_solve = 0.0, t_dot = 0.0;  // FEMI_TONAL_PROF: host wall time in the inner solves / dots
    static double now() {
        return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    }

    // a.b into the device scalar `slot` (default dres); with `out` also to the host (one
    // synchronisation, which also brings back `also` -> `also_host` when given)
    femi_status dot(int64_t n, const double* a, const double* b, double* out, double* slot = nullptr,
                    const double* also = nullptr, double* also_host = nullptr) {
        const double t0 = now();
        struct Acc {
            double& t;
            double t0;
            ~Acc() { t += now() - t0; }
        } acc{t_dot, t0};
        const int nb = 296;
        double* dst = slot ? slot : dres;
        k_dot_part<<<nb, TT, 0, st>>>(n, a, b, part); count_launches(1);
        k_dot_final<<<1, TT, 0, st>>>(nb, part, dst); count_launches(1);
        FEMI_CUDA(cudaGetLastError());
        if (!out) return FEMI_OK;
        FEMI_CUDA(cudaMemcpyAsync(out, dst, sizeof(double), cudaMemcpyDeviceToHost, st));
        if (also) FEMI_CUDA(cudaMemcpyAsync(also_host, also, sizeof(double), cudaMemcpyDeviceToHost, st));
        FEMI_CUDA(cudaStreamSynchronize(st));
        return FEMI_OK;
    }

    void note(femi_status s) {
        if (s != FEMI_OK && status == FEMI_OK) status = s;
    }

    // u_px = B g
    femi_status apply_B(const double* g, double* u_px) {
        femi_cg_opts o = inner;
        o.x0 = 3;  // mask-neighbour fill (reading A11b)
        int32_t it = 0;
        double rr = 0.0;
        int64_t tot = 0;
        femi_system_s* Sv[1] = {S};
        const double* gv[1] = {g};
        double* uvv[1] = {uv};
        const double ts0 = now();
        femi_status s = pcg_solve(1, Sv, gv, nullptr, uvv, o, &it, &rr, st, &tot, ds);
        t_solve += now() - ts0;
        ++solves;
        iters += tot;
        if (s == FEMI_E_NONFINITE || s == FEMI_E_CUDA || s == FEMI_E_OOM) return s;
        note(s);
        const double* uvc[1] = {uv};
        double* pv[1] = {u_px};
        return launch_raster(1, Sv, uvc, nullptr, pv, nullptr, nullptr, nullptr, nullptr, st);
    }

    // s = B^T r
    femi_status apply_BT(const double* r, double* s_out) {
        femi_status ar = launch_adjoint_raster(S, r, tri_w, st);
        if (ar != FEMI_OK) return ar;
        k_vertex_gather<<<grid_for(S->nv), TT, 0, st>>>(S->nv, S->vt_ptr, S->vt_idx, tri_w, w); count_launches(1);
        FEMI_CUDA(cudaGetLastError());
        femi_cg_opts o = inner;
        o.x0 = 0;
        int32_t it = 0;
        double rr = 0.0;
        int64_t tot = 0;
        femi_system_s* Sv[1] = {S};
        const double* bv[1] = {w};
        double* yvv[1] = {yv};
        const double ts0 = now();
        femi_status s = pcg_solve(1, Sv, nullptr, bv, yvv, o, &it, &rr, st, &tot, ds);
        t_solve += now() - ts0;
        ++solves;
        iters += tot;
        if (s == FEMI_E_NONFINITE || s == FEMI_E_CUDA || s == FEMI_E_OOM) return s;
        note(s);
        k_ku<<<grid_for(S->m), TT, 0, st>>>(S->m, S->n_u, S->ku_rowptr, S->ku_src, S->ku_row, S->uk_val, w, yv,
                                            s_out); count_launches(1);
        FEMI_CUDA(cudaGetLastError());
        return FEMI_OK;
    }
};

}  // namespace

struct TonalReadback {
    double gam2, qq;
    DevStats ds;
};
// one pinned readback block per host thread, allocated on first use and kept (cudaMallocHost /
// cudaFreeHost per call cost more than the host round trips they save)
TonalReadback* tonal_readback() {
    struct Holder {
        TonalReadback* p = nullptr;
        ~Holder() {
            if (p) cudaFreeHost(p);
        }
    };
    thread_local Holder h;
    if (!h.p && cudaMallocHost(&h.p, sizeof(TonalReadback)) != cudaSuccess) {
        cudaGetLastError();
        h.p = nullptr;
    }
    return h.p;
}

femi_status tonal_cgls(femi_system_s* S, const double* f, double* g, const femi_tonal_opts& o,
                       femi_tonal_report* rep, cudaStream_t st, const double* sw) {
    const int64_t N = (int64_t)S->W * S->H, m = S->m, nv = S->nv, T = S->T;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t bytes = 3 * al(sizeof(double) * nv) + al(sizeof(double) * 3 * T) + al(sizeof(double) * 300) +
                   al(sizeof(double) * 4) + 3 * al(sizeof(double) * N) + 2 * al(sizeof(double) * m) +
                   al(sizeof(DevStats));
    void* base = nullptr;
    FEMI_CUDA(cudaMallocAsync(&base, bytes, st));
    char* cur = (char*)base;
    auto take = [&](size_t x) {
        char* p = cur;
        cur += al(x);
        return (double*)p;
    };
    Tonal tn;
    tn.S = S;
    tn.st = st;
    tn.inner = o.inner;
    tn.uv = take(sizeof(double) * nv);
    tn.yv = take(sizeof(double) * nv);
    tn.w = take(sizeof(double) * nv);
    tn.tri_w = take(sizeof(double) * 3 * T);
    tn.part = take(sizeof(double) * 300);
    tn.dres = take(sizeof(double) * 4);  // [0] scratch, [1] gam, [2] q.q
    double* u = take(sizeof(double) * N);
    double* r = take(sizeof(double) * N);
    double* q = take(sizeof(double) * N);
    double* s = take(sizeof(double) * m);
    double* p = take(sizeof(double) * m);
    // the inner solves run asynchronously (no host round trip per solve; restarts gated on the
    // device); the host synchronises once per outer iteration for the CGLS scalars
    tn.ds = (DevStats*)take(sizeof(DevStats));
    FEMI_CUDA(cudaMemsetAsync(tn.ds, 0, sizeof(DevStats), st));
    DevStats hds = {};
    TonalReadback* rb = nullptr;
    femi_status rc = FEMI_OK;
#define TRY(x)                      \
    do {                            \
        rc = (x);                   \
        if (rc != FEMI_OK) goto out; \
    } while (0)
    {
        double rr = 0, btf2 = 0, gam = 0, qq = 0, gam2 = 0;
        int outer = 0;
        // sw (IRLS sqrt weights, nullable): minimise || W^1/2 (B g - f) ||: B_w = diag(sw) B
        TRY(tn.apply_B(g, u));
        k_sub<<<grid_for(N), TT, 0, st>>>(N, f, u, r); count_launches(1);
        TRY(tn.dot(N, r, r, &rr));
        rep->mse_before = rr / (double)N;
        if (sw) {
            k_mul<<<grid_for(N), TT, 0, st>>>(N, sw, r, r);
            k_mul_aax<<<grid_for(N), TT, 0, st>>>(N, sw, f, u);  // B_w^T f_w = B^T (sw (sw f))
            count_launches(2);
            TRY(tn.apply_BT(u, s));
        } else {
            TRY(tn.apply_BT(f, s));
        }
        TRY(tn.dot(m, s, s, &btf2));
        const double btf = std::sqrt(btf2);
        if (sw) {
            k_mul<<<grid_for(N), TT, 0, st>>>(N, sw, r, u);
            count_launches(1);
            TRY(tn.apply_BT(u, s));
        } else {
            TRY(tn.apply_BT(r, s));
        }
        FEMI_CUDA(cudaMemcpyAsync(p, s, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
        // gam on the device in two slots by outer-iteration parity (alpha = gam / q.q and
        // beta = gam_new / gam are formed there)
        double* gslot[2] = {tn.dres + 1, tn.dres + 3};
        double* qq_d = tn.dres + 2;
        TRY(tn.dot(m, s, s, &gam, gslot[0]));
        double relg = btf > 0.0 ? std::sqrt(gam) / btf : 0.0;
        // pinned readback of (gam_new, q.q, the inner-solve statistics): one copy batch and one
        // synchronisation per outer iteration
        rb = tonal_readback();
        while (relg >= o.outer_rtol && outer < o.outer_max) {
            double* gam_d = gslot[outer & 1];
            double* gam_n = gslot[(outer + 1) & 1];
            TRY(tn.apply_B(p, q));
            if (sw) {
                k_mul<<<grid_for(N), TT, 0, st>>>(N, sw, q, q);
                count_launches(1);
            }
            TRY(tn.dot(N, q, q, nullptr, qq_d));  // no host round trip: alpha stays on the device
            k_axpy_q<<<grid_for(m), TT, 0, st>>>(m, gam_d, qq_d, 1.0, p, g); count_launches(1);
            k_axpy_q<<<grid_for(N), TT, 0, st>>>(N, gam_d, qq_d, -1.0, q, r); count_launches(1);
            if (sw) {
                k_mul<<<grid_for(N), TT, 0, st>>>(N, sw, r, u);
                count_launches(1);
                TRY(tn.apply_BT(u, s));
            } else {
                TRY(tn.apply_BT(r, s));
            }
            TRY(tn.dot(m, s, s, nullptr, gam_n));  // s.s: the next alpha's numerator
            // p = s + beta p before the host has looked (p is not read after the loop)
            k_xpby_q<<<grid_for(m), TT, 0, st>>>(m, s, gam_n, gam_d, p); count_launches(1);
            if (rb) {
                FEMI_CUDA(cudaMemcpyAsync(&rb->gam2, gam_n, sizeof(double), cudaMemcpyDeviceToHost, st));
                FEMI_CUDA(cudaMemcpyAsync(&rb->qq, qq_d, sizeof(double), cudaMemcpyDeviceToHost, st));
                FEMI_CUDA(cudaMemcpyAsync(&rb->ds, tn.ds, sizeof(DevStats), cudaMemcpyDeviceToHost, st));
                FEMI_CUDA(cudaStreamSynchronize(st));
                gam2 = rb->gam2;
                qq = rb->qq;
                hds = rb->ds;
            } else {
                FEMI_CUDA(cudaMemcpyAsync(&gam2, gam_n, sizeof(double), cudaMemcpyDeviceToHost, st));
                FEMI_CUDA(cudaMemcpyAsync(&qq, qq_d, sizeof(double), cudaMemcpyDeviceToHost, st));
                FEMI_CUDA(cudaMemcpyAsync(&hds, tn.ds, sizeof(DevStats), cudaMemcpyDeviceToHost, st));
                FEMI_CUDA(cudaStreamSynchronize(st));
            }
            if (hds.status == FEMI_E_NONFINITE || hds.status == FEMI_E_NEG_CURVATURE) {
                rc = (femi_status)hds.status;
                goto out;
            }
            if (!(qq > 0.0)) break;  // g and r were left unchanged (k_axpy_q)
            ++outer;
            relg = std::sqrt(gam2) / btf;
            if (!std::isfinite(relg)) {
                rc = FEMI_E_NONFINITE;
                goto out;
            }
            gam = gam2;
            if (relg < o.outer_rtol) break;
        }

        rep->rel_grad_recursive = relg;
        rep->outer_iters = outer;
        TRY(tn.apply_B(g, u));
        k_sub<<<grid_for(N), TT, 0, st>>>(N, f, u, r); count_launches(1);
        TRY(tn.dot(N, r, r, &rr));
        rep->mse_after = rr / (double)N;
        if (sw) {
            k_mul_a2x<<<grid_for(N), TT, 0, st>>>(N, sw, r, u);
            count_launches(1);
            TRY(tn.apply_BT(u, s));
        } else {
            TRY(tn.apply_BT(r, s));
        }
        TRY(tn.dot(m, s, s, &gam2));
        rep->rel_grad = btf > 0.0 ? std::sqrt(gam2) / btf : 0.0;
        if (relg >= o.outer_rtol && outer >= o.outer_max) tn.note(FEMI_E_NOT_CONVERGED);
    }
out:
#undef TRY
    if (std::getenv("FEMI_TONAL_PROF"))
        std::fprintf(stderr, "[femi tonal] solves %lld (%lld CG iterations): %.3f ms in pcg_solve, %.3f ms in dots\n",
                     (long long)tn.solves, (long long)tn.iters, 1e3 * tn.t_solve, 1e3 * tn.t_dot);
    if (cudaMemcpyAsync(&hds, tn.ds, sizeof(DevStats), cudaMemcpyDeviceToHost, st) == cudaSuccess &&
        cudaStreamSynchronize(st) == cudaSuccess) {
        tn.solves = hds.solves;
        tn.iters = (int64_t)hds.iters;
        tn.note((femi_status)hds.status);
    }
    rep->inner_solves = (int32_t)tn.solves;
    rep->inner_iters = tn.iters;
    cudaFreeAsync(base, st);
    if (rc != FEMI_OK) return rc;
    if (tn.status != FEMI_OK) set_error("tonal_optimise: an inner solve or the outer loop did not converge");
    return tn.status;
}

namespace {

// y += a x with a host scalar (the colour loop forms alpha / beta on the host from the
// synchronised per-channel dots: the same IEEE quotients as k_axpy_q / k_xpby)
__global__ void k_axpy_h(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = fma(a, x[i], y[i]);
}

}  // namespace

// Colour tonal optimisation (reading R4): C channels on
// one mesh are C independent CGLS problems (B is block-diagonal over the channels). They run in
// lockstep: every inner solve is ONE batched solve of the active channels' right-hand sides on
// the shared matrix (the multi-RHS graph loop streams the matrix once for all of them), the
// forward raster of all channels is one pass, and the host sees one synchronisation per dot
// round (all channels' scalars together). Each channel follows tonal_cgls's recurrence and
// stopping rule; a converged channel leaves the batch.
femi_status tonal_cgls_channels(femi_system_s* S, int C, const double* const* f, double* const* g,
                                const femi_tonal_opts& o, femi_tonal_report* rep, cudaStream_t st) {
    const int64_t N = (int64_t)S->W * S->H, m = S->m, nv = S->nv, T = S->T;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t per = 3 * al(sizeof(double) * nv) + 3 * al(sizeof(double) * N) + 2 * al(sizeof(double) * m) +
                       al(sizeof(double) * 8);
    size_t bytes = (size_t)C * per + al(sizeof(double) * 3 * std::max<int64_t>(T, 1)) + al(sizeof(double) * 300 * C);
    void* base = nullptr;
    FEMI_CUDA(cudaMallocAsync(&base, bytes, st));
    char* cur = (char*)base;
    auto take = [&](size_t x) {
        char* p = cur;
        cur += al(x);
        return (double*)p;
    };
    std::vector<double*> uv(C), yv(C), w(C), u(C), r(C), q(C), sv(C), p(C), dr(C);
    for (int c = 0; c < C; ++c) {
        uv[c] = take(sizeof(double) * nv);
        yv[c] = take(sizeof(double) * nv);
        w[c] = take(sizeof(double) * nv);
        u[c] = take(sizeof(double) * N);
        r[c] = take(sizeof(double) * N);
        q[c] = take(sizeof(double) * N);
        sv[c] = take(sizeof(double) * m);
        p[c] = take(sizeof(double) * m);
        dr[c] = take(sizeof(double) * 8);
    }
    double* tri_w = take(sizeof(double) * 3 * std::max<int64_t>(T, 1));
    double* part = take(sizeof(double) * 300 * C);
    int64_t solves = 0, inner_iters = 0;
    femi_status note = FEMI_OK;
    auto keep = [&](femi_status s2) {
        if (s2 != FEMI_OK && note == FEMI_OK) note = s2;
    };
    // inner solves of the listed channels, one batched call
    auto solve = [&](const std::vector<int>& ch, bool from_g, const std::vector<const double*>& in,
                     std::vector<double*>& out, int x0) -> femi_status {
        const int B = (int)ch.size();
        if (B == 0) return FEMI_OK;
        std::vector<femi_system_s*> Sv(B, S);
        std::vector<const double*> iv(B);
        std::vector<double*> ov(B);
        for (int b = 0; b < B; ++b) {
            iv[b] = in[ch[b]];
            ov[b] = out[ch[b]];
        }
        femi_cg_opts io = o.inner;
        io.x0 = x0;
        std::vector<int32_t> it(B);
        std::vector<double> rr(B);
        int64_t tot = 0;
        const femi_status s2 = pcg_solve(B, Sv.data(), from_g ? iv.data() : nullptr, from_g ? nullptr : iv.data(),
                                         ov.data(), io, it.data(), rr.data(), st, &tot);
        solves += B;
        inner_iters += tot;
        if (s2 == FEMI_E_NONFINITE || s2 == FEMI_E_CUDA || s2 == FEMI_E_OOM) return s2;
        keep(s2);
        return FEMI_OK;
    };
    // out[c] = B in[c] for the listed channels: one batched solve + one raster pass
    auto apply_B = [&](const std::vector<int>& ch, const std::vector<const double*>& in,
                       std::vector<double*>& out) -> femi_status {
        femi_status s2 = solve(ch, true, in, uv, 3);
        if (s2) return s2;
        const int B = (int)ch.size();
        std::vector<const double*> uvc(B);
        std::vector<double*> po(B);
        for (int b = 0; b < B; ++b) {
            uvc[b] = uv[ch[b]];
            po[b] = out[ch[b]];
        }
        for (int b0 = 0; b0 < B; b0 += 4) {  // raster-only pass, <= 4 channels at a time
            const int nb = std::min(4, B - b0);
            s2 = launch_raster_channels(S, nb, uvc.data() + b0, nullptr, po.data() + b0, nullptr, nullptr, nullptr,
                                        nullptr, st);
            if (s2) return s2;
        }
        return FEMI_OK;
    };
    // s[c] = B^T in[c]
    auto apply_BT = [&](const std::vector<int>& ch, const std::vector<const double*>& in,
                        std::vector<double*>& s_out) -> femi_status {
        for (int c : ch) {
            femi_status s2 = launch_adjoint_raster(S, in[c], tri_w, st);
            if (s2) return s2;
            k_vertex_gather<<<grid_for(nv), TT, 0, st>>>(nv, S->vt_ptr, S->vt_idx, tri_w, w[c]);
            count_launches(1);
        }
        std::vector<const double*> wc(C);
        for (int c = 0; c < C; ++c) wc[c] = w[c];
        femi_status s2 = solve(ch, false, wc, yv, 0);
        if (s2) return s2;
        for (int c : ch) {
            k_ku<<<grid_for(m), TT, 0, st>>>(m, S->n_u, S->ku_rowptr, S->ku_src, S->ku_row, S->uk_val, w[c], yv[c],
                                            s_out[c]);
            count_launches(1);
        }
        FEMI_CUDA(cudaGetLastError());
        return FEMI_OK;
    };
    // host[c] = a[c] . b[c] for the listed channels, one synchronisation
    auto dots = [&](const std::vector<int>& ch, int64_t n, const std::vector<double*>& a, const std::vector<double*>& b,
                    std::vector<double>& host) -> femi_status {
        const int nb = 296;
        for (int c : ch) {
            k_dot_part<<<nb, TT, 0, st>>>(n, a[c], b[c], part + 300 * c);
            k_dot_final<<<1, TT, 0, st>>>(nb, part + 300 * c, dr[c]);
            count_launches(2);
        }
        FEMI_CUDA(cudaGetLastError());
        for (int c : ch) FEMI_CUDA(cudaMemcpyAsync(&host[c], dr[c], sizeof(double), cudaMemcpyDeviceToHost, st));
        FEMI_CUDA(cudaStreamSynchronize(st));
        return FEMI_OK;
    };
    std::vector<int> all(C);
    for (int c = 0; c < C; ++c) all[c] = c;
    std::vector<const double*> gc(g, g + C), fc(f, f + C), pc(C), rc(C);
    for (int c = 0; c < C; ++c) {
        pc[c] = p[c];
        rc[c] = r[c];
    }
    std::vector<double> rr(C), btf2(C), gam(C), gam2(C), qq(C), relg(C);
    std::vector<int> outer(C, 0);
    femi_status rcode = FEMI_OK;
#define TRYC(x)                          \
    do {                                 \
        rcode = (x);                     \
        if (rcode != FEMI_OK) goto done; \
    } while (0)
    {
        TRYC(apply_B(all, gc, u));
        for (int c = 0; c < C; ++c) {
            k_sub<<<grid_for(N), TT, 0, st>>>(N, f[c], u[c], r[c]);
            count_launches(1);
        }
        TRYC(dots(all, N, r, r, rr));
        for (int c = 0; c < C; ++c) rep[c].mse_before = rr[c] / (double)N;
        TRYC(apply_BT(all, fc, sv));
        TRYC(dots(all, m, sv, sv, btf2));
        TRYC(apply_BT(all, rc, sv));
        for (int c = 0; c < C; ++c) FEMI_CUDA(cudaMemcpyAsync(p[c], sv[c], sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
        TRYC(dots(all, m, sv, sv, gam));
        std::vector<int> act;
        for (int c = 0; c < C; ++c) {
            relg[c] = btf2[c] > 0.0 ? std::sqrt(gam[c]) / std::sqrt(btf2[c]) : 0.0;
            if (relg[c] >= o.outer_rtol && o.outer_max > 0) act.push_back(c);
        }
        while (!act.empty()) {
            TRYC(apply_B(act, pc, q));
            TRYC(dots(act, N, q, q, qq));
            std::vector<int> go;
            for (int c : act)
                if (qq[c] > 0.0) go.push_back(c);
            for (int c : go) {
                const double alpha = gam[c] / qq[c];
                k_axpy_h<<<grid_for(m), TT, 0, st>>>(m, alpha, p[c], g[c]);
                k_axpy_h<<<grid_for(N), TT, 0, st>>>(N, -alpha, q[c], r[c]);
                count_launches(2);
            }
            TRYC(apply_BT(go, rc, sv));
            TRYC(dots(go, m, sv, sv, gam2));
            std::vector<int> next;
            for (int c : go) {
                ++outer[c];
                relg[c] = std::sqrt(gam2[c]) / std::sqrt(btf2[c]);
                if (!std::isfinite(relg[c])) {
                    rcode = FEMI_E_NONFINITE;
                    goto done;
                }
                if (relg[c] < o.outer_rtol) {
                    gam[c] = gam2[c];
                    continue;
                }
                if (outer[c] < o.outer_max) {
                    k_xpby<<<grid_for(m), TT, 0, st>>>(m, sv[c], gam2[c] / gam[c], p[c]);
                    count_launches(1);
                    next.push_back(c);
                }
                gam[c] = gam2[c];
            }
            act = next;
        }
        for (int c = 0; c < C; ++c) {
            rep[c].rel_grad_recursive = relg[c];
            rep[c].outer_iters = outer[c];
        }
        TRYC(apply_B(all, gc, u));
        for (int c = 0; c < C; ++c) {
            k_sub<<<grid_for(N), TT, 0, st>>>(N, f[c], u[c], r[c]);
            count_launches(1);
        }
        TRYC(dots(all, N, r, r, rr));
        for (int c = 0; c < C; ++c) rep[c].mse_after = rr[c] / (double)N;
        TRYC(apply_BT(all, rc, sv));
        TRYC(dots(all, m, sv, sv, gam2));
        for (int c = 0; c < C; ++c) {
            rep[c].rel_grad = btf2[c] > 0.0 ? std::sqrt(gam2[c]) / std::sqrt(btf2[c]) : 0.0;
            if (relg[c] >= o.outer_rtol && outer[c] >= o.outer_max) keep(FEMI_E_NOT_CONVERGED);
        }
    }
done:
#undef TRYC
    for (int c = 0; c < C; ++c) {
        rep[c].inner_solves = (int32_t)(solves / C);
        rep[c].inner_iters = inner_iters / C;
    }
    cudaFreeAsync(base, st);
    if (rcode != FEMI_OK) return rcode;
    if (note != FEMI_OK) set_error("tonal_optimise_channels: an inner solve or the outer loop did not converge");
    return note;
}

// The operator alone (femi_apply_B / femi_apply_BT): mode 0 out = B in (pixels), mode 1
// out = B^T in (mask values); one inner solve each, synchronised for its status.
femi_status tonal_apply(femi_system_s* S, int mode, const double* in, double* out, const femi_cg_opts& o,
                        cudaStream_t st) {
    const int64_t nv = S->nv, T = S->T;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    void* base = nullptr;
    FEMI_CUDA(cudaMallocAsync(&base, 3 * al(sizeof(double) * nv) + al(sizeof(double) * 3 * std::max<int64_t>(T, 1)) +
                                         al(sizeof(double) * 300) + al(sizeof(double) * 4),
                              st));
    char* cur = (char*)base;
    auto take = [&](size_t x) {
        char* p = cur;
        cur += al(x);
        return (double*)p;
    };
    Tonal tn;
    tn.S = S;
    tn.st = st;
    tn.inner = o;
    tn.uv = take(sizeof(double) * nv);
    tn.yv = take(sizeof(double) * nv);
    tn.w = take(sizeof(double) * nv);
    tn.tri_w = take(sizeof(double) * 3 * std::max<int64_t>(T, 1));
    tn.part = take(sizeof(double) * 300);
    tn.dres = take(sizeof(double) * 4);
    femi_status rc = mode == 0 ? tn.apply_B(in, out) : tn.apply_BT(in, out);
    if (rc == FEMI_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "apply: sync");
    cudaFreeAsync(base, st);
    if (rc != FEMI_OK) return rc;
    if (tn.status != FEMI_OK) set_error("apply: the inner solve did not converge");
    return tn.status;
}

// L1 tonal optimisation by IRLS (reading R3): `irls`
// reweightings, each computing r = f - B g, sqrt weights 1/sqrt(max(|r|, eps)) and a weighted
// CGLS from the current g; the L1 error mean|f - B g| is reported before and after.
femi_status tonal_irls(femi_system_s* S, const double* f, double* g, const femi_tonal_opts& o, int irls, double eps,
                       femi_tonal_l1_report* rep, cudaStream_t st) {
    const int64_t N = (int64_t)S->W * S->H, nv = S->nv;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    void* base = nullptr;
    FEMI_CUDA(cudaMallocAsync(&base, 2 * al(sizeof(double) * N) + al(sizeof(double) * nv) + al(sizeof(double) * 300),
                              st));
    double* u = (double*)base;
    double* sw = (double*)((char*)u + al(sizeof(double) * N));
    double* uv = (double*)((char*)sw + al(sizeof(double) * N));
    double* part = (double*)((char*)uv + al(sizeof(double) * nv));
    femi_status rc = FEMI_OK, note = FEMI_OK;
    *rep = femi_tonal_l1_report{};
    for (int k = 0; k <= irls; ++k) {
        // u = B g (one inner solve + raster)
        femi_cg_opts io = o.inner;
        io.x0 = 3;
        int32_t it = 0;
        double rr = 0.0;
        int64_t tot = 0;
        femi_system_s* Sv[1] = {S};
        const double* gv[1] = {g};
        double* uvv[1] = {uv};
        femi_status s1 = pcg_solve(1, Sv, gv, nullptr, uvv, io, &it, &rr, st, &tot);
        rep->inner_solves += 1;
        rep->inner_iters += tot;
        if (s1 == FEMI_E_NONFINITE || s1 == FEMI_E_CUDA || s1 == FEMI_E_OOM) {
            rc = s1;
            break;
        }
        if (s1 != FEMI_OK && note == FEMI_OK) note = s1;
        const double* uvc[1] = {uv};
        double* upx[1] = {u};
        if ((rc = launch_raster(1, Sv, uvc, nullptr, upx, nullptr, nullptr, nullptr, nullptr, st))) break;
        const int nb = 296;
        k_irls_weights<<<nb, TT, 0, st>>>(N, f, u, eps, k < irls ? sw : nullptr, part);
        count_launches(1);
        std::vector<double> hp(nb);
        if (cudaMemcpyAsync(hp.data(), part, sizeof(double) * nb, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            rc = cuda_fail(cudaGetLastError(), "tonal_l1: readback");
            break;
        }
        double l1 = 0.0;
        for (double v : hp) l1 += v;
        l1 /= (double)N;
        if (k == 0) rep->l1_before = l1;
        if (k == irls) {
            rep->l1_after = l1;
            break;
        }
        femi_tonal_report r2{};
        femi_status s2 = tonal_cgls(S, f, g, o, &r2, st, sw);
        if (k == 0) rep->mse_before = r2.mse_before;
        rep->mse_after = r2.mse_after;
        rep->irls_steps += 1;
        rep->outer_iters += r2.outer_iters;
        rep->inner_solves += r2.inner_solves;
        rep->inner_iters += r2.inner_iters;
        if (s2 == FEMI_E_NONFINITE || s2 == FEMI_E_CUDA || s2 == FEMI_E_OOM) {
            rc = s2;
            break;
        }
        if (s2 != FEMI_OK && note == FEMI_OK) note = s2;
    }
    cudaFreeAsync(base, st);
    if (rc != FEMI_OK) return rc;
    return note;
}

}  // namespace femi

FEMI_DCHECK_READER(dcheck_tonal)
