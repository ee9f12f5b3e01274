// assemble.cu -- S1: P1 stiffness assembly on the device.
//
// Edge-gather formulation (no atomics): every CSR entry (i,j) of A_uu / A_uk knows the
// (at most two) vertices opposite the mesh edge ij (host table from mesh_build), so one
// thread per unknown row computes its entries in place:
//   A_ij = c(o1) + c(o2),  c(o) = -1/2 * dot(p_i - p_o, p_j - p_o) / |cross(p_i - p_o, p_j - p_o)|
// with exact integer dot/cross and one rounded division (reading A6), then the diagonal
//   A_ii = -(sum of A_uu off-diagonals by ascending column, then A_uk by ascending column)
// i.e. zero row sums of the full matrix (natural Neumann border, Eq. (3)). The sum of the
// two contributions is commutative, so the values are bit-identical to any correct
// implementation that follows reading A6. A second pass builds the Jacobi-scaled solver
// matrix s_i a_ij s_j (off-diagonal only; s = diag^-1/2).
#include <functional>

#include "device.cuh"

namespace femi {
namespace {

__device__ __forceinline__ double half_cot(int W, int32_t pi, int32_t pj, int32_t po) {
    long long xi = pi % W, yi = pi / W, xj = pj % W, yj = pj / W, xo = po % W, yo = po / W;
    long long dot = (xi - xo) * (xj - xo) + (yi - yo) * (yj - yo);
    long long cross = (xi - xo) * (yj - yo) - (yi - yo) * (xj - xo);
    if (cross < 0) cross = -cross;
    return -0.5 * ((double)dot / (double)cross);
}

__global__ void k_tri_records(int64_t T, int W, const int32_t* __restrict__ tri, const uint32_t* __restrict__ flags,
                              const int32_t* __restrict__ vpix, TriRec* __restrict__ out) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
        TriRec R;
        for (int k = 0; k < 3; ++k) {
            int32_t v = tri[3 * t + k];
            int32_t p = vpix[v];
            R.v[k] = v;
            R.x[k] = (int16_t)(p % W);
            R.y[k] = (int16_t)(p / W);
        }
        R.flags = flags[t];
        R.pad = 0;
        out[t] = R;
    }
}

__global__ void k_assemble_rows(int64_t n_u, int W, const int32_t* __restrict__ vpix,
                                const int32_t* __restrict__ urp, const int32_t* __restrict__ uci,
                                const int32_t* __restrict__ uop, double* __restrict__ uval,
                                const int32_t* __restrict__ krp, const int32_t* __restrict__ kci,
                                const int32_t* __restrict__ kop, double* __restrict__ kval,
                                double* __restrict__ s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_u; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t pi = vpix[i];
        double acc = 0.0;
        int32_t dpos = -1;
        for (int32_t e = urp[i]; e < urp[i + 1]; ++e) {
            int32_t j = uci[e];
            if (j == i) {
                dpos = e;
                continue;
            }
            const int32_t pj = vpix[j];
            int32_t o1 = uop[2 * e], o2 = uop[2 * e + 1];
            FEMI_DCHECK(j >= 0 && j < n_u && o1 >= 0, 2);
            double v = half_cot(W, pi, pj, vpix[o1]);
            if (o2 >= 0) v = v + half_cot(W, pi, pj, vpix[o2]);
            uval[e] = v;
            acc = acc + v;
        }
        for (int32_t e = krp[i]; e < krp[i + 1]; ++e) {
            const int32_t pj = vpix[n_u + kci[e]];
            int32_t o1 = kop[2 * e], o2 = kop[2 * e + 1];
            double v = half_cot(W, pi, pj, vpix[o1]);
            if (o2 >= 0) v = v + half_cot(W, pi, pj, vpix[o2]);
            kval[e] = v;
            acc = acc + v;
        }
        const double d = -acc;
        uval[dpos] = d;
        s[i] = 1.0 / sqrt(d);
    }
}

__global__ void k_scaled_offdiag(int64_t n_u, const int32_t* __restrict__ urp, const int32_t* __restrict__ uci,
                                 const double* __restrict__ uval, const double* __restrict__ s,
                                 int32_t* __restrict__ orp, int32_t* __restrict__ oci, double* __restrict__ oval) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_u; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = urp[i] - (int32_t)i;  // one diagonal per earlier row
        orp[i] = b;
        if (i == n_u - 1) orp[n_u] = urp[n_u] - (int32_t)n_u;
        const double si = s[i];
        int32_t o = b;
        for (int32_t e = urp[i]; e < urp[i + 1]; ++e) {
            int32_t j = uci[e];
            if (j == i) continue;
            oci[o] = j;
            oval[o] = (uval[e] * si) * s[j];
            ++o;
        }
    }
}

__global__ void k_sell_values(int64_t ne, const int32_t* __restrict__ src, const double* __restrict__ oval,
                              double* __restrict__ sval) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t q = src[e];
        sval[e] = q >= 0 ? oval[q] : 0.0;
    }
}

__global__ void k_gather_s(int64_t n, int64_t npad, const int32_t* __restrict__ inv, const double* __restrict__ s,
                           double* __restrict__ s_int, double* __restrict__ q_int) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npad; i += (int64_t)gridDim.x * blockDim.x) {
        const double si = i < n ? s[inv[i]] : 1.0;  // padding rows: harmless finite values
        s_int[i] = si;
        q_int[i] = 1.0 / si;
    }
}

}  // namespace

femi_status launch_sell_values(femi_system_s* S, const int32_t* d_src, cudaStream_t st) {
    if (S->n_u == 0) return FEMI_OK;
    if (S->sell_nnz > 0) {
        int g = (int)std::min<int64_t>((S->sell_nnz + 255) / 256, 148 * 16);
        k_sell_values<<<g, 256, 0, st>>>(S->sell_nnz, d_src, S->o_val, S->sell_val);
        count_launches(1);
    }
    if (S->ukI_val) {
        const int64_t ne = S->nnz_uk;
        k_sell_values<<<(int)std::min<int64_t>((ne + 255) / 256, 148 * 16), 256, 0, st>>>(ne, S->ukI_src_tmp,
                                                                                          S->uk_val, S->ukI_val);
        count_launches(1);
    }
    if (S->uuI_val) {
        const int64_t ne = S->nnz_uu;
        k_sell_values<<<(int)std::min<int64_t>((ne + 255) / 256, 148 * 16), 256, 0, st>>>(ne, S->uuI_src_tmp,
                                                                                          S->uu_val, S->uuI_val);
        count_launches(1);
    }
    if (S->jds_nnz > 0) {
        int gj = (int)std::min<int64_t>((S->jds_nnz + 255) / 256, 148 * 16);
        k_sell_values<<<gj, 256, 0, st>>>(S->jds_nnz, S->jds_src_tmp, S->o_val, S->jds_val);
        count_launches(1);
    }
    int g = (int)std::min<int64_t>((S->n_u + 255) / 256, 148 * 16);
    const int64_t npad = (S->n_u + kJdsRows - 1) / kJdsRows * kJdsRows;
    k_gather_s<<<g, 256, 0, st>>>(S->n_u, npad, S->sell_inv, S->s, S->s_int, S->q_int);
    count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    return FEMI_OK;
}

femi_status launch_tri_records(femi_system_s* S, const int32_t* d_tri, const uint32_t* d_flags, cudaStream_t st) {
    if (S->T > 0) {
        int g = (int)std::min<int64_t>((S->T + 255) / 256, 148 * 16);
        k_tri_records<<<g, 256, 0, st>>>(S->T, S->W, d_tri, d_flags, S->vpix, S->tri); count_launches(1);
        FEMI_CUDA(cudaGetLastError());
    }
    return FEMI_OK;
}

femi_status launch_assemble_values(femi_system_s* S, cudaStream_t st) {
    if (S->n_u == 0) return FEMI_OK;
    int g = (int)std::min<int64_t>((S->n_u + 127) / 128, 148 * 32);
    k_assemble_rows<<<g, 128, 0, st>>>(S->n_u, S->W, S->vpix, S->uu_rowptr, S->uu_col, S->uu_opp, S->uu_val,
                                       S->uk_rowptr, S->uk_col, S->uk_opp, S->uk_val, S->s); count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    k_scaled_offdiag<<<g, 128, 0, st>>>(S->n_u, S->uu_rowptr, S->uu_col, S->uu_val, S->s, S->o_rowptr, S->o_col,
                                        S->o_val); count_launches(1);
    FEMI_CUDA(cudaGetLastError());
    return FEMI_OK;
}

// ---- solver layouts built on the device (S1, systems below graph-mode size; FEMI_SELL_HOST=1
// keeps the host construction): from the internal order pi (internal row -> canonical unknown)
// and the natural CSR patterns already on the device, the SELL-32-sigma slices of the scaled
// off-diagonal pattern (lengths, offsets, int16 / int32 columns in the internal numbering, the
// o_val source of every entry) and the internal-order copies of A_uu / A_uk rows -- the same
// arrays the host construction produced, entry for entry.
namespace {

constexpr int LB = 256;

__global__ void k_lay_pos(int n, const int32_t* __restrict__ pi, int32_t* __restrict__ pos) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) pos[pi[i]] = i;
}

// warp per slice: len = the longest off-diagonal row of the slice; *fits16 cleared when a column
// of the slice lies farther than int16 from its window's first row
__global__ void k_lay_len(int n, int nsl, const int32_t* __restrict__ pi, const int32_t* __restrict__ rp,
                          const int32_t* __restrict__ uc, const int32_t* __restrict__ pos, int32_t* __restrict__ len,
                          int32_t* __restrict__ fits16) {
    const int lane = threadIdx.x & 31;
    for (int sl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < nsl; sl += (gridDim.x * blockDim.x) >> 5) {
        const int ri = 32 * sl + lane;
        int L = 0;
        bool ok = true;
        if (ri < n) {
            const int row = pi[ri];
            L = rp[row + 1] - rp[row] - 1;
            const int wbase = (32 * sl / kSellSigma) * kSellSigma;
            for (int e = rp[row]; e < rp[row + 1]; ++e) {
                const int d = pos[uc[e]] - wbase;
                if (d < -32768 || d > 32767) ok = false;
            }
        }
        L = __reduce_max_sync(0xffffffffu, L);
        if (!__all_sync(0xffffffffu, ok) && lane == 0) atomicAnd(fits16, 0);
        if (lane == 0) len[sl] = L;
    }
}

// exclusive scan of mul * in[0..n) into out[0..n] (out[n] = total), one block
__global__ void __launch_bounds__(1024) k_lay_scan(int n, const int32_t* __restrict__ in, int mul,
                                                   int32_t* __restrict__ out) {
    __shared__ int32_t ws[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int ch = (n + 1023) / 1024;
    const int a = min(n, tid * ch), b = min(n, a + ch);
    int loc = 0;
    for (int i = a; i < b; ++i) loc += mul * in[i];
    int inc = loc;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) ws[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int v = ws[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        ws[lane] = v;
    }
    __syncthreads();
    int run = (wid > 0 ? ws[wid - 1] : 0) + inc - loc;
    for (int i = a; i < b; ++i) {
        out[i] = run;
        run += mul * in[i];
    }
    if (tid == 1023) out[n] = run;
}

// thread per slice lane: the slice's entries of this lane (column-major inside the slice)
__global__ void k_lay_fill(int n, int nsl, const int32_t* __restrict__ pi, const int32_t* __restrict__ rp,
                           const int32_t* __restrict__ uc, const int32_t* __restrict__ pos,
                           const int32_t* __restrict__ len, const int32_t* __restrict__ base,
                           int32_t* __restrict__ c32, int16_t* __restrict__ c16, int32_t* __restrict__ src) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 32LL * nsl;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int sl = (int)(t >> 5), lane = (int)(t & 31), ri = 32 * sl + lane;
        const int L = len[sl], wbase = (32 * sl / kSellSigma) * kSellSigma;
        int row = -1, r0 = 0, Lr = 0, dpos = 0;
        if (ri < n) {
            row = pi[ri];
            r0 = rp[row];
            Lr = rp[row + 1] - r0 - 1;
            while (uc[r0 + dpos] != row) ++dpos;
        }
        for (int k = 0; k < L; ++k) {
            const int64_t q = base[sl] + 32LL * k + lane;
            int col = min(ri, n - 1), sidx = -1;
            if (k < Lr) {
                col = pos[uc[r0 + k + (k >= dpos ? 1 : 0)]];
                sidx = (r0 - row) + k;  // index into o_val (natural CSR of the off-diagonals)
            }
            c32[q] = col;
            c16[q] = (int16_t)(col - wbase);
            src[q] = sidx;
        }
    }
}

__global__ void k_lay_rowlen(int n, const int32_t* __restrict__ pi, const int32_t* __restrict__ rp,
                             int32_t* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = pi[i];
        out[i] = rp[r + 1] - rp[r];
    }
}

// internal-order copy of a CSR pattern: columns and the natural entry index of every entry
__global__ void k_lay_rows(int n, const int32_t* __restrict__ pi, const int32_t* __restrict__ rp,
                           const int32_t* __restrict__ col, const int32_t* __restrict__ irp,
                           int32_t* __restrict__ icol, int32_t* __restrict__ isrc) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = pi[i];
        int o = irp[i];
        for (int e = rp[r]; e < rp[r + 1]; ++e, ++o) {
            icol[o] = col[e];
            isrc[o] = e;
        }
    }
}

int lay_grid(int64_t work) { return (int)std::max<int64_t>(1, std::min<int64_t>((work + LB - 1) / LB, 148 * 8)); }

}  // namespace

femi_status sell_layout_device(femi_system_s* S, int64_t n, const int32_t* d_pi, cudaStream_t st,
                               const std::function<femi_status(void**, size_t)>& alloc_dev, int32_t* n_slices,
                               int64_t* n_entries, bool* fits16) {
    const int nsl = (int)((n + 31) / 32);
    int32_t *pos = nullptr, *len = nullptr, *base = nullptr, *flag = nullptr, *tmp = nullptr;
    FEMI_CUDA(cudaMallocAsync(&pos, sizeof(int32_t) * std::max<int64_t>(n, 1), st));
    FEMI_CUDA(cudaMallocAsync(&tmp, sizeof(int32_t) * (std::max<int64_t>(n, 1) + 1), st));
    femi_status s;
    if ((s = alloc_dev((void**)&len, sizeof(int32_t) * std::max(nsl, 1)))) return s;
    if ((s = alloc_dev((void**)&base, sizeof(int32_t) * (nsl + 1)))) return s;
    FEMI_CUDA(cudaMallocAsync(&flag, sizeof(int32_t), st));
    const int32_t one = 1;
    FEMI_CUDA(cudaMemcpyAsync(flag, &one, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    k_lay_pos<<<lay_grid(n), LB, 0, st>>>((int)n, d_pi, pos);
    k_lay_len<<<lay_grid(32LL * nsl), LB, 0, st>>>((int)n, nsl, d_pi, S->uu_rowptr, S->uu_col, pos, len, flag);
    k_lay_scan<<<1, 1024, 0, st>>>(nsl, len, 32, base);
    // the slice offsets on the host (they size the resident solver) with the entry count and the
    // int16 verdict
    S->sell_base_h.assign(nsl + 1, 0);
    int32_t fl = 1;
    FEMI_CUDA(cudaMemcpyAsync(S->sell_base_h.data(), base, sizeof(int32_t) * (nsl + 1), cudaMemcpyDeviceToHost, st));
    FEMI_CUDA(cudaMemcpyAsync(&fl, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    FEMI_CUDA(cudaStreamSynchronize(st));
    const int64_t ent = S->sell_base_h[nsl];
    int32_t *c32 = nullptr, *src = nullptr;
    int16_t* c16 = nullptr;
    if ((s = alloc_dev((void**)&c32, sizeof(int32_t) * std::max<int64_t>(ent, 1)))) return s;
    if ((s = alloc_dev((void**)&c16, sizeof(int16_t) * std::max<int64_t>(ent, 1)))) return s;
    if ((s = alloc_dev((void**)&src, sizeof(int32_t) * std::max<int64_t>(ent, 1)))) return s;
    k_lay_fill<<<lay_grid(32LL * nsl), LB, 0, st>>>((int)n, nsl, d_pi, S->uu_rowptr, S->uu_col, pos, len, base, c32,
                                                      c16, src);
    // internal-order rows of A_uk and A_uu
    if ((s = alloc_dev((void**)&S->ukI_rowptr, sizeof(int32_t) * (n + 1)))) return s;
    if ((s = alloc_dev((void**)&S->uuI_rowptr, sizeof(int32_t) * (n + 1)))) return s;
    k_lay_rowlen<<<lay_grid(n), LB, 0, st>>>((int)n, d_pi, S->uk_rowptr, tmp);
    k_lay_scan<<<1, 1024, 0, st>>>((int)n, tmp, 1, S->ukI_rowptr);
    k_lay_rowlen<<<lay_grid(n), LB, 0, st>>>((int)n, d_pi, S->uu_rowptr, tmp);
    k_lay_scan<<<1, 1024, 0, st>>>((int)n, tmp, 1, S->uuI_rowptr);
    if (S->nnz_uk > 0) {
        if ((s = alloc_dev((void**)&S->ukI_col, sizeof(int32_t) * S->nnz_uk))) return s;
        if ((s = alloc_dev((void**)&S->ukI_src_tmp, sizeof(int32_t) * S->nnz_uk))) return s;
        if ((s = alloc_dev((void**)&S->ukI_val, sizeof(double) * S->nnz_uk))) return s;
        k_lay_rows<<<lay_grid(n), LB, 0, st>>>((int)n, d_pi, S->uk_rowptr, S->uk_col, S->ukI_rowptr, S->ukI_col,
                                                 S->ukI_src_tmp);
    }
    if (S->nnz_uu > 0) {
        if ((s = alloc_dev((void**)&S->uuI_col, sizeof(int32_t) * S->nnz_uu))) return s;
        if ((s = alloc_dev((void**)&S->uuI_src_tmp, sizeof(int32_t) * S->nnz_uu))) return s;
        if ((s = alloc_dev((void**)&S->uuI_val, sizeof(double) * S->nnz_uu))) return s;
        k_lay_rows<<<lay_grid(n), LB, 0, st>>>((int)n, d_pi, S->uu_rowptr, S->uu_col, S->uuI_rowptr, S->uuI_col,
                                                 S->uuI_src_tmp);
    }
    count_launches(10);
    FEMI_CUDA(cudaGetLastError());
    FEMI_CUDA(cudaFreeAsync(pos, st));
    FEMI_CUDA(cudaFreeAsync(tmp, st));
    FEMI_CUDA(cudaFreeAsync(flag, st));
    S->sell_len = len;
    S->sell_base = base;
    S->sell_c16 = fl ? c16 : nullptr;
    S->sell_c32 = fl ? nullptr : c32;
    S->sell_src_tmp = src;
    *n_slices = nsl;
    *n_entries = ent;
    *fits16 = fl != 0;
    return FEMI_OK;
}

}  // namespace femi

FEMI_DCHECK_READER(dcheck_assemble)
