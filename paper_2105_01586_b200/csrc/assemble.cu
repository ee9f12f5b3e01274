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

}  // namespace femi

FEMI_DCHECK_READER(dcheck_assemble)
