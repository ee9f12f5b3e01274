// femi_internal.h -- internal types of libfemi (product path). Not part of the ABI.
#pragma once
#include <algorithm>
#include <cstdint>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "../../include/femi.h"

namespace femi {

void set_error(const std::string& msg);

// Host worker pool (up to 16 threads, created once): run_chunks(n, fn) calls fn(k) for
// k in [0, n) on the pool and the calling thread, and returns when all have finished. A
// densification step's tables at C3 size are ~0.1 ms passes, so spawning 16 threads per pass
// (~0.3 ms) used to cost more than the work. A call made while another parallel region runs
// (from a worker, or from a second host thread) runs its chunks inline.
void run_chunks(int n, const std::function<void(int)>& fn);
int pool_threads();

// fn(lo, hi) over contiguous chunks of [0, n) on up to 16 host threads (one chunk when n is
// below two grains)
template <class F>
void parallel_ranges(int64_t n, F&& fn, int64_t grain = 1 << 14) {
    const int64_t hw = pool_threads();
    const int nt = (int)std::min<int64_t>(hw, std::max<int64_t>(1, n / std::max<int64_t>(1, grain)));
    if (nt <= 1) {
        if (n > 0) fn((int64_t)0, n);
        return;
    }
    run_chunks(nt, [&](int k) { fn(n * k / nt, n * (k + 1) / nt); });
}

// Host mesh (S0). Canonical numbering: unknowns (ascending pix) then masks (ascending pix).
struct Mesh {
    int32_t W = 0, H = 0;
    int64_t n_u = 0, m = 0, nv = 0, T = 0;
    std::vector<int32_t> vpix;       // nv
    std::vector<int32_t> tri;        // 3T canonical vertex indices (CCW, smallest pix first)
    std::vector<int32_t> nbr;        // 3T triangle across the edge opposite vertex k, -1 on the border
    std::vector<uint32_t> flags;     // T: bit k (0..2) owns edge opposite k; bit 3+k owns vertex k
    std::vector<int32_t> uu_rowptr;  // n_u+1 (diagonal included)
    std::vector<int32_t> uu_col;     // nnz_uu
    std::vector<int32_t> uu_opp;     // 2*nnz_uu: vertices opposite the edge (i,col); -1 none; diag -1,-1
    std::vector<int32_t> uk_rowptr;  // n_u+1
    std::vector<int32_t> uk_col;     // nnz_uk (mask index)
    std::vector<int32_t> uk_opp;     // 2*nnz_uk
    std::vector<int32_t> ku_rowptr;  // m+1 transpose of A_uk
    std::vector<int32_t> ku_src;     // index into uk arrays
    std::vector<int32_t> ku_row;     // unknown index
    std::vector<int32_t> vt_ptr;     // nv+1 vertex -> incident corners
    std::vector<int32_t> vt_idx;     // 3T entries: t*3+k, ascending t
    double build_seconds = 0.0;
    int32_t threads = 1;
    int32_t strips = 1;         // horizontal strips triangulated in parallel
    int32_t strip_retries = 0;  // strips re-run with a doubled margin
};

femi_status build_mesh(int32_t W, int32_t H, const int32_t* mask_px, int64_t m, const int32_t* unknown_px,
                       int64_t p, Mesh& out);
femi_status insert_mesh(const Mesh& prev, const int32_t* new_mask_px, int64_t b, Mesh& out);

}  // namespace femi

struct femi_mesh_s {
    femi::Mesh mesh;
};
