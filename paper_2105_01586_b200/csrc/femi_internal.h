// femi_internal.h -- internal types of libfemi (product path). Not part of the ABI.
#pragma once
#include <algorithm>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "../../include/femi.h"

namespace femi {

void set_error(const std::string& msg);

// fn(lo, hi) over contiguous chunks of [0, n) on up to 16 host threads (one chunk when n is
// below two grains)
template <class F>
void parallel_ranges(int64_t n, F&& fn, int64_t grain = 1 << 14) {
    const int64_t hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const int nt = (int)std::min<int64_t>(hw, std::max<int64_t>(1, n / std::max<int64_t>(1, grain)));
    if (nt <= 1) {
        if (n > 0) fn((int64_t)0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int k = 0; k < nt; ++k) th.emplace_back([&, k] { fn(n * k / nt, n * (k + 1) / nt); });
    for (auto& x : th) x.join();
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
