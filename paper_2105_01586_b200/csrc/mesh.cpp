// mesh.cpp -- S0 mesh_build: host setup stage of the FEM inpainting path.
//
// PAPER.md:L211-227 (§2.2): every mask pixel is a vertex, plus "unknown vertices"; "a
// Delaunay triangulation is constructed from the point set formed by the vertices";
// "the mesh can be reconstructed only from the mask pixels and unknown vertices".
// Reading A3 makes the triangulation unique on the maximally cocircular pixel
// grid: lifted heights z_i = x_i^2 + y_i^2 - eps^(pix_i+1) (symbolic), i.e. an exact
// integer in-circle test with the smallest-pixel tie-break. Uniqueness means any correct
// algorithm gives the same mesh; this one is Bowyer-Watson (cavity re-triangulation)
// with biased randomised insertion order (BRIO rounds, Hilbert order within a round) and
// a remembering visibility walk, followed by canonical numbering and the CSR/ownership
// tables the device kernels consume.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <numeric>
#include <thread>

#include "femi_internal.h"

namespace femi {
namespace {

struct Pt {
    int32_t x, y, pix;
};

inline int64_t orient(const Pt& a, const Pt& b, const Pt& c) {
    return (int64_t)(b.x - a.x) * (c.y - a.y) - (int64_t)(b.y - a.y) * (c.x - a.x);
}

// d strictly inside the (symbolically perturbed) circumcircle of CCW (a,b,c)?
// Coordinates < 2^14: |lift| < 2^29, |cross| < 2^29, |det| < 3*2^58 -> int64 exact.
inline bool incircle(const Pt& a, const Pt& b, const Pt& c, const Pt& d) {
    int64_t adx = a.x - d.x, ady = a.y - d.y;
    int64_t bdx = b.x - d.x, bdy = b.y - d.y;
    int64_t cdx = c.x - d.x, cdy = c.y - d.y;
    int64_t al = adx * adx + ady * ady, bl = bdx * bdx + bdy * bdy, cl = cdx * cdx + cdy * cdy;
    int64_t det = al * (bdx * cdy - cdx * bdy) + bl * (cdx * ady - adx * cdy) + cl * (adx * bdy - bdx * ady);
    if (det != 0) return det > 0;
    // cocircular: the point with the smallest pixel index is lowered the most
    int32_t s = std::min(std::min(a.pix, b.pix), std::min(c.pix, d.pix));
    if (s == d.pix) return true;
    if (s == a.pix) return orient(b, c, d) < 0;
    if (s == b.pix) return orient(c, a, d) < 0;
    return orient(a, b, d) < 0;
}

inline uint64_t hilbert_key(uint32_t x, uint32_t y) {
    const uint32_t n = 1u << 14;
    uint64_t d = 0;
    for (uint32_t s = n >> 1; s > 0; s >>= 1) {
        uint32_t rx = (x & s) ? 1u : 0u, ry = (y & s) ? 1u : 0u;
        d += (uint64_t)s * s * ((3u * rx) ^ ry);
        if (ry == 0) {
            if (rx == 1) {
                x = n - 1 - x;
                y = n - 1 - y;
            }
            std::swap(x, y);
        }
    }
    return d;
}

inline uint32_t mix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x7feb352dU;
    h ^= h >> 15;
    h *= 0x846ca68bU;
    h ^= h >> 16;
    return h;
}

struct Tri {
    int32_t v[3];
    int32_t n[3];
};

class BowyerWatson {
  public:
    BowyerWatson(const std::vector<Pt>& P) : P_(P) {
        tris_.reserve(2 * P.size() + 8);
        stamp_.reserve(2 * P.size() + 8);
    }

    // corners: indices of (0,0), (W-1,0), (W-1,H-1), (0,H-1)
    void init(int32_t c0, int32_t c1, int32_t c2, int32_t c3) {
        tris_.push_back({{c0, c1, c2}, {-1, 1, -1}});
        tris_.push_back({{c0, c2, c3}, {-1, -1, 0}});
        stamp_.assign(2, 0);
        if (incircle(P_[c0], P_[c1], P_[c2], P_[c3])) {  // SoS picks the other diagonal
            tris_[0] = {{c1, c2, c3}, {-1, 1, -1}};
            tris_[1] = {{c1, c3, c0}, {-1, -1, 0}};
        }
        last_ = 0;
    }

    void insert(int32_t pi) {
        const Pt& p = P_[pi];
        int32_t t0 = locate(p);
        ++epoch_;
        cavity_.clear();
        stack_.clear();
        stack_.push_back(t0);
        stamp_[t0] = epoch_;
        while (!stack_.empty()) {
            int32_t t = stack_.back();
            stack_.pop_back();
            cavity_.push_back(t);
            const Tri& T = tris_[t];
            for (int k = 0; k < 3; ++k) {
                int32_t nb = T.n[k];
                if (nb < 0 || stamp_[nb] == epoch_) continue;
                const Tri& N = tris_[nb];
                if (incircle(P_[N.v[0]], P_[N.v[1]], P_[N.v[2]], p)) {
                    stamp_[nb] = epoch_;
                    stack_.push_back(nb);
                }
            }
        }
        // boundary edges of the cavity, in the CCW sense of their cavity triangle
        bnd_.clear();
        for (int32_t t : cavity_) {
            const Tri& T = tris_[t];
            for (int k = 0; k < 3; ++k) {
                int32_t nb = T.n[k];
                if (nb >= 0 && stamp_[nb] == epoch_) continue;
                int32_t u = T.v[(k + 1) % 3], w = T.v[(k + 2) % 3];
                if (nb < 0 && orient(P_[u], P_[w], p) == 0) continue;  // p on this hull edge
                bnd_.push_back({u, w, nb, t});
            }
        }
        // new fan (p, u, w): reuse the cavity slots first
        size_t nc = cavity_.size();
        for (size_t q = 0; q < bnd_.size(); ++q) {
            int32_t id;
            if (q < nc) {
                id = cavity_[q];
            } else {
                id = (int32_t)tris_.size();
                tris_.push_back(Tri{});
                stamp_.push_back(0);
            }
            bnd_[q].id = id;
        }
        for (size_t q = 0; q < bnd_.size(); ++q) {
            Edge& e = bnd_[q];
            Tri& T = tris_[e.id];
            T.v[0] = pi;
            T.v[1] = e.u;
            T.v[2] = e.w;
            T.n[0] = e.out;
            T.n[1] = -1;  // across (w,p): the fan triangle starting at w
            T.n[2] = -1;  // across (p,u): the fan triangle ending at u
            for (size_t r = 0; r < bnd_.size(); ++r) {
                if (bnd_[r].u == e.w) T.n[1] = bnd_[r].id;
                if (bnd_[r].w == e.u) T.n[2] = bnd_[r].id;
            }
            if (e.out >= 0) {
                Tri& O = tris_[e.out];
                for (int k = 0; k < 3; ++k)
                    if (O.n[k] == e.old) {
                        // the outside triangle's edge (w,u) may border several cavity
                        // triangles only through distinct edges; match the vertex pair
                        int32_t a = O.v[(k + 1) % 3], b = O.v[(k + 2) % 3];
                        if (a == e.w && b == e.u) {
                            O.n[k] = e.id;
                            break;
                        }
                    }
            }
        }
        last_ = bnd_.empty() ? t0 : bnd_[0].id;
    }

    const std::vector<Tri>& tris() const { return tris_; }

  private:
    struct Edge {
        int32_t u, w, out, old;
        int32_t id = -1;
    };

    int32_t locate(const Pt& p) {
        int32_t t = last_, from = -1;
        uint32_t rot = 0;
        for (;;) {
            const Tri& T = tris_[t];
            int32_t next = -1;
            rot = rot * 1103515245u + 12345u;
            int k0 = (int)((rot >> 16) % 3u);
            for (int j = 0; j < 3; ++j) {
                int k = (k0 + j) % 3;
                int32_t nb = T.n[k];
                if (nb == from && nb >= 0) continue;
                if (orient(P_[T.v[(k + 1) % 3]], P_[T.v[(k + 2) % 3]], p) < 0) {
                    next = nb;
                    break;
                }
            }
            if (next < 0) {
                // either inside t, or the only failing edge is the one we came through
                bool inside = true;
                for (int k = 0; k < 3 && inside; ++k)
                    if (orient(P_[T.v[(k + 1) % 3]], P_[T.v[(k + 2) % 3]], p) < 0) inside = false;
                if (inside) return t;
                next = from;  // step back (cannot happen in a valid Delaunay walk)
            }
            from = t;
            t = next;
        }
    }

    const std::vector<Pt>& P_;
    std::vector<Tri> tris_;
    std::vector<uint32_t> stamp_;
    uint32_t epoch_ = 0;
    int32_t last_ = 0;
    std::vector<int32_t> cavity_, stack_;
    std::vector<Edge> bnd_;
};

}  // namespace

femi_status build_mesh(int32_t W, int32_t H, const int32_t* mask_px, int64_t m, const int32_t* unknown_px,
                       int64_t p, Mesh& M) {
    auto t_start = std::chrono::steady_clock::now();
    if ((m > 0 && !mask_px) || (p > 0 && !unknown_px) || m < 0 || p < 0) {
        set_error("mesh_build: NULL array or negative count");
        return FEMI_E_ARG;
    }
    if (W < 2 || H < 2) {
        set_error("mesh_build: W and H must be >= 2 (all vertices collinear otherwise)");
        return FEMI_E_DEGENERATE;
    }
    if (W > 16384 || H > 16384) {
        set_error("mesh_build: W and H must be <= 16384 (exact int64 predicates)");
        return FEMI_E_SIZE;
    }
    if (m == 0) {
        set_error("mesh_build: at least one mask pixel is required (A_uu singular otherwise)");
        return FEMI_E_NO_MASK;
    }
    const int64_t N = (int64_t)W * H;
    std::vector<uint8_t> role(N, 0);  // 1 mask, 2 unknown
    for (int64_t i = 0; i < m; ++i) {
        int32_t q = mask_px[i];
        if (q < 0 || q >= N || role[q]) {
            set_error("mesh_build: mask pixel out of range or duplicated");
            return FEMI_E_SIZE;
        }
        role[q] = 1;
    }
    for (int64_t i = 0; i < p; ++i) {
        int32_t q = unknown_px[i];
        if (q < 0 || q >= N || role[q]) {
            set_error("mesh_build: unknown pixel out of range, duplicated, or also a mask pixel");
            return FEMI_E_SIZE;
        }
        role[q] = 2;
    }
    const int32_t corners[4] = {0, W - 1, (H - 1) * W + (W - 1), (H - 1) * W};
    for (int c = 0; c < 4; ++c)
        if (!role[corners[c]]) role[corners[c]] = 2;  // reading A2
    // canonical vertex order: unknowns ascending, then masks ascending (role-map scan)
    std::vector<int32_t> unk, msk;
    unk.reserve(p + 4);
    msk.reserve(m);
    for (int64_t q = 0; q < N; ++q) {
        if (role[q] == 2) unk.push_back((int32_t)q);
        else if (role[q] == 1) msk.push_back((int32_t)q);
    }
    M.W = W;
    M.H = H;
    M.n_u = (int64_t)unk.size();
    M.m = (int64_t)msk.size();
    M.nv = M.n_u + M.m;
    M.vpix.resize(M.nv);
    std::copy(unk.begin(), unk.end(), M.vpix.begin());
    std::copy(msk.begin(), msk.end(), M.vpix.begin() + M.n_u);
    std::vector<int32_t>().swap(unk);
    std::vector<int32_t>().swap(msk);

    const int64_t nv = M.nv;
    std::vector<Pt> P(nv);
    for (int64_t v = 0; v < nv; ++v) P[v] = {M.vpix[v] % W, M.vpix[v] / W, M.vpix[v]};
    int32_t cidx[4];
    for (int c = 0; c < 4; ++c) {
        cidx[c] = (int32_t)(std::lower_bound(M.vpix.begin(), M.vpix.begin() + M.n_u, corners[c]) - M.vpix.begin());
        if (cidx[c] >= M.n_u || M.vpix[cidx[c]] != corners[c])
            cidx[c] = (int32_t)(std::lower_bound(M.vpix.begin() + M.n_u, M.vpix.end(), corners[c]) - M.vpix.begin());
    }

    // ---- insertion order: BRIO rounds (geometric sizes), Hilbert order inside a round
    std::vector<std::pair<uint64_t, int32_t>> order;
    order.reserve(nv);
    const int R = 24;
    for (int64_t v = 0; v < nv; ++v) {
        if (v == cidx[0] || v == cidx[1] || v == cidx[2] || v == cidx[3]) continue;
        uint32_t h = mix32((uint32_t)M.vpix[v] * 2654435761u + 0x9e3779b9u);
        int tz = h ? __builtin_ctz(h) : 31;
        uint64_t round = (uint64_t)(R - std::min(tz, R));  // rare (many trailing zeros) first
        order.push_back({(round << 40) | hilbert_key((uint32_t)P[v].x, (uint32_t)P[v].y), (int32_t)v});
    }
    std::sort(order.begin(), order.end());

    BowyerWatson bw(P);
    bw.init(cidx[0], cidx[1], cidx[2], cidx[3]);
    for (auto& kv : order) bw.insert(kv.second);
    std::vector<std::pair<uint64_t, int32_t>>().swap(order);

    // ---- canonical triangles: CCW, smallest pix first, lexicographic by pix triple
    const auto& TR = bw.tris();
    const int64_t T = (int64_t)TR.size();
    M.T = T;
    struct Key {
        int32_t a, b, c;
        int32_t src;
    };
    std::vector<Key> keys(T);
    for (int64_t t = 0; t < T; ++t) {
        const int32_t* v = TR[t].v;
        int k = 0;
        if (M.vpix[v[1]] < M.vpix[v[k]]) k = 1;
        if (M.vpix[v[2]] < M.vpix[v[k]]) k = 2;
        keys[t] = {v[k], v[(k + 1) % 3], v[(k + 2) % 3], (int32_t)t};
    }
    const int32_t* vp = M.vpix.data();
    std::sort(keys.begin(), keys.end(), [vp](const Key& x, const Key& y) {
        if (vp[x.a] != vp[y.a]) return vp[x.a] < vp[y.a];
        if (vp[x.b] != vp[y.b]) return vp[x.b] < vp[y.b];
        return vp[x.c] < vp[y.c];
    });
    M.tri.resize(3 * T);
    for (int64_t t = 0; t < T; ++t) {
        M.tri[3 * t] = keys[t].a;
        M.tri[3 * t + 1] = keys[t].b;
        M.tri[3 * t + 2] = keys[t].c;
    }
    std::vector<Key>().swap(keys);

    // ---- vertex -> incident corners (ascending triangle index)
    M.vt_ptr.assign(nv + 1, 0);
    for (int64_t q = 0; q < 3 * T; ++q) M.vt_ptr[M.tri[q] + 1]++;
    for (int64_t v = 0; v < nv; ++v) M.vt_ptr[v + 1] += M.vt_ptr[v];
    M.vt_idx.resize(3 * T);
    {
        std::vector<int32_t> fill(M.vt_ptr.begin(), M.vt_ptr.end() - 1);
        for (int64_t q = 0; q < 3 * T; ++q) M.vt_idx[fill[M.tri[q]]++] = (int32_t)q;
    }

    // ---- neighbours across edges, ownership flags (reading A7)
    M.nbr.assign(3 * T, -1);
    M.flags.assign(T, 0);
    const int nthreads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    M.threads = nthreads;
    auto parallel = [nthreads](int64_t n, auto&& fn) {
        std::vector<std::thread> th;
        for (int k = 0; k < nthreads; ++k)
            th.emplace_back([&, k] {
                int64_t lo = n * k / nthreads, hi = n * (k + 1) / nthreads;
                for (int64_t i = lo; i < hi; ++i) fn(i);
            });
        for (auto& x : th) x.join();
    };
    parallel(T, [&](int64_t t) {
        uint32_t fl = 0;
        for (int k = 0; k < 3; ++k) {
            int32_t a = M.tri[3 * t + (k + 1) % 3], b = M.tri[3 * t + (k + 2) % 3];
            int32_t nb = -1;
            for (int32_t q = M.vt_ptr[a]; q < M.vt_ptr[a + 1]; ++q) {
                int32_t s = M.vt_idx[q] / 3;
                if (s == t) continue;
                if (M.tri[3 * s] == b || M.tri[3 * s + 1] == b || M.tri[3 * s + 2] == b) {
                    nb = s;
                    break;
                }
            }
            M.nbr[3 * t + k] = nb;
            if (nb < 0 || t < nb) fl |= 1u << k;
            int32_t vk = M.tri[3 * t + k];
            if (M.vt_idx[M.vt_ptr[vk]] / 3 == t) fl |= 1u << (3 + k);  // lowest incident triangle
        }
        M.flags[t] = fl;
    });

    // ---- CSR patterns of A_uu (with diagonal) and A_uk, with opposite-vertex tables
    const int64_t n_u = M.n_u;
    std::vector<int32_t> cnt_uu(n_u, 0), cnt_uk(n_u, 0);
    auto row_entries = [&](int64_t i, std::vector<std::pair<int32_t, int32_t>>& e) {
        e.clear();
        for (int32_t q = M.vt_ptr[i]; q < M.vt_ptr[i + 1]; ++q) {
            int32_t t = M.vt_idx[q] / 3, k = M.vt_idx[q] % 3;
            int32_t j1 = M.tri[3 * t + (k + 1) % 3], j2 = M.tri[3 * t + (k + 2) % 3];
            e.push_back({j1, j2});  // edge (i,j1) has opposite vertex j2 in t
            e.push_back({j2, j1});
        }
        std::sort(e.begin(), e.end());
    };
    parallel(nthreads, [&](int64_t k) {
        std::vector<std::pair<int32_t, int32_t>> e;
        int64_t lo = n_u * k / nthreads, hi = n_u * (k + 1) / nthreads;
        for (int64_t i = lo; i < hi; ++i) {
            row_entries(i, e);
            int32_t cu = 1, ck = 0;  // diagonal
            for (size_t q = 0; q < e.size(); ++q) {
                if (q > 0 && e[q].first == e[q - 1].first) continue;
                if (e[q].first < n_u) ++cu;
                else ++ck;
            }
            cnt_uu[i] = cu;
            cnt_uk[i] = ck;
        }
    });
    M.uu_rowptr.assign(n_u + 1, 0);
    M.uk_rowptr.assign(n_u + 1, 0);
    for (int64_t i = 0; i < n_u; ++i) {
        M.uu_rowptr[i + 1] = M.uu_rowptr[i] + cnt_uu[i];
        M.uk_rowptr[i + 1] = M.uk_rowptr[i] + cnt_uk[i];
    }
    const int64_t nuu = M.uu_rowptr[n_u], nuk = M.uk_rowptr[n_u];
    M.uu_col.resize(nuu);
    M.uu_opp.resize(2 * nuu);
    M.uk_col.resize(nuk);
    M.uk_opp.resize(2 * nuk);
    parallel(nthreads, [&](int64_t k) {
        std::vector<std::pair<int32_t, int32_t>> e;
        int64_t lo = n_u * k / nthreads, hi = n_u * (k + 1) / nthreads;
        for (int64_t i = lo; i < hi; ++i) {
            row_entries(i, e);
            int32_t pu = M.uu_rowptr[i], pk = M.uk_rowptr[i];
            bool diag_done = false;
            for (size_t q = 0; q < e.size();) {
                int32_t j = e[q].first, o1 = e[q].second, o2 = -1;
                size_t r = q + 1;
                if (r < e.size() && e[r].first == j) {
                    o2 = e[r].second;
                    ++r;
                }
                q = r;
                if (j < n_u) {
                    if (!diag_done && j > i) {
                        M.uu_col[pu] = (int32_t)i;
                        M.uu_opp[2 * pu] = -1;
                        M.uu_opp[2 * pu + 1] = -1;
                        ++pu;
                        diag_done = true;
                    }
                    M.uu_col[pu] = j;
                    M.uu_opp[2 * pu] = o1;
                    M.uu_opp[2 * pu + 1] = o2;
                    ++pu;
                } else {
                    M.uk_col[pk] = (int32_t)(j - n_u);
                    M.uk_opp[2 * pk] = o1;
                    M.uk_opp[2 * pk + 1] = o2;
                    ++pk;
                }
            }
            if (!diag_done) {
                M.uu_col[pu] = (int32_t)i;
                M.uu_opp[2 * pu] = -1;
                M.uu_opp[2 * pu + 1] = -1;
            }
        }
    });

    // ---- transpose of A_uk (rows = masks), for B^T in tonal optimisation
    M.ku_rowptr.assign(M.m + 1, 0);
    for (int64_t q = 0; q < nuk; ++q) M.ku_rowptr[M.uk_col[q] + 1]++;
    for (int64_t k = 0; k < M.m; ++k) M.ku_rowptr[k + 1] += M.ku_rowptr[k];
    M.ku_src.resize(nuk);
    M.ku_row.resize(nuk);
    {
        std::vector<int32_t> fill(M.ku_rowptr.begin(), M.ku_rowptr.end() - 1);
        for (int64_t i = 0; i < n_u; ++i)
            for (int32_t q = M.uk_rowptr[i]; q < M.uk_rowptr[i + 1]; ++q) {
                int32_t d = fill[M.uk_col[q]]++;
                M.ku_src[d] = q;
                M.ku_row[d] = (int32_t)i;
            }
    }
    M.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    return FEMI_OK;
}

}  // namespace femi
