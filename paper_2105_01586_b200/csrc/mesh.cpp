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
// a remembering visibility walk, run on overlapping row strips in parallel with a
// certification step (build_mesh), followed by canonical numbering and the CSR/ownership
// tables the device kernels consume.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>

#include "femi_internal.h"

namespace femi {

namespace {
struct ThreadPool {
    std::mutex run_m;  // one parallel region at a time
    std::mutex m;
    std::condition_variable cv, cv_done;
    std::vector<std::thread> th;
    const std::function<void(int)>* job = nullptr;
    int nchunks = 0, pending = 0, active = 0;
    std::atomic<uint64_t> next{0};  // (region generation << 32) | next chunk index
    uint64_t gen = 0;
    explicit ThreadPool(int n) {
        for (int k = 0; k < n; ++k) th.emplace_back([this] { worker(); });
    }
    // claims chunks of region `g` only: a worker that took its snapshot late never runs a chunk
    // index of a later region with an earlier region's function
    void drain(const std::function<void(int)>* j, int nc, uint64_t g) {
        int done = 0;
        for (;;) {
            uint64_t v = next.load();
            int k = -1;
            while ((v >> 32) == (g & 0xffffffffu) && (int)(v & 0xffffffffu) < nc) {
                if (next.compare_exchange_weak(v, v + 1)) {
                    k = (int)(v & 0xffffffffu);
                    break;
                }
            }
            if (k < 0) break;
            (*j)(k);
            ++done;
        }
        std::lock_guard<std::mutex> l(m);
        pending -= done;
        if (pending == 0) cv_done.notify_all();
    }
    void worker() {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)>* j;
            int nc;
            {
                std::unique_lock<std::mutex> l(m);
                cv.wait(l, [&] { return gen != seen; });
                seen = gen;
                j = job;
                nc = nchunks;
                ++active;  // run() does not return (nor start the next region) while we hold j
            }
            drain(j, nc, seen);
            std::lock_guard<std::mutex> l(m);
            if (--active == 0) cv_done.notify_all();
        }
    }
    void run(int n, const std::function<void(int)>& fn) {
        std::unique_lock<std::mutex> r(run_m, std::try_to_lock);
        if (!r.owns_lock()) {  // nested or concurrent region: inline
            for (int k = 0; k < n; ++k) fn(k);
            return;
        }
        {
            std::lock_guard<std::mutex> l(m);
            job = &fn;
            nchunks = n;
            pending = n;
            ++gen;
            next.store((gen & 0xffffffffu) << 32);
        }
        cv.notify_all();
        drain(&fn, n, gen);
        std::unique_lock<std::mutex> l(m);
        cv_done.wait(l, [&] { return pending == 0 && active == 0; });
        job = nullptr;
    }
};
ThreadPool* g_pool() {
    // never destroyed: workers stay blocked on the condition variable until process exit
    static ThreadPool* p = new ThreadPool(std::max(0, pool_threads() - 1));
    return p;
}
}  // namespace

int pool_threads() {
    static const int n = [] {  // FEMI_POOL_THREADS=k caps the pool (diagnostics)
        int k = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        if (const char* e = std::getenv("FEMI_POOL_THREADS")) k = std::max(1, std::min(k, std::atoi(e)));
        return k;
    }();
    return n;
}

void run_chunks(int n, const std::function<void(int)>& fn) {
    if (n <= 0) return;
    if (n == 1 || pool_threads() == 1) {
        for (int k = 0; k < n; ++k) fn(k);
        return;
    }
    g_pool()->run(n, fn);
}
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

// Rows of the closed circumdisk of CCW (a,b,c), widened by one pixel and clipped to the
// columns [0, W): [*lo, *hi] (empty when *lo > *hi). Border triangles have huge circles
// centred outside the image whose part inside it is a thin sliver; the column clip keeps
// only that part. Returns false for a degenerate (non-CCW) triangle.
struct Disk {
    double ox, oy, r;
};
inline bool disk_of(const Pt& a, const Pt& b, const Pt& c, Disk& D) {
    int64_t bx = b.x - a.x, by = b.y - a.y, cx = c.x - a.x, cy = c.y - a.y;
    int64_t d = 2 * (bx * cy - by * cx);
    if (d <= 0) return false;
    int64_t b2 = bx * bx + by * by, c2 = cx * cx + cy * cy;
    double ux = (double)(cy * b2 - by * c2) / (double)d, uy = (double)(bx * c2 - cx * b2) / (double)d;
    D = {a.x + ux, a.y + uy, std::sqrt(ux * ux + uy * uy) + 1.0};
    return true;
}
// x-interval of the (widened) disk on row y, clipped to [0, W); false when it misses the row
inline bool disk_row(const Disk& D, double y, int32_t W, int32_t& x0, int32_t& x1) {
    double dy = std::fabs(y - D.oy);
    if (dy >= D.r) return false;
    double w = std::sqrt(D.r * D.r - dy * dy);
    x0 = (int32_t)std::max(0.0, std::floor(D.ox - w));
    x1 = (int32_t)std::min((double)(W - 1), std::ceil(D.ox + w));
    return x0 <= x1;
}
inline void disk_rows(const Disk& D, int32_t W, int32_t H, int32_t& lo, int32_t& hi) {
    double dx = D.ox < 0.0 ? -D.ox : (D.ox > W - 1 ? D.ox - (W - 1) : 0.0);
    dx = std::max(0.0, dx - 1.0);
    double h = dx >= D.r ? -1.0 : std::sqrt(D.r * D.r - dx * dx);
    lo = (int32_t)std::max(0.0, std::floor(D.oy - h));
    hi = (int32_t)std::min((double)(H - 1), std::ceil(D.oy + h));
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

    // continue from an existing triangulation (CCW triangles, n[k] across the edge opposite
    // v[k]) of a subset of the points
    void adopt(std::vector<Tri>&& t) {
        tris_ = std::move(t);
        tris_.reserve(tris_.size() + 2 * (P_.size() - tris_.size() / 2) + 8);
        stamp_.assign(tris_.size(), 0);
        last_ = 0;
    }

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

// ascending sort of a short range (a vertex's corners, a row's edge pairs: ~6-12 entries):
// insertion sort, longer ranges std::sort
template <class T>
inline void small_sort(T* a, T* b) {
    if (b - a > 32) {
        std::sort(a, b);
        return;
    }
    for (T* p = a + 1; p < b; ++p) {
        const T x = *p;
        T* q = p;
        while (q > a && x < *(q - 1)) {
            *q = *(q - 1);
            --q;
        }
        *q = x;
    }
}

// Everything after the triangulation (M.tri canonical; M.vpix, counts set): vertex ->
// incident corners, neighbours and ownership flags, the CSR patterns of A_uu / A_uk with the
// opposite-vertex tables, and the transpose of A_uk. Shared by build_mesh and insert_mesh.
template <class Stamp>
void mesh_tables(Mesh& M, int nthreads_max, Stamp&& stamp) {
    const int64_t nv = M.nv, T = M.T;
    // tiny meshes run on fewer pool threads
    const int nthreads = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads_max, T / 2048));
    auto parallel = [nthreads](int64_t n, auto&& fn) {
        run_chunks(nthreads, [&](int k) {
            const int64_t lo = n * k / nthreads, hi = n * (k + 1) / nthreads;
            for (int64_t i = lo; i < hi; ++i) fn(i);
        });
    };
    // ---- vertex -> incident corners (ascending triangle index): atomic counting sort,
    // then each vertex's short list sorted
    M.vt_ptr.assign(nv + 1, 0);
    M.vt_idx.resize(3 * T);
    if (T < (1 << 21)) {
        // sequential counting sort: the corners are visited in ascending order, so every
        // vertex's list comes out ascending -- no atomics (a locked add costs ~20 cycles even
        // uncontended) and no per-vertex sort
        int32_t* cnt = M.vt_ptr.data() + 1;
        for (int64_t q = 0; q < 3 * T; ++q) ++cnt[M.tri[q]];
        for (int64_t v = 0; v < nv; ++v) M.vt_ptr[v + 1] += M.vt_ptr[v];
        std::vector<int32_t> fill(M.vt_ptr.begin(), M.vt_ptr.end() - 1);
        for (int64_t q = 0; q < 3 * T; ++q) M.vt_idx[fill[M.tri[q]]++] = (int32_t)q;
    } else {
        int32_t* cnt = M.vt_ptr.data() + 1;
        parallel(3 * T, [&](int64_t q) { __atomic_fetch_add(&cnt[M.tri[q]], 1, __ATOMIC_RELAXED); });
        for (int64_t v = 0; v < nv; ++v) M.vt_ptr[v + 1] += M.vt_ptr[v];
        std::vector<int32_t> fill(M.vt_ptr.begin(), M.vt_ptr.end() - 1);
        parallel(3 * T, [&](int64_t q) {
            M.vt_idx[__atomic_fetch_add(&fill[M.tri[q]], 1, __ATOMIC_RELAXED)] = (int32_t)q;
        });
        parallel(nv, [&](int64_t v) { small_sort(M.vt_idx.data() + M.vt_ptr[v], M.vt_idx.data() + M.vt_ptr[v + 1]); });
    }
    stamp("vt");
    // ---- neighbours across edges, ownership flags (reading A7)
    M.nbr.assign(3 * T, -1);
    M.flags.assign(T, 0);
    parallel(T, [&](int64_t t) {
        uint32_t fl = 0;
        for (int k = 0; k < 3; ++k) {
            int32_t a = M.tri[3 * t + (k + 1) % 3], b = M.tri[3 * t + (k + 2) % 3];
            // the neighbour holds the edge as b -> a: its corner at a (vt entry 3s + j) has the
            // previous vertex b -- one compare per incident corner
            int32_t nb = -1;
            for (int32_t q = M.vt_ptr[a]; q < M.vt_ptr[a + 1]; ++q) {
                const int32_t c = M.vt_idx[q], s = c / 3, j = c - 3 * s;
                if (s != t && M.tri[3 * s + (j + 2) % 3] == b) {
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

    stamp("nbr");
    // ---- CSR patterns of A_uu (with diagonal) and A_uk, with opposite-vertex tables
    const int64_t n_u = M.n_u;
    // ONE pass over the rows: each chunk of rows writes its rows' entries (column, two opposite
    // vertices; the diagonal in place, A_uu and A_uk apart) into a chunk buffer and counts them;
    // after the row-pointer prefix the buffers are copied into place
    auto row_entries = [&](int64_t i, std::vector<std::pair<int32_t, int32_t>>& e) {
        e.clear();
        for (int32_t q = M.vt_ptr[i]; q < M.vt_ptr[i + 1]; ++q) {
            int32_t t = M.vt_idx[q] / 3, k = M.vt_idx[q] % 3;
            int32_t j1 = M.tri[3 * t + (k + 1) % 3], j2 = M.tri[3 * t + (k + 2) % 3];
            e.push_back({j1, j2});  // edge (i,j1) has opposite vertex j2 in t
            e.push_back({j2, j1});
        }
        small_sort(e.data(), e.data() + e.size());
    };
    struct Ent {
        int32_t j, o1, o2;
    };
    std::vector<int32_t> cnt_uu(n_u, 0), cnt_uk(n_u, 0);
    std::vector<std::vector<Ent>> buf_uu(nthreads), buf_uk(nthreads);
    parallel(nthreads, [&](int64_t k) {
        std::vector<std::pair<int32_t, int32_t>> e;
        std::vector<Ent>& bu = buf_uu[k];
        std::vector<Ent>& bk = buf_uk[k];
        const int64_t lo = n_u * k / nthreads, hi = n_u * (k + 1) / nthreads;
        bu.reserve(7 * (hi - lo));
        bk.reserve(4 * (hi - lo));
        for (int64_t i = lo; i < hi; ++i) {
            row_entries(i, e);
            int32_t cu = 0, ck = 0;
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
                        bu.push_back({(int32_t)i, -1, -1});
                        ++cu;
                        diag_done = true;
                    }
                    bu.push_back({j, o1, o2});
                    ++cu;
                } else {
                    bk.push_back({(int32_t)(j - n_u), o1, o2});
                    ++ck;
                }
            }
            if (!diag_done) {
                bu.push_back({(int32_t)i, -1, -1});
                ++cu;
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
        const int64_t lo = n_u * k / nthreads;
        int64_t pu = M.uu_rowptr[lo], pk = M.uk_rowptr[lo];
        for (const Ent& x : buf_uu[k]) {
            M.uu_col[pu] = x.j;
            M.uu_opp[2 * pu] = x.o1;
            M.uu_opp[2 * pu + 1] = x.o2;
            ++pu;
        }
        for (const Ent& x : buf_uk[k]) {
            M.uk_col[pk] = x.j;
            M.uk_opp[2 * pk] = x.o1;
            M.uk_opp[2 * pk + 1] = x.o2;
            ++pk;
        }
        std::vector<Ent>().swap(buf_uu[k]);
        std::vector<Ent>().swap(buf_uk[k]);
    });

    stamp("csr");
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
    stamp("transpose");
}

femi_status build_mesh(int32_t W, int32_t H, const int32_t* mask_px, int64_t m, const int32_t* unknown_px,
                       int64_t p, Mesh& M) {
    auto t_start = std::chrono::steady_clock::now();
    const bool prof = std::getenv("FEMI_MESH_PROF") != nullptr;
    auto stamp = [&](const char* what) {
        if (prof)
            std::fprintf(stderr, "mesh_build %-12s %.3f ms\n", what, 1e3 *
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
    };
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
    const int nthreads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    M.threads = nthreads;
    auto parallel = [nthreads](int64_t n, auto&& fn) {
        run_chunks(nthreads, [&](int k) {
            const int64_t lo = n * k / nthreads, hi = n * (k + 1) / nthreads;
            for (int64_t i = lo; i < hi; ++i) fn(i);
        });
    };

    // canonical vertex order: unknowns ascending, then masks ascending; plus the vertex ids
    // in pixel (row-major) order and per-row pointers. Role-map scan in row chunks: count,
    // prefix, fill.
    std::vector<int64_t> cu(nthreads + 1, 0), cm(nthreads + 1, 0);
    parallel(nthreads, [&](int64_t k) {
        const uint8_t* r0 = role.data() + (int64_t)W * (H * k / nthreads);
        const uint8_t* r1 = role.data() + (int64_t)W * (H * (k + 1) / nthreads);
        int64_t u = 0, mm = 0;
        for (const uint8_t* r = r0; r < r1; ++r) {
            u += *r == 2;
            mm += *r == 1;
        }
        cu[k + 1] = u;
        cm[k + 1] = mm;
    });
    for (int k = 0; k < nthreads; ++k) {
        cu[k + 1] += cu[k];
        cm[k + 1] += cm[k];
    }
    M.W = W;
    M.H = H;
    M.n_u = cu[nthreads];
    M.m = cm[nthreads];
    M.nv = M.n_u + M.m;
    const int64_t nv = M.nv;
    M.vpix.resize(nv);
    std::vector<int32_t> byrow(nv);
    std::vector<int64_t> rowptr(H + 1, 0);
    std::vector<Pt> P(nv);
    parallel(nthreads, [&](int64_t k) {
        int64_t iu = cu[k], im = cm[k];
        for (int32_t y = (int32_t)(H * k / nthreads); y < (int32_t)(H * (k + 1) / nthreads); ++y) {
            const uint8_t* r = role.data() + (int64_t)y * W;
            for (int32_t x = 0; x < W; ++x) {
                if (!r[x]) continue;
                const int32_t q = y * W + x;
                const int64_t v = r[x] == 2 ? iu++ : M.n_u + im++;
                M.vpix[v] = q;
                P[v] = {x, y, q};
                byrow[iu + im - 1] = (int32_t)v;
            }
            rowptr[y + 1] = iu + im;
        }
    });
    std::vector<uint8_t>().swap(role);
    const int32_t cidx[4] = {byrow[0], byrow[rowptr[1] - 1], byrow[nv - 1], byrow[rowptr[H - 1]]};
    stamp("order");

    // ---- triangulation in horizontal strips, one Bowyer-Watson per strip, in parallel.
    // A strip owns rows [y0, y1) and triangulates the points of rows [y0-g, y1+g) plus the
    // points of the two border column bands (x < margin, x >= W - margin) within 8g rows of
    // them and the four image corners, so its local hull is the image rectangle and no local
    // triangle runs along a border past points the strip does not see. A local triangle is
    // certified when no global point outside the strip's rows lies in its SoS circumcircle:
    // trivially when its closed circumdisk (clipped to the image columns) stays inside those
    // rows, else by testing the points of the few outside rows the disk reaches (border
    // slivers). Certified local triangles are Delaunay for the global set, so they belong to
    // the unique global mesh (reading A3). If every local triangle incident to a core vertex
    // is certified, the local star of each core vertex is its global star, and the strip
    // emits exactly the global triangles whose smallest-pixel vertex lies in its core;
    // otherwise it retries with g doubled (once the rows cover the image every triangle is
    // certified). Strips own ascending row ranges, so each strip's triangles sorted by
    // (pix a, pix b, pix c) concatenate into the canonical order directly; the Euler count
    // T = 2 nv - 2 - (border vertices) is checked at the end.
    struct Key {
        int32_t a, b, c;
    };
    const double spacing = std::sqrt((double)W * H / (double)nv);
    int32_t margin = (int32_t)std::ceil(4.0 * spacing) + 4;
    int32_t nstrips = 1;
    if (nv >= 4000) nstrips = std::max(1, std::min((int32_t)(2 * nthreads), H / std::max(1, 4 * margin)));
    if (const char* e = std::getenv("FEMI_MESH_STRIPS")) nstrips = std::max(1, std::min(H, std::atoi(e)));
    if (const char* e = std::getenv("FEMI_MESH_MARGIN")) margin = std::max(1, std::atoi(e));
    std::vector<std::vector<Key>> strip_keys(nstrips);
    std::vector<int32_t> strip_retries(nstrips, 0);
    const int32_t* vp = M.vpix.data();
    // points of the two border column bands (x < margin or x >= W - margin), pixel order
    std::vector<int32_t> border;
    for (int32_t v : byrow)
        if (P[v].x < margin || P[v].x >= W - margin) border.push_back(v);
    // Is no point outside rows [ry0, ry1) inside the SoS circumcircle of (a,b,c)? The rows of
    // the disk are scanned directly when they leave the region by at most a few margins
    // (border slivers); a disk reaching further fails and the strip grows instead.
    auto certified = [&](const Pt& a, const Pt& b, const Pt& c, int32_t ry0, int32_t ry1) {
        Disk D;
        if (!disk_of(a, b, c, D)) return false;
        int32_t lo, hi;
        disk_rows(D, W, H, lo, hi);
        if (lo >= ry0 && hi <= ry1 - 1) return true;
        if ((int64_t)std::max(0, ry0 - lo) + std::max(0, hi - (ry1 - 1)) > 8 * (int64_t)margin) return false;
        for (int32_t y = lo; y <= hi; ++y) {
            if (y >= ry0 && y < ry1) continue;
            int32_t x0, x1;
            if (!disk_row(D, (double)y, W, x0, x1)) continue;
            const int32_t* rb = byrow.data() + rowptr[y];
            const int32_t* re = byrow.data() + rowptr[y + 1];
            const int32_t q0 = y * W + x0, q1 = y * W + x1;
            const int32_t* it = std::lower_bound(rb, re, q0, [vp](int32_t v, int32_t q) { return vp[v] < q; });
            for (; it != re && vp[*it] <= q1; ++it) {
                const Pt& d = P[*it];
                if (d.pix == a.pix || d.pix == b.pix || d.pix == c.pix) continue;
                if (incircle(a, b, c, d)) return false;
            }
        }
        return true;
    };
    auto run_strip = [&](int32_t s) {
        const int32_t y0 = (int32_t)((int64_t)H * s / nstrips), y1 = (int32_t)((int64_t)H * (s + 1) / nstrips);
        std::vector<Key>& out = strip_keys[s];
        std::vector<int32_t> gid;
        std::vector<Pt> LP;
        std::vector<std::pair<uint64_t, int32_t>> order;
        for (int32_t g = margin;; g *= 2) {
            const int32_t ry0 = std::max(0, y0 - g), ry1 = (int32_t)std::min<int64_t>(H, (int64_t)y1 + g);
            const bool whole = ry0 == 0 && ry1 == H;
            // rows [ry0, ry1), plus every point of the two border columns outside them (the
            // image corners among them): the local hull is then the global one, so no
            // local triangle runs along a border past points the strip does not see
            gid.clear();
            const int64_t by0 = (int64_t)ry0 - 8 * (int64_t)g, by1 = (int64_t)ry1 + 8 * (int64_t)g;
            auto keep = [&](int32_t v) {
                return (P[v].y >= by0 && P[v].y < by1) || v == cidx[0] || v == cidx[1] || v == cidx[2] || v == cidx[3];
            };
            for (int32_t v : border)
                if (P[v].y < ry0 && keep(v)) gid.push_back(v);
            gid.insert(gid.end(), byrow.begin() + rowptr[ry0], byrow.begin() + rowptr[ry1]);
            for (int32_t v : border)
                if (P[v].y >= ry1 && keep(v)) gid.push_back(v);
            int32_t lc[4] = {-1, -1, -1, -1};
            for (int64_t k = 0; k < (int64_t)gid.size(); ++k)
                for (int c = 0; c < 4; ++c)
                    if (gid[k] == cidx[c]) lc[c] = (int32_t)k;
            const int64_t nl = (int64_t)gid.size();
            LP.resize(nl);
            for (int64_t k = 0; k < nl; ++k) LP[k] = P[gid[k]];
            // insertion order: BRIO rounds (geometric sizes), Hilbert order inside a round
            order.clear();
            const int R = 24;
            for (int64_t k = 0; k < nl; ++k) {
                if (k == lc[0] || k == lc[1] || k == lc[2] || k == lc[3]) continue;
                uint32_t h = mix32((uint32_t)LP[k].pix * 2654435761u + 0x9e3779b9u);
                int tz = h ? __builtin_ctz(h) : 31;
                uint64_t round = (uint64_t)(R - std::min(tz, R));  // rare (many trailing zeros) first
                order.push_back({(round << 40) | hilbert_key((uint32_t)LP[k].x, (uint32_t)LP[k].y), (int32_t)k});
            }
            std::sort(order.begin(), order.end());
            BowyerWatson bw(LP);
            bw.init(lc[0], lc[1], lc[2], lc[3]);
            for (auto& kv : order) bw.insert(kv.second);
            out.clear();
            bool ok = true;
            for (const Tri& T : bw.tris()) {
                const Pt &A = LP[T.v[0]], &B = LP[T.v[1]], &C = LP[T.v[2]];
                bool core = (A.y >= y0 && A.y < y1) || (B.y >= y0 && B.y < y1) || (C.y >= y0 && C.y < y1);
                if (!core) continue;
                if (!whole && !certified(A, B, C, ry0, ry1)) {
                    ok = false;
                    break;
                }
                int k = 0;
                if (LP[T.v[1]].pix < LP[T.v[k]].pix) k = 1;
                if (LP[T.v[2]].pix < LP[T.v[k]].pix) k = 2;
                if (LP[T.v[k]].y < y0 || LP[T.v[k]].y >= y1) continue;  // owned by an earlier strip
                out.push_back({gid[T.v[k]], gid[T.v[(k + 1) % 3]], gid[T.v[(k + 2) % 3]]});
            }
            if (ok) break;
            ++strip_retries[s];
        }
        std::sort(out.begin(), out.end(), [vp](const Key& x, const Key& y) {
            if (vp[x.a] != vp[y.a]) return vp[x.a] < vp[y.a];
            if (vp[x.b] != vp[y.b]) return vp[x.b] < vp[y.b];
            return vp[x.c] < vp[y.c];
        });
    };
    {
        std::atomic<int32_t> next{0};
        run_chunks(std::min<int>(nthreads, nstrips), [&](int) {
            for (int32_t s; (s = next.fetch_add(1)) < nstrips;) run_strip(s);
        });
    }
    if (prof) {
        int32_t tot = 0;
        for (int32_t r : strip_retries) tot += r;
        std::fprintf(stderr, "mesh_build strips %d margin %d retries %d\n", nstrips, margin, tot);
    }
    stamp("triangulate");
    M.strips = nstrips;
    M.strip_retries = 0;
    for (int32_t r : strip_retries) M.strip_retries += r;

    // ---- canonical triangles: CCW, smallest pix first, lexicographic by pix triple
    std::vector<int64_t> toff(nstrips + 1, 0);
    for (int32_t s = 0; s < nstrips; ++s) toff[s + 1] = toff[s] + (int64_t)strip_keys[s].size();
    const int64_t T = toff[nstrips];
    // Euler check on the rectangle hull: T = 2 nv - 2 - (vertices on the image border)
    int64_t hull = 0;
    for (int64_t v = 0; v < nv; ++v) {
        int32_t x = P[v].x, y = P[v].y;
        hull += (x == 0 || y == 0 || x == W - 1 || y == H - 1);
    }
    if (T != 2 * nv - 2 - hull) {
        set_error("mesh_build: internal error, strip triangulation count mismatch");
        return FEMI_E_ARG;
    }
    M.T = T;
    M.tri.resize(3 * T);
    {
        run_chunks(nthreads, [&](int k) {
            for (int32_t s = k; s < nstrips; s += nthreads) {
                int64_t o = toff[s];
                for (const Key& q : strip_keys[s]) {
                    M.tri[3 * o] = q.a;
                    M.tri[3 * o + 1] = q.b;
                    M.tri[3 * o + 2] = q.c;
                    ++o;
                }
                std::vector<Key>().swap(strip_keys[s]);
            }
        });
    }
    stamp("canonical");

    mesh_tables(M, nthreads, stamp);
    M.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    return FEMI_OK;
}

// S0 incremental (densification): prev's vertices plus b new MASK
// pixels. The new points are inserted into prev's triangulation by the same Bowyer-Watson
// (Hilbert order); by reading A3 the result is the unique triangulation of the union, i.e.
// exactly what build_mesh gives for the union -- only the canonical numbering (unknowns keep
// their indices, masks are re-ranked) and the tables are rebuilt.
femi_status insert_mesh(const Mesh& prev, const int32_t* px, int64_t b, Mesh& M) {
    auto t_start = std::chrono::steady_clock::now();
    const bool prof = std::getenv("FEMI_MESH_PROF") != nullptr;
    auto stamp = [&](const char* what) {
        if (prof)
            std::fprintf(stderr, "mesh_insert %-12s %.3f ms\n", what, 1e3 *
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
    };
    if (b < 0 || (b > 0 && !px)) {
        set_error("mesh_insert: NULL array or negative count");
        return FEMI_E_ARG;
    }
    const int32_t W = prev.W, H = prev.H;
    const int64_t N = (int64_t)W * H, n_u = prev.n_u, m_old = prev.m;
    std::vector<int32_t> add(px, px + b);
    std::sort(add.begin(), add.end());
    for (int64_t i = 0; i < b; ++i) {
        const int32_t q = add[i];
        const bool vert = std::binary_search(prev.vpix.begin(), prev.vpix.begin() + n_u, q) ||
                          std::binary_search(prev.vpix.begin() + n_u, prev.vpix.end(), q);
        if (q < 0 || q >= N || (i > 0 && add[i - 1] == q) || vert) {
            set_error("mesh_insert: pixel out of range, duplicated, or already a vertex");
            return FEMI_E_SIZE;
        }
    }
    const int nthreads = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    M.W = W;
    M.H = H;
    M.threads = nthreads;
    M.n_u = n_u;
    M.m = m_old + b;
    M.nv = n_u + M.m;
    const int64_t nv = M.nv;
    // masks re-ranked: merge of prev's (ascending) and the new pixels (ascending)
    M.vpix.resize(nv);
    std::copy(prev.vpix.begin(), prev.vpix.begin() + n_u, M.vpix.begin());
    std::vector<int32_t> old_to_new(m_old), ins_id(b);
    {
        int64_t i = 0, j = 0, o = 0;
        while (i < m_old || j < b) {
            if (j >= b || (i < m_old && prev.vpix[n_u + i] < add[j])) {
                old_to_new[i] = (int32_t)(n_u + o);
                M.vpix[n_u + o++] = prev.vpix[n_u + i++];
            } else {
                ins_id[j] = (int32_t)(n_u + o);
                M.vpix[n_u + o++] = add[j++];
            }
        }
    }
    std::vector<Pt> P(nv);
    // (x, y) of every vertex without a division per vertex: unknowns and masks are two
    // ascending pixel runs, so the row advances monotonically within each
    for (int64_t r0 : {(int64_t)0, n_u}) {
        const int64_t r1 = r0 == 0 ? n_u : nv;
        int32_t y = r1 > r0 ? M.vpix[r0] / W : 0;
        for (int64_t v = r0; v < r1; ++v) {
            const int32_t p = M.vpix[v];
            while (p >= (y + 1) * W) ++y;
            P[v] = {p - y * W, y, p};
        }
    }
    stamp("renumber");
    // prev's triangles with the new vertex ids, then the new points
    std::vector<Tri> tr(prev.T);
    for (int64_t t = 0; t < prev.T; ++t)
        for (int k = 0; k < 3; ++k) {
            const int32_t v = prev.tri[3 * t + k];
            tr[t].v[k] = v < n_u ? v : old_to_new[v - n_u];
            tr[t].n[k] = prev.nbr[3 * t + k];
        }
    BowyerWatson bw(P);
    bw.adopt(std::move(tr));
    {
        std::vector<std::pair<uint64_t, int32_t>> order(b);
        for (int64_t j = 0; j < b; ++j)
            order[j] = {hilbert_key((uint32_t)P[ins_id[j]].x, (uint32_t)P[ins_id[j]].y), ins_id[j]};
        std::sort(order.begin(), order.end());
        for (auto& kv : order) bw.insert(kv.second);
    }
    stamp("insert");
    // canonical triangles: rotate (smallest pix first), order by (pix a, pix b, pix c) -- a
    // counting sort by the pixel rank of a (the vertex ranks by pixel merge the two ascending
    // runs, unknowns and masks), then the few triangles sharing one a by (pix b, pix c):
    // O(T + nv), no comparison sort of random keys
    const auto& TR = bw.tris();
    const int64_t T = (int64_t)TR.size();
    struct Key {
        int32_t a, b, c, pb, pc;
    };
    const int32_t* vp = M.vpix.data();
    std::vector<int32_t> prank(nv);
    {
        int64_t i = 0, j = n_u, o = 0;
        while (i < n_u || j < nv) {
            if (j >= nv || (i < n_u && vp[i] < vp[j])) prank[i++] = (int32_t)o++;
            else prank[j++] = (int32_t)o++;
        }
    }
    std::vector<Key> keys(T);
    std::vector<int32_t> off(nv + 1, 0);
    parallel_ranges(T, [&](int64_t lo, int64_t hi) {
        for (int64_t t = lo; t < hi; ++t) {
            const int32_t* v = TR[t].v;
            int k = 0;
            if (vp[v[1]] < vp[v[k]]) k = 1;
            if (vp[v[2]] < vp[v[k]]) k = 2;
            const int32_t a = v[k], b = v[(k + 1) % 3], c = v[(k + 2) % 3];
            keys[t] = {a, b, c, vp[b], vp[c]};
        }
    }, 16384);
    for (int64_t t = 0; t < T; ++t) ++off[prank[keys[t].a] + 1];
    for (int64_t r = 0; r < nv; ++r) off[r + 1] += off[r];
    std::vector<Key> sorted(T);
    {
        std::vector<int32_t> fill(off.begin(), off.end() - 1);
        for (int64_t t = 0; t < T; ++t) sorted[fill[prank[keys[t].a]]++] = keys[t];
    }
    std::vector<Key>().swap(keys);
    M.T = T;
    M.tri.resize(3 * T);
    parallel_ranges(nv, [&](int64_t lo, int64_t hi) {
        for (int64_t r = lo; r < hi; ++r) {  // insertion sort of each (small) group of one a
            for (int32_t q = off[r] + 1; q < off[r + 1]; ++q) {
                const Key x = sorted[q];
                int32_t z = q - 1;
                while (z >= off[r] && (sorted[z].pb > x.pb || (sorted[z].pb == x.pb && sorted[z].pc > x.pc))) {
                    sorted[z + 1] = sorted[z];
                    --z;
                }
                sorted[z + 1] = x;
            }
            for (int32_t q = off[r]; q < off[r + 1]; ++q) {
                M.tri[3 * q] = sorted[q].a;
                M.tri[3 * q + 1] = sorted[q].b;
                M.tri[3 * q + 2] = sorted[q].c;
            }
        }
    }, 8192);
    stamp("canonical");
    mesh_tables(M, nthreads, stamp);
    M.strips = 0;
    M.strip_retries = 0;
    M.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    return FEMI_OK;
}

}  // namespace femi
