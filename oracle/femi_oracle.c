/*
 * femi_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the FEM
 * harmonic-inpainting hot path of Chizhov & Weickert (arXiv 2105.01586).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2105_01586_b200/) never links, imports or calls it, and this file shares no
 * code, header, table or helper with it.
 *
 * Single-threaded, fp64, built with -O2 -ffp-contract=off (reading A18).
 * Every function cites the PAPER.md passage (and the DESIGN.md reading) it follows.
 *
 * Coordinates: pixel pix = y*W + x sits at the integer point (x, y) (reading A1).
 * orient(a,b,c) = (b-a) x (c-a); "CCW" means orient > 0.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;
typedef int32_t i32;

enum { ORC_OK = 0, ORC_E_ARG = 1, ORC_E_DEGENERATE = 2, ORC_E_NO_MASK = 3,
       ORC_E_NOT_CONVERGED = 4, ORC_E_NONFINITE = 5, ORC_E_NOT_SPD = 6, ORC_E_OOM = 9 };

/* ------------------------------------------------------------------------- */
/* Exact predicates ("Delaunay triangulation"; reading A3)  */
/* ------------------------------------------------------------------------- */

static i64 orient(int W, i32 a, i32 b, i32 c) {
    i64 ax = a % W, ay = a / W, bx = b % W, by = b / W, cx = c % W, cy = c / W;
    return (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
}

/* Is d strictly inside the circumcircle of the CCW triangle (a,b,c), under the
 * symbolic lowering z_i = x_i^2 + y_i^2 - eps^(pix_i + 1) (reading A3)? */
static int incircle_sos(int W, i32 a, i32 b, i32 c, i32 d) {
    i64 dx = d % W, dy = d / W;
    i64 adx = a % W - dx, ady = a / W - dy;
    i64 bdx = b % W - dx, bdy = b / W - dy;
    i64 cdx = c % W - dx, cdy = c / W - dy;
    __int128 al = (__int128)(adx * adx + ady * ady);
    __int128 bl = (__int128)(bdx * bdx + bdy * bdy);
    __int128 cl = (__int128)(cdx * cdx + cdy * cdy);
    __int128 det = al * (__int128)(bdx * cdy - cdx * bdy)
                 + bl * (__int128)(cdx * ady - adx * cdy)
                 + cl * (__int128)(adx * bdy - bdx * ady);
    if (det > 0) return 1;
    if (det < 0) return 0;
    /* cocircular: the smallest pixel index carries the dominant perturbation */
    i32 s = a;
    if (b < s) s = b;
    if (c < s) s = c;
    if (d < s) s = d;
    if (s == d) return 1;                        /* lowering d puts it inside      */
    if (s == a) return orient(W, b, c, d) < 0;   /* cofactor of z_a = orient(b,c,d) */
    if (s == b) return orient(W, c, a, d) < 0;
    return orient(W, a, b, d) < 0;
}

/* ------------------------------------------------------------------------- */
/* Canonical triangle order (reading A3/S0): CCW, smallest pix first, lexicographic */
/* ------------------------------------------------------------------------- */

static const i32* g_sort_vpix; /* qsort context (single-threaded oracle) */

static int cmp_tri(const void* A, const void* B) {
    const i32* p = (const i32*)A;
    const i32* q = (const i32*)B;
    for (int k = 0; k < 3; ++k) {
        i32 u = g_sort_vpix[p[k]], v = g_sort_vpix[q[k]];
        if (u != v) return u < v ? -1 : 1;
    }
    return 0;
}

static void canonicalise(const i32* vpix, i64 T, i32* tri) {
    for (i64 t = 0; t < T; ++t) {
        i32* v = tri + 3 * t;
        int k = 0;
        if (vpix[v[1]] < vpix[v[k]]) k = 1;
        if (vpix[v[2]] < vpix[v[k]]) k = 2;
        i32 a = v[k], b = v[(k + 1) % 3], c = v[(k + 2) % 3];
        v[0] = a; v[1] = b; v[2] = c;
    }
    g_sort_vpix = vpix;
    qsort(tri, (size_t)T, 3 * sizeof(i32), cmp_tri);
}

/* Brute force O(V^4): a CCW triple is a triangle iff no other vertex is inside its
 * (perturbed) circumcircle. PAPER.md:L220-227; reading A3. Tiny inputs only. */
i64 orc_delaunay_brute(int W, i64 n, const i32* vpix, i32* tri, i64 cap) {
    i64 T = 0;
    for (i64 i = 0; i < n; ++i)
        for (i64 j = i + 1; j < n; ++j)
            for (i64 k = j + 1; k < n; ++k) {
                i64 o = orient(W, vpix[i], vpix[j], vpix[k]);
                if (o == 0) continue;
                i64 a = i, b = o > 0 ? j : k, c = o > 0 ? k : j;
                int empty = 1;
                for (i64 d = 0; d < n && empty; ++d) {
                    if (d == a || d == b || d == c) continue;
                    if (incircle_sos(W, vpix[a], vpix[b], vpix[c], vpix[d])) empty = 0;
                }
                if (!empty) continue;
                if (T >= cap) return -ORC_E_OOM;
                tri[3 * T] = (i32)a; tri[3 * T + 1] = (i32)b; tri[3 * T + 2] = (i32)c;
                ++T;
            }
    canonicalise(vpix, T, tri);
    return T;
}

/* ------------------------------------------------------------------------- */
/* Incremental Delaunay by Lawson flips (textbook: insert, split, legalise).   */
/* Start: the two triangles of the four image corners (reading A2).            */
/* ------------------------------------------------------------------------- */

typedef struct {
    int W;
    const i32* vpix;
    i32* tv; /* 3 vertices per triangle (indices into vpix), CCW       */
    i32* tn; /* tn[3t+k] = triangle across the edge opposite tv[3t+k] */
    i64 T, cap;
} Lawson;

static i32 PX(const Lawson* L, i32 v) { return L->vpix[v]; }

static void set_tri(Lawson* L, i64 t, i32 a, i32 b, i32 c, i32 na, i32 nb, i32 nc) {
    L->tv[3 * t] = a; L->tv[3 * t + 1] = b; L->tv[3 * t + 2] = c;
    L->tn[3 * t] = na; L->tn[3 * t + 1] = nb; L->tn[3 * t + 2] = nc;
}

/* in triangle n, replace the neighbour pointer `from` by `to` */
static void repoint(Lawson* L, i32 n, i32 from, i32 to) {
    if (n < 0) return;
    for (int k = 0; k < 3; ++k)
        if (L->tn[3 * n + k] == from) { L->tn[3 * n + k] = to; return; }
}

/* triangle t has the new point p at slot 0; legalise its edge opposite p */
static void legalise(Lawson* L, i32 t) {
    i32 p = L->tv[3 * t], a = L->tv[3 * t + 1], b = L->tv[3 * t + 2];
    i32 n = L->tn[3 * t];
    if (n < 0) return;
    int j = 0;
    while (L->tn[3 * n + j] != t) ++j;
    i32 d = L->tv[3 * n + j];
    if (!incircle_sos(L->W, PX(L, p), PX(L, a), PX(L, b), PX(L, d))) return;
    /* n = (d, b, a) CCW; its neighbours: opposite b -> edge (a,d), opposite a -> edge (d,b) */
    i32 N_ad = -1, N_db = -1;
    for (int k = 0; k < 3; ++k) {
        if (L->tv[3 * n + k] == b) N_ad = L->tn[3 * n + k];
        if (L->tv[3 * n + k] == a) N_db = L->tn[3 * n + k];
    }
    i32 N_bp = L->tn[3 * t + 1]; /* opposite a in t: edge (b,p) */
    i32 N_pa = L->tn[3 * t + 2]; /* opposite b in t: edge (p,a) */
    /* t' = (p,a,d), n' = (p,d,b) */
    set_tri(L, t, p, a, d, N_ad, n, N_pa);
    set_tri(L, n, p, d, b, N_db, N_bp, t);
    repoint(L, N_ad, n, t);
    repoint(L, N_bp, t, n);
    legalise(L, t);
    legalise(L, n);
}

static i32 locate(Lawson* L, i32 start, i32 p, int* edge_k) {
    i32 t = start;
    i64 steps = 0, limit = 4 * L->T + 16;
    for (;;) {
        int moved = 0;
        for (int k = 0; k < 3; ++k) {
            i32 a = L->tv[3 * t + (k + 1) % 3], b = L->tv[3 * t + (k + 2) % 3];
            if (orient(L->W, PX(L, a), PX(L, b), PX(L, p)) < 0) {
                t = L->tn[3 * t + k];
                moved = 1;
                break;
            }
        }
        if (!moved) break;
        if (t < 0 || ++steps > limit) { /* should not happen; fall back to a linear scan */
            for (t = 0; t < L->T; ++t) {
                int ok = 1;
                for (int k = 0; k < 3 && ok; ++k)
                    if (orient(L->W, PX(L, L->tv[3 * t + (k + 1) % 3]), PX(L, L->tv[3 * t + (k + 2) % 3]), PX(L, p)) < 0) ok = 0;
                if (ok) break;
            }
            break;
        }
    }
    *edge_k = -1;
    for (int k = 0; k < 3; ++k) {
        i32 a = L->tv[3 * t + (k + 1) % 3], b = L->tv[3 * t + (k + 2) % 3];
        if (orient(L->W, PX(L, a), PX(L, b), PX(L, p)) == 0) *edge_k = k;
    }
    return t;
}

static i32 insert_point(Lawson* L, i32 start, i32 p) {
    int k;
    i32 t = locate(L, start, p, &k);
    if (k < 0) { /* strictly inside t = (a,b,c) */
        i32 a = L->tv[3 * t], b = L->tv[3 * t + 1], c = L->tv[3 * t + 2];
        i32 na = L->tn[3 * t], nb = L->tn[3 * t + 1], nc = L->tn[3 * t + 2];
        i32 t1 = (i32)L->T++, t2 = (i32)L->T++;
        set_tri(L, t, p, a, b, nc, t1, t2);  /* (a,b,p) stored as (p,a,b) */
        set_tri(L, t1, p, b, c, na, t2, t);  /* (b,c,p) */
        set_tri(L, t2, p, c, a, nb, t, t1);  /* (c,a,p) */
        repoint(L, na, t, t1);
        repoint(L, nb, t, t2);
        legalise(L, t);
        legalise(L, t1);
        legalise(L, t2);
        return t;
    }
    /* p on the edge (a,b) opposite c = tv[t][k] */
    i32 c = L->tv[3 * t + k], a = L->tv[3 * t + (k + 1) % 3], b = L->tv[3 * t + (k + 2) % 3];
    i32 n = L->tn[3 * t + k];
    i32 N_bc = L->tn[3 * t + (k + 1) % 3]; /* opposite a: edge (b,c) */
    i32 N_ca = L->tn[3 * t + (k + 2) % 3]; /* opposite b: edge (c,a) */
    i32 t2 = (i32)L->T++;
    if (n < 0) { /* hull edge */
        set_tri(L, t, p, c, a, N_ca, -1, t2);  /* (c,a,p) */
        set_tri(L, t2, p, b, c, N_bc, t, -1);  /* (c,p,b) */
        repoint(L, N_bc, t, t2);
        legalise(L, t);
        legalise(L, t2);
        return t;
    }
    int j = 0;
    while (L->tn[3 * n + j] != t) ++j;
    i32 d = L->tv[3 * n + j];
    i32 N_ad = -1, N_db = -1;
    for (int q = 0; q < 3; ++q) {
        if (L->tv[3 * n + q] == b) N_ad = L->tn[3 * n + q];
        if (L->tv[3 * n + q] == a) N_db = L->tn[3 * n + q];
    }
    i32 n1 = (i32)L->T++;
    /* t1=(c,a,p) [t], t2=(c,p,b), n1=(d,b,p), n2=(d,p,a) [n]; all stored with p first */
    set_tri(L, t, p, c, a, N_ca, n, t2);
    set_tri(L, t2, p, b, c, N_bc, t, n1);
    set_tri(L, n1, p, d, b, N_db, t2, n);
    set_tri(L, n, p, a, d, N_ad, n1, t);
    repoint(L, N_bc, t, t2);
    repoint(L, N_db, n, n1);
    legalise(L, t);
    legalise(L, t2);
    legalise(L, n1);
    legalise(L, n);
    return t;
}

static uint64_t morton(i64 x, i64 y) {
    uint64_t k = 0;
    for (int b = 0; b < 16; ++b)
        k |= ((uint64_t)((x >> b) & 1) << (2 * b)) | ((uint64_t)((y >> b) & 1) << (2 * b + 1));
    return k;
}

typedef struct { uint64_t key; i32 v; } KeyV;
static int cmp_keyv(const void* A, const void* B) {
    const KeyV* p = (const KeyV*)A;
    const KeyV* q = (const KeyV*)B;
    if (p->key != q->key) return p->key < q->key ? -1 : 1;
    return p->v < q->v ? -1 : (p->v > q->v);
}

/* Returns T >= 0, or -status. vpix must contain the four corner pixels. */
i64 orc_delaunay(int W, int H, i64 n, const i32* vpix, i32* tri, i64 cap) {
    if (W < 2 || H < 2) return -ORC_E_DEGENERATE;
    i32 cpix[4] = {0, W - 1, (H - 1) * W + W - 1, (H - 1) * W};
    i32 cidx[4] = {-1, -1, -1, -1};
    for (i64 i = 0; i < n; ++i)
        for (int c = 0; c < 4; ++c)
            if (vpix[i] == cpix[c]) cidx[c] = (i32)i;
    for (int c = 0; c < 4; ++c)
        if (cidx[c] < 0) return -ORC_E_ARG;
    Lawson L;
    L.W = W; L.vpix = vpix; L.cap = 2 * n + 8; L.T = 0;
    L.tv = (i32*)malloc(sizeof(i32) * 3 * L.cap);
    L.tn = (i32*)malloc(sizeof(i32) * 3 * L.cap);
    KeyV* order = (KeyV*)malloc(sizeof(KeyV) * (size_t)(n > 0 ? n : 1));
    if (!L.tv || !L.tn || !order) { free(L.tv); free(L.tn); free(order); return -ORC_E_OOM; }
    /* corners c0=(0,0) c1=(W-1,0) c2=(W-1,H-1) c3=(0,H-1): (c0,c1,c2), (c0,c2,c3), then legalise */
    set_tri(&L, 0, cidx[0], cidx[1], cidx[2], -1, 1, -1);
    set_tri(&L, 1, cidx[0], cidx[2], cidx[3], -1, -1, 0);
    L.T = 2;
    if (incircle_sos(W, cpix[0], cpix[1], cpix[2], cpix[3])) { /* flip to diagonal c1-c3 */
        set_tri(&L, 0, cidx[1], cidx[2], cidx[3], -1, 1, -1);
        set_tri(&L, 1, cidx[1], cidx[3], cidx[0], -1, -1, 0);
    }
    i64 m = 0;
    for (i64 i = 0; i < n; ++i) {
        int corner = 0;
        for (int c = 0; c < 4; ++c) corner |= (i == cidx[c]);
        if (corner) continue;
        order[m].key = morton(vpix[i] % W, vpix[i] / W);
        order[m].v = (i32)i;
        ++m;
    }
    qsort(order, (size_t)m, sizeof(KeyV), cmp_keyv);
    i32 last = 0;
    for (i64 i = 0; i < m; ++i) last = insert_point(&L, last, order[i].v);
    free(order);
    i64 T = L.T;
    if (T > cap) { free(L.tv); free(L.tn); return -ORC_E_OOM; }
    memcpy(tri, L.tv, sizeof(i32) * 3 * (size_t)T);
    free(L.tv); free(L.tn);
    canonicalise(vpix, T, tri);
    return T;
}

/* ------------------------------------------------------------------------- */
/* The system on one mesh: P1 stiffness, Dirichlet reduction */
/* ------------------------------------------------------------------------- */

typedef struct {
    int W, H;
    i64 n_u, m, nv, T;
    i32* vpix;  /* canonical: unknowns (ascending pix), then masks (ascending pix) */
    i32* tri;   /* canonical triangles, vertex indices */
    i32* vmap;  /* pixel -> vertex index or -1 */
    i32* owner; /* pixel -> owning triangle (reading A7) */
    i64 *uu_ptr, *uk_ptr;
    i32 *uu_col, *uk_col;
    double *uu_val, *uk_val;
    double* chol; /* dense Cholesky factor of A_uu (n_u <= 1000) or NULL */
} OrcSys;

typedef struct { i32 r, c; double v; } Trip;
static int cmp_trip(const void* A, const void* B) {
    const Trip* p = (const Trip*)A;
    const Trip* q = (const Trip*)B;
    if (p->r != q->r) return p->r < q->r ? -1 : 1;
    if (p->c != q->c) return p->c < q->c ? -1 : 1;
    return 0;
}

/* Local P1 stiffness ([Johnson2009]; reading A6): for the CCW
 * triangle (i,j,k) the entry (i,j) receives -1/2 cot(angle at k), with
 * cot = dot(p_i-p_k, p_j-p_k) / cross, cross = orient(i,j,k) = 2*area (exact integers). */
static double half_cot(int W, i32 pi, i32 pj, i32 pk) {
    i64 xi = pi % W, yi = pi / W, xj = pj % W, yj = pj / W, xk = pk % W, yk = pk / W;
    i64 dot = (xi - xk) * (xj - xk) + (yi - yk) * (yj - yk);
    i64 cross = (xi - xk) * (yj - yk) - (yi - yk) * (xj - xk);
    return -0.5 * ((double)dot / (double)cross);
}

/* Owner map (reading A7): loop triangles in canonical order, pixels inside the closed
 * triangle take the first (lowest) index. PAPER.md:L239-241, L264-265. */
static void build_owner(OrcSys* S) {
    i64 N = (i64)S->W * S->H;
    for (i64 i = 0; i < N; ++i) S->owner[i] = -1;
    for (i64 t = 0; t < S->T; ++t) {
        i32 a = S->vpix[S->tri[3 * t]], b = S->vpix[S->tri[3 * t + 1]], c = S->vpix[S->tri[3 * t + 2]];
        int x0 = a % S->W, x1 = x0, y0 = a / S->W, y1 = y0;
        i32 vs[2] = {b, c};
        for (int q = 0; q < 2; ++q) {
            int x = vs[q] % S->W, y = vs[q] / S->W;
            if (x < x0) x0 = x;
            if (x > x1) x1 = x;
            if (y < y0) y0 = y;
            if (y > y1) y1 = y;
        }
        for (int y = y0; y <= y1; ++y)
            for (int x = x0; x <= x1; ++x) {
                i32 p = y * S->W + x;
                if (S->owner[p] >= 0) continue;
                if (orient(S->W, b, c, p) >= 0 && orient(S->W, c, a, p) >= 0 && orient(S->W, a, b, p) >= 0)
                    S->owner[p] = (i32)t;
            }
    }
}

void orc_sys_free(OrcSys* S) {
    if (!S) return;
    free(S->vpix); free(S->tri); free(S->vmap); free(S->owner);
    free(S->uu_ptr); free(S->uk_ptr); free(S->uu_col); free(S->uk_col);
    free(S->uu_val); free(S->uk_val); free(S->chol);
    free(S);
}

/* Assemble the full stiffness matrix from the triangles, then split it into the
 * unknown-unknown block A_uu and the unknown-mask block A_uk (Dirichlet elimination of
 * Eq. (2); natural Neumann border Eq. (3)).
 * Diagonal = -(sum of A_uu off-diagonals by ascending column, then A_uk by ascending
 * column) (reading A6: zero row sums). */
OrcSys* orc_sys_new(int W, int H, i64 n_u, i64 m, const i32* vpix, i64 T, const i32* tri) {
    OrcSys* S = (OrcSys*)calloc(1, sizeof(OrcSys));
    if (!S) return NULL;
    i64 nv = n_u + m, N = (i64)W * H;
    S->W = W; S->H = H; S->n_u = n_u; S->m = m; S->nv = nv; S->T = T;
    S->vpix = (i32*)malloc(sizeof(i32) * (size_t)(nv + 1));
    S->tri = (i32*)malloc(sizeof(i32) * (size_t)(3 * T + 1));
    S->vmap = (i32*)malloc(sizeof(i32) * (size_t)N);
    S->owner = (i32*)malloc(sizeof(i32) * (size_t)N);
    Trip* tr = (Trip*)malloc(sizeof(Trip) * (size_t)(6 * T + 1));
    if (!S->vpix || !S->tri || !S->vmap || !S->owner || !tr) { free(tr); orc_sys_free(S); return NULL; }
    memcpy(S->vpix, vpix, sizeof(i32) * (size_t)nv);
    memcpy(S->tri, tri, sizeof(i32) * (size_t)(3 * T));
    for (i64 i = 0; i < N; ++i) S->vmap[i] = -1;
    for (i64 v = 0; v < nv; ++v) S->vmap[vpix[v]] = (i32)v;
    i64 nt = 0;
    for (i64 t = 0; t < T; ++t) {
        i32 v[3] = {tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]};
        for (int k = 0; k < 3; ++k) {
            i32 i = v[(k + 1) % 3], j = v[(k + 2) % 3], o = v[k];
            double c = half_cot(W, vpix[i], vpix[j], vpix[o]);
            tr[nt].r = i; tr[nt].c = j; tr[nt].v = c; ++nt;
            tr[nt].r = j; tr[nt].c = i; tr[nt].v = c; ++nt;
        }
    }
    qsort(tr, (size_t)nt, sizeof(Trip), cmp_trip);
    /* combine the (at most two) contributions of each edge */
    i64 ne = 0;
    for (i64 q = 0; q < nt;) {
        i64 r = q + 1;
        double v = tr[q].v;
        while (r < nt && tr[r].r == tr[q].r && tr[r].c == tr[q].c) { v = v + tr[r].v; ++r; }
        tr[ne].r = tr[q].r; tr[ne].c = tr[q].c; tr[ne].v = v; ++ne;
        q = r;
    }
    S->uu_ptr = (i64*)calloc((size_t)(n_u + 1), sizeof(i64));
    S->uk_ptr = (i64*)calloc((size_t)(n_u + 1), sizeof(i64));
    i64 nuu = n_u, nuk = 0; /* diagonal always present (reading A5) */
    for (i64 q = 0; q < ne; ++q) {
        if (tr[q].r >= n_u) continue;
        if (tr[q].c < n_u) { ++nuu; S->uu_ptr[tr[q].r + 1]++; }
        else { ++nuk; S->uk_ptr[tr[q].r + 1]++; }
    }
    for (i64 i = 0; i < n_u; ++i) {
        S->uu_ptr[i + 1] += S->uu_ptr[i] + 1;
        S->uk_ptr[i + 1] += S->uk_ptr[i];
    }
    S->uu_col = (i32*)malloc(sizeof(i32) * (size_t)(nuu + 1));
    S->uu_val = (double*)malloc(sizeof(double) * (size_t)(nuu + 1));
    S->uk_col = (i32*)malloc(sizeof(i32) * (size_t)(nuk + 1));
    S->uk_val = (double*)malloc(sizeof(double) * (size_t)(nuk + 1));
    if (!S->uu_ptr || !S->uk_ptr || !S->uu_col || !S->uu_val || !S->uk_col || !S->uk_val) {
        free(tr); orc_sys_free(S); return NULL;
    }
    i64 q = 0;
    for (i64 i = 0; i < n_u; ++i) {
        while (q < ne && tr[q].r < i) ++q;
        i64 puu = S->uu_ptr[i], puk = S->uk_ptr[i], dpos = -1;
        double acc = 0.0;
        i64 q0 = q;
        for (; q < ne && tr[q].r == i && tr[q].c < n_u; ++q) {
            if (dpos < 0 && tr[q].c > i) { dpos = puu; S->uu_col[puu] = (i32)i; ++puu; }
            S->uu_col[puu] = tr[q].c; S->uu_val[puu] = tr[q].v; acc = acc + tr[q].v; ++puu;
        }
        if (dpos < 0) { dpos = puu; S->uu_col[puu] = (i32)i; ++puu; }
        for (; q < ne && tr[q].r == i; ++q) {
            S->uk_col[puk] = (i32)(tr[q].c - n_u); S->uk_val[puk] = tr[q].v; acc = acc + tr[q].v; ++puk;
        }
        (void)q0;
        S->uu_val[dpos] = -acc;
    }
    free(tr);
    build_owner(S);
    return S;
}

void orc_sys_counts(const OrcSys* S, i64* out) {
    out[0] = S->uu_ptr[S->n_u];
    out[1] = S->uk_ptr[S->n_u];
}

void orc_sys_export(const OrcSys* S, i64* uu_ptr, i32* uu_col, double* uu_val,
                    i64* uk_ptr, i32* uk_col, double* uk_val, i32* owner) {
    i64 nuu = S->uu_ptr[S->n_u], nuk = S->uk_ptr[S->n_u];
    memcpy(uu_ptr, S->uu_ptr, sizeof(i64) * (size_t)(S->n_u + 1));
    memcpy(uk_ptr, S->uk_ptr, sizeof(i64) * (size_t)(S->n_u + 1));
    memcpy(uu_col, S->uu_col, sizeof(i32) * (size_t)nuu);
    memcpy(uu_val, S->uu_val, sizeof(double) * (size_t)nuu);
    memcpy(uk_col, S->uk_col, sizeof(i32) * (size_t)nuk);
    memcpy(uk_val, S->uk_val, sizeof(double) * (size_t)nuk);
    if (owner) memcpy(owner, S->owner, sizeof(i32) * (size_t)S->W * S->H);
}

/* ------------------------------------------------------------------------- */
/* Solve A_uu x = -A_uk g (SPD, conjugate gradients)        */
/* ------------------------------------------------------------------------- */

static void matvec_uu(const OrcSys* S, const double* x, double* y) {
    for (i64 i = 0; i < S->n_u; ++i) {
        double acc = 0.0;
        for (i64 q = S->uu_ptr[i]; q < S->uu_ptr[i + 1]; ++q) acc = acc + S->uu_val[q] * x[S->uu_col[q]];
        y[i] = acc;
    }
}

static double dot(i64 n, const double* a, const double* b) {
    double s = 0.0;
    for (i64 i = 0; i < n; ++i) s = s + a[i] * b[i];
    return s;
}

static int factor_dense(OrcSys* S) {
    i64 n = S->n_u;
    double* A = (double*)calloc((size_t)(n * n), sizeof(double));
    if (!A) return ORC_E_OOM;
    for (i64 i = 0; i < n; ++i)
        for (i64 q = S->uu_ptr[i]; q < S->uu_ptr[i + 1]; ++q) A[i * n + S->uu_col[q]] = S->uu_val[q];
    for (i64 j = 0; j < n; ++j) { /* plain Cholesky, lower triangle */
        double d = A[j * n + j];
        for (i64 k = 0; k < j; ++k) d = d - A[j * n + k] * A[j * n + k];
        if (!(d > 0.0)) { free(A); return ORC_E_NOT_SPD; }
        d = sqrt(d);
        A[j * n + j] = d;
        for (i64 i = j + 1; i < n; ++i) {
            double s = A[i * n + j];
            for (i64 k = 0; k < j; ++k) s = s - A[i * n + k] * A[j * n + k];
            A[i * n + j] = s / d;
        }
    }
    S->chol = A;
    return ORC_OK;
}

/* Preconditioned CG [Sa03, Alg. 9.1] with the Jacobi preconditioner M = diag(A_uu).
 * r holds b - A x on entry; p, q are scratch. Stops like the plain CG below: when the
 * recursive ||r|| <= rtol ||b||, the true residual is recomputed and the iteration restarts
 * from it if it misses (reading A11). */
static int pcg_jacobi(const OrcSys* S, const double* b, double* x, double* r, double* p, double* q, double bn,
                      double rtol, int max_iter, int* iters_out) {
    i64 n = S->n_u;
    double* dinv = (double*)malloc(sizeof(double) * (size_t)n);
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    if (!dinv || !z) { free(dinv); free(z); return ORC_E_OOM; }
    for (i64 i = 0; i < n; ++i) {
        double d = 0.0;
        for (i64 e = S->uu_ptr[i]; e < S->uu_ptr[i + 1]; ++e) if (S->uu_col[e] == i) d = S->uu_val[e];
        dinv[i] = 1.0 / d;
    }
    int status = ORC_OK, it = 0;
    for (i64 i = 0; i < n; ++i) { z[i] = dinv[i] * r[i]; p[i] = z[i]; }
    double rz = dot(n, r, z);
    while (it < max_iter) {
        matvec_uu(S, p, q);
        double pq = dot(n, p, q);
        if (!(pq > 0.0)) { status = isfinite(pq) ? ORC_E_NOT_SPD : ORC_E_NONFINITE; break; }
        double alpha = rz / pq;
        for (i64 i = 0; i < n; ++i) { x[i] = x[i] + alpha * p[i]; r[i] = r[i] - alpha * q[i]; }
        ++it;
        double rr = dot(n, r, r);
        if (!isfinite(rr)) { status = ORC_E_NONFINITE; break; }
        if (sqrt(rr) <= rtol * bn) {
            matvec_uu(S, x, q);
            for (i64 i = 0; i < n; ++i) r[i] = b[i] - q[i];
            rr = dot(n, r, r);
            if (sqrt(rr) <= rtol * bn) break;
            for (i64 i = 0; i < n; ++i) { z[i] = dinv[i] * r[i]; p[i] = z[i]; }
            rz = dot(n, r, z);
            continue;
        }
        for (i64 i = 0; i < n; ++i) z[i] = dinv[i] * r[i];
        double rz2 = dot(n, r, z);
        double beta = rz2 / rz;
        for (i64 i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        rz = rz2;
    }
    *iters_out = it;
    free(dinv); free(z);
    return status;
}

/* method: 0 auto (dense Cholesky when n_u <= 1000, else CG), 1 Cholesky, 2 CG, 3 Jacobi PCG.
 * Solves A_uu x = b. x holds the initial guess on entry (reading A11). The method stops
 * on the true relative residual ||b - A x|| / ||b|| <= rtol. */
static int solve_uu(OrcSys* S, const double* b, double* x, double rtol, int max_iter, int method,
                    int* iters_out, double* relres_out) {
    i64 n = S->n_u;
    *iters_out = 0;
    *relres_out = 0.0;
    if (n == 0) return ORC_OK;
    double bn = sqrt(dot(n, b, b));
    if (!isfinite(bn)) return ORC_E_NONFINITE;
    if (bn == 0.0) { for (i64 i = 0; i < n; ++i) x[i] = 0.0; return ORC_OK; }
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    double* p = (double*)malloc(sizeof(double) * (size_t)n);
    double* q = (double*)malloc(sizeof(double) * (size_t)n);
    if (!r || !p || !q) { free(r); free(p); free(q); return ORC_E_OOM; }
    matvec_uu(S, x, q);
    for (i64 i = 0; i < n; ++i) r[i] = b[i] - q[i];
    double rn = sqrt(dot(n, r, r));
    int status = ORC_OK;
    if (rn <= rtol * bn) goto done; /* initial guess already solves (reading A16) */
    if (method == 0) method = (n <= 1000) ? 1 : 2;
    if (method == 1) {
        if (!S->chol) { status = factor_dense(S); if (status) goto done; }
        const double* L = S->chol;
        for (i64 i = 0; i < n; ++i) { /* L y = b */
            double s = b[i];
            for (i64 k = 0; k < i; ++k) s = s - L[i * n + k] * p[k];
            p[i] = s / L[i * n + i];
        }
        for (i64 i = n - 1; i >= 0; --i) { /* L^T x = y */
            double s = p[i];
            for (i64 k = i + 1; k < n; ++k) s = s - L[k * n + i] * x[k];
            x[i] = s / L[i * n + i];
        }
        *iters_out = 1;
        matvec_uu(S, x, q);
        for (i64 i = 0; i < n; ++i) r[i] = b[i] - q[i];
        rn = sqrt(dot(n, r, r));
        goto done;
    }
    if (method == 3) { /* Jacobi-preconditioned CG (reading A11: changes iterates, not the solution) */
        status = pcg_jacobi(S, b, x, r, p, q, bn, rtol, max_iter, iters_out);
        matvec_uu(S, x, q);
        for (i64 i = 0; i < n; ++i) r[i] = b[i] - q[i];
        rn = sqrt(dot(n, r, r));
        if (status == ORC_OK && !(rn <= rtol * bn)) status = ORC_E_NOT_CONVERGED;
        goto done;
    }
    /* plain conjugate gradients [Sa03], restarted from the true residual if the
     * recursive residual converges early */
    for (i64 i = 0; i < n; ++i) p[i] = r[i];
    double rr = dot(n, r, r);
    int it = 0;
    while (it < max_iter) {
        matvec_uu(S, p, q);
        double pq = dot(n, p, q);
        if (!(pq > 0.0)) { status = isfinite(pq) ? ORC_E_NOT_SPD : ORC_E_NONFINITE; break; }
        double alpha = rr / pq;
        for (i64 i = 0; i < n; ++i) { x[i] = x[i] + alpha * p[i]; r[i] = r[i] - alpha * q[i]; }
        double rr2 = dot(n, r, r);
        ++it;
        if (!isfinite(rr2)) { status = ORC_E_NONFINITE; break; }
        if (sqrt(rr2) <= rtol * bn) {
            matvec_uu(S, x, q);
            for (i64 i = 0; i < n; ++i) r[i] = b[i] - q[i];
            rr2 = dot(n, r, r);
            if (sqrt(rr2) <= rtol * bn) break;
            for (i64 i = 0; i < n; ++i) p[i] = r[i];
            rr = rr2;
            continue;
        }
        double beta = rr2 / rr;
        for (i64 i = 0; i < n; ++i) p[i] = r[i] + beta * p[i];
        rr = rr2;
    }
    *iters_out = it;
    matvec_uu(S, x, q);
    for (i64 i = 0; i < n; ++i) r[i] = b[i] - q[i];
    rn = sqrt(dot(n, r, r));
    if (status == ORC_OK && !(rn <= rtol * bn)) status = ORC_E_NOT_CONVERGED;
done:
    *relres_out = rn / bn;
    free(r); free(p); free(q);
    return status;
}

/* right-hand side b = -A_uk g (Eq. (2) eliminated) */
static void rhs(const OrcSys* S, const double* g, double* b) {
    for (i64 i = 0; i < S->n_u; ++i) {
        double acc = 0.0;
        for (i64 q = S->uk_ptr[i]; q < S->uk_ptr[i + 1]; ++q) acc = acc + S->uk_val[q] * g[S->uk_col[q]];
        b[i] = -acc;
    }
}

static double midrange(i64 m, const double* g) {
    double lo = g[0], hi = g[0];
    for (i64 k = 1; k < m; ++k) { if (g[k] < lo) lo = g[k]; if (g[k] > hi) hi = g[k]; }
    return 0.5 * (lo + hi);
}

/* Harmonic inpainting on the mesh (Eqs. (1)-(3)):
 * u_vert = [x (unknowns) ; g (masks)], x from A_uu x = -A_uk g with x0 = midrange(g).
 * x0_in (optional) overrides the initial guess. */
int orc_sys_solve(OrcSys* S, const double* g, const double* x0_in, double rtol, int max_iter, int method,
                  double* u_vert, int* iters, double* relres) {
    if (S->m == 0) return ORC_E_NO_MASK;
    for (i64 k = 0; k < S->m; ++k) if (!isfinite(g[k])) return ORC_E_NONFINITE;
    double* b = (double*)malloc(sizeof(double) * (size_t)(S->n_u + 1));
    if (!b) return ORC_E_OOM;
    rhs(S, g, b);
    double x0 = midrange(S->m, g);
    for (i64 i = 0; i < S->n_u; ++i) u_vert[i] = x0_in ? x0_in[i] : x0;
    int st = solve_uu(S, b, u_vert, rtol, max_iter, method, iters, relres);
    for (i64 k = 0; k < S->m; ++k) u_vert[S->n_u + k] = g[k];
    free(b);
    return st;
}

/* ------------------------------------------------------------------------- */
/* Rasterisation and error (L262-265 "e_i = (u_i - f_i)^2",   */
/* "total L2 error in each triangle"; readings A7, A8)                         */
/* ------------------------------------------------------------------------- */

/* value of u at pixel p from its owner triangle (S3): a vertex pixel takes that vertex's
 * value; otherwise u_a + lb (u_b - u_a) + lc (u_c - u_a), lb = orient(c,a,p)/D,
 * lc = orient(a,b,p)/D, D = orient(a,b,c). */
static double pixel_value(const OrcSys* S, i32 p, const double* u_vert) {
    if (S->vmap[p] >= 0) return u_vert[S->vmap[p]];
    i64 t = S->owner[p];
    i32 va = S->tri[3 * t], vb = S->tri[3 * t + 1], vc = S->tri[3 * t + 2];
    i32 a = S->vpix[va], b = S->vpix[vb], c = S->vpix[vc];
    double D = (double)orient(S->W, a, b, c);
    double lb = (double)orient(S->W, c, a, p) / D;
    double lc = (double)orient(S->W, a, b, p) / D;
    double ua = u_vert[va];
    double t1 = lb * (u_vert[vb] - ua);
    double t2 = lc * (u_vert[vc] - ua);
    return (ua + t1) + t2;
}

void orc_sys_raster(const OrcSys* S, const double* u_vert, const double* f, double* u_px, double* e_px,
                    double* tri_err, i32* best, double* sse) {
    i64 N = (i64)S->W * S->H;
    double* best_e = (double*)malloc(sizeof(double) * (size_t)(S->T + 1));
    for (i64 t = 0; t < S->T; ++t) { tri_err[t] = 0.0; best[t] = -1; best_e[t] = -1.0; }
    double s = 0.0;
    for (i64 p = 0; p < N; ++p) {
        double u = pixel_value(S, (i32)p, u_vert);
        double d = u - f[p];
        double e = d * d;
        if (u_px) u_px[p] = u;
        if (e_px) e_px[p] = e;
        s = s + e;
        i64 t = S->owner[p];
        tri_err[t] = tri_err[t] + e;
        if (S->vmap[p] < 0 && e > best_e[t]) { best_e[t] = e; best[t] = (i32)p; } /* ties: lowest pix */
    }
    *sse = s;
    free(best_e);
}

/* Colour ("Extending the method to colour images is straightforward"):
 * C channels on one mesh; the error map is the channel sum e = sum_c (u_c - f_c)^2, added in
 * channel order (SPEC.md:L74, L83 convention); per-triangle sums, arg-max and SSE as in
 * orc_sys_raster. u_vert, f: C pointers; u_px: NULL or C pointers (entries may be NULL). */
void orc_sys_raster_channels(const OrcSys* S, int C, const double* const* u_vert, const double* const* f,
                             double* const* u_px, double* e_px, double* tri_err, i32* best, double* sse) {
    i64 N = (i64)S->W * S->H;
    double* best_e = (double*)malloc(sizeof(double) * (size_t)(S->T + 1));
    for (i64 t = 0; t < S->T; ++t) { tri_err[t] = 0.0; best[t] = -1; best_e[t] = -1.0; }
    double s = 0.0;
    for (i64 p = 0; p < N; ++p) {
        double e = 0.0;
        for (int c = 0; c < C; ++c) {
            double u = pixel_value(S, (i32)p, u_vert[c]);
            double d = u - f[c][p];
            double dd = d * d;
            e = (c == 0) ? dd : e + dd;
            if (u_px && u_px[c]) u_px[c][p] = u;
        }
        if (e_px) e_px[p] = e;
        s = s + e;
        i64 t = S->owner[p];
        tri_err[t] = tri_err[t] + e;
        if (S->vmap[p] < 0 && e > best_e[t]) { best_e[t] = e; best[t] = (i32)p; } /* ties: lowest pix */
    }
    *sse = s;
    free(best_e);
}

/* ------------------------------------------------------------------------- */
/* Densification selection (readings A8-A10)                 */
/* ------------------------------------------------------------------------- */

typedef struct { double e; i64 idx; } EI;
static int cmp_ei_desc(const void* A, const void* B) {
    const EI* p = (const EI*)A;
    const EI* q = (const EI*)B;
    if (p->e != q->e) return p->e > q->e ? -1 : 1;
    return p->idx < q->idx ? -1 : (p->idx > q->idx);
}
static int cmp_i32(const void* A, const void* B) {
    i32 a = *(const i32*)A, b = *(const i32*)B;
    return a < b ? -1 : (a > b);
}

/* "insert a single mask pixel in each triangle, in descending order of the L2 error ...
 * at the empty location with the largest pointwise error": order triangles by (tri_err
 * desc, index asc), skip tri_err == 0 or no empty pixel, take the first b; fill any
 * shortfall with the globally largest-e empty pixels (ties: lowest pix). Output sorted
 * ascending. `is_vertex[p]` marks current mesh vertices. Returns the count written. */
i64 orc_select(i64 T, const double* tri_err, const i32* best, i64 N, const double* e_px,
               const uint8_t* is_vertex, i64 b, i32* out) {
    EI* cand = (EI*)malloc(sizeof(EI) * (size_t)(T + 1));
    i64 nc = 0;
    for (i64 t = 0; t < T; ++t)
        if (tri_err[t] > 0.0 && best[t] >= 0) { cand[nc].e = tri_err[t]; cand[nc].idx = t; ++nc; }
    qsort(cand, (size_t)nc, sizeof(EI), cmp_ei_desc);
    i64 k = 0;
    for (i64 q = 0; q < nc && k < b; ++q) out[k++] = best[cand[q].idx];
    free(cand);
    if (k < b) {
        uint8_t* taken = (uint8_t*)calloc((size_t)N, 1);
        for (i64 q = 0; q < k; ++q) taken[out[q]] = 1;
        EI* pc = (EI*)malloc(sizeof(EI) * (size_t)N);
        i64 np = 0;
        for (i64 p = 0; p < N; ++p)
            if (!is_vertex[p] && !taken[p]) { pc[np].e = e_px[p]; pc[np].idx = p; ++np; }
        qsort(pc, (size_t)np, sizeof(EI), cmp_ei_desc);
        for (i64 q = 0; q < np && k < b; ++q) out[k++] = (i32)pc[q].idx;
        free(pc); free(taken);
    }
    qsort(out, (size_t)k, sizeof(i32), cmp_i32);
    return k;
}

/* ------------------------------------------------------------------------- */
/* Tonal optimisation (Eqs. (4)-(5); reading A13)            */
/* B g = P_k g + P_u A_uu^{-1} (-A_uk g);  B^T r = P_k^T r - A_uk^T A_uu^{-1} P_u^T r */
/* ------------------------------------------------------------------------- */

typedef struct { int rtol_set; double rtol; int max_iter; int method; i64 solves; i64 iters; int status; } Inner;

static void apply_B(OrcSys* S, const double* g, double* u_px, double* u_vert, Inner* in) {
    int it; double rr;
    int st = orc_sys_solve(S, g, NULL, in->rtol, in->max_iter, in->method, u_vert, &it, &rr);
    if (st && !in->status) in->status = st;
    in->solves++; in->iters += it;
    i64 N = (i64)S->W * S->H;
    for (i64 p = 0; p < N; ++p) u_px[p] = pixel_value(S, (i32)p, u_vert);
}

/* P^T r: each pixel spreads r with its barycentric weights (vertex pixels: weight 1) */
static void raster_adjoint(const OrcSys* S, const double* r, double* w) {
    i64 N = (i64)S->W * S->H;
    for (i64 v = 0; v < S->nv; ++v) w[v] = 0.0;
    for (i64 p = 0; p < N; ++p) {
        if (S->vmap[p] >= 0) { w[S->vmap[p]] = w[S->vmap[p]] + r[p]; continue; }
        i64 t = S->owner[p];
        i32 va = S->tri[3 * t], vb = S->tri[3 * t + 1], vc = S->tri[3 * t + 2];
        i32 a = S->vpix[va], b = S->vpix[vb], c = S->vpix[vc];
        double D = (double)orient(S->W, a, b, c);
        double la = (double)orient(S->W, b, c, (i32)p) / D;
        double lb = (double)orient(S->W, c, a, (i32)p) / D;
        double lc = (double)orient(S->W, a, b, (i32)p) / D;
        w[va] = w[va] + la * r[p];
        w[vb] = w[vb] + lb * r[p];
        w[vc] = w[vc] + lc * r[p];
    }
}

static void apply_BT(OrcSys* S, const double* r, double* s, double* w, double* y, Inner* in) {
    raster_adjoint(S, r, w);
    for (i64 i = 0; i < S->n_u; ++i) y[i] = 0.0;
    int it; double rr;
    int st = solve_uu(S, w, y, in->rtol, in->max_iter, in->method, &it, &rr);
    if (st && !in->status) in->status = st;
    in->solves++; in->iters += it;
    for (i64 k = 0; k < S->m; ++k) s[k] = w[S->n_u + k];
    for (i64 i = 0; i < S->n_u; ++i)
        for (i64 q = S->uk_ptr[i]; q < S->uk_ptr[i + 1]; ++q)
            s[S->uk_col[q]] = s[S->uk_col[q]] - S->uk_val[q] * y[i];
}

int orc_sys_apply_B(OrcSys* S, const double* g, double* u_px, double rtol) {
    double* uv = (double*)malloc(sizeof(double) * (size_t)S->nv);
    Inner in = {1, rtol, 100000, 0, 0, 0, 0};
    apply_B(S, g, u_px, uv, &in);
    free(uv);
    return in.status;
}

int orc_sys_apply_BT(OrcSys* S, const double* r, double* s, double rtol) {
    double* w = (double*)malloc(sizeof(double) * (size_t)S->nv);
    double* y = (double*)malloc(sizeof(double) * (size_t)(S->n_u + 1));
    Inner in = {1, rtol, 100000, 0, 0, 0, 0};
    apply_BT(S, r, s, w, y, &in);
    free(w); free(y);
    return in.status;
}

/* CGLS form of CG on the normal equations B^T B g = B^T f (Eq. (5)), started from
 * g0 = f at the mask pixels (g_inout on entry), stopped when ||B^T(f - B g)|| /
 * ||B^T f|| < outer_tol on the recursive gradient; at exit the gradient and MSE are
 * recomputed with fresh solves. report[0..7] = outer_iters, inner_solves, inner_iters,
 * rel_grad, mse_before, mse_after, status, rel_grad_recursive. */
/* Weighted CGLS (IRLS step, NEXT-2): minimise || W^1/2 (B g - f) ||^2 with per-pixel sqrt
 * weights sw (NULL = all ones: plain tonal optimisation). B_w = diag(sw) B, f_w = sw f. */
int orc_sys_tonal_w(OrcSys* S, const double* f, const double* sw, double* g, double outer_tol, int outer_max,
                    double inner_rtol, int inner_method, double* report);

int orc_sys_tonal(OrcSys* S, const double* f, double* g, double outer_tol, int outer_max,
                  double inner_rtol, int inner_method, double* report) {
    return orc_sys_tonal_w(S, f, NULL, g, outer_tol, outer_max, inner_rtol, inner_method, report);
}

int orc_sys_tonal_w(OrcSys* S, const double* f, const double* sw, double* g, double outer_tol, int outer_max,
                    double inner_rtol, int inner_method, double* report) {
    i64 N = (i64)S->W * S->H, m = S->m;
    double* u = (double*)malloc(sizeof(double) * (size_t)N);
    double* r = (double*)malloc(sizeof(double) * (size_t)N);
    double* q = (double*)malloc(sizeof(double) * (size_t)N);
    double* s = (double*)malloc(sizeof(double) * (size_t)m);
    double* pdir = (double*)malloc(sizeof(double) * (size_t)m);
    double* uv = (double*)malloc(sizeof(double) * (size_t)S->nv);
    double* w = (double*)malloc(sizeof(double) * (size_t)S->nv);
    double* y = (double*)malloc(sizeof(double) * (size_t)(S->n_u + 1));
    Inner in = {1, inner_rtol, 100000, inner_method, 0, 0, 0};
    double* fw = (double*)malloc(sizeof(double) * (size_t)N); /* W^1/2 f */
    for (i64 p = 0; p < N; ++p) fw[p] = sw ? sw[p] * f[p] : f[p];
    apply_B(S, g, u, uv, &in);
    for (i64 p = 0; p < N; ++p) r[p] = f[p] - u[p];
    double mse_before = dot(N, r, r) / (double)N;
    if (sw) for (i64 p = 0; p < N; ++p) r[p] = sw[p] * r[p];
    for (i64 p = 0; p < N; ++p) q[p] = sw ? sw[p] * fw[p] : fw[p]; /* B_w^T f_w = B^T (W f) */
    apply_BT(S, q, s, w, y, &in); /* ||B_w^T f_w|| for the relative stopping rule */
    double btf = sqrt(dot(m, s, s));
    for (i64 p = 0; p < N; ++p) q[p] = sw ? sw[p] * r[p] : r[p];
    apply_BT(S, q, s, w, y, &in);
    for (i64 k = 0; k < m; ++k) pdir[k] = s[k];
    double gam = dot(m, s, s);
    int outer = 0;
    double relg = btf > 0.0 ? sqrt(gam) / btf : 0.0;
    while (relg >= outer_tol && outer < outer_max) {
        apply_B(S, pdir, q, uv, &in);
        if (sw) for (i64 p = 0; p < N; ++p) q[p] = sw[p] * q[p];
        double qq = dot(N, q, q);
        if (!(qq > 0.0)) break;
        double alpha = gam / qq;
        for (i64 k = 0; k < m; ++k) g[k] = g[k] + alpha * pdir[k];
        for (i64 p = 0; p < N; ++p) r[p] = r[p] - alpha * q[p];
        if (sw) {
            for (i64 p = 0; p < N; ++p) q[p] = sw[p] * r[p];
            apply_BT(S, q, s, w, y, &in);
        } else {
            apply_BT(S, r, s, w, y, &in);
        }
        double gam2 = dot(m, s, s);
        ++outer;
        relg = sqrt(gam2) / btf;
        if (relg < outer_tol) { gam = gam2; break; }
        double beta = gam2 / gam;
        for (i64 k = 0; k < m; ++k) pdir[k] = s[k] + beta * pdir[k];
        gam = gam2;
    }
    double relg_rec = relg;
    apply_B(S, g, u, uv, &in);
    for (i64 p = 0; p < N; ++p) r[p] = f[p] - u[p];
    double mse_after = dot(N, r, r) / (double)N;
    for (i64 p = 0; p < N; ++p) q[p] = sw ? (sw[p] * sw[p]) * r[p] : r[p];
    apply_BT(S, q, s, w, y, &in);
    report[0] = outer; report[1] = (double)in.solves; report[2] = (double)in.iters;
    report[3] = btf > 0.0 ? sqrt(dot(m, s, s)) / btf : 0.0;
    report[4] = mse_before; report[5] = mse_after; report[6] = in.status; report[7] = relg_rec;
    free(u); free(r); free(q); free(s); free(pdir); free(uv); free(w); free(y); free(fw);
    return in.status;
}

/* L1 tonal optimisation by iteratively reweighted least squares ("optimised
 * the L1 error instead of the L2 one"; the method is unstated there, IRLS with weights
 * w_i = 1 / max(|r_i|, eps) is SPEC.md:L366-374's reading, R3): each of `irls`
 * steps computes r = f - B g, sets sqrt weights 1/sqrt(max(|r_i|, eps)) and runs the weighted
 * CGLS from the current g. report: [0] outer iterations (all steps), [1] inner solves,
 * [2] inner CG iterations, [3] L1 before, [4] L1 after (mean |f - B g|), [5] MSE after. */
int orc_sys_tonal_l1(OrcSys* S, const double* f, double* g, int irls, double eps, double outer_tol, int outer_max,
                     double inner_rtol, double* report) {
    i64 N = (i64)S->W * S->H;
    double* u = (double*)malloc(sizeof(double) * (size_t)N);
    double* sw = (double*)malloc(sizeof(double) * (size_t)N);
    double* uv = (double*)malloc(sizeof(double) * (size_t)S->nv);
    double rep[8];
    int st = 0;
    double outer = 0, solves = 0, iters = 0, l1_before = 0.0;
    Inner in = {1, inner_rtol, 100000, 0, 0, 0, 0};
    for (int k = 0; k <= irls; ++k) {
        apply_B(S, g, u, uv, &in);
        double l1 = 0.0;
        for (i64 p = 0; p < N; ++p) l1 = l1 + fabs(f[p] - u[p]);
        if (k == 0) l1_before = l1 / (double)N;
        if (k == irls) {
            double mse = 0.0;
            for (i64 p = 0; p < N; ++p) mse = mse + (f[p] - u[p]) * (f[p] - u[p]);
            report[4] = l1 / (double)N;
            report[5] = mse / (double)N;
            break;
        }
        for (i64 p = 0; p < N; ++p) {
            double a = fabs(f[p] - u[p]);
            sw[p] = 1.0 / sqrt(a > eps ? a : eps);
        }
        int s1 = orc_sys_tonal_w(S, f, sw, g, outer_tol, outer_max, inner_rtol, 0, rep);
        if (s1 && !st) st = s1;
        outer += rep[0];
        solves += rep[1];
        iters += rep[2];
    }
    report[0] = outer; report[1] = solves + (double)in.solves; report[2] = iters + (double)in.iters;
    report[3] = l1_before;
    if (in.status && !st) st = in.status;
    free(u); free(sw); free(uv);
    return st;
}

