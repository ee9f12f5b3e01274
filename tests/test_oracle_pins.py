"""Pins of the oracle to what the paper and mathematics fix.

Each test checks the oracle against something other than itself: closed forms, a
different formula for the same quantity (gradient-form stiffness vs the oracle's cotangent
form), brute force, library routines, invariants. CPU only.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
from synth import make_config
from synth.generate import draw_mask, draw_unknowns

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")))


def xy(p, W):
    return (int(p) % W, int(p) // W)


def random_system(seed, W=12, H=10, m=8, p=10, brute=False):
    rng = np.random.default_rng(seed)
    mk = draw_mask(rng, W * H, m)
    un = draw_unknowns(rng, W, H, mk, p)
    return oracle.System(W, H, mk, un, brute=brute)


def full_matrix_gradient_form(S):
    """Independent assembly: K_T = area * G^T G with G the barycentric gradients from a
    3x3 inverse (not the cotangent formula the oracle uses)."""
    K = np.zeros((S.nv, S.nv))
    for t in S.tri:
        P = np.array([xy(S.vpix[v], S.W) for v in t], dtype=float)
        M = np.column_stack([np.ones(3), P])
        C = np.linalg.inv(M)  # column i = coefficients of phi_i
        G = C[1:, :]
        area = 0.5 * abs(np.linalg.det(M))
        K[np.ix_(t, t)] += area * G.T @ G
    return K


# ---------------------------------------------------------------- P1 / assembly pins

def test_p1_unit_right_triangle_local_matrix():
    """SPEC.md:L199. A 2x2 image is two unit right triangles."""
    g = GOLD["p1_unit_right_triangle"]
    Kloc = np.array(g["local_stiffness"])
    # corners (0,0)=0,(1,0)=1,(0,1)=2,(1,1)=3; SoS split keeps the diagonal through pix 0
    S = oracle.System(2, 2, [3], [0, 1, 2])
    assert sorted(map(tuple, S.tri_px().tolist())) == [(0, 1, 3), (0, 3, 2)]
    K = np.zeros((4, 4))
    # triangle (0,0),(1,0),(1,1): right angle at (1,0); map the closed form's right-angle vertex
    for tri_px, right in (((0, 1, 3), 1), ((0, 3, 2), 2)):
        others = [v for v in tri_px if v != right]
        order = [right] + others  # closed form lists the right-angle vertex first
        K[np.ix_(order, order)] += Kloc
    A = np.zeros((4, 4))
    A[:3, :3] = S.dense_uu()
    A[:3, 3:] = S.dense_uk()
    np.testing.assert_array_equal(A[:3], K[:3])


@pytest.mark.parametrize("seed", range(6))
def test_assembly_equals_gradient_form(seed):
    """cotangent assembly (oracle) == area * grad.grad assembly (independent), 1e-13."""
    S = random_system(seed, W=14, H=11, m=10, p=12)
    K = full_matrix_gradient_form(S)
    n = S.n_u
    np.testing.assert_allclose(S.dense_uu(), K[:n, :n], rtol=0, atol=1e-13)
    np.testing.assert_allclose(S.dense_uk(), K[:n, n:], rtol=0, atol=1e-13)


@pytest.mark.parametrize("seed", range(10))
def test_p2_symmetry_zero_rowsum_spd(seed):
    """SPEC.md:L200, L210, L231-232; PAPER.md:L236-237 (SPD with >= 1 mask pixel)."""
    S = random_system(100 + seed, W=16, H=13, m=7, p=15)
    A = S.dense_uu()
    np.testing.assert_array_equal(A, A.T)
    rows = A.sum(1) + S.dense_uk().sum(1)
    scale = np.abs(A).max()
    assert np.abs(rows).max() <= 1e-12 * scale
    np.linalg.cholesky(A)  # raises if not SPD


def test_csr_pattern_structural_zero_and_diagonal():
    """Reading A5: every unknown-unknown mesh edge is an entry even if its value is 0."""
    W = H = 4
    un = np.arange(W * H)
    un = un[un != 5]
    S = oracle.System(W, H, [5], un)
    # full grid: diagonal-neighbour edges (x,y)-(x+1,y+1) are structural zeros
    for i in range(S.n_u):
        cols = S.uu_col[S.uu_ptr[i]:S.uu_ptr[i + 1]]
        assert i in cols and np.all(np.diff(cols) > 0)
    zeros = np.sum(S.uu_val == 0.0)
    assert zeros > 0


# ---------------------------------------------------------------- P3 / P4 triangulation pins

def _incircle_exact(a, b, c, d):
    adx, ady = a[0] - d[0], a[1] - d[1]
    bdx, bdy = b[0] - d[0], b[1] - d[1]
    cdx, cdy = c[0] - d[0], c[1] - d[1]
    return ((adx * adx + ady * ady) * (bdx * cdy - cdx * bdy) + (bdx * bdx + bdy * bdy) * (cdx * ady - adx * cdy)
            + (cdx * cdx + cdy * cdy) * (adx * bdy - bdx * ady))


def _orient(a, b, c):
    return (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])


def check_triangulation(S, brute_empty=True):
    W, H = S.W, S.H
    P = [xy(p, W) for p in S.vpix]
    T = S.tri
    # CCW and canonical rotation/order
    for t in T:
        assert _orient(P[t[0]], P[t[1]], P[t[2]]) > 0
        assert S.vpix[t[0]] < S.vpix[t[1]] and S.vpix[t[0]] < S.vpix[t[2]]
    keys = [tuple(S.vpix[t]) for t in T]
    assert keys == sorted(keys)
    # areas tile the rectangle
    area2 = sum(_orient(P[t[0]], P[t[1]], P[t[2]]) for t in T)
    assert area2 == 2 * (W - 1) * (H - 1)
    # Euler: T = 2v - 2 - h, h = number of vertices on the border
    h = sum(1 for (x, y) in P if x in (0, W - 1) or y in (0, H - 1))
    assert len(T) == 2 * len(P) - 2 - h
    # each edge used by at most two triangles, border edges by one
    edges = {}
    for t in T:
        for k in range(3):
            e = tuple(sorted((t[(k + 1) % 3], t[(k + 2) % 3])))
            edges[e] = edges.get(e, 0) + 1
    assert max(edges.values()) <= 2
    if brute_empty:  # classical Delaunay: no vertex strictly inside any circumcircle
        for t in T:
            a, b, c = (P[v] for v in t)
            for q in P:
                assert _incircle_exact(a, b, c, q) <= 0


@pytest.mark.parametrize("seed", range(25))
def test_p3_delaunay_brute_force(seed):
    """empty circumcircles (exact), tiling, Euler, edge manifoldness;
    incremental (Lawson, Morton order) == brute force (no order) bit-exactly."""
    rng = np.random.default_rng(seed)
    W, H = int(rng.integers(3, 9)), int(rng.integers(3, 9))
    N = W * H
    m = int(rng.integers(1, max(2, N // 3)))
    p = int(rng.integers(4, max(5, N // 2)))
    mk = draw_mask(rng, N, m)
    if N - m < p:
        p = N - m
    un = draw_unknowns(rng, W, H, mk, min(p, N - m))
    S = oracle.System(W, H, mk, un)
    Sb = oracle.System(W, H, mk, un, brute=True)
    np.testing.assert_array_equal(S.tri, Sb.tri)
    check_triangulation(S)


def test_p3_sos_full_grid_main_diagonal():
    """Reading A3 consequence: the full grid splits every cell along (x,y)-(x+1,y+1);
    in each cocircular quad the diagonal through the smallest pixel wins."""
    W, H = 7, 5
    allpx = np.arange(W * H)
    S = oracle.System(W, H, [8], allpx[allpx != 8])
    check_triangulation(S)
    diag = set()
    for t in S.tri_px():
        for k in range(3):
            a, b = sorted((t[k], t[(k + 1) % 3]))
            (ax, ay), (bx, by) = xy(a, W), xy(b, W)
            if abs(ax - bx) == 1 and abs(ay - by) == 1:
                diag.add((a, b))
                assert bx == ax + 1 and by == ay + 1
    assert len(diag) == (W - 1) * (H - 1)


def test_p3_cocircular_diamond_and_octagon():
    """8 cocircular lattice points (x^2+y^2 = 25 family shifted) -> 6 triangles; diamond
    quad -> diagonal through the smallest pixel."""
    W, H = 11, 11
    c = (5, 5)
    ring = [(c[0] + dx, c[1] + dy) for dx, dy in
            [(3, 4), (4, 3), (4, -3), (3, -4), (-3, -4), (-4, -3), (-4, 3), (-3, 4)]]
    ring_px = [y * W + x for x, y in ring]
    vpix = np.array(sorted(ring_px), dtype=np.int32)
    tri = oracle.delaunay(W, H, vpix, brute=True)
    assert tri.shape[0] == 6
    # every triangle uses the smallest-pix point (fan from it), as the SoS rule implies
    assert all(0 in t for t in tri)
    quad = sorted([2 * W + 5, 5 * W + 2, 5 * W + 8, 8 * W + 5])  # diamond around (5,5)
    tri = oracle.delaunay(W, H, np.array(quad, np.int32), brute=True)
    assert tri.shape[0] == 2 and all(0 in t for t in tri)


def _segments_cross(p, q, r, s):
    d1, d2 = _orient(p, q, r), _orient(p, q, s)
    d3, d4 = _orient(r, s, p), _orient(r, s, q)
    return d1 * d2 < 0 and d3 * d4 < 0


def _all_triangulations(P):
    n = len(P)
    segs = [(i, j) for i in range(n) for j in range(i + 1, n)]
    cross = {(a, b): _segments_cross(P[a[0]], P[a[1]], P[b[0]], P[b[1]]) for a in segs for b in segs}
    out = []

    def rec(k, chosen):
        if k == len(segs):
            if all(any(cross[(s, c)] for c in chosen) for s in segs if s not in chosen):
                out.append(list(chosen))
            return
        s = segs[k]
        if not any(cross[(s, c)] for c in chosen):
            chosen.append(s)
            rec(k + 1, chosen)
            chosen.pop()
        rec(k + 1, chosen)

    rec(0, [])
    tris = []
    for E in out:
        Es = set(E)
        T = []
        for a, b, c in itertools.combinations(range(n), 3):
            if (a, b) in Es and (a, c) in Es and (b, c) in Es and _orient(P[a], P[b], P[c]) != 0:
                inside = any(all(o > 0 for o in (_orient(P[a], P[b], P[d]), _orient(P[b], P[c], P[d]),
                                                 _orient(P[c], P[a], P[d]))) or
                             all(o < 0 for o in (_orient(P[a], P[b], P[d]), _orient(P[b], P[c], P[d]),
                                                 _orient(P[c], P[a], P[d])))
                             for d in range(n) if d not in (a, b, c))
                if not inside:
                    T.append((a, b, c))
        tris.append(T)
    return tris


def _min_angle(P, T):
    best = math.pi
    for t in T:
        for k in range(3):
            a, b, c = (np.array(P[t[(k + j) % 3]], float) for j in range(3))
            u, v = b - a, c - a
            ang = math.acos(max(-1.0, min(1.0, u @ v / (np.linalg.norm(u) * np.linalg.norm(v)))))
            best = min(best, ang)
    return best


@pytest.mark.parametrize("seed", range(6))
def test_p4_max_min_angle_exhaustive(seed):
    """PAPER.md:L222-223 "maximising the minimum angle": exhaustive over all
    triangulations of <= 7 points in general position."""
    rng = np.random.default_rng(1000 + seed)
    W = H = 9
    while True:
        px = np.sort(rng.choice(W * H, size=int(rng.integers(5, 8)), replace=False))
        P = [xy(p, W) for p in px]
        ok = all(_orient(*c) != 0 for c in itertools.combinations(P, 3))
        ok = ok and all(_incircle_exact(*c) != 0 for c in itertools.combinations(P, 4))
        if ok:
            break
    tri = oracle.delaunay(W, H, px.astype(np.int32), brute=True)
    dmin = _min_angle(P, [tuple(t) for t in tri])
    for T in _all_triangulations(P):
        assert _min_angle(P, T) <= dmin + 1e-12


# ---------------------------------------------------------------- P5 full grid = FDM

def test_p5_full_grid_rows_are_fdm_stencil():
    """all non-mask pixels unknown -> 5-point FDM stencil (row-scaled
    1/2 on borders, 1/4 at corners)."""
    gr = GOLD["full_grid_rows"]
    W, H = 6, 5
    allpx = np.arange(W * H)
    mask = [W * H - 1]  # one Dirichlet pixel (corner) so that A_uu exists for every other row
    S = oracle.System(W, H, mask, allpx[:-1])
    A = np.zeros((W * H, W * H))
    A[: S.n_u, : S.n_u] = S.dense_uu()
    A[: S.n_u, S.n_u:] = S.dense_uk()
    for p in range(W * H - 1):
        x, y = xy(p, W)
        row = A[p]
        bx, by = x in (0, W - 1), y in (0, H - 1)
        if not bx and not by:
            assert row[p] == gr["interior"]["diag"]
            for q in (p - 1, p + 1, p - W, p + W):
                assert row[q] == gr["interior"]["axis"]
            assert row[p + W + 1] == 0.0 and row[p - W - 1] == 0.0
            assert np.count_nonzero(row) == 5
        elif bx and by:
            s = gr["corner"]["scale"]
            assert row[p] == s * gr["corner"]["diag"]
            assert np.count_nonzero(row) == 3 and row.sum() == 0.0
            assert set(row[row != 0][row[row != 0] < 0]) == {s * gr["corner"]["neighbours"]}
        else:
            s = gr["border"]["scale"]
            assert row[p] == s * gr["border"]["diag"]
            inward = (p + 1 if x == 0 else p - 1) if bx else (p + W if y == 0 else p - W)
            assert row[inward] == s * gr["border"]["inward"]
            assert np.count_nonzero(row) == 4


@pytest.mark.parametrize("seed", range(4))
def test_p5_full_grid_inpainting_equals_dense_fdm(seed):
    """FEM inpainting on the full grid == dense 5-point FDM with reflecting boundary."""
    rng = np.random.default_rng(seed)
    W, H = 16, 12
    f = rng.uniform(0, 255, (H, W))
    mk = draw_mask(rng, W * H, 12)
    allpx = np.arange(W * H)
    R = oracle.inpaint(W, H, f, mk, np.setdiff1d(allpx, mk))
    ufdm = oracle.fdm_inpaint_dense(f, mk)
    assert np.abs(R["u_px"] - ufdm.reshape(-1)).max() <= 1e-9


# ---------------------------------------------------------------- P6 closed forms for the solve

def test_p6_single_unknown_on_grid_is_axis_mean():
    W = H = 3
    f = np.arange(9, dtype=float).reshape(3, 3) ** 1.5
    mk = [0, 1, 2, 3, 5, 6, 7, 8]
    R = oracle.inpaint(W, H, f, mk, [4])
    fv = f.reshape(-1)
    assert abs(R["u_vert"][0] - (fv[1] + fv[3] + fv[5] + fv[7]) / 4) <= 1e-14


@pytest.mark.parametrize("seed", range(5))
def test_p6_single_unknown_cotan_weighted_mean(seed):
    """one unknown with mask neighbours -> sum w_j g_j / sum w_j with
    w_j = (cot a + cot b)/2 computed here from angles (arctan2), not integer formulas."""
    rng = np.random.default_rng(seed)
    W = H = 9
    centre = 4 * W + 4
    others = rng.choice(np.setdiff1d(np.arange(W * H), [centre, 0, 8, 72, 80]), size=8, replace=False)
    mk = np.concatenate([[0, 8, 72, 80], others])
    g_img = rng.uniform(0, 255, W * H)
    S = oracle.System(W, H, mk, [centre])
    u, st, it, rr = S.solve(g_img[S.mask_px])
    P = {p: np.array(xy(p, W), float) for p in S.vpix}
    wsum, acc = 0.0, 0.0
    nbr = {}
    for t in S.tri_px():
        if centre not in t:
            continue
        k = list(t).index(centre)
        a, b = t[(k + 1) % 3], t[(k + 2) % 3]
        for j, o in ((a, b), (b, a)):
            u1, u2 = P[centre] - P[o], P[j] - P[o]
            ang = math.atan2(abs(u1[0] * u2[1] - u1[1] * u2[0]), u1 @ u2)
            nbr[j] = nbr.get(j, 0.0) + 0.5 / math.tan(ang)
    for j, w in nbr.items():
        wsum += w
        acc += w * g_img[j]
    assert abs(u[0] - acc / wsum) <= 1e-10


def test_p6_cholesky_and_cg_agree():
    c = make_config(1)
    S = oracle.System(c["W"], c["H"], c["mask"], c["unknowns"])
    g = c["f"].reshape(-1)[S.mask_px]
    u1, *_ = S.solve(g, method=1)
    u2, st, it, rr = S.solve(g, method=2, rtol=1e-13)
    A = S.dense_uu()
    x = np.linalg.solve(A, -S.dense_uk() @ g)
    assert np.abs(u1[: S.n_u] - x).max() <= 1e-9
    assert np.abs(u2[: S.n_u] - x).max() <= 1e-9


@pytest.mark.parametrize("seed", range(3))
def test_jacobi_pcg_reaches_the_same_solution(seed):
    """Reading A11: Jacobi preconditioning changes the iterates, not the solution. The oracle's
    Jacobi-PCG (method 3) meets the true relative residual and agrees with numpy's dense solve
    (a library routine, independent of the oracle's C code) and with the dense FDM on the full
    grid (P5); a constant image still exits at 0 iterations (A16)."""
    rng = np.random.default_rng(seed)
    c = make_config(4, W=48, H=40, seed=70 + seed)
    S = oracle.System(48, 40, c["mask"], c["unknowns"])
    g = c["f"].reshape(-1)[S.mask_px]
    u3, st, it, rr = S.solve(g, method=3, rtol=1e-12)
    assert st == 0 and rr <= 1e-12 and it > 0
    x = np.linalg.solve(S.dense_uu(), -S.dense_uk() @ g)
    assert np.abs(u3[: S.n_u] - x).max() <= 1e-8
    u2, _, it2, _ = S.solve(g, method=2, rtol=1e-12)
    assert it < it2  # preconditioning pays on these meshes (kappa 477 -> 24 class)
    W, H = 16, 12
    f = rng.uniform(0, 255, (H, W))
    mk = draw_mask(rng, W * H, 12)
    Sf = oracle.System(W, H, mk, np.setdiff1d(np.arange(W * H), mk))
    uf, *_ = Sf.solve(f.reshape(-1)[Sf.mask_px], method=3, rtol=1e-13)
    Rf = Sf.raster(uf, f)
    assert np.abs(Rf["u_px"] - oracle.fdm_inpaint_dense(f, mk).reshape(-1)).max() <= 1e-9
    uc, st, itc, _ = S.solve(np.full(S.m, 42.5), method=3)
    assert itc == 0 and np.all(uc == 42.5)


def test_cg_2x2_golden_via_dense():
    """SPEC.md:L218 closed form; confirms the numpy dense path used in these pins."""
    g = GOLD["cg_2x2"]
    x = np.linalg.solve(np.array(g["A"]), np.array(g["b"]))
    np.testing.assert_allclose(x, g["x"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(x, [1 / 11, 7 / 11], rtol=0, atol=1e-15)


# ---------------------------------------------------------------- P7 / P8 special cases

@pytest.mark.parametrize("c0", [0.0, 17.25, 254.999])
def test_p7_constant_image_exact(c0):
    """Constants are harmonic and linear elements reproduce them exactly (reading A16)."""
    cfg = make_config(1)
    f = np.full((cfg["H"], cfg["W"]), c0)
    R = oracle.inpaint(cfg["W"], cfg["H"], f, cfg["mask"], cfg["unknowns"])
    assert np.all(R["u_px"] == c0) and R["sse"] == 0.0 and R["iters"] == 0


def test_p7_single_mask_pixel_constant():
    """one Dirichlet pixel + Neumann border -> constant image."""
    rng = np.random.default_rng(3)
    W, H = 20, 15
    f = rng.uniform(0, 255, (H, W))
    mk = [7 * W + 9]
    un = draw_unknowns(rng, W, H, np.array(mk), 30)
    R = oracle.inpaint(W, H, f, mk, un)
    assert np.all(R["u_px"] == f.reshape(-1)[mk[0]])


def test_p8_full_mask_returns_image():
    """Every pixel a mask vertex (n_u = 0) -> u = f bit-exactly, MSE 0."""
    rng = np.random.default_rng(4)
    W, H = 9, 7
    f = rng.uniform(0, 255, (H, W))
    R = oracle.inpaint(W, H, f, np.arange(W * H), [])
    assert R["system"].n_u == 0
    assert np.array_equal(R["u_px"], f.reshape(-1)) and R["sse"] == 0.0


# ---------------------------------------------------------------- P9 linearity, P10 barycentrics

def test_p9_linearity():
    S = random_system(7, W=20, H=16, m=20, p=25)
    rng = np.random.default_rng(0)
    g1, g2 = rng.uniform(0, 255, S.m), rng.uniform(0, 255, S.m)
    u1 = S.solve(g1)[0]
    u2 = S.solve(g2)[0]
    u3 = S.solve(0.3 * g1 - 1.7 * g2)[0]
    assert np.abs(u3 - (0.3 * u1 - 1.7 * u2)).max() <= 1e-9


def test_p10_owner_partition_and_vertex_values():
    S = random_system(8, W=24, H=19, m=25, p=25)
    assert np.all(S.owner >= 0) and np.all(S.owner < S.T)
    counts = np.bincount(S.owner, minlength=S.T)
    assert counts.sum() == S.W * S.H
    # owner is the lowest-index closed triangle (reading A7), checked by exhaustive scan
    P = {p: xy(p, S.W) for p in S.vpix}
    for pix in range(S.W * S.H):
        q = xy(pix, S.W)
        for t, tp in enumerate(S.tri_px()):
            a, b, c = (P[v] for v in tp)
            if _orient(b, c, q) >= 0 and _orient(c, a, q) >= 0 and _orient(a, b, q) >= 0:
                assert S.owner[pix] == t
                break
    rng = np.random.default_rng(1)
    u = rng.uniform(0, 255, S.nv)
    R = S.raster(u, np.zeros(S.W * S.H))
    assert np.array_equal(R["u_px"][S.vpix], u)


def test_p10_centroid_barycentrics():
    """(0,0),(3,0),(3,3) is a mesh triangle (diagonal through pix 0, reading A3) with centroid
    pixel (2,1): u there = mean of its vertex values (1e-12)."""
    W = H = 4
    S = oracle.System(W, H, [0], [3, 12, 15])
    u = np.array([11.0, 40.0, 95.0, 3.0])  # unknowns 3,12,15 then mask 0
    R = S.raster(u, np.zeros(W * H))
    assert (0, 3, 15) in [tuple(t) for t in S.tri_px()]
    assert abs(R["u_px"][1 * W + 2] - (3.0 + 11.0 + 95.0) / 3) <= 1e-12


# ---------------------------------------------------------------- P11 error identities

def test_p11_mse_golden_and_sums():
    g = GOLD["mse_example"]
    assert np.mean((np.array(g["a"]) - np.array(g["b"])) ** 2) == g["mse"]
    c = make_config(1)
    R = oracle.inpaint(c["W"], c["H"], c["f"], c["mask"], c["unknowns"])
    N = c["W"] * c["H"]
    e = (R["u_px"] - c["f"].reshape(-1)) ** 2
    np.testing.assert_array_equal(R["e_px"], e)
    assert abs(R["e_px"].sum() - N * R["mse"]) <= 1e-12 * N * R["mse"]
    assert abs(R["tri_err"].sum() - R["sse"]) <= 1e-12 * R["sse"]
    S = R["system"]
    # per-triangle sums and argmax by brute force over the owner map
    isv = S.is_vertex()
    for t in range(0, S.T, 7):
        pix = np.nonzero(S.owner == t)[0]
        assert abs(R["tri_err"][t] - e[pix].sum()) <= 1e-12 * max(1.0, e[pix].sum())
        cand = pix[isv[pix] == 0]
        if cand.size == 0:
            assert R["best"][t] == -1
        else:
            assert R["best"][t] == cand[np.argmax(e[cand])]


# ---------------------------------------------------------------- L1 tonal via IRLS (NEXT-2)

def test_weighted_tonal_unit_weights_is_tonal():
    """W = I: the weighted CGLS is the plain one, bit for bit (x 1.0 is exact)."""
    cfg = make_config(4, W=40, H=32, seed=12)
    S = oracle.System(40, 32, cfg["mask"], cfg["unknowns"])
    g0, r0 = S.tonal(cfg["f"], outer_tol=1e-8)
    g1, r1 = oracle.tonal_weighted(S, cfg["f"], np.ones(40 * 32), outer_tol=1e-8)
    np.testing.assert_array_equal(g0, g1)
    assert r0["outer_iters"] == r1["outer_iters"]


@pytest.mark.parametrize("seed", range(3))
def test_weighted_tonal_matches_weighted_dense_lstsq(seed):
    """IRLS step = argmin ||W^1/2 (B g - f)|| by lstsq on the materialised dense B (<= 16x16)."""
    cfg = make_config(4, W=16, H=16, seed=70 + seed)
    S = oracle.System(16, 16, cfg["mask"], cfg["unknowns"])
    B = oracle.materialise_B(S)
    f = cfg["f"].reshape(-1)
    sw = np.random.default_rng(seed).uniform(0.2, 3.0, f.size)
    gstar = np.linalg.lstsq(sw[:, None] * B, sw * f, rcond=None)[0]
    g, rep = oracle.tonal_weighted(S, f, sw, outer_tol=1e-11)
    assert np.abs(g - gstar).max() <= 1e-4


def test_irls_uniform_weights_is_l2_and_l1_improves():
    """eps >= max |r| makes every IRLS weight 1/eps: the weighted minimiser is the L2 one
    (SPEC.md:L374); with eps = 1 three IRLS steps end with an L1 error no larger than the L2
    solution's."""
    cfg = make_config(4, W=48, H=40, seed=21)
    S = oracle.System(48, 40, cfg["mask"], cfg["unknowns"])
    f = cfg["f"].reshape(-1)
    g2, _ = S.tonal(cfg["f"], outer_tol=1e-10)
    gu, rep_u = oracle.tonal_l1(S, f, irls=1, eps=1e6, outer_tol=1e-10)
    assert np.abs(gu - g2).max() <= 1e-6
    g1, rep1 = oracle.tonal_l1(S, f, irls=3, eps=1.0, outer_tol=1e-10)
    l1_of_l2 = np.abs(f - S.apply_B(g2)).mean()
    assert rep1["l1_after"] <= l1_of_l2 + 1e-9
    assert rep1["l1_after"] <= rep1["l1_before"]
    assert abs(rep1["l1_after"] - np.abs(f - S.apply_B(g1)).mean()) <= 1e-9


# ---------------------------------------------------------------- colour (NEXT-1)

def test_colour_raster_pins():
    """PAPER.md:L521-524 colour = channels on one mesh; error map = channel sum.
    Pinned against the grey raster: one channel equals it bit for bit; C channels give the
    channel-order sum of the per-channel error maps, per-triangle sums in pixel order, the
    first strict maximum over non-vertex pixels, and SSE as the pixel-order sum."""
    c = make_config(1)
    W, H = c["W"], c["H"]
    N = W * H
    S = oracle.System(W, H, c["mask"], c["unknowns"])
    rng = np.random.default_rng(3)
    fs = [c["f"].reshape(-1), rng.uniform(0, 255, N), np.full(N, 17.0)]
    us = [S.solve(f[S.mask_px])[0] for f in fs]
    R1 = S.raster(us[0], fs[0])
    C1 = S.raster_channels(us[:1], fs[:1])
    for k in ("e_px", "tri_err", "best"):
        np.testing.assert_array_equal(C1[k], R1[k])
    np.testing.assert_array_equal(C1["u_px"][0], R1["u_px"])
    assert C1["sse"] == R1["sse"]
    per = [S.raster(u, f) for u, f in zip(us, fs)]
    C3 = S.raster_channels(us, fs)
    e = (per[0]["e_px"] + per[1]["e_px"]) + per[2]["e_px"]
    np.testing.assert_array_equal(C3["e_px"], e)
    for k in range(3):
        np.testing.assert_array_equal(C3["u_px"][k], per[k]["u_px"])
    te = np.zeros(S.T)
    np.add.at(te, S.owner, e)  # unbuffered, in pixel order
    np.testing.assert_array_equal(C3["tri_err"], te)
    isv = S.is_vertex()
    for t in range(S.T):
        pix = np.nonzero(S.owner == t)[0]
        cand = pix[isv[pix] == 0]
        assert C3["best"][t] == (cand[np.argmax(e[cand])] if cand.size else -1)
    assert C3["sse"] == float(np.cumsum(e)[-1])
    # three identical channels: e = fl(3 e_1) (2 e_1 is exact)
    C33 = S.raster_channels([us[0]] * 3, [fs[0]] * 3)
    np.testing.assert_array_equal(C33["e_px"], 3.0 * R1["e_px"])


# ---------------------------------------------------------------- P12 conditional DMP

def _m_matrix(S):
    offd = S.dense_uu() - np.diag(np.diag(S.dense_uu()))
    return offd.max() <= 0.0 and (S.uk_val.size == 0 or S.uk_val.max() <= 0.0)


@pytest.mark.parametrize("seed", range(30))
def test_p12_dmp_on_m_matrix_meshes(seed):
    """Reading A12: the DMP holds when all off-diagonals are <= 0; asserted only then."""
    rng = np.random.default_rng(500 + seed)
    W, H = int(rng.integers(4, 9)), int(rng.integers(4, 9))
    N = W * H
    mk = draw_mask(rng, N, int(rng.integers(2, N // 3)))
    un = np.setdiff1d(np.arange(N), mk) if seed % 2 == 0 else draw_unknowns(rng, W, H, mk, (N - mk.size) // 2)
    f = rng.uniform(0, 255, (H, W))
    R = oracle.inpaint(W, H, f, mk, un)
    if _m_matrix(R["system"]):
        g = f.reshape(-1)[mk]
        assert R["u_px"].min() >= g.min() - 1e-9 and R["u_px"].max() <= g.max() + 1e-9


def test_p12_full_grid_is_m_matrix_and_dmp():
    rng = np.random.default_rng(9)
    W, H = 12, 10
    mk = draw_mask(rng, W * H, 9)
    f = rng.uniform(0, 255, (H, W))
    R = oracle.inpaint(W, H, f, mk, np.setdiff1d(np.arange(W * H), mk))
    assert _m_matrix(R["system"])
    g = f.reshape(-1)[mk]
    assert R["u_px"].min() >= g.min() - 1e-9 and R["u_px"].max() <= g.max() + 1e-9


# ---------------------------------------------------------------- P13-P15 tonal

@pytest.mark.parametrize("seed", range(3))
def test_p13_tonal_matches_dense_lstsq(seed):
    """PAPER.md:L290-302 Eqs. (4)-(5): CGLS g == argmin ||Bg - f|| by lstsq on dense B."""
    rng = np.random.default_rng(seed)
    W, H = 16, 16
    cfg = make_config(4, W=W, H=H, seed=40 + seed)
    S = oracle.System(W, H, cfg["mask"], cfg["unknowns"])
    B = oracle.materialise_B(S)
    f = cfg["f"].reshape(-1)
    gstar = np.linalg.lstsq(B, f, rcond=None)[0]
    g, rep = S.tonal(cfg["f"], outer_tol=1e-10)
    assert np.abs(g - gstar).max() <= 1e-4
    assert rep["mse_after"] <= rep["mse_before"] + 1e-12
    # B has identity rows at the mask pixels -> B^T B >= I
    assert np.linalg.eigvalsh(B.T @ B).min() >= 1.0 - 1e-9
    np.testing.assert_array_equal(B[S.mask_px], np.eye(S.m))


def test_colour_tonal_is_the_joint_least_squares():
    """NEXT-1 colour tonal (reading R4): the joint problem min sum_c ||B g_c - f_c||^2 over all
    channels, solved densely as ONE block-diagonal least-squares system with numpy, equals the
    oracle's per-channel solutions (and a channel permutation permutes them)."""
    cfg = make_config(4, W=14, H=12, seed=77)
    S = oracle.System(14, 12, cfg["mask"], cfg["unknowns"])
    rng = np.random.default_rng(77)
    fs = [cfg["f"].reshape(-1), rng.uniform(0, 255, 14 * 12), np.clip(cfg["f"].reshape(-1) * 0.5 + 40, 0, 255)]
    B = oracle.materialise_B(S)
    Z = np.zeros_like(B)
    Bj = np.block([[B, Z, Z], [Z, B, Z], [Z, Z, B]])
    gj = np.linalg.lstsq(Bj, np.concatenate(fs), rcond=None)[0]
    gs, reps = oracle.tonal_channels(S, fs, outer_tol=1e-10)
    for c in range(3):
        assert np.abs(gs[c] - gj[c * S.m:(c + 1) * S.m]).max() <= 1e-4
        assert reps[c]["mse_after"] <= reps[c]["mse_before"]
    gp, _ = oracle.tonal_channels(S, [fs[2], fs[0], fs[1]], outer_tol=1e-10)
    np.testing.assert_array_equal(gp[1], gs[0])


def test_p14_adjoint_identity_and_partition_of_unity():
    cfg = make_config(4, W=40, H=32, seed=77)
    S = oracle.System(40, 32, cfg["mask"], cfg["unknowns"])
    rng = np.random.default_rng(2)
    for _ in range(4):
        x = rng.normal(size=S.m)
        y = rng.normal(size=S.W * S.H)
        lhs = S.apply_B(x) @ y
        rhs = x @ S.apply_BT(y)
        assert abs(lhs - rhs) <= 1e-9 * (abs(lhs) + abs(rhs))
    one = S.apply_B(np.ones(S.m))
    assert np.all(one == 1.0)


def test_p15_tonal_consistent_system_and_monotone():
    cfg = make_config(4, W=48, H=40, seed=5)
    S = oracle.System(48, 40, cfg["mask"], cfg["unknowns"])
    rng = np.random.default_rng(3)
    g0 = rng.uniform(0, 255, S.m)
    f = S.apply_B(g0)
    g, rep = S.tonal(f, g0=np.zeros(S.m), outer_tol=1e-10)
    assert rep["mse_after"] <= 1e-12
    g, rep = S.tonal(cfg["f"], outer_tol=1e-8)
    assert rep["mse_after"] <= rep["mse_before"]
    assert rep["rel_grad"] < 1e-7
    assert rep["inner_solves"] == 3 + 2 * rep["outer_iters"] + 2


# ---------------------------------------------------------------- P16 densification + select

def _select_bruteforce(tri_err, best, e_px, isv, b):
    order = sorted([t for t in range(len(tri_err)) if tri_err[t] > 0 and best[t] >= 0],
                   key=lambda t: (-tri_err[t], t))
    out = [int(best[t]) for t in order[:b]]
    if len(out) < b:
        taken = set(out)
        rest = sorted([p for p in range(len(e_px)) if not isv[p] and p not in taken], key=lambda p: (-e_px[p], p))
        out += rest[: b - len(out)]
    return sorted(out)


@pytest.mark.parametrize("seed", range(4))
def test_select_matches_bruteforce(seed):
    c = make_config(3, W=48, H=40, seed=seed)
    S = oracle.System(48, 40, c["mask0"], c["unknowns"])
    f = c["f"].reshape(-1)
    u = S.solve(f[S.mask_px])[0]
    R = S.raster(u, f)
    for b in (1, 5, 40, S.T + 50):
        got = oracle.select(R["tri_err"], R["best"], R["e_px"], S.is_vertex(), b)
        assert got.tolist() == _select_bruteforce(R["tri_err"], R["best"], R["e_px"], S.is_vertex(), b)


def test_p16_densify_properties():
    c = make_config(3, W=64, H=48, seed=11)
    W, H, m = 64, 48, c["m"]
    mask, recs, mse = oracle.densify(W, H, c["f"], c["mask0"], c["unknowns"], c["schedule"])
    assert mask.size == m and np.unique(mask).size == m
    assert np.intersect1d(mask, c["unknowns"]).size == 0
    assert recs[-1]["mse"] >= mse  # more masks did not hurt on this image
    mask2, _, _ = oracle.densify(W, H, c["f"], c["mask0"], c["unknowns"], c["schedule"])
    np.testing.assert_array_equal(mask, mask2)  # deterministic
    # constant image: every error is zero -> global-fill path, still exactly m masks
    fc = np.full((H, W), 42.0)
    mask3, recs3, mse3 = oracle.densify(W, H, fc, c["mask0"], c["unknowns"], c["schedule"])
    assert mask3.size == m and mse3 == 0.0
    # n = 1: the random initial mask is the whole mask
    from synth import schedule
    assert schedule(m, 1) == [m]
