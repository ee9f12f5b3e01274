"""S0 mesh_build (host C++ stage of the product library) vs the oracle: bit-exact topology
and CSR patterns (BASELINE.json north_star correctness criterion). CPU only: mesh_build
runs on the host, so no GPU is needed to call it through the C ABI."""
import numpy as np
import pytest

import oracle
from paper_2105_01586_b200 import femi
from synth import make_config
from synth.generate import draw_mask, draw_unknowns


def product_mesh(W, H, mk, un):
    M = femi.Mesh(W, H, mk, un)
    return M, M.export()


def assert_same(W, H, mk, un):
    M, E = product_mesh(W, H, mk, un)
    S = oracle.System(W, H, mk, un)
    np.testing.assert_array_equal(E["vert_px"], S.vpix)
    np.testing.assert_array_equal(E["tri"], S.tri)
    np.testing.assert_array_equal(E["uu_rowptr"], S.uu_ptr)
    np.testing.assert_array_equal(E["uu_col"], S.uu_col)
    np.testing.assert_array_equal(E["uk_rowptr"], S.uk_ptr)
    np.testing.assert_array_equal(E["uk_col"], S.uk_col)
    assert M.info["n_unknown"] == S.n_u and M.info["n_mask"] == S.m and M.info["n_tri"] == S.T
    return M, S


def test_abi_exports_every_declared_symbol():
    L = femi.lib()
    import re
    hdr = open(__file__.replace("tests/test_mesh_host.py", "include/femi.h")).read()
    declared = set(re.findall(r"\b(femi_[A-Za-z0-9_]+)\s*\(", hdr))
    assert declared == set(femi.SYMBOLS)
    for name in declared:
        assert hasattr(L, name)
    assert "sm_100a" in femi.version()


@pytest.mark.parametrize("seed", range(40))
def test_mesh_bit_exact_small_random(seed):
    rng = np.random.default_rng(seed)
    W, H = int(rng.integers(2, 24)), int(rng.integers(2, 24))
    N = W * H
    m = int(rng.integers(1, max(2, N // 2)))
    mk = draw_mask(rng, N, m)
    p = int(rng.integers(0, N - m + 1))
    un = draw_unknowns(rng, W, H, mk, min(max(p, 4), N - m)) if N - m >= 4 else np.setdiff1d(np.arange(N), mk)
    # input order must not matter
    assert_same(W, H, rng.permutation(mk), rng.permutation(un))


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_mesh_bit_exact_configs(cfg):
    c = make_config(cfg)
    if cfg == 2:
        for b in (0, 7, 31):
            assert_same(c["W"], c["H"], c["masks"][b], c["unknowns"][b])
    elif cfg == 3:
        assert_same(c["W"], c["H"], c["mask0"], c["unknowns"])
    else:
        assert_same(c["W"], c["H"], c["mask"], c["unknowns"])


def test_mesh_bit_exact_config4():
    c = make_config(4)
    assert_same(c["W"], c["H"], c["mask"], c["unknowns"])


def test_full_grid_and_full_mask():
    W, H = 17, 9
    allpx = np.arange(W * H)
    assert_same(W, H, [40], np.setdiff1d(allpx, [40]))  # maximal cocircular degeneracy
    M, E = product_mesh(W, H, allpx, [])
    assert M.info["n_unknown"] == 0 and M.info["nnz_uu"] == 0


@pytest.mark.parametrize("W,H,mk,un,err", [
    (1, 5, [0], [], 2), (5, 1, [0], [], 2), (4, 4, [], [1], 3), (4, 4, [16], [], 7), (4, 4, [3, 3], [], 7),
    (4, 4, [5], [5], 7), (20000, 4, [0], [], 7)])
def test_mesh_errors(W, H, mk, un, err):
    with pytest.raises(femi.FemiError) as ei:
        femi.Mesh(W, H, np.array(mk, np.int32), np.array(un, np.int32))
    assert ei.value.status == err


def test_mesh_large_structure():
    """2048^2 with ~168K vertices: Delaunay local property on every interior edge (exact
    SoS in-circle, reimplemented in numpy int64), plus area and Euler counts."""
    W = H = 2048
    rng = np.random.default_rng(12)
    mk = draw_mask(rng, W * H, 83886)
    un = draw_unknowns(rng, W, H, mk, 83886)
    M, E = product_mesh(W, H, mk, un)
    S_tri = oracle.delaunay(W, H, E["vert_px"])
    np.testing.assert_array_equal(E["tri"], S_tri)
    # the shared mesh itself, checked from scratch in numpy (not through either C code):
    vp = E["vert_px"].astype(np.int64)
    tri = E["tri"].astype(np.int64)
    X, Y = vp % W, vp // W
    nv, T = vp.size, tri.shape[0]

    def orient(a, b, c):
        return (X[b] - X[a]) * (Y[c] - Y[a]) - (Y[b] - Y[a]) * (X[c] - X[a])

    a, b, c = tri[:, 0], tri[:, 1], tri[:, 2]
    o = orient(a, b, c)
    assert np.all(o > 0)  # every triangle CCW and non-degenerate
    assert o.sum() == 2 * (W - 1) * (H - 1)  # areas tile the image domain (reading A1)
    on_border = (X == 0) | (X == W - 1) | (Y == 0) | (Y == H - 1)
    assert T == 2 * nv - 2 - int(on_border.sum())  # Euler count with h hull (border) points
    # edges: each used by <= 2 triangles; edges used once lie on the image border
    ev = np.concatenate([np.stack([tri[:, (k + 1) % 3], tri[:, (k + 2) % 3]], 1) for k in range(3)])
    opp = np.concatenate([tri[:, k] for k in range(3)])
    own = np.concatenate([np.arange(T)] * 3)
    key = np.minimum(ev[:, 0], ev[:, 1]) * nv + np.maximum(ev[:, 0], ev[:, 1])
    order = np.argsort(key, kind="stable")
    ks = key[order]
    _, cnt = np.unique(ks, return_counts=True)
    assert cnt.max() <= 2
    single = np.ones(ks.size, bool)
    dup = ks[1:] == ks[:-1]
    single[1:] &= ~dup
    single[:-1] &= ~dup
    se = ev[order[single]]
    bx = ((X[se[:, 0]] == 0) & (X[se[:, 1]] == 0)) | ((X[se[:, 0]] == W - 1) & (X[se[:, 1]] == W - 1))
    by = ((Y[se[:, 0]] == 0) & (Y[se[:, 1]] == 0)) | ((Y[se[:, 0]] == H - 1) & (Y[se[:, 1]] == H - 1))
    assert np.all(bx | by)
    # local SoS-Delaunay property (reading A3) on every interior edge, both directions
    i1, i2 = order[:-1][dup], order[1:][dup]

    def sos_inside(t, d):
        ta, tb, tc = tri[t, 0], tri[t, 1], tri[t, 2]
        adx, ady = X[ta] - X[d], Y[ta] - Y[d]
        bdx, bdy = X[tb] - X[d], Y[tb] - Y[d]
        cdx, cdy = X[tc] - X[d], Y[tc] - Y[d]
        det = ((adx * adx + ady * ady) * (bdx * cdy - bdy * cdx) - (bdx * bdx + bdy * bdy) * (adx * cdy - ady * cdx)
               + (cdx * cdx + cdy * cdy) * (adx * bdy - ady * bdx))
        res = det > 0
        z = det == 0
        if np.any(z):
            P = np.stack([vp[ta], vp[tb], vp[tc], vp[d]], 1)
            smin = P.argmin(1)
            verts = np.stack([ta, tb, tc], 1)
            k = np.minimum(smin, 2)
            t1 = verts[np.arange(t.size), (k + 1) % 3]
            t2 = verts[np.arange(t.size), (k + 2) % 3]
            tie = np.where(smin == 3, True, orient(t1, t2, d) < 0)
            res = np.where(z, tie, res)
        return res

    assert not np.any(sos_inside(own[i1], opp[i2]))
    assert not np.any(sos_inside(own[i2], opp[i1]))


@pytest.mark.parametrize("strips,margin", [(2, None), (7, 1), (16, 2), (40, 3)])
def test_mesh_strip_decomposition(monkeypatch, capfd, strips, margin):
    """The parallel strip triangulation (mesh.cpp: local Bowyer-Watson per row strip,
    circumdisk certification, retry with a doubled margin) gives the unique SoS mesh for any
    strip count; tiny margins force the retry path."""
    monkeypatch.setenv("FEMI_MESH_STRIPS", str(strips))
    monkeypatch.setenv("FEMI_MESH_PROF", "1")
    if margin is not None:
        monkeypatch.setenv("FEMI_MESH_MARGIN", str(margin))
    retries = 0
    for seed in range(3):
        rng = np.random.default_rng(100 + seed)
        W, H = int(rng.integers(40, 160)), int(rng.integers(40, 160))
        N = W * H
        mk = draw_mask(rng, N, int(rng.integers(1, N // 8)))
        un = draw_unknowns(rng, W, H, mk, int(rng.integers(4, N // 10)))
        assert_same(W, H, mk, un)
        err = capfd.readouterr().err
        line = [x for x in err.splitlines() if x.startswith("mesh_build strips")]
        assert line and int(line[-1].split()[2]) == min(strips, H)
        retries += int(line[-1].split()[-1])
    c = make_config(3)
    assert_same(c["W"], c["H"], c["mask0"], c["unknowns"])
    if margin is not None:
        assert retries > 0


def test_mesh_strips_sparse_and_clustered(monkeypatch):
    """Strips on point sets far from uniform: a sparse mask with all vertices in one corner
    region plus long empty bands (huge circumcircles cross many strips)."""
    monkeypatch.setenv("FEMI_MESH_STRIPS", "12")
    W, H = 300, 240
    rng = np.random.default_rng(5)
    xs, ys = rng.integers(0, 60, 400), rng.integers(0, 50, 400)
    pts = np.unique(ys * W + xs)
    mk = pts[: len(pts) // 2]
    un = np.concatenate([pts[len(pts) // 2:], [120 * W + 150, 200 * W + 299, 239 * W + 10]])
    assert_same(W, H, mk, un)


def _same_export(A, B):
    EA, EB = A.export(), B.export()
    for k in ("vert_px", "tri", "uu_rowptr", "uu_col", "uk_rowptr", "uk_col"):
        np.testing.assert_array_equal(EA[k], EB[k], err_msg=k)
    assert A.info == B.info


@pytest.mark.parametrize("seed", range(12))
def test_mesh_insert_equals_rebuild(seed):
    """S0 incremental (femi_mesh_insert): inserting new mask pixels into a mesh gives exactly
    the mesh built from scratch on the union (reading A3: the SoS triangulation is unique)."""
    rng = np.random.default_rng(500 + seed)
    W, H = int(rng.integers(8, 90)), int(rng.integers(8, 90))
    N = W * H
    mk = draw_mask(rng, N, int(rng.integers(1, max(2, N // 10))))
    un = draw_unknowns(rng, W, H, mk, int(rng.integers(4, max(5, N // 8))))
    prev = femi.Mesh(W, H, mk, un)
    free = np.setdiff1d(np.arange(N), np.concatenate([mk, prev.export()["vert_px"]]))
    add = rng.choice(free, size=min(free.size, int(rng.integers(1, max(2, N // 12)))), replace=False)
    new = prev.insert(rng.permutation(add))
    ref = femi.Mesh(W, H, np.concatenate([mk, add]), un)
    _same_export(new, ref)
    # prev is unchanged
    _same_export(prev, femi.Mesh(W, H, mk, un))


def test_mesh_insert_densification_sequence():
    """A C3-like schedule: nine insertions of ~1% of the pixels, each equal to a rebuild."""
    c = make_config(3)
    W, H = c["W"], c["H"]
    rng = np.random.default_rng(33)
    mask = np.sort(c["mask0"])
    M = femi.Mesh(W, H, mask, c["unknowns"])
    verts = set(M.export()["vert_px"].tolist())
    for t in range(9):
        cand = np.array([q for q in rng.choice(W * H, 2000, replace=False) if q not in verts][:1300])
        M = M.insert(cand)
        mask = np.sort(np.concatenate([mask, cand]))
        verts.update(cand.tolist())
        if t in (0, 4, 8):
            _same_export(M, femi.Mesh(W, H, mask, c["unknowns"]))


def test_mesh_insert_cocircular_lattice():
    """Maximal cocircular degeneracy: a lattice of unknowns, lattice points inserted as masks."""
    W, H = 33, 29
    lat = np.array([y * W + x for y in range(0, H, 4) for x in range(0, W, 4)])
    mk = lat[::3]
    un = np.setdiff1d(lat, mk)
    prev = femi.Mesh(W, H, mk, un)
    add = np.array([y * W + x for y in range(2, H, 4) for x in range(2, W, 4)])
    _same_export(prev.insert(add), femi.Mesh(W, H, np.concatenate([mk, add]), un))


def test_mesh_insert_errors():
    W, H = 20, 20
    M = femi.Mesh(W, H, [21, 55, 300], [5, 77])
    for bad in ([21], [5], [0], [400], [-1], [100, 100]):
        with pytest.raises(femi.FemiError) as ei:
            M.insert(np.array(bad, np.int32))
        assert ei.value.status == 7
    _same_export(M.insert(np.array([], np.int32)), M)
