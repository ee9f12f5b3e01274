"""Plain fp64 CPU oracle of the FEM harmonic-inpainting hot path (arXiv 2105.01586).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The product path
(``paper_2105_01586_b200``) never imports it, and the two share no code; they share only
the seeded input generator ``synth`` (which holds none of the method's arithmetic).

The arithmetic lives in ``femi_oracle.c`` (single-threaded C, fp64, ``-O2
-ffp-contract=off``); this module is ctypes marshalling plus a few NumPy pins
(dense FDM inpainting, dense B materialisation, dense least squares).

Parity status per function:
  delaunay / delaunay_brute ........ pinned (P3, P4, brute force, closed forms)
  assemble ......................... pinned (P1, P2, P5, P6)
  solve ............................ pinned (P5 FDM, P6, P7, P8, P9, dense Cholesky)
  raster / error ................... pinned (P10, P11, P7, P8)
  raster_channels (colour) ......... pinned (C = 1 equals raster; channel sum of per-channel maps)
  select ........................... pinned (P16, brute-force re-derivation on tiny cases)
  tonal ............................ pinned (P13 dense lstsq, P14, P15)
  tonal_channels (colour) .......... pinned (joint block-diagonal dense lstsq equals the per-channel solutions)
  tonal_weighted / tonal_l1 (IRLS) . pinned (unit weights = tonal bit for bit; weighted dense lstsq;
                                     uniform weights = L2 solution; L1 error <= the L2 solution's)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "femi_oracle.c")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, -ffp-contract=off, reading A18)."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.orc_delaunay_brute.restype = ctypes.c_int64
        L.orc_delaunay_brute.argtypes = [ctypes.c_int, ctypes.c_int64, i32p, i32p, ctypes.c_int64]
        L.orc_delaunay.restype = ctypes.c_int64
        L.orc_delaunay.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, i32p, i32p, ctypes.c_int64]
        L.orc_sys_new.restype = ctypes.c_void_p
        L.orc_sys_new.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, i32p,
                                  ctypes.c_int64, i32p]
        L.orc_sys_free.argtypes = [ctypes.c_void_p]
        L.orc_sys_counts.argtypes = [ctypes.c_void_p, i64p]
        L.orc_sys_export.argtypes = [ctypes.c_void_p, i64p, i32p, f64p, i64p, i32p, f64p, i32p]
        L.orc_sys_solve.restype = ctypes.c_int
        L.orc_sys_solve.argtypes = [ctypes.c_void_p, f64p, ctypes.c_void_p, ctypes.c_double, ctypes.c_int,
                                    ctypes.c_int, f64p, ctypes.POINTER(ctypes.c_int),
                                    ctypes.POINTER(ctypes.c_double)]
        L.orc_sys_raster.argtypes = [ctypes.c_void_p, f64p, f64p, f64p, f64p, f64p, i32p,
                                     ctypes.POINTER(ctypes.c_double)]
        L.orc_sys_raster_channels.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                              ctypes.c_void_p, f64p, f64p, i32p, ctypes.POINTER(ctypes.c_double)]
        L.orc_sys_raster_channels.restype = None
        L.orc_sys_tonal_w.argtypes = [ctypes.c_void_p, f64p, ctypes.c_void_p, f64p, ctypes.c_double, ctypes.c_int,
                                      ctypes.c_double, ctypes.c_int, f64p]
        L.orc_sys_tonal_w.restype = ctypes.c_int
        L.orc_sys_tonal_l1.argtypes = [ctypes.c_void_p, f64p, f64p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_int, ctypes.c_double, f64p]
        L.orc_sys_tonal_l1.restype = ctypes.c_int
        L.orc_select.restype = ctypes.c_int64
        L.orc_select.argtypes = [ctypes.c_int64, f64p, i32p, ctypes.c_int64, f64p, u8p, ctypes.c_int64, i32p]
        L.orc_sys_apply_B.restype = ctypes.c_int
        L.orc_sys_apply_B.argtypes = [ctypes.c_void_p, f64p, f64p, ctypes.c_double]
        L.orc_sys_apply_BT.restype = ctypes.c_int
        L.orc_sys_apply_BT.argtypes = [ctypes.c_void_p, f64p, f64p, ctypes.c_double]
        L.orc_sys_tonal.restype = ctypes.c_int
        L.orc_sys_tonal.argtypes = [ctypes.c_void_p, f64p, f64p, ctypes.c_double, ctypes.c_int,
                                    ctypes.c_double, ctypes.c_int, f64p]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


# --------------------------------------------------------------------------------------
# Vertex set and triangulation (readings A2, A3)
# --------------------------------------------------------------------------------------

def vertex_set(W: int, H: int, mask_px, unknown_px):
    """Canonical vertices: unknowns (ascending pix, missing corners added), then masks
    (ascending pix). Returns (vpix int32, n_u, m)."""
    mask = np.unique(np.asarray(mask_px, dtype=np.int64))
    unk = np.unique(np.asarray(unknown_px, dtype=np.int64))
    corners = np.unique(np.array([0, W - 1, (H - 1) * W, H * W - 1], dtype=np.int64))
    unk = np.union1d(unk, np.setdiff1d(corners, mask))
    if np.intersect1d(mask, unk).size:
        raise OracleError("mask and unknown sets overlap")
    vpix = np.concatenate([unk, mask]).astype(np.int32)
    return vpix, int(unk.size), int(mask.size)


def delaunay(W: int, H: int, vpix: np.ndarray, brute: bool = False) -> np.ndarray:
    """Canonical SoS-Delaunay triangles [T,3] as indices into vpix."""
    vpix = np.ascontiguousarray(vpix, dtype=np.int32)
    n = vpix.size
    cap = 2 * n + 8
    tri = np.zeros(3 * cap, dtype=np.int32)
    if brute:
        T = lib().orc_delaunay_brute(W, n, vpix, tri, cap)
    else:
        T = lib().orc_delaunay(W, H, n, vpix, tri, cap)
    if T < 0:
        raise OracleError(f"delaunay failed: status {-T}")
    return tri[: 3 * T].reshape(T, 3).copy()


class System:
    """The FEM system on one mesh: A_uu, A_uk, owner map."""

    def __init__(self, W: int, H: int, mask_px, unknown_px, brute: bool = False, tri=None):
        self.W, self.H = W, H
        self.vpix, self.n_u, self.m = vertex_set(W, H, mask_px, unknown_px)
        self.nv = self.vpix.size
        self.tri = delaunay(W, H, self.vpix, brute) if tri is None else np.ascontiguousarray(tri, np.int32)
        self.T = self.tri.shape[0]
        h = lib().orc_sys_new(W, H, self.n_u, self.m, self.vpix, self.T, self.tri.reshape(-1))
        if not h:
            raise OracleError("orc_sys_new failed")
        self._h = h
        cnt = np.zeros(2, dtype=np.int64)
        lib().orc_sys_counts(h, cnt)
        self.nnz_uu, self.nnz_uk = int(cnt[0]), int(cnt[1])
        self.uu_ptr = np.zeros(self.n_u + 1, np.int64)
        self.uk_ptr = np.zeros(self.n_u + 1, np.int64)
        self.uu_col = np.zeros(max(self.nnz_uu, 1), np.int32)
        self.uu_val = np.zeros(max(self.nnz_uu, 1), np.float64)
        self.uk_col = np.zeros(max(self.nnz_uk, 1), np.int32)
        self.uk_val = np.zeros(max(self.nnz_uk, 1), np.float64)
        self.owner = np.zeros(W * H, np.int32)
        lib().orc_sys_export(h, self.uu_ptr, self.uu_col, self.uu_val, self.uk_ptr, self.uk_col,
                             self.uk_val, self.owner)
        self.uu_col, self.uu_val = self.uu_col[: self.nnz_uu], self.uu_val[: self.nnz_uu]
        self.uk_col, self.uk_val = self.uk_col[: self.nnz_uk], self.uk_val[: self.nnz_uk]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.orc_sys_free(h)
            self._h = None

    @property
    def mask_px(self):
        return self.vpix[self.n_u:]

    @property
    def unknown_px(self):
        return self.vpix[: self.n_u]

    def tri_px(self) -> np.ndarray:
        return self.vpix[self.tri]

    def dense_uu(self) -> np.ndarray:
        A = np.zeros((self.n_u, self.n_u))
        for i in range(self.n_u):
            s, e = self.uu_ptr[i], self.uu_ptr[i + 1]
            A[i, self.uu_col[s:e]] = self.uu_val[s:e]
        return A

    def dense_uk(self) -> np.ndarray:
        A = np.zeros((self.n_u, self.m))
        for i in range(self.n_u):
            s, e = self.uk_ptr[i], self.uk_ptr[i + 1]
            A[i, self.uk_col[s:e]] = self.uk_val[s:e]
        return A

    # ---- solve ----
    def solve(self, g, rtol: float = 1e-12, max_iter: int = 100000, method: int = 0, x0=None):
        g = np.ascontiguousarray(g, np.float64)
        u = np.zeros(self.nv, np.float64)
        it, rr = ctypes.c_int(0), ctypes.c_double(0.0)
        x0p = None
        if x0 is not None:
            x0a = np.ascontiguousarray(x0, np.float64)
            x0p = x0a.ctypes.data_as(ctypes.c_void_p)
        st = lib().orc_sys_solve(self._h, g, x0p, rtol, max_iter, method, u, ctypes.byref(it), ctypes.byref(rr))
        return u, st, it.value, rr.value

    # ---- raster + error ----
    def raster(self, u_vert, f):
        u_vert = np.ascontiguousarray(u_vert, np.float64)
        f = np.ascontiguousarray(f, np.float64).reshape(-1)
        N = self.W * self.H
        u_px = np.zeros(N)
        e_px = np.zeros(N)
        tri_err = np.zeros(max(self.T, 1))
        best = np.zeros(max(self.T, 1), np.int32)
        sse = ctypes.c_double(0.0)
        lib().orc_sys_raster(self._h, u_vert, f, u_px, e_px, tri_err, best, ctypes.byref(sse))
        return dict(u_px=u_px, e_px=e_px, tri_err=tri_err[: self.T], best=best[: self.T], sse=sse.value,
                    mse=sse.value / N)

    def raster_channels(self, u_list, f_list):
        """Colour raster: channels on this mesh, e = sum_c (u_c - f_c)^2."""
        C = len(u_list)
        N = self.W * self.H
        us = [np.ascontiguousarray(u, np.float64) for u in u_list]
        fs = [np.ascontiguousarray(f, np.float64).reshape(-1) for f in f_list]
        ups = [np.zeros(N) for _ in range(C)]
        arr = lambda xs: (ctypes.c_void_p * C)(*[x.ctypes.data for x in xs])  # noqa: E731
        e_px = np.zeros(N)
        tri_err = np.zeros(max(self.T, 1))
        best = np.zeros(max(self.T, 1), np.int32)
        sse = ctypes.c_double(0.0)
        lib().orc_sys_raster_channels(self._h, C, arr(us), arr(fs), arr(ups), e_px, tri_err, best, ctypes.byref(sse))
        return dict(u_px=ups, e_px=e_px, tri_err=tri_err[: self.T], best=best[: self.T], sse=sse.value,
                    mse=sse.value / N)

    def is_vertex(self) -> np.ndarray:
        v = np.zeros(self.W * self.H, np.uint8)
        v[self.vpix] = 1
        return v

    # ---- tonal ----
    def apply_B(self, g, rtol: float = 1e-12):
        out = np.zeros(self.W * self.H)
        st = lib().orc_sys_apply_B(self._h, np.ascontiguousarray(g, np.float64), out, rtol)
        if st:
            raise OracleError(f"apply_B status {st}")
        return out

    def apply_BT(self, r, rtol: float = 1e-12):
        out = np.zeros(self.m)
        st = lib().orc_sys_apply_BT(self._h, np.ascontiguousarray(r, np.float64).reshape(-1), out, rtol)
        if st:
            raise OracleError(f"apply_BT status {st}")
        return out

    def tonal(self, f, g0=None, outer_tol: float = 1e-8, outer_max: int = 1000, inner_rtol: float = 1e-12,
              inner_method: int = 0):
        f = np.ascontiguousarray(f, np.float64).reshape(-1)
        g = np.array(f[self.mask_px] if g0 is None else g0, dtype=np.float64)
        rep = np.zeros(8)
        st = lib().orc_sys_tonal(self._h, f, g, outer_tol, outer_max, inner_rtol, inner_method, rep)
        return g, dict(outer_iters=int(rep[0]), inner_solves=int(rep[1]), inner_iters=int(rep[2]),
                       rel_grad=rep[3], mse_before=rep[4], mse_after=rep[5], status=int(st),
                       rel_grad_recursive=rep[7])


def tonal_weighted(S, f, sw, g0=None, outer_tol: float = 1e-8, outer_max: int = 1000, inner_rtol: float = 1e-12):
    """Weighted CGLS: min || diag(sw) (B g - f) ||^2 (one IRLS step; sw = None: plain tonal)."""
    f = np.ascontiguousarray(f, np.float64).reshape(-1)
    g = np.array(f[S.mask_px] if g0 is None else g0, dtype=np.float64)
    swa = None if sw is None else np.ascontiguousarray(sw, np.float64).reshape(-1)
    rep = np.zeros(8)
    st = lib().orc_sys_tonal_w(S._h, f, None if swa is None else swa.ctypes.data_as(ctypes.c_void_p), g, outer_tol,
                               outer_max, inner_rtol, 0, rep)
    return g, dict(outer_iters=int(rep[0]), inner_solves=int(rep[1]), rel_grad=rep[3], mse_before=rep[4],
                   mse_after=rep[5], status=int(st))


def tonal_l1(S, f, irls: int = 3, eps: float = 1.0, g0=None, outer_tol: float = 1e-8, outer_max: int = 1000,
             inner_rtol: float = 1e-12):
    """L1 tonal optimisation by IRLS (reading R3)."""
    f = np.ascontiguousarray(f, np.float64).reshape(-1)
    g = np.array(f[S.mask_px] if g0 is None else g0, dtype=np.float64)
    rep = np.zeros(8)
    st = lib().orc_sys_tonal_l1(S._h, f, g, irls, eps, outer_tol, outer_max, inner_rtol, rep)
    return g, dict(outer_iters=int(rep[0]), inner_solves=int(rep[1]), inner_iters=int(rep[2]), l1_before=rep[3],
                   l1_after=rep[4], mse_after=rep[5], status=int(st))


def tonal_channels(S, f_list, **kw):
    """Colour tonal optimisation (reading R4): the channels share the mesh
    and B acts on each channel alone, so the colour least-squares problem min sum_c ||B g_c -
    f_c||^2 separates into one tonal problem per channel. Returns ([g_c], [report_c])."""
    out = [S.tonal(f, **kw) for f in f_list]
    return [g for g, _ in out], [r for _, r in out]


def select(tri_err, best, e_px, is_vertex, b: int) -> np.ndarray:
    """Densification selection (readings A8-A10). Ascending pix."""
    tri_err = np.ascontiguousarray(tri_err, np.float64)
    best = np.ascontiguousarray(best, np.int32)
    e_px = np.ascontiguousarray(e_px, np.float64).reshape(-1)
    is_vertex = np.ascontiguousarray(is_vertex, np.uint8)
    out = np.zeros(max(b, 1), np.int32)
    k = lib().orc_select(tri_err.size, tri_err, best, e_px.size, e_px, is_vertex, b, out)
    return out[:k].copy()


def inpaint(W, H, f, mask_px, unknown_px, rtol=1e-12, brute=False):
    """One harmonic inpainting with g = f at the mask (config 1 workload)."""
    S = System(W, H, mask_px, unknown_px, brute=brute)
    f = np.asarray(f, np.float64).reshape(-1)
    u, st, it, rr = S.solve(f[S.mask_px], rtol=rtol)
    R = S.raster(u, f)
    R.update(system=S, u_vert=u, status=st, iters=it, relres=rr)
    return R


def densify(W, H, f, mask0, unknowns, schedule, rtol=1e-12, lockstep_masks=None, method=0):
    """Error-map densification: iteration 0 = the random mask0; each
    later iteration inpaints on the current mesh and inserts b_t pixels. Returns the final
    mask and per-iteration records. With `lockstep_masks` (list of masks per iteration)
    each iteration starts from the given mask instead of the oracle's own (reading A15)."""
    f = np.asarray(f, np.float64).reshape(-1)
    mask = np.sort(np.asarray(mask0, np.int64))
    recs = []
    for t in range(1, len(schedule)):
        if lockstep_masks is not None:
            mask = np.sort(np.asarray(lockstep_masks[t - 1], np.int64))
        S = System(W, H, mask, unknowns)
        u, st, it, rr = S.solve(f[S.mask_px], rtol=rtol, method=method)
        R = S.raster(u, f)
        new = select(R["tri_err"], R["best"], R["e_px"], S.is_vertex(), schedule[t])
        recs.append(dict(mask=mask.copy(), mse=R["mse"], iters=it, new=new, tri_err=R["tri_err"],
                         best=R["best"], T=S.T))
        mask = np.sort(np.concatenate([mask, new.astype(np.int64)]))
    S = System(W, H, mask, unknowns)
    u, st, it, rr = S.solve(f[S.mask_px], rtol=rtol, method=method)
    R = S.raster(u, f)
    return mask, recs, R["mse"]


# --------------------------------------------------------------------------------------
# NumPy pins (independent of the C code above)
# --------------------------------------------------------------------------------------

def fdm_inpaint_dense(f2d: np.ndarray, mask_px) -> np.ndarray:
    """5-point FDM harmonic inpainting with reflecting boundary, dense solve
    ("standard (5-point stencil) FDM"; Eq. (3)). The domain is
    [0,W-1]x[0,H-1] with pixel centres on its border (reading A1), so the reflecting
    (Neumann) ghost value across a border pixel is its mirror neighbour (u_{-1} = u_1).
    Small images only."""
    H, W = f2d.shape
    N = W * H
    assert N <= 4096
    mask = np.zeros(N, bool)
    mask[np.asarray(mask_px)] = True
    L = np.zeros((N, N))
    for y in range(H):
        for x in range(W):
            i = y * W + x
            for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                xx, yy = x + dx, y + dy
                if not 0 <= xx < W:
                    xx = x - dx  # mirror about the border pixel centre
                if not 0 <= yy < H:
                    yy = y - dy
                L[i, i] += 1.0
                L[i, yy * W + xx] -= 1.0
    fv = f2d.reshape(-1)
    unk = ~mask
    u = fv.copy()
    u[unk] = np.linalg.solve(L[np.ix_(unk, unk)], -L[np.ix_(unk, mask)] @ fv[mask])
    return u.reshape(H, W)


def materialise_B(S: System, rtol: float = 1e-12) -> np.ndarray:
    """Dense B ("the matrix B is dense"): column j = B e_j. Tiny only."""
    assert S.W * S.H <= 4096 and S.m <= 256
    B = np.zeros((S.W * S.H, S.m))
    for j in range(S.m):
        e = np.zeros(S.m)
        e[j] = 1.0
        B[:, j] = S.apply_B(e, rtol)
    return B
