"""ctypes binding of libfemi (include/femi.h). Argument marshalling only: every step of the
hot path runs in the CUDA kernels behind the C ABI. There is no CPU fallback: if the
library or a B200 is missing, the calls raise.

Device buffers are torch CUDA tensors (fp64 / int32, contiguous); host buffers are numpy
arrays. Streams default to torch's current stream.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FEMI_LIB selects another build of the same library (e.g. libfemi_check.so, the device-
# bounds-checked build the GPU tests can run under); default: the in-tree libfemi.so
LIB_PATH = os.path.join(_HERE, os.environ.get("FEMI_LIB", "libfemi.so"))

FEMI_OK = 0
STATUS = {0: "OK", 1: "E_ARG", 2: "E_DEGENERATE", 3: "E_NO_MASK", 4: "E_NOT_CONVERGED", 5: "E_NONFINITE",
          6: "E_NEG_CURVATURE", 7: "E_SIZE", 8: "E_CUDA", 9: "E_OOM"}


class FemiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"femi status {status} ({STATUS.get(status, '?')}): {msg}")
        self.status = status


class MeshInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("width", "height", "n_vert", "n_unknown", "n_mask", "n_tri", "nnz_uu", "nnz_uk")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class CgOpts(ctypes.Structure):
    _fields_ = [("rtol", ctypes.c_double), ("max_iter", ctypes.c_int32), ("precond", ctypes.c_int32),
                ("x0", ctypes.c_int32), ("check_every", ctypes.c_int32)]


class TonalOpts(ctypes.Structure):
    _fields_ = [("outer_rtol", ctypes.c_double), ("outer_max", ctypes.c_int32), ("inner", CgOpts),
                ("warm_start", ctypes.c_int32)]


class TonalReport(ctypes.Structure):
    _fields_ = [("outer_iters", ctypes.c_int32), ("inner_solves", ctypes.c_int32), ("inner_iters", ctypes.c_int64),
                ("rel_grad", ctypes.c_double), ("rel_grad_recursive", ctypes.c_double),
                ("mse_before", ctypes.c_double), ("mse_after", ctypes.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class BandInfo(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("n_unknown", ctypes.c_int64),
                ("row0", ctypes.c_int64), ("row1", ctypes.c_int64), ("n_halo", ctypes.c_int64),
                ("n_send", ctypes.c_int64), ("nnz_uu", ctypes.c_int64), ("nnz_uk", ctypes.c_int64),
                ("n_peers", ctypes.c_int32), ("pad", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


class TonalL1Report(ctypes.Structure):
    _fields_ = [("irls_steps", ctypes.c_int32), ("outer_iters", ctypes.c_int32), ("inner_solves", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("inner_iters", ctypes.c_int64), ("l1_before", ctypes.c_double),
                ("l1_after", ctypes.c_double), ("mse_before", ctypes.c_double), ("mse_after", ctypes.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "pad"}


_lib = None
P = ctypes.c_void_p
I32P = ctypes.POINTER(ctypes.c_int32)

# every symbol include/femi.h declares
SYMBOLS = ["femi_last_error", "femi_version", "femi_kernel_launches", "femi_mesh_build", "femi_mesh_info_get", "femi_mesh_export",
           "femi_mesh_timing", "femi_mesh_free", "femi_assemble", "femi_system_info_get", "femi_system_export",
           "femi_system_free", "femi_inpaint_solve_batched", "femi_rasterise_error", "femi_rasterise_error_batched",
           "femi_densify_step", "femi_tonal_optimise", "femi_rasterise_error_channels",
           "femi_densify_step_channels", "femi_tonal_optimise_l1", "femi_mesh_insert",
           "femi_system_solver_path", "femi_apply_B", "femi_apply_BT", "femi_device_check_failures",
           "femi_tonal_optimise_channels", "femi_band_plan", "femi_band_plan_export", "femi_band_create",
           "femi_band_info_get", "femi_band_set_buffers", "femi_band_begin", "femi_band_pack", "femi_band_spmv",
           "femi_band_update", "femi_band_restart", "femi_band_status", "femi_band_result", "femi_band_free",
           "femi_band_raster_system"]

# femi_system_solver_path values (include/femi.h)
PATH_NAMES = {0: "none", 1: "resident", 2: "persistent", 3: "graph_sell", 4: "graph_tma", 5: "graph_multi"}


def lib():
    """Load libfemi.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FemiError(8, f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.femi_last_error.restype = ctypes.c_char_p
        L.femi_version.restype = ctypes.c_char_p
        L.femi_kernel_launches.restype = ctypes.c_int64
        L.femi_device_check_failures.restype = ctypes.c_int64
        L.femi_mesh_build.argtypes = [ctypes.c_int32, ctypes.c_int32, P, ctypes.c_int64, P, ctypes.c_int64,
                                      ctypes.POINTER(P)]
        L.femi_mesh_info_get.argtypes = [P, ctypes.POINTER(MeshInfo)]
        L.femi_mesh_export.argtypes = [P, P, P, P, P, P, P]
        L.femi_mesh_timing.argtypes = [P, ctypes.POINTER(ctypes.c_double), I32P]
        L.femi_mesh_free.argtypes = [P]
        L.femi_mesh_insert.argtypes = [P, P, ctypes.c_int64, ctypes.POINTER(P)]
        L.femi_mesh_free.restype = None
        L.femi_assemble.argtypes = [P, P, ctypes.POINTER(P)]
        L.femi_system_info_get.argtypes = [P, ctypes.POINTER(MeshInfo)]
        L.femi_system_export.argtypes = [P, P, P, P]
        L.femi_system_free.argtypes = [P]
        L.femi_system_free.restype = None
        L.femi_inpaint_solve_batched.argtypes = [ctypes.c_int32, P, P, P, ctypes.POINTER(CgOpts), P, P, P]
        L.femi_rasterise_error.argtypes = [P, P, P, P, P, P, P, P, P]
        L.femi_rasterise_error_batched.argtypes = [ctypes.c_int32, P, P, P, P, P, P, P, P, P]
        L.femi_densify_step.argtypes = [P, P, P, ctypes.c_int64, P, ctypes.POINTER(ctypes.c_int64), P]
        L.femi_tonal_optimise.argtypes = [P, P, P, ctypes.POINTER(TonalOpts), ctypes.POINTER(TonalReport), P]
        L.femi_rasterise_error_channels.argtypes = [P, ctypes.c_int32, P, P, P, P, P, P, P, P]
        L.femi_densify_step_channels.argtypes = [P, ctypes.c_int32, P, P, ctypes.c_int64, P,
                                                 ctypes.POINTER(ctypes.c_int64), P]
        L.femi_tonal_optimise_l1.argtypes = [P, P, P, ctypes.POINTER(TonalOpts), ctypes.c_int32, ctypes.c_double,
                                             ctypes.POINTER(TonalL1Report), P]
        L.femi_system_solver_path.argtypes = [P, I32P]
        L.femi_tonal_optimise_channels.argtypes = [P, ctypes.c_int32, P, P, ctypes.POINTER(TonalOpts), P, P]
        L.femi_device_check_failures.argtypes = [ctypes.POINTER(ctypes.c_int64)]
        L.femi_apply_B.argtypes = [P, P, P, ctypes.POINTER(CgOpts), P]
        L.femi_apply_BT.argtypes = [P, P, P, ctypes.POINTER(CgOpts), P]
        L.femi_band_plan.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(BandInfo)]
        L.femi_band_plan_export.argtypes = [P, ctypes.c_int32, ctypes.c_int32, P, P, P, P, P, P, P]
        L.femi_band_create.argtypes = [P, ctypes.c_int32, ctypes.c_int32, P, ctypes.POINTER(P)]
        L.femi_band_info_get.argtypes = [P, ctypes.POINTER(BandInfo)]
        L.femi_band_set_buffers.argtypes = [P, P, P, P]
        L.femi_band_begin.argtypes = [P, P, ctypes.c_double, P]
        L.femi_band_pack.argtypes = [P, ctypes.c_int32, P]
        L.femi_band_spmv.argtypes = [P, ctypes.c_int32, P]
        L.femi_band_update.argtypes = [P, P]
        L.femi_band_restart.argtypes = [P, P]
        L.femi_band_status.argtypes = [P, P, I32P, I32P, P]
        L.femi_band_result.argtypes = [P, P, P]
        L.femi_band_free.argtypes = [P]
        L.femi_band_free.restype = None
        L.femi_band_raster_system.argtypes = [P, ctypes.c_int32, ctypes.c_int32, P, ctypes.POINTER(P),
                                              ctypes.POINTER(ctypes.c_int64 * 4)]
        for name in SYMBOLS:
            if name not in ("femi_last_error", "femi_version", "femi_mesh_free", "femi_system_free", "femi_band_free",
                            "femi_kernel_launches", "femi_device_check_failures"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != FEMI_OK:
        raise FemiError(status, lib().femi_last_error().decode())


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _dptr(t, dtype=None):
    """Device pointer of a contiguous CUDA tensor (or None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise FemiError(1, "expected a contiguous CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise FemiError(1, f"expected dtype {dtype}, got {t.dtype}")
    return ctypes.c_void_p(t.data_ptr())


def _hptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = None if p is None else (p.value if isinstance(p, ctypes.c_void_p) else p)
    return arr


def version() -> str:
    return lib().femi_version().decode()


def kernel_launches() -> int:
    """Kernels launched by libfemi so far (process-wide)."""
    return int(lib().femi_kernel_launches())


class Mesh:
    """S0 mesh_build (host setup stage)."""

    def __init__(self, W: int, H: int, mask_px, unknown_px):
        mk = np.ascontiguousarray(np.asarray(mask_px).reshape(-1), dtype=np.int32)
        un = np.ascontiguousarray(np.asarray(unknown_px).reshape(-1), dtype=np.int32)
        h = ctypes.c_void_p()
        self._lib = lib()  # kept: close() may run at interpreter shutdown
        _check(self._lib.femi_mesh_build(W, H, _hptr(mk), mk.size, _hptr(un), un.size, ctypes.byref(h)))
        self._h = h
        info = MeshInfo()
        _check(lib().femi_mesh_info_get(h, ctypes.byref(info)))
        self.info = info.as_dict()
        sec, thr = ctypes.c_double(), ctypes.c_int32()
        _check(lib().femi_mesh_timing(h, ctypes.byref(sec), ctypes.byref(thr)))
        self.build_seconds, self.build_threads = sec.value, thr.value

    def insert(self, new_mask_px) -> "Mesh":
        """S0 incremental: a new Mesh with the given pixels added as mask vertices (identical
        to building the union from scratch; this mesh is unchanged)."""
        add = np.ascontiguousarray(np.asarray(new_mask_px).reshape(-1), dtype=np.int32)
        h = ctypes.c_void_p()
        _check(self._lib.femi_mesh_insert(self._h, _hptr(add), add.size, ctypes.byref(h)))
        return Mesh._from_handle(h, self._lib)

    @classmethod
    def _from_handle(cls, h, L):
        M = cls.__new__(cls)
        M._lib = L
        M._h = h
        info = MeshInfo()
        _check(L.femi_mesh_info_get(h, ctypes.byref(info)))
        M.info = info.as_dict()
        sec, thr = ctypes.c_double(), ctypes.c_int32()
        _check(L.femi_mesh_timing(h, ctypes.byref(sec), ctypes.byref(thr)))
        M.build_seconds, M.build_threads = sec.value, thr.value
        return M

    def export(self) -> dict:
        i = self.info
        out = dict(vert_px=np.zeros(i["n_vert"], np.int32), tri=np.zeros(3 * i["n_tri"], np.int32),
                   uu_rowptr=np.zeros(i["n_unknown"] + 1, np.int32), uu_col=np.zeros(i["nnz_uu"], np.int32),
                   uk_rowptr=np.zeros(i["n_unknown"] + 1, np.int32), uk_col=np.zeros(i["nnz_uk"], np.int32))
        _check(lib().femi_mesh_export(self._h, *(_hptr(out[k]) for k in
                                                 ("vert_px", "tri", "uu_rowptr", "uu_col", "uk_rowptr", "uk_col"))))
        out["tri"] = out["tri"].reshape(-1, 3)
        return out

    def vert_px(self) -> np.ndarray:
        """Pixel index of every vertex, canonical order (export()'s vert_px alone)."""
        v = np.zeros(self.info["n_vert"], np.int32)
        _check(lib().femi_mesh_export(self._h, _hptr(v), None, None, None, None, None))
        return v

    def close(self):
        if getattr(self, "_h", None):
            self._lib.femi_mesh_free(self._h)
            self._h = None

    def __del__(self):
        self.close()


class System:
    """S1 assemble: device matrices and raster tables of one mesh."""

    def __init__(self, mesh: Mesh, stream=None):
        h = ctypes.c_void_p()
        self._lib = lib()
        _check(self._lib.femi_assemble(mesh._h, _stream(stream), ctypes.byref(h)))
        self._h = h
        info = MeshInfo()
        _check(lib().femi_system_info_get(h, ctypes.byref(info)))
        self.info = info.as_dict()
        self.W, self.H = self.info["width"], self.info["height"]
        self.n_u, self.m, self.nv, self.T = (self.info[k] for k in ("n_unknown", "n_mask", "n_vert", "n_tri"))

    def export_values(self, stream=None):
        uu = np.zeros(self.info["nnz_uu"], np.float64)
        uk = np.zeros(self.info["nnz_uk"], np.float64)
        _check(lib().femi_system_export(self._h, _hptr(uu), _hptr(uk), _stream(stream)))
        return uu, uk

    def close(self):
        if getattr(self, "_h", None):
            self._lib.femi_system_free(self._h)
            self._h = None

    def __del__(self):
        self.close()


def cg_opts(rtol=1e-10, max_iter=100000, precond=1, x0=3, check_every=0) -> CgOpts:
    """x0: 0 zeros, 1 midrange(g), 2 caller-provided (u_vert), 3 mask-neighbour fill (default,
    reading A11b)."""
    return CgOpts(rtol, max_iter, precond, x0, check_every)


def _dptr_array(L, dtype):
    """ctypes array of the device pointers of a list of contiguous CUDA tensors (None -> NULL)."""
    if L is None:
        return None
    ptrs = []
    for t in L:
        if t is None:
            ptrs.append(None)
            continue
        if not (t.is_cuda and t.dtype == dtype and t.is_contiguous()):
            raise FemiError(1, f"expected contiguous CUDA tensors of dtype {dtype}")
        ptrs.append(t.data_ptr())
    return (ctypes.c_void_p * len(ptrs))(*ptrs)


class SolvePlan:
    """The arguments of one batched solve, marshalled once (pointer arrays, result buffers);
    run() is then a single C call -- for small batched workloads whose host-side marshalling
    would otherwise show up between the launches. The tensors must stay alive and in place."""

    def __init__(self, systems, g_list, u_list, opts: CgOpts | None = None):
        import torch
        self.B = len(systems)
        self.opts = opts or cg_opts()
        self._keep = (list(systems), list(g_list), list(u_list))
        self.sys_arr = _ptr_array([s._h for s in systems])
        self.g_arr = _dptr_array(g_list, torch.float64)
        self.u_arr = _dptr_array(u_list, torch.float64)
        self.iters = np.zeros(self.B, np.int32)
        self.rel = np.zeros(self.B, np.float64)
        self._pi, self._pr = _hptr(self.iters), _hptr(self.rel)

    def run(self, stream=None):
        st = lib().femi_inpaint_solve_batched(self.B, self.sys_arr, self.g_arr, self.u_arr, ctypes.byref(self.opts),
                                              self._pi, self._pr, _stream(stream))
        if st not in (FEMI_OK, 4):
            _check(st)
        return st, self.iters.copy(), self.rel.copy()


def inpaint_solve_batched(systems, g_list, u_list, opts: CgOpts | None = None, stream=None):
    """S2. Returns (status, iters[B], relres[B]); raises on hard errors."""
    return SolvePlan(systems, g_list, u_list, opts).run(stream)


class RasterPlan:
    """rasterise_error_batched with its arguments marshalled once (see SolvePlan)."""

    def __init__(self, systems, u_list, f_list, sse_list, u_px=None, e_px=None, tri_err=None, best=None):
        import torch
        self.B = len(systems)
        self._keep = (list(systems), u_list, f_list, sse_list, u_px, e_px, tri_err, best)
        f64 = torch.float64
        self.args = (_ptr_array([s._h for s in systems]), _dptr_array(u_list, f64), _dptr_array(f_list, f64),
                     _dptr_array(u_px, f64), _dptr_array(e_px, f64), _dptr_array(tri_err, f64),
                     _dptr_array(best, torch.int32), _dptr_array(sse_list, f64))

    def run(self, stream=None):
        _check(lib().femi_rasterise_error_batched(self.B, *self.args, _stream(stream)))


def rasterise_error_batched(systems, u_list, f_list, sse_list, u_px=None, e_px=None, tri_err=None, best=None,
                            stream=None):
    """S3+S4 (enqueue only)."""
    RasterPlan(systems, u_list, f_list, sse_list, u_px, e_px, tri_err, best).run(stream)


def rasterise_error(system, u_vert, f, sse, u_px=None, e_px=None, tri_err=None, best=None, stream=None):
    import torch
    _check(lib().femi_rasterise_error(system._h, _dptr(u_vert, torch.float64), _dptr(f, torch.float64),
                                      _dptr(u_px, torch.float64), _dptr(e_px, torch.float64),
                                      _dptr(tri_err, torch.float64), _dptr(best, torch.int32),
                                      _dptr(sse, torch.float64), _stream(stream)))


def densify_step(system, f, u_vert, b: int, stream=None) -> np.ndarray:
    """S5: new mask pixels (ascending) chosen from the per-triangle error of u_vert."""
    import torch
    out = np.zeros(max(b, 1), np.int32)
    n = ctypes.c_int64(0)
    _check(lib().femi_densify_step(system._h, _dptr(f, torch.float64), _dptr(u_vert, torch.float64), b, _hptr(out),
                                   ctypes.byref(n), _stream(stream)))
    return out[: n.value].copy()


def rasterise_error_channels(system, u_list, f_list, sse=None, u_px=None, e_px=None, tri_err=None, best=None,
                             stream=None):
    """Colour S3+S4 (enqueue only): channels on one mesh, e = sum_c (u_c - f_c)^2."""
    import torch
    C = len(u_list)
    ua = _ptr_array([_dptr(u, torch.float64) for u in u_list])
    fa = _ptr_array([_dptr(f, torch.float64) for f in f_list]) if f_list is not None else None
    pa = _ptr_array([_dptr(u, torch.float64) for u in u_px]) if u_px is not None else None
    _check(lib().femi_rasterise_error_channels(system._h, C, ua, fa, pa, _dptr(e_px, torch.float64),
                                               _dptr(tri_err, torch.float64), _dptr(best, torch.int32),
                                               _dptr(sse, torch.float64), _stream(stream)))


def densify_step_channels(system, f_list, u_list, b: int, stream=None) -> np.ndarray:
    """Colour S5: new mask pixels chosen from the channel-summed error."""
    import torch
    out = np.zeros(max(b, 1), np.int32)
    n = ctypes.c_int64(0)
    fa = _ptr_array([_dptr(f, torch.float64) for f in f_list])
    ua = _ptr_array([_dptr(u, torch.float64) for u in u_list])
    _check(lib().femi_densify_step_channels(system._h, len(f_list), fa, ua, b, _hptr(out), ctypes.byref(n),
                                            _stream(stream)))
    return out[: n.value].copy()


def tonal_optimise(system, f, g, outer_rtol=1e-8, outer_max=1000, inner: CgOpts | None = None, stream=None):
    """S6: g (device, in/out) <- argmin ||B g - f||^2. Returns (status, report dict)."""
    import torch
    inner = inner or cg_opts(rtol=1e-12)
    o = TonalOpts(outer_rtol, outer_max, inner, 0)
    rep = TonalReport()
    st = lib().femi_tonal_optimise(system._h, _dptr(f, torch.float64), _dptr(g, torch.float64), ctypes.byref(o),
                                   ctypes.byref(rep), _stream(stream))
    if st not in (FEMI_OK, 4):
        _check(st)
    return st, rep.as_dict()


def tonal_optimise_l1(system, f, g, irls=3, eps=1.0, outer_rtol=1e-8, outer_max=1000, inner: CgOpts | None = None,
                      stream=None):
    """NEXT-2: L1 tonal optimisation by IRLS (g device, in/out). Returns (status, report dict)."""
    import torch
    inner = inner or cg_opts(rtol=1e-12)
    o = TonalOpts(outer_rtol, outer_max, inner, 0)
    rep = TonalL1Report()
    st = lib().femi_tonal_optimise_l1(system._h, _dptr(f, torch.float64), _dptr(g, torch.float64), ctypes.byref(o),
                                      irls, eps, ctypes.byref(rep), _stream(stream))
    if st not in (FEMI_OK, 4):
        _check(st)
    return st, rep.as_dict()


def solver_path(system) -> str:
    """Which solver the last solve on `system` ran (diagnostic; include/femi.h FEMI_PATH_*)."""
    v = ctypes.c_int32(0)
    _check(lib().femi_system_solver_path(system._h, ctypes.byref(v)))
    return PATH_NAMES.get(v.value, str(v.value))


def apply_B(system, g, u_px, inner: CgOpts | None = None, stream=None):
    """u_px (device, W*H) <- B g (Eq. (4): inpainting from mask values g, rasterised)."""
    import torch
    inner = inner or cg_opts(rtol=1e-12)
    _check(lib().femi_apply_B(system._h, _dptr(g, torch.float64), _dptr(u_px, torch.float64), ctypes.byref(inner),
                              _stream(stream)))


def apply_BT(system, r, s, inner: CgOpts | None = None, stream=None):
    """s (device, n_mask) <- B^T r (the adjoint of apply_B)."""
    import torch
    inner = inner or cg_opts(rtol=1e-12)
    _check(lib().femi_apply_BT(system._h, _dptr(r, torch.float64), _dptr(s, torch.float64), ctypes.byref(inner),
                               _stream(stream)))


def device_check_failures():
    """(count, first failing site) of the device bounds checks since the last call (always
    (0, 0) unless the library is the checked build, FEMI_LIB=libfemi_check.so)."""
    site = ctypes.c_int64(0)
    n = lib().femi_device_check_failures(ctypes.byref(site))
    return int(n), int(site.value)


def tonal_optimise_channels(system, f_list, g_list, outer_rtol=1e-8, outer_max=1000, inner: CgOpts | None = None,
                            stream=None):
    """NEXT-1 colour tonal optimisation: C channels (device f_c, g_c in/out) on one mesh.
    Returns (status, [report dict per channel])."""
    import torch
    C = len(f_list)
    inner = inner or cg_opts(rtol=1e-12)
    o = TonalOpts(outer_rtol, outer_max, inner, 0)
    reps = (TonalReport * C)()
    fa = _ptr_array([_dptr(f, torch.float64) for f in f_list])
    ga = _ptr_array([_dptr(g, torch.float64) for g in g_list])
    st = lib().femi_tonal_optimise_channels(system._h, C, fa, ga, ctypes.byref(o), reps, _stream(stream))
    if st not in (FEMI_OK, 4):
        _check(st)
    return st, [r.as_dict() for r in reps]


# ------------------------------------------------------------------ row-band multi-GPU (NEXT-4)
def band_plan(mesh: Mesh, nranks: int, rank: int) -> dict:
    """HOST only: the band plan of `rank` (sizes and arrays; femi_band_plan / _export)."""
    info = BandInfo()
    _check(lib().femi_band_plan(mesh._h, nranks, rank, ctypes.byref(info)))
    d = info.as_dict()
    nloc = d["row1"] - d["row0"]
    out = dict(info=d, peer=np.zeros(d["n_peers"], np.int32), recv_off=np.zeros(d["n_peers"] + 1, np.int64),
               send_off=np.zeros(d["n_peers"] + 1, np.int64), halo_id=np.zeros(d["n_halo"], np.int64),
               send_row=np.zeros(d["n_send"], np.int32), rowptr=np.zeros(nloc + 1, np.int32),
               col=np.zeros(d["nnz_uu"], np.int32))
    _check(lib().femi_band_plan_export(mesh._h, nranks, rank, *(_hptr(out[k]) for k in (
        "peer", "recv_off", "send_off", "halo_id", "send_row", "rowptr", "col"))))
    return out


class Band:
    """One rank's band of a row-band solve (femi_band_*): the communication buffers are torch
    tensors owned here and handed to the library; the exchange / all-reduce are the caller's
    (paper_2105_01586_b200.multi)."""

    def __init__(self, mesh: Mesh, nranks: int, rank: int, stream=None):
        import torch
        self._lib = lib()
        h = ctypes.c_void_p()
        _check(self._lib.femi_band_create(mesh._h, nranks, rank, _stream(stream), ctypes.byref(h)))
        self._h = h
        info = BandInfo()
        _check(self._lib.femi_band_info_get(h, ctypes.byref(info)))
        self.info = info.as_dict()
        plan = band_plan(mesh, nranks, rank)
        self.peer, self.recv_off, self.send_off = plan["peer"], plan["recv_off"], plan["send_off"]
        dev = torch.device("cuda", torch.cuda.current_device())
        self.halo = torch.zeros(max(self.info["n_halo"], 1), dtype=torch.float64, device=dev)
        self.send = torch.zeros(max(self.info["n_send"], 1), dtype=torch.float64, device=dev)
        self.dots = torch.zeros(4, dtype=torch.float64, device=dev)
        _check(self._lib.femi_band_set_buffers(h, _dptr(self.halo), _dptr(self.send), _dptr(self.dots)))
        self.row0, self.row1 = self.info["row0"], self.info["row1"]

    def begin(self, g, rtol, stream=None):
        _check(self._lib.femi_band_begin(self._h, _dptr(g, _f64()), float(rtol), _stream(stream)))

    def pack(self, which, stream=None):
        _check(self._lib.femi_band_pack(self._h, int(which), _stream(stream)))

    def spmv(self, which, stream=None):
        _check(self._lib.femi_band_spmv(self._h, int(which), _stream(stream)))

    def update(self, stream=None):
        _check(self._lib.femi_band_update(self._h, _stream(stream)))

    def restart(self, stream=None):
        _check(self._lib.femi_band_restart(self._h, _stream(stream)))

    def status(self, stream=None):
        done, iters = ctypes.c_int32(), ctypes.c_int32()
        d = np.zeros(4, np.float64)
        _check(self._lib.femi_band_status(self._h, _stream(stream), ctypes.byref(done), ctypes.byref(iters), _hptr(d)))
        return bool(done.value), int(iters.value), d

    def result(self, u_local, stream=None):
        _check(self._lib.femi_band_result(self._h, _dptr(u_local, _f64()), _stream(stream)))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.femi_band_free(self._h)
            self._h = None

    def __del__(self):
        self.close()


def band_raster_system(mesh: Mesh, nranks: int, rank: int, stream=None):
    """Raster-only System over rank `rank`'s triangle share (femi_band_raster_system); returns
    (system, {'t0', 't1', 'y0', 'rows'})."""
    h = ctypes.c_void_p()
    info = (ctypes.c_int64 * 4)()
    _check(lib().femi_band_raster_system(mesh._h, nranks, rank, _stream(stream), ctypes.byref(h), ctypes.byref(info)))
    S = System.__new__(System)
    S._lib = lib()
    S._h = h
    mi = MeshInfo()
    _check(lib().femi_system_info_get(h, ctypes.byref(mi)))
    S.info = mi.as_dict()
    S.W, S.H = S.info["width"], S.info["height"]
    S.n_u, S.m, S.nv, S.T = (S.info[k] for k in ("n_unknown", "n_mask", "n_vert", "n_tri"))
    return S, dict(zip(("t0", "t1", "y0", "rows"), (int(v) for v in info)))


def _f64():
    import torch
    return torch.float64
