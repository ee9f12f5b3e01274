"""Host-side drivers composed from the C-ABI calls (no arithmetic of the method here).

    inpaint()  -- mesh_build -> assemble -> inpaint_solve_batched -> rasterise_error
    densify()  -- PAPER.md:L257-268: iteration 0 is the random initial mask; each later
                  iteration inpaints on the current mesh and inserts b_t pixels chosen by
                  densify_step; the host merges the mask and re-meshes.
    tonal()    -- tonal_optimise on a fixed mesh with g0 = f at the mask.
    inpaint_channels() / densify_channels() -- colour: channels on one
                  mesh, one shared-matrix multi-RHS solve, channel-summed error map.
"""
from __future__ import annotations

import numpy as np

from . import femi


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise femi.FemiError(8, "no CUDA device: the FEM inpainting path has no CPU fallback")
    return torch


def mask_values(f_dev, mesh_or_sys_vert_px, n_u):
    """g = f at the mask vertices in canonical (ascending pix) order, gathered on the device."""
    torch = _torch()
    idx = torch.as_tensor(np.asarray(mesh_or_sys_vert_px[n_u:], dtype=np.int64), device=f_dev.device)
    return f_dev.reshape(-1).index_select(0, idx).contiguous()


def inpaint(W, H, f_dev, mask_px, unknown_px, rtol=1e-10, want_images=True, stream=None, x0_unknown=None,
            mesh=None, x0=3):
    """x0_unknown: optional initial guess at the unknown vertices (canonical order, e.g. the
    previous densification iteration's solution: the unknown set is fixed, reading A4).
    mesh: a prebuilt femi.Mesh of exactly these vertices (e.g. from Mesh.insert)."""
    torch = _torch()
    if mesh is None:
        mesh = femi.Mesh(W, H, mask_px, unknown_px)
    sysm = femi.System(mesh, stream)
    vert = mesh.vert_px()
    g = mask_values(f_dev, vert, sysm.n_u)
    u_vert = torch.empty(sysm.nv, dtype=torch.float64, device=f_dev.device)
    if x0_unknown is not None and x0_unknown.numel() == sysm.n_u:
        u_vert[: sysm.n_u] = x0_unknown
        x0 = 2
    st, iters, rel = femi.inpaint_solve_batched([sysm], [g], [u_vert], femi.cg_opts(rtol=rtol, x0=x0), stream)
    sse = torch.zeros(1, dtype=torch.float64, device=f_dev.device)
    u_px = e_px = None
    if want_images:
        u_px = torch.empty(W * H, dtype=torch.float64, device=f_dev.device)
        e_px = torch.empty(W * H, dtype=torch.float64, device=f_dev.device)
    tri_err = torch.empty(max(sysm.T, 1), dtype=torch.float64, device=f_dev.device)
    best = torch.empty(max(sysm.T, 1), dtype=torch.int32, device=f_dev.device)
    femi.rasterise_error(sysm, u_vert, f_dev.reshape(-1), sse, u_px, e_px, tri_err, best, stream)
    return dict(mesh=mesh, system=sysm, vert_px=vert, u_vert=u_vert, u_px=u_px, e_px=e_px, tri_err=tri_err[: sysm.T],
                best=best[: sysm.T], sse=sse, status=st, iters=int(iters[0]), relres=float(rel[0]))


def densify(W, H, f_dev, mask0, unknown_px, schedule, rtol=1e-10, lockstep_masks=None, stream=None,
            warm_start=False, incremental_mesh=True, x0=3):
    """Returns (final mask, per-iteration records, final MSE). warm_start: each solve starts
    from the previous iteration's solution at the (fixed, reading A4) unknown vertices
    (changes iterates, not the solution). incremental_mesh: each mesh is
    the previous one plus the new mask pixels (Mesh.insert, identical to a rebuild)."""
    _torch()
    mask = np.sort(np.asarray(mask0, dtype=np.int64))
    recs = []
    f1 = f_dev.reshape(-1)
    x_prev = None
    mesh, new = None, None
    for t in range(1, len(schedule)):
        if lockstep_masks is not None:
            mask = np.sort(np.asarray(lockstep_masks[t - 1], dtype=np.int64))
            mesh = None
        elif incremental_mesh and mesh is not None:
            mesh = mesh.insert(new)
        R = inpaint(W, H, f_dev, mask, unknown_px, rtol=rtol, want_images=False, stream=stream,
                    x0_unknown=x_prev if warm_start else None, mesh=mesh, x0=x0)
        mesh = R["mesh"] if incremental_mesh else None
        x_prev = R["u_vert"][: R["system"].n_u].clone()
        new = femi.densify_step(R["system"], f1, R["u_vert"], int(schedule[t]), stream)
        recs.append(dict(mask=mask.copy(), mse=float(R["sse"].item()) / (W * H), iters=R["iters"], new=new,
                         T=R["system"].T, mesh_seconds=R["mesh"].build_seconds))
        mask = np.sort(np.concatenate([mask, new.astype(np.int64)]))
    if incremental_mesh and mesh is not None and lockstep_masks is None:
        mesh = mesh.insert(new)
    else:
        mesh = None
    R = inpaint(W, H, f_dev, mask, unknown_px, rtol=rtol, want_images=False, stream=stream,
                x0_unknown=x_prev if warm_start else None, mesh=mesh, x0=x0)
    return mask, recs, float(R["sse"].item()) / (W * H)


def tonal(W, H, f_dev, mask_px, unknown_px, outer_rtol=1e-8, outer_max=1000, inner_rtol=1e-12, stream=None):
    _torch()
    mesh = femi.Mesh(W, H, mask_px, unknown_px)
    sysm = femi.System(mesh, stream)
    vert = mesh.vert_px()
    g = mask_values(f_dev, vert, sysm.n_u)
    st, rep = femi.tonal_optimise(sysm, f_dev.reshape(-1), g, outer_rtol, outer_max, femi.cg_opts(rtol=inner_rtol),
                                  stream)
    return g, rep, dict(mesh=mesh, system=sysm, vert_px=vert, status=st)


def inpaint_channels(W, H, f_list, mask_px, unknown_px, rtol=1e-10, want_images=True, stream=None):
    """Colour inpainting: every channel on the same mask/mesh; the error is the channel sum."""
    torch = _torch()
    mesh = femi.Mesh(W, H, mask_px, unknown_px)
    sysm = femi.System(mesh, stream)
    vert = mesh.vert_px()
    dev = f_list[0].device
    gs = [mask_values(f, vert, sysm.n_u) for f in f_list]
    us = [torch.empty(sysm.nv, dtype=torch.float64, device=dev) for _ in f_list]
    st, iters, rel = femi.inpaint_solve_batched([sysm] * len(f_list), gs, us, femi.cg_opts(rtol=rtol), stream)
    sse = torch.zeros(1, dtype=torch.float64, device=dev)
    u_px = [torch.empty(W * H, dtype=torch.float64, device=dev) for _ in f_list] if want_images else None
    e_px = torch.empty(W * H, dtype=torch.float64, device=dev) if want_images else None
    femi.rasterise_error_channels(sysm, us, [f.reshape(-1) for f in f_list], sse, u_px, e_px, stream=stream)
    return dict(mesh=mesh, system=sysm, vert_px=vert, u_vert=us, u_px=u_px, e_px=e_px, sse=sse, status=st,
                iters=[int(i) for i in iters], relres=[float(r) for r in rel])


def densify_channels(W, H, f_list, mask0, unknown_px, schedule, rtol=1e-10, stream=None):
    """Colour densification: insertion driven by the channel-summed error map."""
    _torch()
    mask = np.sort(np.asarray(mask0, dtype=np.int64))
    for t in range(1, len(schedule)):
        R = inpaint_channels(W, H, f_list, mask, unknown_px, rtol=rtol, want_images=False, stream=stream)
        new = femi.densify_step_channels(R["system"], [f.reshape(-1) for f in f_list], R["u_vert"], int(schedule[t]),
                                         stream)
        mask = np.sort(np.concatenate([mask, new.astype(np.int64)]))
    return mask
