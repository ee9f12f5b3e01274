"""Host-stage breakdown of one densification iteration (C3) and of the C5 setup on the GPU
box: mesh_build, assemble, export, gather, solve, raster, select (wall clock with syncs)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2105_01586_b200 import femi, pipeline  # noqa: E402
from synth import make_config  # noqa: E402


def stamp(t):
    torch.cuda.synchronize()
    return time.perf_counter() - t


def iteration(W, H, f, mask, unk, b, st):
    T = {}
    t = time.perf_counter()
    mesh = femi.Mesh(W, H, mask, unk)
    T["mesh"] = stamp(t)
    t = time.perf_counter()
    sysm = femi.System(mesh, st)
    T["assemble"] = stamp(t)
    t = time.perf_counter()
    vert = mesh.export()["vert_px"]
    g = pipeline.mask_values(f, vert, sysm.n_u)
    T["export+gather"] = stamp(t)
    t = time.perf_counter()
    u = torch.empty(sysm.nv, dtype=torch.float64, device=f.device)
    femi.inpaint_solve_batched([sysm], [g], [u], femi.cg_opts(rtol=1e-10), st)
    T["solve"] = stamp(t)
    t = time.perf_counter()
    sse = torch.zeros(1, dtype=torch.float64, device=f.device)
    femi.rasterise_error(sysm, u, f.reshape(-1), sse, None, None, None, None, st)
    T["raster"] = stamp(t)
    t = time.perf_counter()
    new = femi.densify_step(sysm, f.reshape(-1), u, b, st) if b else None
    T["select"] = stamp(t)
    return T, new, mesh.build_seconds


def main():
    st = torch.cuda.current_stream().cuda_stream
    c = make_config(3)
    W, H = c["W"], c["H"]
    f = torch.as_tensor(c["f"], device="cuda").reshape(-1)
    mask = np.sort(c["mask0"].astype(np.int64))
    iteration(W, H, f, mask, c["unknowns"], 0, st)  # warm-up (context, graphs)
    tot = {}
    for t in range(1, len(c["schedule"])):
        T, new, mb = iteration(W, H, f, mask, c["unknowns"], int(c["schedule"][t]), st)
        for k, v in T.items():
            tot[k] = tot.get(k, 0.0) + v
        mask = np.sort(np.concatenate([mask, new.astype(np.int64)]))
    n = len(c["schedule"]) - 1
    print("C3 per iteration (ms):", {k: round(1e3 * v / n, 3) for k, v in tot.items()})
    c = make_config(5)
    W, H = c["W"], c["H"]
    f = torch.as_tensor(c["f"], device="cuda").reshape(-1)
    for rep in range(2):
        T, _, mb = iteration(W, H, f, c["mask0"], c["unknowns"], 0, st)
        print("C5 mask0 (s):", {k: round(v, 4) for k, v in T.items()}, "mesh_build_seconds", round(mb, 4))


if __name__ == "__main__":
    main()
