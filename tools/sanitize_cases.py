"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck), one per case:
  c1     C1: mesh, assemble, resident on-chip solve (k_cgr, one CTA), raster, densify_step,
         3 tonal iterations
  c2     C2 shape: 4 distinct 256^2 meshes as one block-diagonal batch (k_cgr clusters) + rasters
  graph  2880^2 C5 recipe: graph-mode solve (k_gu / k_gt with PDL and TMA), raster
  dmulti densify_step on the multi-kernel selection (FEMI_SEL_MULTI) incl. the shortfall fill
  tonal  2 tonal CGLS iterations on the graph-mode system (adjoint raster, gathers, inner solves)
Exit code 0 when every call returned OK; the sanitizer's own summary decides the verdict."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_01586_b200 import femi, pipeline  # noqa: E402
from synth import make_config  # noqa: E402

DEV = "cuda:0"


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=DEV)


def c1():
    c = make_config(1)
    f = dev(c["f"])
    R = pipeline.inpaint(64, 64, f, c["mask"], c["unknowns"])
    assert R["status"] == 0
    femi.densify_step(R["system"], f.reshape(-1), R["u_vert"], 20)
    g, rep, _ = pipeline.tonal(64, 64, f, c["mask"], c["unknowns"], outer_rtol=1e-12, outer_max=3)
    print("c1 ok", femi.solver_path(R["system"]), rep["outer_iters"])


def c2():
    c = make_config(2)
    W, H = c["W"], c["H"]
    f = dev(c["f"]).reshape(-1)
    systems = [femi.System(femi.Mesh(W, H, c["masks"][b], c["unknowns"][b])) for b in range(4)]
    gs = [pipeline.mask_values(f, femi.Mesh(W, H, c["masks"][b], c["unknowns"][b]).export()["vert_px"], s.n_u)
          for b, s in enumerate(systems)]
    us = [torch.empty(s.nv, dtype=torch.float64, device=DEV) for s in systems]
    st, it, rel = femi.inpaint_solve_batched(systems, gs, us, femi.cg_opts(rtol=1e-10))
    assert st == 0
    sse = [torch.zeros(1, dtype=torch.float64, device=DEV) for _ in systems]
    femi.rasterise_error_batched(systems, us, [f] * 4, sse)
    torch.cuda.synchronize()
    print("c2 ok", femi.solver_path(systems[0]), list(it))


def _graph_system():
    W = 2880
    c = make_config(5, W=W, H=W, seed=58)
    f = dev(c["f"])
    mask, _, _ = pipeline.densify(W, W, f, c["mask0"], c["unknowns"], c["schedule"][:2])
    return W, c, f, mask


def graph():
    W, c, f, mask = _graph_system()
    R = pipeline.inpaint(W, W, f, mask, c["unknowns"])
    assert R["status"] == 0
    print("graph ok", femi.solver_path(R["system"]), R["iters"])


def dmulti():
    os.environ["FEMI_SEL_MULTI"] = "1"
    c = make_config(3)
    f = dev(c["f"])
    R = pipeline.inpaint(512, 512, f, c["mask0"], c["unknowns"], want_images=False)
    a = femi.densify_step(R["system"], f.reshape(-1), R["u_vert"], int(c["schedule"][1]))
    b = femi.densify_step(R["system"], f.reshape(-1), R["u_vert"], R["system"].T + 100)
    print("dmulti ok", a.size, b.size)


def tonal():
    W, c, f, mask = _graph_system()
    M = femi.Mesh(W, W, mask, c["unknowns"])
    S = femi.System(M)
    g = pipeline.mask_values(f, M.export()["vert_px"], S.n_u)
    st, rep = femi.tonal_optimise(S, f.reshape(-1), g, outer_rtol=1e-300, outer_max=2)
    print("tonal ok", femi.solver_path(S), rep["outer_iters"], st)


if __name__ == "__main__":
    globals()[sys.argv[1]]()
