"""Band solve vs the single-GPU solver: iteration counts and solutions (R bands, loopback).
    python tools/diag_band.py CONFIG [R...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from synth import make_config  # noqa: E402
from paper_2105_01586_b200 import femi, multi, pipeline  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
Rs = [int(a) for a in sys.argv[2:]] or [1, 4]
c = make_config(cfg)
W, H = c["W"], c["H"]
f = torch.as_tensor(c["f"], dtype=torch.float64, device="cuda").reshape(-1)
if c["kind"].startswith("densify"):
    mask, _, _ = pipeline.densify(W, H, f, c["mask0"], c["unknowns"], c["schedule"][:2], rtol=1e-10)
else:
    mask = c["mask"]
M = femi.Mesh(W, H, mask, c["unknowns"])
S = femi.System(M)
vert = M.vert_px()
n_u = M.info["n_unknown"]
g = f[torch.as_tensor(vert[n_u:], dtype=torch.int64, device="cuda")].contiguous()
for x0 in (1, 3):
    uv = torch.empty(S.nv, dtype=torch.float64, device="cuda")
    st, it, rel = femi.inpaint_solve_batched([S], [g], [uv], femi.cg_opts(rtol=1e-10, x0=x0))
    print(f"single-GPU solver x0={x0}: iters {int(it[0])} relres {float(rel[0]):.3e}")
ref = uv[:n_u].clone()
for R in Rs:
    bands = [femi.Band(M, R, r) for r in range(R)]
    for ce in (1, 8):
        rep = multi.band_solve(multi.LoopbackComm(bands), g, rtol=1e-10, check_every=ce)
        u = torch.empty(n_u, dtype=torch.float64, device="cuda")
        for b in bands:
            b.result(u[b.row0:b.row1])
        print(f"band R={R} check_every={ce}: {rep} max|u - single| = {float((u - ref).abs().max()):.3e}")
