"""Set up one inpainting workload and run `--steps` solve+raster steps inside a
cudaProfilerStart/Stop range (for `ncu --profile-from-start off`).

Usage: python tools/profile_step.py --config 5 --steps 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2105_01586_b200 import femi, pipeline  # noqa: E402
from synth import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--densify", type=int, default=1)
a = ap.parse_args()
c = make_config(a.config)
W, H = c["W"], c["H"]
f = torch.as_tensor(c["f"], dtype=torch.float64, device="cuda").reshape(-1)
if c["kind"].startswith("densify") and a.densify:
    mask, _, _ = pipeline.densify(W, H, f, c["mask0"], c["unknowns"], c["schedule"][:2])
else:
    mask = c.get("mask", c.get("mask0"))
mesh = femi.Mesh(W, H, mask, c["unknowns"])
S = femi.System(mesh)
g = pipeline.mask_values(f, mesh.export()["vert_px"], S.n_u)
u = torch.empty(S.nv, dtype=torch.float64, device="cuda")
upx = torch.empty(W * H, dtype=torch.float64, device="cuda")
epx = torch.empty(W * H, dtype=torch.float64, device="cuda")
te = torch.empty(S.T, dtype=torch.float64, device="cuda")
bs = torch.empty(S.T, dtype=torch.int32, device="cuda")
sse = torch.zeros(1, dtype=torch.float64, device="cuda")
for _ in range(2):  # warm-up outside the profiled range
    femi.inpaint_solve_batched([S], [g], [u], femi.cg_opts(rtol=1e-10))
    femi.rasterise_error(S, u, f, sse, upx, epx, te, bs)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(a.steps):
    st, it, rel = femi.inpaint_solve_batched([S], [g], [u], femi.cg_opts(rtol=1e-10))
    femi.rasterise_error(S, u, f, sse, upx, epx, te, bs)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("iters", it, "relres", rel, "mse", sse.item() / (W * H), "launches", femi.kernel_launches())
