"""Diagnose GPU vs oracle tonal CGLS at 2880^2 (graph mode): operator agreement and g drift
per outer iteration count."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_2105_01586_b200 import femi, pipeline
from synth import make_config
W = int(sys.argv[1]) if len(sys.argv) > 1 else 2880
dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda:0")
c = make_config(5, W=W, H=W, seed=58)
fd = dev(c["f"])
mask, _, _ = pipeline.densify(W, W, fd, c["mask0"], c["unknowns"], c["schedule"][:2])
M = femi.Mesh(W, W, mask, c["unknowns"]); S = femi.System(M)
O = oracle.System(W, W, mask, c["unknowns"])
vert = M.export()["vert_px"]
rng = np.random.default_rng(5)
x = rng.uniform(0, 255, S.m); y = rng.uniform(-50, 50, W * W)
Bx = torch.empty(W * W, dtype=torch.float64, device="cuda:0"); BTy = torch.empty(S.m, dtype=torch.float64, device="cuda:0")
opts = femi.cg_opts(rtol=1e-12)
femi.apply_B(S, dev(x), Bx, opts); femi.apply_BT(S, dev(y), BTy, opts)
print("path", femi.solver_path(S))
oBx = O.apply_B(x); oBTy = O.apply_BT(y)
print("apply_B max diff", np.abs(Bx.cpu().numpy() - oBx).max(), "max |Bx|", np.abs(oBx).max())
d = np.abs(BTy.cpu().numpy() - oBTy)
print("apply_BT max diff", d.max(), "at", d.argmax(), "val", oBTy[d.argmax()], "max |BTy|", np.abs(oBTy).max(), "rel", d.max() / np.abs(oBTy).max())
lhs = float(Bx.cpu().numpy() @ y); rhs = float(x @ BTy.cpu().numpy())
print("adjoint gpu rel", abs(lhs - rhs) / abs(lhs))
for K in (1, 2, 5, 10, 20):
    g = pipeline.mask_values(fd, vert, S.n_u)
    st, rep = femi.tonal_optimise(S, fd.reshape(-1), g, outer_rtol=1e-300, outer_max=K, inner=opts)
    go, orep = O.tonal(c["f"], outer_tol=1e-300, outer_max=K, inner_rtol=1e-12, inner_method=3)
    gg = g.cpu().numpy(); dd = np.abs(gg - go)
    print(f"K={K} max|dg| {dd.max():.3e} at {dd.argmax()} g {go[dd.argmax()]:.4f} max|g| {np.abs(go).max():.2f} "
          f"mse gpu {rep['mse_after']:.10f} ora {orep['mse_after']:.10f} relg {rep['rel_grad']:.3e} {orep['rel_grad']:.3e}")
