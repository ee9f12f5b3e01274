"""Prologue / epilogue cost of one C5 graph-mode solve: event time of a full solve against a
0-iteration solve (rtol so loose that x0 meets it) for the fill and the midrange starts."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_01586_b200 import femi, pipeline
from synth import make_config
W = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
c = make_config(5, W=W, H=W)
f = torch.as_tensor(c["f"], dtype=torch.float64, device="cuda:0").reshape(-1)
mask, _, _ = pipeline.densify(W, W, f, c["mask0"], c["unknowns"], c["schedule"][:2])
M = femi.Mesh(W, W, mask, c["unknowns"]); S = femi.System(M)
g = pipeline.mask_values(f, M.export()["vert_px"], S.n_u)
u = torch.empty(S.nv, dtype=torch.float64, device="cuda:0")
st = torch.cuda.current_stream()
def timed(opts, reps=5):
    ts = []
    for k in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); s2, it, rel = femi.inpaint_solve_batched([S], [g], [u], opts); b.record(st)
        torch.cuda.synchronize()
        if k >= 2: ts.append(a.elapsed_time(b))
    return float(np.median(ts)), int(it[0])
for name, o in [("fill full", femi.cg_opts(rtol=1e-10, x0=3)), ("fill 0-iter", femi.cg_opts(rtol=1e300, x0=3)),
                ("midrange full", femi.cg_opts(rtol=1e-10, x0=1)), ("midrange 0-iter", femi.cg_opts(rtol=1e300, x0=1))]:
    ms, it = timed(o)
    print(f"{name:16s} {ms:8.3f} ms  iters {it}")
sse = torch.zeros(1, dtype=torch.float64, device="cuda:0")
ts = []
for k in range(7):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); femi.rasterise_error(S, u, f, sse); b.record(st); torch.cuda.synchronize()
    if k >= 2: ts.append(a.elapsed_time(b))
print(f"raster sse/tri only {np.median(ts):.3f} ms")
