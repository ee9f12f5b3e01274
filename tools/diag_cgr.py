"""Resident solver (k_cgp / k_cgr) timing on the C1, C2 (32-item batch) and C4 systems: event time
of a full solve and of a 0-iteration solve (the fixed per-solve cost), median of 20.
Run with FEMI_CG_PIPE=0/1 and FEMI_PCG_TIMERS=1 for the per-phase split."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_01586_b200 import femi, pipeline
from synth import make_config
dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda:0")
st = torch.cuda.current_stream()
def timed(Ss, gs, us, o, reps=None):
    reps = REPS if reps is None else reps
    ts = []
    for k in range(reps + 3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st); _, it, rel = femi.inpaint_solve_batched(Ss, gs, us, o); b.record(st)
        torch.cuda.synchronize()
        if k >= 3: ts.append(a.elapsed_time(b))
    return float(np.median(ts)), np.asarray(it), np.asarray(rel)
CFGS = [int(a) for a in sys.argv[1].split(',')] if len(sys.argv) > 1 else [1, 2, 4]
REPS = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for k in CFGS:
    c = make_config(k)
    f = dev(c["f"]).reshape(-1)
    items = ([dict(mask=a, unknowns=b) for a, b in zip(c["masks"], c["unknowns"])] if "masks" in c
             else [dict(mask=c.get("mask", c.get("mask0")), unknowns=c["unknowns"])])
    Ss, gs, us = [], [], []
    for itm in items:
        M = femi.Mesh(c["W"], c["H"], itm["mask"], itm["unknowns"]); S = femi.System(M)
        Ss.append(S); gs.append(pipeline.mask_values(f, M.export()["vert_px"], S.n_u))
        us.append(torch.empty(S.nv, dtype=torch.float64, device="cuda:0"))
    for rt in (1e-10, 1e-12):
        ms, it, rel = timed(Ss, gs, us, femi.cg_opts(rtol=rt))
        print(f"C{k} rtol {rt:g}: {ms*1e3:9.1f} us  iters max {it.max()} mean {it.mean():.1f}  relres max {rel.max():.2e}  path {femi.solver_path(Ss[0])}")
    ms0, _, _ = timed(Ss, gs, us, femi.cg_opts(rtol=1e300))
    print(f"C{k} 0-iteration solve: {ms0*1e3:9.1f} us")
