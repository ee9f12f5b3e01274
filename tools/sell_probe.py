"""Solve a few systems (C1, C2 items 0-3, C3 first mesh, C4) and save u_vert + iteration counts
to an .npz (used by tests/test_gpu_parity.py::test_device_layouts_match_host to compare the
device-built solver layouts with FEMI_SELL_HOST=1 in a second process)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_01586_b200 import femi, pipeline
from synth import make_config
out = {}
dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda:0")
cases = []
c = make_config(1); cases.append(("c1", c, c["mask"], c["unknowns"]))
c2 = make_config(2)
for b in range(4):
    cases.append((f"c2_{b}", c2, c2["masks"][b], c2["unknowns"][b]))
c = make_config(3); cases.append(("c3", c, c["mask0"], c["unknowns"]))
c = make_config(4); cases.append(("c4", c, c["mask"], c["unknowns"]))
for name, c, mk, un in cases:
    f = dev(c["f"]).reshape(-1)
    M = femi.Mesh(c["W"], c["H"], mk, un)
    S = femi.System(M)
    g = pipeline.mask_values(f, M.export()["vert_px"], S.n_u)
    u = torch.empty(S.nv, dtype=torch.float64, device="cuda:0")
    st, it, rel = femi.inpaint_solve_batched([S], [g], [u], femi.cg_opts(rtol=1e-10))
    sse = torch.zeros(1, dtype=torch.float64, device="cuda:0")
    femi.rasterise_error(S, u, f, sse)
    out[name + "_u"] = u.cpu().numpy()
    out[name + "_it"] = np.array([it[0], st])
    out[name + "_sse"] = sse.cpu().numpy()
np.savez(sys.argv[1], **out)
print("ok", len(cases))
