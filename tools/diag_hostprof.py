import sys, time, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2105_01586_b200 import femi, pipeline
from synth import make_config
c = make_config(1)
f = torch.as_tensor(c['f'], dtype=torch.float64, device='cuda').reshape(-1)
M = femi.Mesh(64, 64, c['mask'], c['unknowns']); S = femi.System(M)
g = pipeline.mask_values(f, M.export()['vert_px'], S.n_u)
u = torch.empty(S.nv, dtype=torch.float64, device='cuda')
P = femi.SolvePlan([S], [g], [u], femi.cg_opts(rtol=1e-10))
for k in range(30): P.run()
torch.cuda.synchronize()
t = time.perf_counter()
for k in range(200): P.run()
print("host wall per solve us", (time.perf_counter() - t) / 200 * 1e6)
t = time.perf_counter()
for k in range(2000): femi.version()
print("ctypes call us", (time.perf_counter() - t) / 2000 * 1e6)
P0 = femi.SolvePlan([S], [g], [u], femi.cg_opts(rtol=1e300))
t = time.perf_counter()
for k in range(200): P0.run()
print("0-iteration host wall per solve us", (time.perf_counter() - t) / 200 * 1e6)
os.environ["X"] = "1"
