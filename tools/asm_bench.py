"""Repeated assemble of one mesh (C3 size): wall time of System() and of its release."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2105_01586_b200 import femi  # noqa: E402
from synth import make_config  # noqa: E402

c = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
mk = c.get("mask0", c.get("mask"))
mesh = femi.Mesh(c["W"], c["H"], mk, c["unknowns"])
st = torch.cuda.current_stream().cuda_stream
torch.cuda.synchronize()
ta, tf = [], []
for r in range(12):
    t = time.perf_counter()
    s = femi.System(mesh, st)
    torch.cuda.synchronize()
    ta.append(time.perf_counter() - t)
    t = time.perf_counter()
    s.close() if hasattr(s, "close") else None
    del s
    torch.cuda.synchronize()
    tf.append(time.perf_counter() - t)
print("assemble ms", np.round(1e3 * np.array(ta), 2))
print("free ms", np.round(1e3 * np.array(tf), 2))
