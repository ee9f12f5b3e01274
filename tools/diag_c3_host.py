"""Host-side split of one C3 densification run (BASELINE configs[2]): per iteration, the time
of each host stage around the GPU work, to find what the C3 end-to-end time is made of.
    python tools/diag_c3_host.py [reps]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from synth import make_config  # noqa: E402
from paper_2105_01586_b200 import femi, pipeline  # noqa: E402


def run(c, f_dev, tm):
    W, H = c["W"], c["H"]
    sched = c["schedule"]
    mask = np.sort(np.asarray(c["mask0"], dtype=np.int64))
    M, new, S = None, None, None
    t_all = time.perf_counter()
    for t in range(1, len(sched) + 1):
        t0 = time.perf_counter()
        M = femi.Mesh(W, H, mask, c["unknowns"]) if M is None else M.insert(new)
        t1 = time.perf_counter()
        S_old, S = S, None
        del S_old
        t2 = time.perf_counter()
        S = femi.System(M)
        t3 = time.perf_counter()
        vert = M.vert_px()
        g = pipeline.mask_values(f_dev, vert, S.n_u)
        u = torch.empty(S.nv, dtype=torch.float64, device="cuda")
        sse = torch.zeros(1, dtype=torch.float64, device="cuda")
        tri = torch.empty(max(S.T, 1), dtype=torch.float64, device="cuda")
        bst = torch.empty(max(S.T, 1), dtype=torch.int32, device="cuda")
        t4 = time.perf_counter()
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        femi.inpaint_solve_batched([S], [g], [u], femi.cg_opts(rtol=1e-10))
        t6 = time.perf_counter()
        femi.rasterise_error(S, u, f_dev, sse, tri_err=tri, best=bst)
        new = femi.densify_step(S, f_dev, u, int(sched[t])) if t < len(sched) else None
        torch.cuda.synchronize()
        t7 = time.perf_counter()
        if new is not None:
            mask = np.sort(np.concatenate([mask, new.astype(np.int64)]))
        t8 = time.perf_counter()
        for k, v in zip(("mesh", "free_old", "assemble", "export+g+alloc", "sync", "solve", "raster+select",
                         "mask_update"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t7 - t6, t8 - t7)):
            tm.setdefault(k, []).append(v)
    torch.cuda.synchronize()
    return time.perf_counter() - t_all


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    c = make_config(3)
    f_dev = torch.as_tensor(c["f"], dtype=torch.float64, device="cuda").reshape(-1)
    for _ in range(2):
        run(c, f_dev, {})
    tot, tm = [], {}
    for _ in range(reps):
        tot.append(run(c, f_dev, tm))
    print(f"C3 run (n={len(c['schedule'])}): median {1e3 * np.median(tot):.2f} ms end to end (min {1e3 * min(tot):.2f})")
    n = len(c["schedule"])
    for k, v in tm.items():
        v = np.array(v).reshape(reps, n)
        print(f"  {k:15s} {1e3 * np.median(v.sum(1)):8.2f} ms/run   first iter {1e3 * np.median(v[:, 0]):7.2f} ms")


if __name__ == "__main__":
    main()
