"""A/B bit-identity check of the solver across a library change.

    FEMI_LIB=<lib.so> python tools/ab_bits.py dump out.npz
    python tools/ab_bits.py compare a.npz b.npz

`dump` runs one solve per path and initial-guess mode (graph single-RHS, graph multi-RHS,
batched non-graph, the given-b operator pair B / B^T) on seeded synthetic inputs and stores
u_vert, iteration counts and relative residuals; `compare` requires every array to be
bitwise equal."""
import sys

import numpy as np


def dump(out):
    import torch
    sys.path.insert(0, ".")
    from synth import make_config
    from paper_2105_01586_b200 import femi, pipeline

    dev = "cuda:0"
    res = {}
    c = make_config(5, W=2880, H=2880, seed=58)
    W = 2880
    fd = torch.as_tensor(c["f"], dtype=torch.float64, device=dev)
    M = femi.Mesh(W, W, c["mask0"], c["unknowns"])
    S = femi.System(M)
    vert = M.export()["vert_px"]
    g = pipeline.mask_values(fd, vert, S.n_u)
    rng = np.random.default_rng(3)
    for x0 in (0, 1, 2, 3):
        u = torch.zeros(S.n_u + S.m, dtype=torch.float64, device=dev)
        if x0 == 2:
            u[: S.n_u] = torch.as_tensor(rng.uniform(0, 255, S.n_u), device=dev)
        st, it, rel = femi.inpaint_solve_batched([S], [g], [u], femi.cg_opts(x0=x0))
        res[f"single_x0{x0}"] = u.cpu().numpy()
        res[f"single_x0{x0}_it"] = np.array([st, *it, *rel])
        res[f"single_x0{x0}_path"] = np.array([ord(ch) for ch in femi.solver_path(S)])
    gs = [g, g * 0.5 + 3.0, 255.0 - g]
    for x0 in (1, 3):
        us = [torch.zeros(S.n_u + S.m, dtype=torch.float64, device=dev) for _ in gs]
        st, it, rel = femi.inpaint_solve_batched([S, S, S], gs, us, femi.cg_opts(x0=x0))
        for k, u in enumerate(us):
            res[f"multi_x0{x0}_{k}"] = u.cpu().numpy()
        res[f"multi_x0{x0}_it"] = np.array([st, *it, *rel])
    small = []
    cs = make_config(2)
    fs = torch.as_tensor(cs["f"], dtype=torch.float64, device=dev)
    for k in range(3):
        Ms = femi.Mesh(cs["W"], cs["H"], cs["masks"][k], cs["unknowns"][k])
        Ss = femi.System(Ms)
        small.append((Ss, pipeline.mask_values(fs, Ms.export()["vert_px"], Ss.n_u)))
    for x0 in (1, 3):
        us = [torch.zeros(s.n_u + s.m, dtype=torch.float64, device=dev) for s, _ in small]
        st, it, rel = femi.inpaint_solve_batched([s for s, _ in small], [gg for _, gg in small], us,
                                                 femi.cg_opts(x0=x0))
        for k, u in enumerate(us):
            res[f"batched_x0{x0}_{k}"] = u.cpu().numpy()
        res[f"batched_x0{x0}_it"] = np.array([st, *it, *rel])
    x = torch.as_tensor(rng.uniform(0, 255, S.m), device=dev)
    y = torch.as_tensor(rng.uniform(-50, 50, W * W), device=dev)
    Bx = torch.empty(W * W, dtype=torch.float64, device=dev)
    BTy = torch.empty(S.m, dtype=torch.float64, device=dev)
    femi.apply_B(S, x, Bx, femi.cg_opts(rtol=1e-12))
    femi.apply_BT(S, y, BTy, femi.cg_opts(rtol=1e-12))
    res["apply_B"] = Bx.cpu().numpy()
    res["apply_BT"] = BTy.cpu().numpy()
    np.savez(out, **res)
    print(f"wrote {out}: {len(res)} arrays")


def compare(a, b):
    A, B = np.load(a), np.load(b)
    bad = 0
    for k in sorted(set(A.files) | set(B.files)):
        if k not in A.files or k not in B.files:
            print(f"{k}: missing on one side")
            bad += 1
            continue
        x, y = A[k], B[k]
        same = x.shape == y.shape and np.array_equal(x.view(np.uint8), y.view(np.uint8))
        if not same:
            bad += 1
            d = np.abs(x - y).max() if x.shape == y.shape else float("nan")
            print(f"{k}: DIFFERS (max |d| = {d:.3e})")
        elif k.endswith("_it"):
            print(f"{k}: identical {x.tolist()}")
    print("ALL BIT-IDENTICAL" if bad == 0 else f"{bad} arrays differ")
    return bad


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(sys.argv[2])
    else:
        sys.exit(1 if compare(sys.argv[2], sys.argv[3]) else 0)
