"""Row-band multi-GPU solve (NEXT-4; include/femi.h femi_band_*).

CPU (not gpu): the band plan (host C code through the ABI) partitions the unknowns, its halo
is exactly the off-band columns of the band's rows, every send segment equals the peer's halo
segment for it, and the band algorithm run over the plan in numpy -- in one process and over
gloo at world_size 2 (halo exchange = point-to-point send/recv, dots = all_reduce) -- reaches
the dense direct solution of the oracle's matrices.
GPU: the library's band kernels over R = 1..4 bands of one process (LoopbackComm) against the
oracle's solve."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2105_01586_b200 import femi, multi
from synth import make_config
from synth.generate import draw_image, draw_mask, draw_unknowns


def _case(W=40, H=32, m=60, p=200, seed=5):
    rng = np.random.default_rng(seed)
    mk = draw_mask(rng, W * H, m)
    un = draw_unknowns(rng, W, H, mk, p)
    f = draw_image(rng, W, H).reshape(-1)
    return W, H, mk, un, f


def _plans(M, R):
    return [femi.band_plan(M, R, r) for r in range(R)]


@pytest.mark.parametrize("R", [1, 2, 3, 5])
def test_band_plan_structure(R):
    W, H, mk, un, _ = _case()
    M = femi.Mesh(W, H, mk, un)
    E = M.export()
    n = M.info["n_unknown"]
    rp, uc = E["uu_rowptr"], E["uu_col"]
    P = _plans(M, R)
    # bands partition [0, n) in rank order, balanced
    assert P[0]["info"]["row0"] == 0 and P[-1]["info"]["row1"] == n
    for a, b in zip(P, P[1:]):
        assert a["info"]["row1"] == b["info"]["row0"]
    sizes = [p["info"]["row1"] - p["info"]["row0"] for p in P]
    assert max(sizes) - min(sizes) <= 1
    owner = np.concatenate([np.full(s, r) for r, s in enumerate(sizes)])
    for r, p in enumerate(P):
        i0, i1 = p["info"]["row0"], p["info"]["row1"]
        cols = uc[rp[i0]:rp[i1]]
        off = np.unique(cols[(cols < i0) | (cols >= i1)])
        np.testing.assert_array_equal(p["halo_id"], off)  # halo = off-band columns, ascending
        # local CSR: same row lengths; local columns map back to the canonical ones
        np.testing.assert_array_equal(p["rowptr"], rp[i0:i1 + 1] - rp[i0])
        loc = p["col"].astype(np.int64)
        nloc = i1 - i0
        hal = np.concatenate([p["halo_id"], [0]])  # (a dummy slot for R = 1)
        glob = np.where(loc < nloc, loc + i0, hal[np.maximum(loc - nloc, 0)])
        np.testing.assert_array_equal(glob, cols)
        # peers = owners of the halo, recv segments grouped by owner
        for k, q in enumerate(p["peer"]):
            seg = p["halo_id"][p["recv_off"][k]:p["recv_off"][k + 1]]
            assert len(seg) > 0 and np.all(owner[seg] == q)
            # what q sends to r is exactly r's halo segment owned by q
            pq = P[q]
            kk = list(pq["peer"]).index(r)
            sent = pq["send_row"][pq["send_off"][kk]:pq["send_off"][kk + 1]] + pq["info"]["row0"]
            np.testing.assert_array_equal(sent, seg)
        if len(p["peer"]):
            assert p["recv_off"][-1] == p["info"]["n_halo"]
        else:
            assert p["info"]["n_halo"] == 0 and R == 1


def _band_cg_numpy(blocks, exchange, allreduce, rtol=1e-12, max_iter=5000):
    """The femi_band_* iteration (single-reduction Jacobi-PCG, x0 = midrange(g)) over the plan,
    in numpy: `blocks` = list of per-band dicts (A_loc over own + halo columns, A_uk rows, plan);
    exchange(vecs) fills each band's halo from its peers; allreduce(list of 4-vectors)."""
    for B in blocks:
        B["x"] = np.full(B["n"], B["c"])
        B["r"] = -(B["Auk"] @ (B["g"] - B["c"]))
        B["b"] = -(B["Auk"] @ B["g"])
        B["u"] = B["r"] / B["d"]
        B["p"] = np.zeros(B["n"])
        B["s"] = np.zeros(B["n"])
    bb = allreduce([np.array([0, 0, 0, B["b"] @ B["b"]]) for B in blocks])[3]

    def spmv():
        halos = exchange([B["u"] for B in blocks])
        dots = []
        for B, h in zip(blocks, halos):
            B["w"] = B["A"] @ np.concatenate([B["u"], h])
            dots.append(np.array([B["r"] @ B["u"], B["w"] @ B["u"], B["r"] @ B["r"], 0.0]))
        return allreduce(dots)

    d = spmv()
    gam_prev = alpha_prev = None
    for k in range(max_iter):
        gamma, delta, rho = d[:3]
        if rho <= rtol * rtol * bb:
            return k
        if k == 0:
            beta, alpha = 0.0, gamma / delta
        else:
            beta = gamma / gam_prev
            alpha = gamma / (delta - beta * gamma / alpha_prev)
        for B in blocks:
            B["p"] = B["u"] + beta * B["p"]
            B["s"] = B["w"] + beta * B["s"]
            B["x"] = B["x"] + alpha * B["p"]
            B["r"] = B["r"] - alpha * B["s"]
            B["u"] = B["r"] / B["d"]
        gam_prev, alpha_prev = gamma, alpha
        d = spmv()
    return max_iter


def _blocks(M, S, g, R, ranks=None):
    Auu, Auk = S.dense_uu(), S.dense_uk()
    c = 0.5 * (g.min() + g.max())
    out = []
    for r in (range(R) if ranks is None else ranks):
        p = femi.band_plan(M, R, r)
        i0, i1 = p["info"]["row0"], p["info"]["row1"]
        cols = np.concatenate([np.arange(i0, i1), p["halo_id"]]).astype(np.int64)
        out.append(dict(plan=p, n=i1 - i0, A=Auu[i0:i1][:, cols], Auk=Auk[i0:i1], d=np.diag(Auu)[i0:i1].copy(),
                        g=g, c=c, rank=r))
    return out


def _loop_exchange(blocks):
    by = {B["rank"]: B for B in blocks}

    def ex(vecs):
        vec = {B["rank"]: v for B, v in zip(blocks, vecs)}
        halos = []
        for B in blocks:
            p = B["plan"]
            h = np.zeros(p["info"]["n_halo"])
            for k, q in enumerate(p["peer"]):
                pq = by[int(q)]["plan"]
                kk = list(pq["peer"]).index(B["rank"])
                h[p["recv_off"][k]:p["recv_off"][k + 1]] = vec[int(q)][pq["send_row"][pq["send_off"][kk]:pq["send_off"][kk + 1]]]
            halos.append(h)
        return halos
    return ex


@pytest.mark.parametrize("R", [1, 2, 4])
def test_band_algorithm_numpy_reaches_dense_solution(R):
    W, H, mk, un, f = _case(seed=11)
    M = femi.Mesh(W, H, mk, un)
    S = oracle.System(W, H, mk, un)
    g = f[np.sort(mk)]
    blocks = _blocks(M, S, g, R)
    it = _band_cg_numpy(blocks, _loop_exchange(blocks), lambda ds: np.sum(ds, axis=0))
    x = np.concatenate([B["x"] for B in blocks])
    ref = np.linalg.solve(S.dense_uu(), -S.dense_uk() @ g)
    assert it < 5000
    assert np.max(np.abs(x - ref)) <= 1e-8 * max(1.0, np.max(np.abs(ref)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, H, mk, un, f = _case(seed=11)
        M = femi.Mesh(W, H, mk, un)
        S = oracle.System(W, H, mk, un)
        g = f[np.sort(mk)]
        (B,) = _blocks(M, S, g, world, ranks=[rank])
        p = B["plan"]

        def ex(vecs):
            (v,) = vecs
            h = torch.zeros(p["info"]["n_halo"], dtype=torch.float64)
            ops = []
            for k, peer in enumerate(p["peer"]):
                send = torch.as_tensor(v[p["send_row"][p["send_off"][k]:p["send_off"][k + 1]]].copy())
                ops.append(dist.P2POp(dist.isend, send, int(peer)))
                ops.append(dist.P2POp(dist.irecv, h[p["recv_off"][k]:p["recv_off"][k + 1]], int(peer)))
            if ops:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
            return [h.numpy()]

        def ar(ds):
            t = torch.as_tensor(ds[0].copy())
            dist.all_reduce(t)
            return t.numpy()

        it = _band_cg_numpy([B], ex, ar)
        q.put((rank, p["info"]["row0"], B["x"].tolist(), it))
    finally:
        dist.destroy_process_group()


def test_band_algorithm_gloo_world2():
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    x = np.concatenate([np.array(v) for _, _, v, _ in res])
    assert res[0][3] == res[1][3]  # the same iteration count on both ranks (same all-reduced dots)
    W, H, mk, un, f = _case(seed=11)
    S = oracle.System(W, H, mk, un)
    g = f[np.sort(mk)]
    ref = np.linalg.solve(S.dense_uu(), -S.dense_uk() @ g)
    assert np.max(np.abs(x - ref)) <= 1e-8 * max(1.0, np.max(np.abs(ref)))


# ------------------------------------------------------------------ GPU: the library's band kernels
def _gpu_band_case(W, H, mk, un, f, R, rtol=1e-10):
    import torch
    M = femi.Mesh(W, H, mk, un)
    g_h = np.asarray(f).reshape(-1)[np.sort(mk)]
    g = torch.as_tensor(g_h, dtype=torch.float64, device="cuda")
    bands = [femi.Band(M, R, r) for r in range(R)]
    rep = multi.band_solve(multi.LoopbackComm(bands), g, rtol=rtol)
    u = torch.empty(M.info["n_unknown"], dtype=torch.float64, device="cuda")
    for b in bands:
        b.result(u[b.row0:b.row1])
    torch.cuda.synchronize()
    return M, rep, u.cpu().numpy(), g_h


@pytest.mark.gpu
@pytest.mark.parametrize("R", [1, 2, 3, 4])
def test_gpu_band_solve_matches_oracle(R):
    W, H, mk, un, f = _case(W=96, H=80, m=300, p=900, seed=3)
    M, rep, u, g = _gpu_band_case(W, H, mk, un, f, R)
    S = oracle.System(W, H, mk, un)
    ref = np.linalg.solve(S.dense_uu(), -S.dense_uk() @ g)
    assert rep["converged"] and rep["rel_res"] <= 1e-10
    assert np.max(np.abs(u - ref)) <= 1e-6, (R, rep)
    # the oracle's own CG solve agrees to the parity tolerance
    uo = S.solve(g, rtol=1e-12)[0]
    assert np.max(np.abs(u - uo[: len(u)])) <= 1e-4


@pytest.mark.gpu
def test_gpu_band_solve_config3_shape_equals_single_gpu_solution():
    """C3-recipe image (512^2, 5 % mask), R = 4 bands: the band solution equals the single-GPU
    solver's within the solve tolerance, and the oracle's at the parity tolerance."""
    import torch
    c = make_config(3)
    W, H = c["W"], c["H"]
    mk = np.asarray(c["mask0"])
    M, rep, u, g = _gpu_band_case(W, H, mk, c["unknowns"], c["f"], 4)
    assert rep["converged"]
    S1 = femi.System(M)
    uv = torch.empty(S1.nv, dtype=torch.float64, device="cuda")
    gd = torch.as_tensor(g, device="cuda")
    # the same algorithm as the single-GPU solver from the same start (x0 = midrange, Jacobi, the
    # same stopping test): the same iteration count up to rounding-order effects
    _, it1, _ = femi.inpaint_solve_batched([S1], [gd], [uv], femi.cg_opts(rtol=1e-10, x0=1))
    assert abs(rep["iters"] - int(it1[0])) <= 2, (rep, int(it1[0]))
    bands = [femi.Band(M, 4, r) for r in range(4)]
    for ce in (1, 8):  # the count does not depend on how often the host polls
        assert multi.band_solve(multi.LoopbackComm(bands), gd, rtol=1e-10, check_every=ce)["iters"] == rep["iters"]
    femi.inpaint_solve_batched([S1], [gd], [uv], femi.cg_opts(rtol=1e-12))
    u1 = uv.cpu().numpy()[: len(u)]
    assert np.max(np.abs(u - u1)) <= 1e-6 * max(1.0, np.abs(u1).max())
    O = oracle.System(W, H, mk, c["unknowns"])
    uo = O.solve(g, rtol=1e-12)[0]
    assert np.max(np.abs(u - uo[: len(u)])) <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("R", [1, 3])
def test_gpu_band_raster_partitions_the_image(R):
    """femi_band_raster_system: R triangle shares rasterised into one image through their row
    offsets give u_px, e_px, tri_err and best bit-identical to the whole mesh's raster on the same
    u_vert; the band SSEs sum to the image's; the band pipeline (band solve + band raster) meets
    the oracle's MSE."""
    import torch
    c = make_config(3)
    W, H = c["W"], c["H"]
    mk = np.asarray(c["mask0"])
    M = femi.Mesh(W, H, mk, c["unknowns"])
    S1 = femi.System(M)
    f = torch.as_tensor(c["f"], dtype=torch.float64, device="cuda").reshape(-1)
    vert = M.vert_px()
    n_u = M.info["n_unknown"]
    g = f[torch.as_tensor(vert[n_u:], dtype=torch.int64, device="cuda")].contiguous()
    uv = torch.empty(S1.nv, dtype=torch.float64, device="cuda")
    femi.inpaint_solve_batched([S1], [g], [uv], femi.cg_opts(rtol=1e-12))
    N = W * H
    ref = dict(u=torch.zeros(N, dtype=torch.float64, device="cuda"), e=torch.zeros(N, dtype=torch.float64, device="cuda"),
               t=torch.zeros(S1.T, dtype=torch.float64, device="cuda"), b=torch.zeros(S1.T, dtype=torch.int32, device="cuda"),
               s=torch.zeros(1, dtype=torch.float64, device="cuda"))
    femi.rasterise_error(S1, uv, f, ref["s"], ref["u"], ref["e"], ref["t"], ref["b"])
    u_img = torch.full((N,), float("nan"), dtype=torch.float64, device="cuda")
    e_img = torch.full((N,), float("nan"), dtype=torch.float64, device="cuda")
    tri = torch.zeros(S1.T, dtype=torch.float64, device="cuda")
    best = torch.zeros(S1.T, dtype=torch.int32, device="cuda")
    sse = 0.0
    for r in range(R):
        Sb, bi = femi.band_raster_system(M, R, r)
        o = bi["y0"] * W
        n = bi["rows"] * W
        fb = f[o:o + n].contiguous()
        ub = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
        eb = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
        tb = torch.zeros(max(Sb.T, 1), dtype=torch.float64, device="cuda")
        bb = torch.zeros(max(Sb.T, 1), dtype=torch.int32, device="cuda")
        sb = torch.zeros(1, dtype=torch.float64, device="cuda")
        femi.rasterise_error(Sb, uv, fb, sb, ub, eb, tb, bb)
        own = ~torch.isnan(ub)
        idx = torch.nonzero(own).reshape(-1) + o
        assert torch.all(torch.isnan(u_img[idx]))  # no pixel written by two shares
        u_img[idx] = ub[own]
        e_img[idx] = eb[own]
        tri[bi["t0"]:bi["t1"]] = tb[:Sb.T]
        best[bi["t0"]:bi["t1"]] = torch.where(bb[:Sb.T] >= 0, bb[:Sb.T] + o, bb[:Sb.T])
        sse += float(sb.item())
        with pytest.raises(femi.FemiError):  # raster-only: no solve
            femi.inpaint_solve_batched([Sb], [g], [uv], femi.cg_opts())
    assert not torch.any(torch.isnan(u_img))  # the shares cover the image
    assert torch.equal(u_img, ref["u"]) and torch.equal(e_img, ref["e"])
    assert torch.equal(tri, ref["t"]) and torch.equal(best, ref["b"])
    assert abs(sse - float(ref["s"].item())) <= 1e-12 * float(ref["s"].item())
    # the whole band pipeline against the oracle
    _, rep, u_b, g_h = _gpu_band_case(W, H, mk, c["unknowns"], c["f"], R)
    O = oracle.inpaint(W, H, c["f"], mk, c["unknowns"], rtol=1e-12)
    uvb = torch.as_tensor(np.concatenate([u_b, g_h]), device="cuda")
    sse_b = 0.0
    for r in range(R):
        Sb, bi = femi.band_raster_system(M, R, r)
        o, n = bi["y0"] * W, bi["rows"] * W
        sb = torch.zeros(1, dtype=torch.float64, device="cuda")
        femi.rasterise_error(Sb, uvb, f[o:o + n].contiguous(), sb)
        sse_b += float(sb.item())
    assert abs(sse_b / N - O["mse"]) <= 1e-6 * O["mse"]


class _FakeBand:
    """CPU stand-in for femi.Band with the real plan: send carries the canonical ids of the sent
    rows, the 'solution' of a row is its canonical id (for the DistComm checks under gloo)."""

    def __init__(self, M, R, r):
        import torch
        p = femi.band_plan(M, R, r)
        self.info = p["info"]
        self.peer, self.recv_off, self.send_off = p["peer"], p["recv_off"], p["send_off"]
        self.row0, self.row1 = self.info["row0"], self.info["row1"]
        self.halo_id = p["halo_id"]
        self.send = torch.as_tensor((p["send_row"] + self.row0).astype(np.float64))
        self.halo = torch.zeros(max(self.info["n_halo"], 1), dtype=torch.float64)
        self.dots = torch.tensor([1.0, 2.0, 3.0, 4.0], dtype=torch.float64) * (r + 1)

    def result(self, u):
        import torch
        u.copy_(torch.arange(self.row0, self.row1, dtype=torch.float64))


def _gloo_comm_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = make_config(3)
        M = femi.Mesh(c["W"], c["H"], np.asarray(c["mask0"]), c["unknowns"])
        b = _FakeBand(M, world, rank)
        comm = multi.DistComm(b)
        comm.exchange()
        halo_ok = bool(np.array_equal(b.halo[: b.info["n_halo"]].numpy(), b.halo_id.astype(np.float64)))
        comm.allreduce()
        nv, n_u = M.info["n_vert"], M.info["n_unknown"]
        u = torch.zeros(nv, dtype=torch.float64)
        g = torch.full((nv - n_u,), -1.0, dtype=torch.float64)
        comm.gather_solution(u, g)
        gather_ok = bool(np.array_equal(u[:n_u].numpy(), np.arange(n_u, dtype=np.float64))) and bool(torch.all(u[n_u:] == -1))
        t = comm.allreduce_scalar(torch.tensor([float(rank + 1)], dtype=torch.float64))
        q.put((rank, halo_ok, b.dots.tolist(), gather_ok, float(t.item()), b.info["n_halo"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distcomm_gloo_exchange_allreduce_gather(world):
    """DistComm over gloo with the real band plans of the C3 mesh: after the exchange every halo
    slot holds its owner's value (here: the canonical id), the dots are summed over ranks, the
    gathered solution is in canonical order on every rank."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    tot = sum(range(1, world + 1))
    for rank, halo_ok, dots, gather_ok, t, nh in res:
        assert nh > 0 and halo_ok and gather_ok
        assert dots == [1.0 * tot, 2.0 * tot, 3.0 * tot, 4.0 * tot]
        assert t == float(tot)
