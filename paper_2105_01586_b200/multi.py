"""Multi-GPU plumbing (host logic only).

The hot path runs on one GPU. Across GPUs there are three modes; the first two have no
collective on the data path:

* replicas -- every rank runs the whole workload (weak scaling; bench.py's default);
* batch sharding -- independent units (C2's 32 masks, colour channels, images) are split
  into contiguous shards, one per rank; the only exchange is gathering the per-unit scalars
  (MSE, iteration counts) at the end.

* row bands (NEXT-4) -- ONE image's solve split over ranks by bands of unknowns (femi_band_*):
  per CG iteration one halo exchange with the neighbouring bands and one all-reduce of four
  doubles. `band_solve` sequences the library calls; the exchange and the all-reduce go through
  a comm object: `DistComm` (torch.distributed: NCCL on GPUs) or `LoopbackComm` (several bands
  in one process, stepped in lockstep -- the single-GPU test stand-in; no kernel waits on
  another).

Device time of a multi-rank run is the MAX over ranks (one all-reduce of a scalar), never
wall clock. Works with any torch.distributed backend (nccl on the GPU box, gloo in the CPU
tests).
"""
from __future__ import annotations

import numpy as np


def shard(n_items: int, rank: int, world: int) -> range:
    """Contiguous, balanced shard of [0, n_items) for `rank` (sizes differ by at most one)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    lo = n_items * rank // world
    hi = n_items * (rank + 1) // world
    return range(lo, hi)


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def max_over_ranks(value: float, device=None) -> float:
    """The job's time: max of a per-rank scalar (identity when not distributed)."""
    dist = _dist()
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_scalars(local: np.ndarray, n_items: int, device=None) -> np.ndarray:
    """Per-unit scalars of every rank's shard, in global unit order (all ranks get them)."""
    local = np.asarray(local, dtype=np.float64)
    dist = _dist()
    if dist is None:
        if local.size != n_items:
            raise ValueError("not distributed: the local shard must hold every unit")
        return local.copy()
    import torch
    world = dist.get_world_size()
    width = max(len(shard(n_items, r, world)) for r in range(world))
    buf = torch.full((width,), float("nan"), dtype=torch.float64, device=device)
    buf[: local.size] = torch.as_tensor(local, dtype=torch.float64)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    parts = [outs[r][: len(shard(n_items, r, world))].cpu().numpy() for r in range(world)]
    return np.concatenate(parts)


# ------------------------------------------------------------------ row bands (NEXT-4)
class LoopbackComm:
    """The bands of one process: the exchange copies every band's send segment for a peer into
    that peer's halo slots for it; the all-reduce sums the bands' dots in rank order (what an
    NCCL all-reduce computes across processes)."""

    def __init__(self, bands):
        self.bands = sorted(bands, key=lambda b: b.info["rank"])
        self.by_rank = {b.info["rank"]: b for b in self.bands}
        self.pairs = []
        for b in self.bands:
            r = b.info["rank"]
            for i, q in enumerate(b.peer):
                dst = self.by_rank[int(q)]
                j = list(dst.peer).index(r)
                s0, s1 = int(b.send_off[i]), int(b.send_off[i + 1])
                d0, d1 = int(dst.recv_off[j]), int(dst.recv_off[j + 1])
                if s1 - s0 != d1 - d0:
                    raise ValueError(f"band plan mismatch: rank {r} sends {s1 - s0} to {q}, which expects {d1 - d0}")
                self.pairs.append((b, s0, s1, dst, d0, d1))

    def exchange(self):
        for b, s0, s1, dst, d0, d1 in self.pairs:
            if s1 > s0:
                dst.halo[d0:d1].copy_(b.send[s0:s1])

    def gather_solution(self, u_vert, g):
        """u_vert (n_vert, canonical) = the bands' solutions + the mask values g."""
        for b in self.bands:
            b.result(u_vert[b.row0:b.row1])
        n_u = self.bands[0].info["n_unknown"]
        u_vert[n_u:].copy_(g)

    def allreduce_scalar(self, t):
        return t

    def allreduce(self):
        tot = self.bands[0].dots.clone()
        for b in self.bands[1:]:
            tot += b.dots
        for b in self.bands:
            b.dots.copy_(tot)


class DistComm:
    """One band per process over torch.distributed (NCCL on the GPU box): the halo exchange is
    one batch of point-to-point send / recv with the peers, the all-reduce a 4-double SUM."""

    def __init__(self, band):
        import torch.distributed as dist
        self.dist, self.band = dist, band

    @property
    def bands(self):
        return [self.band]

    def exchange(self):
        dist, b = self.dist, self.band
        ops = []
        for i, q in enumerate(b.peer):
            s0, s1 = int(b.send_off[i]), int(b.send_off[i + 1])
            r0, r1 = int(b.recv_off[i]), int(b.recv_off[i + 1])
            ops.append(dist.P2POp(dist.isend, b.send[s0:s1], int(q)))
            ops.append(dist.P2POp(dist.irecv, b.halo[r0:r1], int(q)))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def allreduce(self):
        self.dist.all_reduce(self.band.dots)

    def gather_solution(self, u_vert, g):
        """u_vert (n_vert, canonical) on every rank: all-gather of the bands' solutions (padded to
        the largest band) + the mask values g."""
        import torch
        b = self.band
        world = self.dist.get_world_size()
        n_u = b.info["n_unknown"]
        width = max(n_u * (r + 1) // world - n_u * r // world for r in range(world))
        mine = torch.zeros(width, dtype=torch.float64, device=u_vert.device)
        b.result(mine[: b.row1 - b.row0])
        outs = [torch.empty_like(mine) for _ in range(world)]
        self.dist.all_gather(outs, mine)
        for r in range(world):
            lo, hi = n_u * r // world, n_u * (r + 1) // world
            u_vert[lo:hi].copy_(outs[r][: hi - lo])
        u_vert[n_u:].copy_(g)

    def allreduce_scalar(self, t):
        self.dist.all_reduce(t)
        return t


def band_solve(comm, g, rtol=1e-10, max_iter=100000, check_every=8, max_restarts=3):
    """Row-band Jacobi-PCG of one image (femi.h femi_band_*): every band of `comm` steps in
    lockstep; returns {'iters', 'restarts', 'rel_res', 'converged'} (identical on every rank).
    The solution of each band is in band.result()."""
    bands = comm.bands

    def spmv(which):
        for b in bands:
            b.pack(which)
        comm.exchange()
        for b in bands:
            b.spmv(which)
        comm.allreduce()

    for b in bands:
        b.begin(g, rtol)
    comm.allreduce()  # ||b||^2
    spmv(0)
    it, restarts = 0, 0
    while True:
        while True:
            for b in bands:
                b.update()
            it += 1
            if it % check_every == 0 or it >= max_iter:
                done, _, _ = bands[0].status()
                if done or it >= max_iter:
                    break
            spmv(0)
        spmv(1)  # true residual b - A x (reading A11)
        done, iters, d = bands[0].status()
        res2, bb = d[2], d[3]
        ok = bb == 0.0 or res2 <= rtol * rtol * bb
        if ok or restarts >= max_restarts or it >= max_iter:
            break
        restarts += 1
        for b in bands:
            b.restart()
        spmv(0)
    return {"iters": iters, "restarts": restarts, "rel_res": float(np.sqrt(res2 / bb)) if bb > 0 else 0.0,
            "converged": bool(ok)}
