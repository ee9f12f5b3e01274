#!/usr/bin/env python
"""bench.py -- FEM harmonic inpainting hot path on B200 (arXiv 2105.01586).

Workload (default, BASELINE.json configs[4], "C5"): 8192x8192 fp64 synthetic image (bump
sigma x32), 2 % mask from one densification pass (1 % random + 1 % selected by per-triangle
error), p = m unknown vertices. Setup (untimed, reported): image generation, the
densification pass, host mesh_build, assemble. One timed STEP = one full inpainting:
inpaint_solve (Jacobi-PCG to relative residual 1e-10, x0 = midrange(g)) + rasterise_error
(u image, e image, per-triangle error and best pixel, SSE). Inputs (f 537 MB) exceed L2,
so no extra flush is needed between steps.

    value  = whole-job Mpixels/s = ranks * W*H * K / max-over-ranks device time
    e2e    = the same with f and g copied host->device (pinned) and SSE device->host
             inside every step; the copies run on a second stream into double buffers, so
             step k+1's inputs move while step k computes (PCIe-bound: ~10 ms of copies
             against ~4.8 ms of compute at C5)
    roofline: the PCG iteration (k_gu update + k_gt TMA SpMV), algorithmic bytes per iteration
             12 nnz_uu + 4 (n_u+1) + 80 n_u x iterations over
             the solve's device time, against MEASURED_PEAKS.json hbm_gbs.
    cpu_baseline: the fp64 oracle (oracle/, 1 thread) on the same workload, run in a
             separate process on a host core while the GPU part runs.

--impl reference times the oracle alone (the reference arm of this tier).
--gpus N (torchrun): replicas only -- every rank runs its own copy.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import make_config, schedule  # noqa: E402

RTOL = 1e-10


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5,
                    help="1/5: single-image inpainting (the headline); 2: 32-mask batch; 3: densification; "
                         "4: tonal optimisation; 6: colour C5 (3 channels on one mesh, NEXT-1)")
    ap.add_argument("--size", type=int, default=0, help="override W=H (scaled variant of the config)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tonal", action="store_true", help="C5: skip the 20-iteration tonal tail")
    ap.add_argument("--n", type=int, default=0, help="C3: densification iterations (default: the config's 10)")
    ap.add_argument("--warm", action="store_true", help="C3: warm-start each solve from the previous solution")
    ap.add_argument("--rebuild-mesh", action="store_true",
                    help="C3: build every densification mesh from scratch instead of inserting the new pixels")
    ap.add_argument("--band", action="store_true",
                    help="NEXT-4: ONE image over the torchrun ranks in row bands (solve + raster + error; strong scaling)")
    ap.add_argument("--bands", type=int, default=0,
                    help="with --band at N=1: R bands of one process stepped in lockstep (single-GPU check)")
    ap.add_argument("--shard", action="store_true",
                    help="C2 under torchrun: split the 32 masks across ranks (strong scaling) instead of replicas")
    return ap.parse_args()


# ----------------------------------------------------------------------------- inputs

def workload_inputs(cfg: int, size: int = 0):
    """Seeded inputs; for the densify-type config the initial random mask + schedule."""
    c = make_config(cfg, W=size or None, H=size or None)
    return c


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is None:
            return
        time.sleep(0.15)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def summary(self):
        if not getattr(self, "rows", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- oracle (CPU)

def oracle_run(cfg: int, size: int, mode: str, steps: int, warmup: int, q):
    """Runs in a separate process (1 host thread). The oracle solves with its Jacobi-PCG
    (method 3) to the same relative residual as the GPU (1e-10; reading A11: same solution,
    same preconditioner, so the CPU and GPU numbers compare the same algorithm).
    mode 'baseline': setup (the oracle's own densification pass and mesh), then one full step
    (solve + raster + error) timed. mode 'reference': setup, then warmup + steps full steps,
    each timed (no extrapolation)."""
    try:
        import oracle
        c = workload_inputs(cfg, size)
        W, H = c["W"], c["H"]
        f = c["f"].reshape(-1)
        t0 = time.time()
        if c["kind"].startswith("densify"):
            mask, _, _ = oracle.densify(W, H, c["f"], c["mask0"], c["unknowns"], c["schedule"][:2], rtol=RTOL,
                                        method=3)
        else:
            mask = c["mask"]
        S = oracle.System(W, H, mask, c["unknowns"])
        t_setup = time.time() - t0
        g = f[S.mask_px]

        def one_step():
            a = time.perf_counter()
            u, st, iters, rr = S.solve(g, rtol=RTOL, method=3)
            b = time.perf_counter()
            R = S.raster(u, f)
            e = time.perf_counter()
            return dict(solve_s=b - a, raster_s=e - b, iters=iters, mse=R["mse"])

        full = dict(one_step(), setup_s=t_setup, n_u=S.n_u, nnz_uu=S.nnz_uu)
        out = dict(full=full, samples=[])
        if mode == "reference":
            for s in range(warmup + steps):
                r = one_step()
                r["warm"] = s < warmup
                out["samples"].append(r)
        q.put(out)
    except Exception as e:  # report, never hang the bench
        q.put({"error": repr(e)})


def start_oracle(cfg, size, mode, steps=0, warmup=0):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=oracle_run, args=(cfg, size, mode, steps, warmup, q), daemon=True)
    p.start()
    return p, q


# ----------------------------------------------------------------------------- reference arm

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    p, q = start_oracle(args.config, args.size, "reference", args.steps, args.warmup)
    out = q.get()
    p.join(timeout=60)
    c = make_config(args.config, W=args.size or None, H=args.size or None)
    Npx = c["W"] * c["H"]
    if "error" in out:
        print(json.dumps({"impl": "reference", "unavailable": "oracle failed: " + out["error"]}))
        return 0
    full = out["full"]
    timed = [s for s in out["samples"] if not s["warm"]]
    per_step = [s["solve_s"] + s["raster_s"] for s in timed]
    ms = 1e3 * float(np.sum(per_step)) / len(per_step)
    value = Npx / (ms * 1e-3) / 1e6
    line = {
        "impl": "reference", "metric": "FEM inpainting Mpixels/s (solve+raster+error)", "value": value,
        "unit": "Mpx/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, c),
        "cpu_baseline": {"value": value, "unit": "Mpx/s", "cores": 1, "kind": "oracle",
                         "sample": f"every step is the full workload on 1 host thread: oracle Jacobi-PCG to 1e-10 "
                                   f"({timed[0]['iters']} iterations, {float(np.median([s['solve_s'] for s in timed])):.2f} s) "
                                   f"+ raster+error ({float(np.median([s['raster_s'] for s in timed])):.2f} s) on the "
                                   f"oracle's own densified mesh of the same seeded input (setup {full['setup_s']:.1f} s)"},
        "e2e": {"value": value, "unit": "Mpx/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "oracle_mse": full["mse"],
    }
    print(json.dumps(line))
    return 0


def config_dict(args, c):
    return {"workload": f"C{args.config}: {c['W']}x{c['H']} fp64 synthetic, "
                        f"{'2% mask from one densification pass (1% random + 1% selected)' if args.config == 5 else '5% random mask'}, "
                        "p = m unknown vertices; step = PCG solve (rtol 1e-10) + rasterise + error maps + MSE",
            "W": c["W"], "H": c["H"], "global_batch": 1, "parallelism": f"replicas{args.gpus}",
            "l2_flush": "inputs larger than L2 (f = 537 MB)" if c["W"] * c["H"] * 8 > 126 * 2**20 else
                        "L2-resident working set (no flush; latency-bound config)"}


# ----------------------------------------------------------------------------- our arm

def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    from paper_2105_01586_b200 import femi, pipeline

    baseline_proc = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        baseline_proc = start_oracle(args.config, args.size, "baseline")

    # ---- setup (untimed, reported)
    t0 = time.time()
    c = workload_inputs(args.config, args.size)
    W, H = c["W"], c["H"]
    Npx = W * H
    f_dev = torch.as_tensor(c["f"], dtype=torch.float64, device=dev).reshape(-1)
    t_gen = time.time() - t0
    setup = {"generate_s": t_gen}
    if c["kind"].startswith("densify"):
        t0 = time.time()
        mask, recs, _ = pipeline.densify(W, H, f_dev, c["mask0"], c["unknowns"], c["schedule"][:2], rtol=RTOL)
        setup["densify_pass_s"] = time.time() - t0
        setup["densify_mesh_s"] = recs[0]["mesh_seconds"]
    else:
        mask = c["mask"]
    t0 = time.time()
    mesh = femi.Mesh(W, H, mask, c["unknowns"])
    setup["mesh_build_s"] = mesh.build_seconds
    setup["mesh_threads"] = mesh.build_threads
    torch.cuda.synchronize()
    t1 = time.time()
    sysm = femi.System(mesh)
    torch.cuda.synchronize()
    setup["assemble_s"] = time.time() - t1
    vert = mesh.vert_px()
    info = mesh.info
    g_dev = pipeline.mask_values(f_dev, vert, sysm.n_u)
    u_vert = torch.empty(sysm.nv, dtype=torch.float64, device=dev)
    u_px = torch.empty(Npx, dtype=torch.float64, device=dev)
    e_px = torch.empty(Npx, dtype=torch.float64, device=dev)
    tri_err = torch.empty(sysm.T, dtype=torch.float64, device=dev)
    best = torch.empty(sysm.T, dtype=torch.int32, device=dev)
    sse = torch.zeros(1, dtype=torch.float64, device=dev)
    # x0: the mask-neighbour fill (reading A11b; FEMI_BENCH_X0=1: the midrange start of round 1)
    opts = femi.cg_opts(rtol=RTOL, x0=int(os.environ.get("FEMI_BENCH_X0", "3")))
    stream = torch.cuda.current_stream()

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        st, it, rel = femi.inpaint_solve_batched([sysm], [g_dev], [u_vert], opts)
        if ev:
            ev[1].record(stream)
        femi.rasterise_error(sysm, u_vert, f_dev, sse, u_px, e_px, tri_err, best)
        if ev:
            ev[2].record(stream)
        return st, int(it[0]), float(rel[0])

    for _ in range(args.warmup):
        st, iters, rel = step()
    torch.cuda.synchronize()
    assert st == 0 and rel <= RTOL, f"solve failed: status {st} relres {rel}"

    # ---- timed region (device events, barrier + sync both sides)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = femi.kernel_launches()
    it_list = []
    with Clocks(local) as clk:
        torch.cuda.cudart().cudaProfilerStart()  # ncu --profile-from-start off: timed region only
        e_start.record(stream)
        for k in range(args.steps):
            st, iters, rel = step(evs[k])
            it_list.append(iters)
        e_end.record(stream)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    launches = femi.kernel_launches() - launches0
    if world > 1:
        dist.barrier()
    total_ms = e_start.elapsed_time(e_end)
    solve_ms = [e[0].elapsed_time(e[1]) for e in evs]
    raster_ms = [e[1].elapsed_time(e[2]) for e in evs]
    from paper_2105_01586_b200 import multi
    total_ms = multi.max_over_ranks(total_ms, device=dev)  # device time of the job = max over ranks
    ms_per_step = total_ms / args.steps
    value = world * Npx * args.steps / (total_ms * 1e-3) / 1e6
    mse = sse.item() / Npx

    # ---- e2e: host buffers (pinned) in, SSE out, every step
    e2e = None
    if not args.no_e2e:
        f_host = torch.empty(Npx, dtype=torch.float64, pin_memory=True)
        f_host.copy_(torch.as_tensor(c["f"].reshape(-1)))
        g_host = torch.empty(sysm.m, dtype=torch.float64, pin_memory=True)
        g_host.copy_(g_dev.cpu())
        # double-buffered inputs: step k+1's copies (g then f, on a copy stream) are issued
        # right after step k's kernels, so they overlap step k's solve and raster; the raster
        # of a step waits for its f, the solve for its g
        f_d2 = [torch.empty_like(f_dev) for _ in range(2)]
        g_d2 = [torch.empty_like(g_dev) for _ in range(2)]
        sse_host = torch.empty(1, dtype=torch.float64, pin_memory=True)
        cs = torch.cuda.Stream(device=dev)
        g_ready = [torch.cuda.Event() for _ in range(2)]
        f_ready = [torch.cuda.Event() for _ in range(2)]
        used = [torch.cuda.Event() for _ in range(2)]

        def issue_copy(k):
            b = k % 2
            cs.wait_event(used[b])  # step k-2 is done with this buffer
            with torch.cuda.stream(cs):
                g_d2[b].copy_(g_host, non_blocking=True)
                g_ready[b].record(cs)
                f_d2[b].copy_(f_host, non_blocking=True)
                f_ready[b].record(cs)

        def run_e2e(nsteps, ev=None):
            if ev:
                ev[0].record(stream)
            for b in range(2):
                used[b].record(stream)  # the copies start inside the timed region
            issue_copy(0)
            s_val = None
            for k in range(nsteps):
                b = k % 2
                stream.wait_event(g_ready[b])
                femi.inpaint_solve_batched([sysm], [g_d2[b]], [u_vert], opts)
                stream.wait_event(f_ready[b])
                femi.rasterise_error(sysm, u_vert, f_d2[b], sse, u_px, e_px, tri_err, best)
                used[b].record(stream)
                sse_host.copy_(sse, non_blocking=True)
                done = torch.cuda.Event()
                done.record(stream)
                if k + 1 < nsteps:
                    issue_copy(k + 1)
                done.synchronize()
                s_val = float(sse_host[0])
            if ev:
                ev[1].record(stream)
            return s_val

        run_e2e(max(1, args.warmup))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_e2e = run_e2e(args.steps, (a, b))
        torch.cuda.synchronize()
        t_e2e = multi.max_over_ranks(a.elapsed_time(b), device=dev)
        assert abs(s_e2e / Npx - mse) <= 1e-9 * mse
        e2e = {"value": world * Npx * args.steps / (t_e2e * 1e-3) / 1e6, "unit": "Mpx/s",
               "h2d_bytes_per_step": int(8 * Npx + 8 * sysm.m), "d2h_bytes_per_step": 8}

    # ---- roofline of the dominant launch: the solve graph (SURVEY §8(d) algorithmic bytes). Per CG
    # iteration 12 nnz_uu + 4 (n_u + 1) + 80 n_u; plus, once per solve, the prologue / epilogue
    # kernels' algorithmic bytes: the right-hand side (12 nnz_uk + 4 (n_u + 1) + 8 m + 16 n_u), the
    # mask-neighbour fill (one A_uk pass 12 nnz_uk + 4 (n_u + 1) + 8 n_u, two A_uu passes
    # 2 (4 nnz_uu + 8 nnz_uu + 8 n_u)), x^0 + p = s = 0 (40 n_u), the initial residual and the first
    # SpMV (2 (12 nnz_uu + 4 (n_u + 1) + 24 n_u)), finalize (32 n_u + 8 m) and the true residual
    # (12 nnz_uu + 4 (n_u + 1) + 24 n_u)
    n_u, nnz_uu = info["n_unknown"], info["nnz_uu"]
    nnz_uk, m_ = info["nnz_uk"], info["n_mask"]
    bytes_iter = 12 * nnz_uu + 4 * (n_u + 1) + 80 * n_u
    fill = opts.x0 == 3 and n_u >= 8192
    bytes_once = (12 * nnz_uk + 4 * (n_u + 1) + 8 * m_ + 16 * n_u
                  + ((12 * nnz_uk + 4 * (n_u + 1) + 8 * n_u + 2 * (12 * nnz_uu + 8 * n_u)) if fill else 0)
                  + 40 * n_u + (2 if fill else 1) * (12 * nnz_uu + 4 * (n_u + 1) + 24 * n_u)
                  + 32 * n_u + 8 * m_ + 12 * nnz_uu + 4 * (n_u + 1) + 24 * n_u)
    iters = int(np.median(it_list))
    solve_s = float(np.median(solve_ms)) * 1e-3
    achieved = (bytes_iter * iters + bytes_once) / solve_s / 1e9
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    traffic = None  # DRAM bytes of one solve-graph launch (ncu, stored under profiles/)
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"C{args.config}", {}).get("solve_graph_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- C5's tonal tail (BASELINE.json configs[4]: "then 20 tonal CG iterations"), timed
    # separately and reported in detail (not part of the Mpx/s metric)
    tonal = None
    if args.config == 5 and not args.no_tonal:
        # one warm-up run (graph capture, scratch pools), then the median of 3 timed runs
        runs = []
        for k in range(4):
            g_t = g_dev.clone()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st_t, rep = femi.tonal_optimise(sysm, f_dev, g_t, outer_rtol=1e-300, outer_max=20,
                                            inner=femi.cg_opts(rtol=1e-12))
            b.record(stream)
            torch.cuda.synchronize()
            if k:
                runs.append(a.elapsed_time(b) * 1e-3)
        tonal = {"outer_iters": rep["outer_iters"], "inner_solves": rep["inner_solves"],
                 "inner_cg_iters": rep["inner_iters"], "seconds": float(np.median(runs)),
                 "seconds_runs": runs, "mse_before": rep["mse_before"], "mse_after": rep["mse_after"],
                 "inner_rtol": 1e-12, "us_per_inner_cg_iter": 1e6 * float(np.median(runs)) / max(rep["inner_iters"], 1)}

    cpu = None
    if baseline_proc is not None:
        p, q = baseline_proc
        try:
            out = q.get(timeout=900)
        except Exception as e:
            out = {"error": repr(e)}
        p.join(timeout=30)
        if "full" in out:
            fo = out["full"]
            t_cpu = fo["solve_s"] + fo["raster_s"]
            cpu = {"value": Npx / t_cpu / 1e6, "unit": "Mpx/s", "cores": 1, "kind": "oracle",
                   "sample": f"the whole step once: oracle Jacobi-PCG to 1e-10 ({fo['iters']} iterations, "
                             f"{fo['solve_s']:.2f} s; the GPU's algorithm and tolerance) + raster+error "
                             f"({fo['raster_s']:.2f} s) on the oracle's own densified mesh of the same seeded input; "
                             f"oracle MSE {fo['mse']:.6f}",
                   "us_per_cg_iter": 1e6 * fo["solve_s"] / max(fo["iters"], 1)}
        else:
            cpu = {"value": None, "unit": "Mpx/s", "cores": 1, "kind": "oracle", "sample": out.get("error")}

    if rank == 0:
        line = {
            "metric": "FEM inpainting Mpixels/s (solve+raster+error)", "value": value, "unit": "Mpx/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, c),
            "roofline": {"bound": "hbm", "kernel": "solve graph (prologue, PCG iterations k_gur + k_gt in the WHILE loop, epilogue)",
                         "achieved": achieved,
                         "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                         "bytes_per_iter": bytes_iter, "bytes_once_per_solve": bytes_once, "iters": iters,
                         "achieved_is": "algorithmic bytes of the solve launch (SURVEY 8(d): 12 nnz + 4 (n+1) + 80 n per "
                                        "iteration x iterations + the prologue/epilogue kernels' bytes) / its event time "
                                        "-- an effective bandwidth: the CG vectors stay in the 126 MB L2; DRAM moves "
                                        "`traffic` bytes per launch",
                         "dram_gbs": (traffic / solve_s / 1e9) if traffic else None,
                         "dram_frac": (traffic / solve_s / 1e9 / hbm) if traffic else None,
                         "traffic_source": "profiles/traffic.json: ncu dram__bytes_read + _write of one solve-graph launch",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
            "detail": {"solve_ms": float(np.median(solve_ms)), "raster_ms": float(np.median(raster_ms)),
                       "cg_iters": iters, "us_per_cg_iter": 1e3 * float(np.median(solve_ms)) / max(iters, 1),
                       "mse": mse, "n_unknown": n_u, "n_mask": info["n_mask"], "n_tri": info["n_tri"],
                       "nnz_uu": nnz_uu, "nnz_uk": info["nnz_uk"], "setup": setup, "version": femi.version(),
                       "tonal20": tonal,
                       # the second kernel of the step: the fused raster + error pass, 28 B/px
                       # algorithmic (list 4 + f 8 + u 8 + e 8) + 12 B/triangle, over its event time
                       "roofline_raster": {
                           "kernel": "k_raster_grp + k_sse (S3+S4)", "bound": "hbm",
                           "bytes": 28 * Npx + 12 * info["n_tri"],
                           "achieved": (28 * Npx + 12 * info["n_tri"]) / (float(np.median(raster_ms)) * 1e-3) / 1e9,
                           "peak": hbm, "unit": "GB/s",
                           "frac": (28 * Npx + 12 * info["n_tri"]) / (float(np.median(raster_ms)) * 1e-3) / 1e9 / hbm}},
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- configs 2-4

def run_workload(args):
    """BASELINE.json configs[1..3] on the GPU (replicas under torchrun): C2 = one batched
    solve of 32 different meshes + 32 rasters; C3 = the 10-iteration densification (GPU
    stages timed on the device, host re-meshing timed separately, plus the whole run end to
    end in `e2e`); C4 = tonal optimisation
    to ||B^T(f - Bg)|| / ||B^T f|| < 1e-8. All inputs resident on the device."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    from paper_2105_01586_b200 import femi, pipeline

    c = workload_inputs(args.config, args.size)
    W, H = c["W"], c["H"]
    Npx = W * H
    f_dev = torch.as_tensor(c["f"], dtype=torch.float64, device=dev).reshape(-1)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    detail, setup = {}, {}
    launches0 = None
    e2e = None

    from paper_2105_01586_b200 import multi
    if args.config == 2:
        t0 = time.time()
        nb = len(c["masks"])
        mine = multi.shard(nb, rank, world) if (args.shard and world > 1) else range(nb)
        meshes = [femi.Mesh(W, H, c["masks"][b], c["unknowns"][b]) for b in mine]
        setup["mesh_build_s"] = time.time() - t0
        t0 = time.time()
        systems = [femi.System(M) for M in meshes]
        torch.cuda.synchronize()
        setup["assemble_s"] = time.time() - t0
        B = len(systems)
        gs = [pipeline.mask_values(f_dev, M.vert_px(), S.n_u) for M, S in zip(meshes, systems)]
        us = [torch.empty(S.nv, dtype=torch.float64, device=dev) for S in systems]
        sse = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in systems]
        e_px = [torch.empty(Npx, dtype=torch.float64, device=dev) for _ in systems]
        tri = [torch.empty(S.T, dtype=torch.float64, device=dev) for S in systems]
        best = [torch.empty(S.T, dtype=torch.int32, device=dev) for S in systems]
        opts = femi.cg_opts(rtol=RTOL)

        split = []
        # the public API's plan objects: arguments marshalled once, one C call per stage
        solve_plan = femi.SolvePlan(systems, gs, us, opts)
        raster_plan = femi.RasterPlan(systems, us, [f_dev] * B, sse, e_px=e_px, tri_err=tri, best=best)

        def step(evs=None):
            if evs:
                evs[0].record(stream)
            st, it, rel = solve_plan.run()
            if evs:
                evs[1].record(stream)
            raster_plan.run()
            if evs:
                evs[2].record(stream)
                split.append(evs)
            return it

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        launches0 = femi.kernel_launches()
        a, b = ev(), ev()
        with Clocks(local) as clk:
            a.record(stream)
            for _ in range(args.steps):
                it = step()
            b.record(stream)
            torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.steps
        units = B * Npx
        metric, unit, hib = "FEM inpainting Mpixels/s (solve+raster+error)", "Mpx/s", True
        value_one = units / (ms * 1e-3) / 1e6
        mse_all = multi.gather_scalars(np.array([float(x.item()) / Npx for x in sse]), nb if args.shard else B,
                                       device=dev) if (args.shard and world > 1) else \
            np.array([float(x.item()) / Npx for x in sse])
        for _ in range(3):  # solve / raster split, measured after the timed region
            step([ev(), ev(), ev()])
        torch.cuda.synchronize()
        detail.update(solve_ms=float(np.median([e[0].elapsed_time(e[1]) for e in split])),
                      raster_ms=float(np.median([e[1].elapsed_time(e[2]) for e in split])))
        detail.update(solves_per_s=B / (ms * 1e-3), cg_iters_mean=float(np.mean(it)), cg_iters_max=int(np.max(it)),
                      mse_first4=[float(v) for v in mse_all[:4]], batch_per_rank=B,
                      sharded=bool(args.shard and world > 1))
        n_u = sum(S.n_u for S in systems) / B
        nnz = sum(S.info["nnz_uu"] for S in systems) / B
        bytes_iter = B * (12 * nnz + 4 * (n_u + 1) + 80 * n_u)
        iters_roof = float(np.max(it))
        work = "C2: 256x256 fp64 synthetic + noise, 32 independent 4% masks (32 meshes) solved as ONE batch " \
               "(block-diagonal), 32 rasters/error maps/MSEs; step = batched PCG (rtol 1e-10) + 32 rasters"
    elif args.config == 3:
        if args.n:  # longer schedules: same final density, n iterations
            c = make_config(3, W=args.size or None, H=args.size or None, n=args.n)
        sched = c["schedule"]

        def densify_timed(f_host=None):
            if f_host is not None:  # end to end: the image arrives from pinned host memory
                f_dev.copy_(f_host, non_blocking=True)
            mask = np.sort(np.asarray(c["mask0"], dtype=np.int64))
            gpu_ms, host_s, its = 0.0, 0.0, []
            x_prev = None
            M, new = None, None
            for t in range(1, len(sched) + 1):
                h0 = time.time()
                # re-meshing: the previous mesh plus the new mask pixels (femi_mesh_insert,
                # identical to a rebuild); --rebuild-mesh builds each mesh from scratch
                if M is None or args.rebuild_mesh:
                    M = femi.Mesh(W, H, mask, c["unknowns"])
                else:
                    M = M.insert(new)
                S = femi.System(M)
                g = pipeline.mask_values(f_dev, M.vert_px(), S.n_u)
                u = torch.empty(S.nv, dtype=torch.float64, device=dev)
                x0 = 3
                if args.warm and x_prev is not None and x_prev.numel() == S.n_u:
                    u[: S.n_u] = x_prev  # NEXT-4 warm start: previous solution at the fixed unknowns
                    x0 = 2
                opts = femi.cg_opts(rtol=RTOL, x0=x0)
                sse = torch.zeros(1, dtype=torch.float64, device=dev)
                tri = torch.empty(max(S.T, 1), dtype=torch.float64, device=dev)
                bst = torch.empty(max(S.T, 1), dtype=torch.int32, device=dev)
                torch.cuda.synchronize()
                host_s += time.time() - h0
                a, b = ev(), ev()
                a.record(stream)
                st, it, rel = femi.inpaint_solve_batched([S], [g], [u], opts)
                femi.rasterise_error(S, u, f_dev, sse, tri_err=tri, best=bst)
                new = femi.densify_step(S, f_dev, u, int(sched[t])) if t < len(sched) else None
                b.record(stream)
                torch.cuda.synchronize()
                gpu_ms += a.elapsed_time(b)
                its.append(int(it[0]))
                x_prev = u[: S.n_u].clone()
                if new is not None:
                    mask = np.sort(np.concatenate([mask, new.astype(np.int64)]))
            return gpu_ms, host_s, its, float(sse.item()) / Npx, S

        for _ in range(args.warmup):
            densify_timed()
        launches0 = femi.kernel_launches()
        gms, hs_, its = [], [], None
        with Clocks(local) as clk:
            for _ in range(args.steps):
                g_ms, h_s, its, mse, S = densify_timed()
                gms.append(g_ms)
                hs_.append(h_s)
        ms = float(np.mean(gms))
        launches1 = femi.kernel_launches()
        # end to end: one whole run through the public API -- f copied from
        # pinned host memory, every host re-mesh + assemble, the GPU stages, the per-iteration
        # selection read back, the final MSE read back -- wall time on the host, median
        f_pin = torch.from_numpy(np.ascontiguousarray(c["f"], dtype=np.float64).reshape(-1)).pin_memory()
        e2e_s = []
        for _ in range(max(3, args.steps)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            densify_timed(f_pin)  # returns after reading the final SSE back (sse.item())
            e2e_s.append(time.perf_counter() - t0)
        e2e = {"value": float(np.median(e2e_s)), "unit": "s", "h2d_bytes_per_step": int(f_pin.numel() * 8),
               "d2h_bytes_per_step": int(4 * int(np.sum(sched[1:])) + 8),
               "timing": "host wall clock of the whole run (host meshing + assemble + GPU stages), median of "
                         f"{len(e2e_s)} runs"}
        launches0 += femi.kernel_launches() - launches1  # the e2e runs are not in the device-timed count
        units = 1
        metric, unit, hib = (f"densification seconds (n={len(sched)}, 0.5%->5%; GPU stages: solve+raster+select"
                             f"{', warm starts' if args.warm else ''})"), "s", False
        value_one = ms * 1e-3
        detail.update(host_mesh_assemble_s=float(np.mean(hs_)), cg_iters=its, final_mse=mse,
                      mpx_iter_per_s=Npx * len(its) / (ms * 1e-3) / 1e6)
        n_u, nnz = S.n_u, S.info["nnz_uu"]
        bytes_iter = 12 * nnz + 4 * (n_u + 1) + 80 * n_u
        iters_roof = float(np.sum(its))
        work = "C3: 512x512 fp64 synthetic (bumps + disks + ramps), spatial densification 0.5% -> 5% in n = 10 " \
               "iterations (b_t ~ 1311), each iteration: host re-mesh + GPU solve (rtol 1e-10) + raster + select"
    else:  # config 4
        t0 = time.time()
        M = femi.Mesh(W, H, c["mask"], c["unknowns"])
        S = femi.System(M)
        torch.cuda.synchronize()
        setup["mesh_assemble_s"] = time.time() - t0
        g0 = pipeline.mask_values(f_dev, M.vert_px(), S.n_u)

        def run():
            g = g0.clone()
            st, rep = femi.tonal_optimise(S, f_dev, g, outer_rtol=1e-8, outer_max=1000, inner=femi.cg_opts(rtol=1e-12))
            return rep

        for _ in range(args.warmup):
            run()
        torch.cuda.synchronize()
        launches0 = femi.kernel_launches()
        a, b = ev(), ev()
        with Clocks(local) as clk:
            a.record(stream)
            for _ in range(args.steps):
                rep = run()
            b.record(stream)
            torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.steps
        units = 1
        metric, unit, hib = "tonal optimisation seconds to ||grad||/||B^T f|| < 1e-8", "s", False
        value_one = ms * 1e-3
        detail.update(rep)
        detail["inner_solves_per_s"] = rep["inner_solves"] / (ms * 1e-3)
        detail["us_per_inner_cg_iter"] = 1e3 * ms / max(rep["inner_iters"], 1)
        n_u, nnz = S.n_u, S.info["nnz_uu"]
        bytes_iter = 12 * nnz + 4 * (n_u + 1) + 80 * n_u
        iters_roof = float(rep["inner_iters"])
        work = "C4: 1024x1024 fp64 synthetic, fixed 3% random mask, tonal optimisation: CGLS on B^T B g = B^T f, " \
               "inner Jacobi-PCG to rtol 1e-12, until the relative gradient < 1e-8"
    launches = femi.kernel_launches() - launches0
    ms = multi.max_over_ranks(ms, device=dev)  # device time of the job = max over ranks
    sharded = args.config == 2 and args.shard and world > 1
    value = ((1 if sharded else world) * (nb * Npx if sharded else units) / (ms * 1e-3) / 1e6) if hib else ms * 1e-3
    solve_s = ms * 1e-3
    achieved = bytes_iter * iters_roof / solve_s / 1e9
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": hib,
            "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": work, "W": W, "H": H,
                       "parallelism": f"batch-shard{world}" if sharded else f"replicas{world}",
                       "l2_flush": "L2-resident working set (latency-bound config; no flush)"},
            "roofline": {"bound": "hbm", "kernel": "PCG iterations of the workload (L2-resident: latency-bound)",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": None, "bytes_per_iter": bytes_iter,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback"},
            "cpu_baseline": None, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
            "detail": dict(detail, setup=setup, version=femi.version()),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_colour(args):
    """NEXT-1 colour on the C5 recipe: three channels (seeds 505, 506, 507 of the C5
    generator) on one mesh; mask from one colour densification pass (1 % random + 1 %
    selected by the channel-summed error). Step = ONE shared-matrix multi-RHS solve of the 3
    channels (rtol 1e-10) + colour raster (3 u images, summed error map, per-triangle
    reductions, SSE). Metric: colour Mpixels/s (W*H per step)."""
    import torch
    from paper_2105_01586_b200 import femi, pipeline, multi
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    W = args.size or 8192
    cs = [make_config(5, W=W, H=W, seed=505 + k) for k in range(3)]
    c = cs[0]
    fd = [torch.as_tensor(ci["f"], dtype=torch.float64, device=dev).reshape(-1) for ci in cs]
    t0 = time.time()
    mask = pipeline.densify_channels(W, W, fd, c["mask0"], c["unknowns"], c["schedule"][:2], rtol=RTOL)
    setup = {"densify_pass_s": time.time() - t0}
    M = femi.Mesh(W, W, mask, c["unknowns"])
    S = femi.System(M)
    torch.cuda.synchronize()
    vert = M.vert_px()
    gs = [pipeline.mask_values(f, vert, S.n_u) for f in fd]
    us = [torch.empty(S.nv, dtype=torch.float64, device=dev) for _ in range(3)]
    upx = [torch.empty(W * W, dtype=torch.float64, device=dev) for _ in range(3)]
    e_px = torch.empty(W * W, dtype=torch.float64, device=dev)
    te = torch.empty(S.T, dtype=torch.float64, device=dev)
    bs = torch.empty(S.T, dtype=torch.int32, device=dev)
    sse = torch.zeros(1, dtype=torch.float64, device=dev)
    opts = femi.cg_opts(rtol=RTOL)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(e=None):
        if e:
            e[0].record(stream)
        st, it, rel = femi.inpaint_solve_batched([S] * 3, gs, us, opts)
        if e:
            e[1].record(stream)
        femi.rasterise_error_channels(S, us, fd, sse, upx, e_px, te, bs)
        if e:
            e[2].record(stream)
        return st, it, rel

    for _ in range(args.warmup):
        st, it, rel = step()
    torch.cuda.synchronize()
    assert st == 0 and np.all(rel <= RTOL)
    evs = [[ev() for _ in range(3)] for _ in range(args.steps)]
    a, b = ev(), ev()
    launches0 = femi.kernel_launches()
    with Clocks(local) as clk:
        a.record(stream)
        for k in range(args.steps):
            st, it, rel = step(evs[k])
        b.record(stream)
        torch.cuda.synchronize()
    launches = femi.kernel_launches() - launches0
    ms = multi.max_over_ranks(a.elapsed_time(b) / args.steps, device=dev)
    solve_ms = float(np.median([e[0].elapsed_time(e[1]) for e in evs]))
    raster_ms = float(np.median([e[1].elapsed_time(e[2]) for e in evs]))
    info = M.info
    n_u, nnz = info["n_unknown"], info["nnz_uu"]
    iters = int(np.max(it))
    bytes_iter = 12 * nnz + 4 * (n_u + 1) + 80 * 3 * n_u  # shared matrix, 3 right-hand sides
    tonal = None
    if not args.no_tonal:  # NEXT-1 colour tonal: 20 lockstep CGLS iterations of the 3 channels
        runs = []
        for k in range(3):
            gt = [g.clone() for g in gs]
            a2, b2 = ev(), ev()
            a2.record(stream)
            st_t, reps = femi.tonal_optimise_channels(S, fd, gt, outer_rtol=1e-300, outer_max=20)
            b2.record(stream)
            torch.cuda.synchronize()
            if k:
                runs.append(a2.elapsed_time(b2) * 1e-3)
        tonal = {"channels": 3, "outer_iters": [r["outer_iters"] for r in reps],
                 "inner_solves": [r["inner_solves"] for r in reps], "seconds": float(np.median(runs)),
                 "mse_before": [r["mse_before"] for r in reps], "mse_after": [r["mse_after"] for r in reps],
                 "inner_rtol": 1e-12}
    achieved = bytes_iter * iters / (solve_ms * 1e-3) / 1e9
    pk = peaks()
    hbm = pk.get("hbm_gbs", 6650.0)
    if rank == 0:
        line = {
            "metric": "FEM colour inpainting Mpixels/s (3-channel solve+raster+error, shared mesh)",
            "value": world * W * W / (ms * 1e-3) / 1e6, "unit": "Mpx/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"colour C5: {W}x{W} x 3 channels fp64 synthetic (C5 recipe, seeds 505-507), "
                                   "2% mask from one colour densification pass; step = shared-matrix 3-RHS PCG "
                                   "(rtol 1e-10) + colour raster + summed error maps + SSE",
                       "W": W, "H": W, "channels": 3, "parallelism": f"replicas{world}",
                       "l2_flush": "inputs larger than L2 (3 x 537 MB)"},
            "roofline": {"bound": "hbm", "kernel": "3-RHS PCG iteration (k_gum + k_gtm, one matrix stream)",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": None, "bytes_per_iter": bytes_iter, "iters": iters,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in pk else "fallback"},
            "cpu_baseline": None, "e2e": None, "gpu_launches": int(launches), "clocks": clk.summary(),
            "detail": {"solve_ms": solve_ms, "raster_ms": raster_ms, "cg_iters": [int(i) for i in it],
                       "us_per_cg_iter": 1e3 * solve_ms / max(iters, 1), "mse": float(sse.item()) / (W * W),
                       "n_unknown": n_u, "nnz_uu": nnz, "setup": setup, "version": femi.version(),
                       "tonal20": tonal},
        }
        print(json.dumps(line))
    return 0


def run_band(args):
    """NEXT-4: one image's solve split into row bands (femi_band_*, multi.band_solve). Under
    torchrun every rank owns one band (halo exchange + 4-double all-reduce per CG iteration over
    NCCL); with --bands R at N = 1, R bands of one process step in lockstep (LoopbackComm). The
    step is the band solve, the all-gather of the solution, the raster/error of each rank's triangle
    share and the SSE all-reduce; strong scaling."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    from paper_2105_01586_b200 import femi, multi, pipeline

    c = workload_inputs(args.config, args.size)
    W, H = c["W"], c["H"]
    f_dev = torch.as_tensor(c["f"], dtype=torch.float64, device=dev).reshape(-1)
    if c["kind"].startswith("densify"):
        mask, _, _ = pipeline.densify(W, H, f_dev, c["mask0"], c["unknowns"], c["schedule"][:2], rtol=RTOL)
    else:
        mask = c["mask"]
    mesh = femi.Mesh(W, H, mask, c["unknowns"])
    vert = mesh.vert_px()
    n_u = mesh.info["n_unknown"]
    g = f_dev[torch.as_tensor(vert[n_u:], dtype=torch.int64, device=dev)].contiguous()
    R = world if world > 1 else max(1, args.bands)
    ranks = [rank] if world > 1 else list(range(R))
    bands = [femi.Band(mesh, R, r) for r in ranks]
    comm = multi.DistComm(bands[0]) if world > 1 else multi.LoopbackComm(bands)
    # raster shares: triangle ranges over their image rows (femi_band_raster_system)
    rsys = []
    for r in ranks:
        Sb, bi = femi.band_raster_system(mesh, R, r)
        o, n = bi["y0"] * W, bi["rows"] * W
        rsys.append((Sb, f_dev[o:o + n].contiguous(), torch.empty(n, dtype=torch.float64, device=dev),
                     torch.empty(n, dtype=torch.float64, device=dev), torch.zeros(1, dtype=torch.float64, device=dev)))
    u_vert = torch.empty(mesh.info["n_vert"], dtype=torch.float64, device=dev)
    sse_t = torch.zeros(1, dtype=torch.float64, device=dev)

    def step():
        rep = multi.band_solve(comm, g, rtol=RTOL)
        comm.gather_solution(u_vert, g)
        sse_t.zero_()
        for Sb, fb, ub, eb, sb in rsys:
            femi.rasterise_error(Sb, u_vert, fb, sb, ub, eb)
            sse_t.add_(sb)
        comm.allreduce_scalar(sse_t)
        return rep

    for _ in range(args.warmup):
        rep = step()
    torch.cuda.synchronize()
    assert rep["converged"], rep
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        e0.record()
        for _ in range(args.steps):
            rep = step()
        e1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    ms = multi.max_over_ranks(ms, device=dev)
    if rank == 0:
        info = [b.info for b in bands]
        print(json.dumps({
            "metric": "row-band FEM inpainting Mpixels/s (one image over N bands: solve+raster+error)", "value": W * H / (ms * 1e-3) / 1e6,
            "unit": "Mpx/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C{args.config} {W}x{H}: PCG solve (rtol {RTOL}, x0 = midrange) over {R} row "
                                   f"bands + all-gather of the solution + raster/error over {R} triangle shares + "
                                   f"SSE all-reduce ({'NCCL ranks' if world > 1 else 'lockstep bands of one process'})",
                       "W": W, "H": H, "bands": R, "parallelism": f"rowband{R}",
                       "l2_flush": "inputs larger than L2 (f = 537 MB at C5)"},
            "roofline": None, "cpu_baseline": None, "e2e": None,
            "clocks": clk.summary(),
            "detail": {"iters": rep["iters"], "restarts": rep["restarts"], "rel_res": rep["rel_res"],
                       "mse": float(sse_t.item()) / (W * H),
                       "n_unknown": n_u, "halo": [i["n_halo"] for i in info], "send": [i["n_send"] for i in info],
                       "peers": [i["n_peers"] for i in info]}}))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.band:
        return run_band(args)
    if args.config in (2, 3, 4):
        return run_workload(args)
    if args.config == 6:
        return run_colour(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
