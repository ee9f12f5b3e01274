"""Seeded synthetic workloads shaped like the paper's.

The paper's test images (trui, walter, peppers, saomiguel)
are not available. Seeded images with the shapes and mask densities of BASELINE.json's
five configs stand in for them. Draw order is frozen:

1. ramps (C3 only): 2 x (theta~U[0,2pi), a~U[20,60]) adding a*(cos t*x/(W-1) + sin t*y/(H-1))
2. six bumps: (A~U[20,120], sigma~U[4,16]*s, cx~U[0,W), cy~U[0,H)) adding A*exp(-r^2/(2 sigma^2))
3. three disks: (r~U[W/32,W/8], cx~U[0,W), cy~U[0,H), value~U[0,255]) overwriting the disk
4. noise (C2 only): N(0, 2^2) per pixel
5. clip to [0,255]
6. masks: rng.choice(N, m, replace=False)
7. unknowns: corners forced in (unless masked), the rest uniform from non-mask pixels
8. C2 draws its 32 masks/unknown sets from SeedSequence(seed).spawn(32)

Pixel index pix = y*W + x ("f, g, u are vectors").
"""
from __future__ import annotations

import numpy as np

# Seeds per config.
SEEDS = {1: 101, 2: 202, 3: 303, 4: 404, 5: 505}


def half_up(x: float) -> int:
    """floor(x + 1/2): SURVEY A9 reading of "m/n" and "5 %" (half-up, not banker's)."""
    return int(np.floor(x + 0.5))


def schedule(m: int, n: int) -> list[int]:
    """Batch sizes b_t, t = 0..n-1, with sum b_t = m ("m/n"; A9)."""
    return [half_up(m * (t + 1) / n) - half_up(m * t / n) for t in range(n)]


def corner_pixels(W: int, H: int) -> np.ndarray:
    return np.unique(np.array([0, W - 1, (H - 1) * W, (H - 1) * W + W - 1], dtype=np.int64))


def draw_image(rng: np.random.Generator, W: int, H: int, *, ramps: bool = False,
               noise: bool = False, sigma_scale: float = 1.0) -> np.ndarray:
    """fp64 image f[H, W] on the 0..255 scale, drawn in the frozen order."""
    x = np.arange(W, dtype=np.float64)
    y = np.arange(H, dtype=np.float64)
    f = np.zeros((H, W), dtype=np.float64)
    if ramps:
        for _ in range(2):
            theta = rng.uniform(0.0, 2.0 * np.pi)
            a = rng.uniform(20.0, 60.0)
            f += a * (np.cos(theta) * x[None, :] / (W - 1) + np.sin(theta) * y[:, None] / (H - 1))
    for _ in range(6):
        A = rng.uniform(20.0, 120.0)
        sigma = rng.uniform(4.0, 16.0) * sigma_scale
        cx = rng.uniform(0.0, W)
        cy = rng.uniform(0.0, H)
        ex = np.exp(-((x - cx) ** 2) / (2.0 * sigma * sigma))
        ey = np.exp(-((y - cy) ** 2) / (2.0 * sigma * sigma))
        f += A * np.outer(ey, ex)  # separable form of exp(-r^2/2s^2)
    for _ in range(3):
        r = rng.uniform(W / 32.0, W / 8.0)
        cx = rng.uniform(0.0, W)
        cy = rng.uniform(0.0, H)
        value = rng.uniform(0.0, 255.0)
        y0, y1 = max(0, int(np.floor(cy - r)) - 1), min(H, int(np.ceil(cy + r)) + 2)
        x0, x1 = max(0, int(np.floor(cx - r)) - 1), min(W, int(np.ceil(cx + r)) + 2)
        if y0 < y1 and x0 < x1:
            dx2 = (x[x0:x1] - cx) ** 2
            dy2 = (y[y0:y1] - cy) ** 2
            inside = (dy2[:, None] + dx2[None, :]) <= r * r
            f[y0:y1, x0:x1][inside] = value
    if noise:
        f += rng.normal(0.0, 2.0, size=(H, W))
    np.clip(f, 0.0, 255.0, out=f)
    return f


def draw_mask(rng: np.random.Generator, N: int, m: int) -> np.ndarray:
    """m distinct pixel indices, uniform without replacement, ascending."""
    return np.sort(rng.choice(N, size=m, replace=False).astype(np.int64))


def _choose_excluding(rng: np.random.Generator, N: int, k: int, excluded: np.ndarray) -> np.ndarray:
    """k distinct pixels uniform over [0,N) minus `excluded` (sorted, unique)."""
    excluded = np.unique(np.asarray(excluded, dtype=np.int64))
    avail = N - excluded.size
    if k > avail:
        raise ValueError("not enough free pixels")
    ranks = rng.choice(avail, size=k, replace=False).astype(np.int64)
    # rank -> pixel: pixel = rank + #{excluded e : e - idx(e) <= rank}
    adj = excluded - np.arange(excluded.size, dtype=np.int64)
    return np.sort(ranks + np.searchsorted(adj, ranks, side="right"))


def draw_unknowns(rng: np.random.Generator, W: int, H: int, mask: np.ndarray, p: int) -> np.ndarray:
    """p unknown vertices: unmasked corners forced in, the rest uniform."""
    N = W * H
    mask = np.asarray(mask, dtype=np.int64)
    corners = corner_pixels(W, H)
    forced = np.setdiff1d(corners, mask)
    rest = _choose_excluding(rng, N, p - forced.size, np.concatenate([mask, corners]))
    return np.sort(np.concatenate([forced, rest]))


CONFIGS = {
    1: dict(W=64, H=64, density=0.05, kind="inpaint"),
    2: dict(W=256, H=256, density=0.04, kind="batch", batch=32, noise=True),
    3: dict(W=512, H=512, density=0.05, kind="densify", n=10, ramps=True),
    4: dict(W=1024, H=1024, density=0.03, kind="tonal"),
    5: dict(W=8192, H=8192, density=0.02, kind="densify_inpaint_tonal", n=2, sigma_scale=32.0),
}


def make_config(k: int, *, W: int | None = None, H: int | None = None, seed: int | None = None,
                n: int | None = None) -> dict:
    """Inputs of BASELINE.json config k (1-based). W/H/seed overrides give scaled-down
    variants of the same recipe for fast tests; n overrides the number of densification
    iterations (longer schedules). Returns numpy arrays only."""
    c = dict(CONFIGS[k])
    if n is not None and c["kind"].startswith("densify"):
        c["n"] = n
    W = W or c["W"]
    H = H or c["H"]
    seed = SEEDS[k] if seed is None else seed
    N = W * H
    rng = np.random.default_rng(seed)
    f = draw_image(rng, W, H, ramps=c.get("ramps", False), noise=c.get("noise", False),
                   sigma_scale=c.get("sigma_scale", 1.0) * (W / c["W"]))
    m = half_up(c["density"] * N)
    out = dict(config=k, W=W, H=H, seed=seed, f=f, m=m, kind=c["kind"])
    if c["kind"] == "batch":
        masks, unks = [], []
        for child in np.random.SeedSequence(seed).spawn(c["batch"]):
            r = np.random.default_rng(child)
            mk = draw_mask(r, N, m)
            masks.append(mk)
            unks.append(draw_unknowns(r, W, H, mk, m))
        out.update(masks=masks, unknowns=unks)
    elif c["kind"].startswith("densify"):
        n = c["n"]
        b = schedule(m, n)
        mk = draw_mask(rng, N, b[0])
        out.update(n=n, schedule=b, mask0=mk, unknowns=draw_unknowns(rng, W, H, mk, m))
    else:
        mk = draw_mask(rng, N, m)
        out.update(mask=mk, unknowns=draw_unknowns(rng, W, H, mk, m))
    return out
