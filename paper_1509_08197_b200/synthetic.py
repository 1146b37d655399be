"""Seeded synthetic stereo pairs for the BASELINE.json configurations.

BASELINE.json names no public dataset; its five configurations describe a
Voronoi scene model, which this module freezes in code.  The
warp rule follows the reference generator (synthetic.py:54-114 of
``treestereo``): disparities are painted in ascending order so nearer
surfaces overwrite farther ones, unreached right-image pixels keep uniform
noise, and the left-view occlusion mask is derived analytically.

Seed = 1_000_000 * config_id + pair_index (config_id 1..5 as in BASELINE.json).
This is host-side input generation, outside the timed hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .raster_io import DisparityMap, RasterImage, StereoPair


@dataclass(frozen=True)
class SceneSpec:
    config_id: int
    height: int
    width: int
    d_max: int
    segments: int
    slanted: float
    sigma: float
    batch: int
    brightness_frac: float = 0.0  # fraction of pairs with a global right offset
    colour_groups: int = 1  # segments sharing one base colour (greedy adjacency)


# BASELINE.json "configs" (W x H as written there; arrays are H x W).
CONFIGS = {
    1: SceneSpec(1, 96, 128, 16, 8, 0.0, 8.0, 1),
    2: SceneSpec(2, 370, 463, 80, 30, 0.2, 8.0, 8),
    3: SceneSpec(3, 555, 695, 120, 50, 0.3, 6.0, 32, brightness_frac=0.1),
    4: SceneSpec(4, 1110, 1390, 240, 120, 0.3, 8.0, 64, colour_groups=4),
    5: SceneSpec(5, 1988, 2880, 512, 300, 0.4, 8.0, 1),
}


@dataclass(frozen=True)
class Scene:
    pair: StereoPair
    gt_left: DisparityMap
    occlusion: np.ndarray
    brightness_offset: int = 0  # global offset added to the right image (C3)


def _voronoi_labels(h: int, w: int, sx: np.ndarray, sy: np.ndarray) -> np.ndarray:
    """Nearest site per pixel; ties go to the lower site index (first argmin)."""
    labels = np.empty((h, w), np.int32)
    xs = np.arange(w, dtype=np.float64)
    rows_per_chunk = max(1, 2_000_000 // max(1, w * len(sx)))
    for r0 in range(0, h, rows_per_chunk):
        r1 = min(h, r0 + rows_per_chunk)
        ys = np.arange(r0, r1, dtype=np.float64)
        d2 = (xs[None, :, None] - sx[None, None, :]) ** 2 + (ys[:, None, None] - sy[None, None, :]) ** 2
        labels[r0:r1] = np.argmin(d2, axis=2)
    return labels


def _colour_groups(labels: np.ndarray, n: int, group: int) -> np.ndarray:
    """Greedy adjacency grouping: walk segments in index order, each open
    group absorbs up to `group` mutually reachable neighbours."""
    adj = [set() for _ in range(n)]
    a = labels[:, :-1].ravel()
    b = labels[:, 1:].ravel()
    c = labels[:-1, :].ravel()
    d = labels[1:, :].ravel()
    for x, y in ((a, b), (c, d)):
        diff = x != y
        for i, j in set(zip(x[diff].tolist(), y[diff].tolist())):
            adj[i].add(j)
            adj[j].add(i)
    gid = np.full(n, -1, np.int64)
    g = 0
    for s in range(n):
        if gid[s] >= 0:
            continue
        members = [s]
        gid[s] = g
        frontier = sorted(adj[s])
        while frontier and len(members) < group:
            t = frontier.pop(0)
            if gid[t] >= 0:
                continue
            gid[t] = g
            members.append(t)
            frontier.extend(sorted(x for x in adj[t] if gid[x] < 0))
        g += 1
    return gid


def make_scene(spec: SceneSpec, pair_index: int = 0) -> Scene:
    """Render one seeded pair of configuration `spec`."""
    h, w, d_max, n = spec.height, spec.width, spec.d_max, spec.segments
    rng = np.random.default_rng(1_000_000 * spec.config_id + pair_index)
    sx = rng.uniform(0.0, w, n)
    sy = rng.uniform(0.0, h, n)
    base = rng.integers(0, 256, size=(n, 3)).astype(np.float64)
    d0 = rng.integers(0, d_max, size=n)  # uniform in [0, d_max - 1]
    slanted = rng.uniform(0.0, 1.0, n) < spec.slanted
    gx = rng.uniform(-0.05, 0.05, n)
    gy = rng.uniform(-0.05, 0.05, n)
    period = rng.uniform(16.0, 48.0, n)
    theta = rng.uniform(0.0, np.pi, n)
    phi = rng.uniform(0.0, 2.0 * np.pi, n)

    labels = _voronoi_labels(h, w, sx, sy)
    if spec.colour_groups > 1:
        gid = _colour_groups(labels, n, spec.colour_groups)
        first = {}
        for s in range(n):
            first.setdefault(int(gid[s]), s)
        base = base[[first[int(g)] for g in gid]]

    yy, xx = np.meshgrid(np.arange(h, dtype=np.float64), np.arange(w, dtype=np.float64),
                         indexing="ij")
    L = labels
    disp = d0[L].astype(np.float64)
    sl = slanted[L]
    disp = np.where(sl, np.rint(d0[L] + gx[L] * (xx - sx[L]) + gy[L] * (yy - sy[L])), disp)
    disp = np.clip(disp, 0, d_max).astype(np.int32)

    tex = 20.0 * np.sin(2.0 * np.pi * (xx * np.cos(theta[L]) + yy * np.sin(theta[L])) / period[L]
                        + phi[L])
    noise = rng.normal(0.0, spec.sigma, size=(h, w, 3))
    left = np.clip(np.rint(base[L] + tex[:, :, None] + noise), 0, 255).astype(np.uint8)

    right = np.clip(np.rint(rng.uniform(0.0, 255.0, size=(h, w, 3))), 0, 255).astype(np.uint8)
    winner_col = np.full((h, w), -1, np.int64)
    rows_idx, cols_idx = np.meshgrid(np.arange(h), np.arange(w), indexing="ij")
    for d in np.unique(disp).tolist():  # ascending: nearer surfaces overwrite
        on = disp == d
        src_r, src_c = rows_idx[on], cols_idx[on]
        dst_c = src_c - d
        ok = dst_c >= 0
        right[src_r[ok], dst_c[ok]] = left[src_r[ok], src_c[ok]]
        winner_col[src_r[ok], dst_c[ok]] = src_c[ok]
    off = 0
    if spec.brightness_frac > 0.0 and rng.uniform() < spec.brightness_frac:
        off = int(rng.integers(-15, 16))
        right = np.clip(right.astype(np.int32) + off, 0, 255).astype(np.uint8)

    target = cols_idx - disp
    inside = target >= 0
    occluded = ~inside | (winner_col[rows_idx, np.maximum(target, 0)] != cols_idx)
    pair = StereoPair(RasterImage(left), RasterImage(right), d_max,
                      name=f"c{spec.config_id}-{pair_index}")
    gt = DisparityMap(values=disp, valid=np.ones((h, w), bool))
    return Scene(pair=pair, gt_left=gt, occlusion=occluded, brightness_offset=off)


def make_batch(config_id: int, batch: int | None = None, start: int = 0) -> list[Scene]:
    spec = CONFIGS[config_id]
    n = spec.batch if batch is None else batch
    return [make_scene(spec, start + i) for i in range(n)]
