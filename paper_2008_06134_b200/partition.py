"""Contiguous screen bands and the frustum-culled attenuation build.

With the default partition (8-row bands dealt round-robin, frame.py) every
rank's rays cross the whole volume, so every rank needs the whole light
buffer: the build is replicated (or row-sharded and exchanged). Texels are
independent (lightbuffer.py:168-198), and a march reads only the quads its
own lookups reach — so when a rank renders ONE contiguous band of rows, it
can build just the texel-slices its band can read, with no exchange:

- the band's rays lie between two planes through the eye (the pixel rows
  at its top and bottom edge, raycaster.py:53-68 ray directions); widened
  by the lookups' lateral reach (lightbuffer.lookup_reach) they are the
  clip half-spaces of a sparse K1 (``sbrc_build_params.clip``): texels
  whose line misses the band's slab are skipped, and each texel's slice
  recurrence stops after the last layer the band can read. Values written
  are identical to a full build; at 8 ranks a rank runs about half of the
  covered texel-slices instead of all of them (config 3).
- band boundaries are balanced by cost: a per-row cost profile (the
  geometric in-cube ray length at first, then the march's measured tile
  costs, ``sbrc_render_params.tile_steps``) cut into ``world`` contiguous
  ranges of multiples of 8 rows that minimise the largest share.
"""

from __future__ import annotations

import numpy as np

from .scene import camera_frame

ALIGN = 8  # K2 block tiles are 8 rows tall


def ndc_y(settings, row: int) -> float:
    """Camera.rays' vertical coordinate of pixel row ``row`` (raycaster.py:62)."""
    h = int(settings.viewport[1])
    fr = camera_frame(settings.camera, settings.viewport)
    return (1.0 - (row + 0.5) / h * 2.0) * fr["tan_half"]


def frustum_clip(settings, row_begin: int, row_end: int, reach: float) -> tuple:
    """Two half-spaces (a, b, c, d), a*x + b*y + c*z + d >= 0, containing every
    sample of the rays of rows [row_begin, row_end), widened by ``reach``
    (world units: any point within ``reach`` of such a sample satisfies them).

    With q = p - eye and the camera basis (forward, right, up2), a point on
    the ray of vertical coordinate b has q.up2 = b * q.forward (q.forward > 0
    for every sample, t > 0); rows [r0, r1) span b in [b(r1-1), b(r0)], i.e.
    q.(up2 - b_lo forward) >= 0 and q.(b_hi forward - up2) >= 0."""
    fr = camera_frame(settings.camera, settings.viewport)
    eye = np.asarray(settings.camera.position, dtype=np.float64)
    fwd, up2 = np.asarray(fr["forward"], np.float64), np.asarray(fr["up2"], np.float64)
    b_hi, b_lo = ndc_y(settings, row_begin), ndc_y(settings, row_end - 1)
    planes = []
    for n in (up2 - b_lo * fwd, b_hi * fwd - up2):
        norm = float(np.linalg.norm(n))
        # 1e-9 |n| on top of the reach covers the float64 rounding of ray directions and positions
        planes.append((float(n[0]), float(n[1]), float(n[2]), float(-n @ eye) + (reach + 1e-9) * norm))
    return tuple(planes)


def row_costs_geometric(settings, stride: int = 4) -> np.ndarray:
    """(H,) cost profile: per image row, the summed in-cube ray length of every
    ``stride``-th pixel (ray_box_intersect, geometry.py:46-67)."""
    w, h = int(settings.viewport[0]), int(settings.viewport[1])
    fr = camera_frame(settings.camera, settings.viewport)
    eye = np.asarray(settings.camera.position, dtype=np.float64)
    px = np.arange(0, w, stride, dtype=np.float64)
    py = np.arange(h, dtype=np.float64)
    ndc_x = ((px + 0.5) / w * 2.0 - 1.0) * fr["tan_half"] * fr["aspect"]
    ndc_yv = (1.0 - (py + 0.5) / h * 2.0) * fr["tan_half"]
    d = (fr["forward"] + ndc_x[None, :, None] * fr["right"] + ndc_yv[:, None, None] * fr["up2"])
    d = d / np.linalg.norm(d, axis=-1, keepdims=True)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / d
        a = (0.0 - eye) * inv
        b = (1.0 - eye) * inv
    flat = d == 0.0
    inside = (eye >= 0.0) & (eye <= 1.0)
    a = np.where(flat, np.where(inside, -np.inf, np.inf), a)
    b = np.where(flat, np.where(inside, np.inf, -np.inf), b)
    t_in = np.maximum(np.minimum(a, b).max(axis=-1), 0.0)
    t_out = np.maximum(a, b).min(axis=-1)
    return np.where(t_out > t_in, t_out - t_in, 0.0).sum(axis=1)


def row_costs_measured(steps: np.ndarray, grid, row_begin: int, height: int) -> np.ndarray:
    """(H,) cost profile of one rank's contiguous range from its march's tile
    costs: ``steps`` (tiles_y * tiles_x,) longest-ray sample counts over
    ``grid`` = (tiles_x, tiles_y, tile_w, tile_h); a tile's time is its
    longest ray's, spread evenly over its rows. Zero outside the range."""
    tx, ty, _, th = (int(g) for g in grid)
    per_tile_row = np.asarray(steps, dtype=np.float64).reshape(ty, tx).sum(axis=1) / th
    out = np.zeros(height, dtype=np.float64)
    for j in range(ty):
        a, b = row_begin + j * th, min(height, row_begin + (j + 1) * th)
        if a < b:
            out[a:b] = per_tile_row[j]
    return out


def calibrated_profile(shape: np.ndarray, ranges, times) -> np.ndarray:
    """(H,) cost profile whose integral over each rank's range equals that
    rank's measured time, distributed inside the range like ``shape`` (e.g.
    the geometric profile; a floor keeps empty rows from costing nothing)."""
    shape = np.asarray(shape, dtype=np.float64)
    shape = shape + 0.05 * max(float(shape.mean()), 1e-12)
    prof = np.zeros_like(shape)
    for (b, n), t in zip(ranges, times):
        seg = shape[b:b + n]
        prof[b:b + n] = seg * (float(t) / float(seg.sum()))
    return prof


def damped_ranges(old, new, height: int, align: int = ALIGN) -> list[tuple[int, int]]:
    """Move each boundary halfway from ``old`` to ``new`` (rounded to ``align``,
    ranges kept non-empty): re-cuts from measured times converge instead of
    oscillating when a band's time is not proportional to its rows."""
    world = len(old)
    edges = []
    for i in range(1, world):
        o, t = old[i][0], new[i][0]
        step = max(align, (abs(t - o) // (2 * align)) * align) if t != o else 0  # at least one group
        e = o + (step if t > o else -step)
        e = min(max(e, min(o, t)), max(o, t))
        lo = (edges[-1] if edges else 0) + align
        edges.append(min(max(e, lo), height - align * (world - i)))
    edges = [0] + edges + [height]
    return [(edges[i], edges[i + 1] - edges[i]) for i in range(world)]


def balanced_ranges(costs: np.ndarray, world: int, align: int = ALIGN) -> list[tuple[int, int]]:
    """Cut the (H,) cost profile into ``world`` contiguous (row_begin, row_count)
    ranges of multiples of ``align`` rows (the last takes the remainder),
    every rank at least one group, minimising the largest summed cost
    (binary search on the bound with a greedy cut)."""
    h = len(costs)
    groups = -(-h // align)
    if world < 1 or world > groups:
        raise ValueError(f"cannot cut {h} rows into {world} ranges of multiples of {align}")
    g = np.add.reduceat(np.asarray(costs, dtype=np.float64), np.arange(0, h, align))
    g = np.maximum(g, 0.0) + 1e-12 * max(float(g.max()), 1.0)  # empty groups still cost a little

    def cuts(bound):
        """Greedy cut positions (group indices) keeping every range <= bound, or None."""
        out, acc = [], 0.0
        for i, c in enumerate(g):
            if acc > 0.0 and acc + c > bound:
                out.append(i)
                acc = 0.0
                if len(out) > world - 1:
                    return None
            acc += c
        while len(out) < world - 1:  # spare ranks: split the longest range (never raises the maximum)
            edges = [0] + out + [groups]
            j = max(range(len(edges) - 1), key=lambda k: edges[k + 1] - edges[k])
            if edges[j + 1] - edges[j] < 2:
                return None
            out = sorted(out + [(edges[j] + edges[j + 1]) // 2])
        return out

    lo, hi = float(g.max()), float(g.sum()) * (1.0 + 1e-9)
    best = cuts(hi)
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        c = cuts(mid)
        if c is not None:
            best, hi = c, mid
        else:
            lo = mid
    edges = [0] + [b * align for b in best] + [h]
    return [(edges[i], edges[i + 1] - edges[i]) for i in range(world)]


def row_permutation(ranges, height: int, rows_per_rank: int) -> np.ndarray:
    """Raster row y -> row of the gathered (world * rows_per_rank) stack of
    compact rank chunks (chunk r holds rows [b_r, b_r + n_r) at 0..n_r-1)."""
    perm = np.empty(height, dtype=np.int64)
    for r, (b, n) in enumerate(ranges):
        perm[b:b + n] = r * rows_per_rank + np.arange(n)
    return perm
