"""Heavy-first tile scheduling for the march (K2).

The march cannot finish before its slowest blocks — the tiles whose rays
cross the most volume (hundreds of serial samples). With few blocks per SM
(small images, or one rank's share of a multi-GPU frame) those tiles
decide the kernel time if they start late. The block scheduler dispatches
blocks roughly in index order, so the march reads a dispatch table
(``tile_order``) that lists tiles by decreasing estimated cost: the
geometric length of the rays inside the unit cube (ray_box_intersect,
geometry.py:46-67), sampled at the tile's corners and centre.
"""

from __future__ import annotations

import numpy as np

import torch

from . import _native as N
from .scene import camera_frame


def tile_cost(settings, band_rows: int = 8, rank: int = 0, world: int = 1, grid=None,
              row_range=None) -> np.ndarray:
    """(tiles_y, tiles_x) estimated cost (mean in-cube ray length) of the rank-local K2 tiles of
    ``grid`` (tiles_x, tiles_y, tile_w, tile_h: N.render_grid of the launch; default the block grid).
    ``row_range`` = (row_begin, row_count): a contiguous share of the rows instead of bands."""
    w, h = int(settings.viewport[0]), int(settings.viewport[1])
    if grid is None:
        grid = (N.march_grid(w, int(row_range[1]), 8, 0, 1) if row_range is not None
                else N.march_grid(w, h, band_rows if world > 1 else 8, rank, world))
    tx, ty, bw, bh = grid
    fr = camera_frame(settings.camera, settings.viewport)
    eye = np.asarray(settings.camera.position, dtype=np.float64)
    # sample pixels: corners and centre of every tile
    offs = np.array([[0.0, 0.0], [bw - 1, 0.0], [0.0, bh - 1], [bw - 1, bh - 1], [bw / 2, bh / 2]])
    gx, gy = np.meshgrid(np.arange(tx) * bw, np.arange(ty) * bh)
    px = np.clip(gx[..., None] + offs[:, 0], 0, w - 1)
    lr = gy[..., None] + offs[:, 1]
    if row_range is not None:
        py = np.clip(int(row_range[0]) + lr, 0, h - 1)
    else:
        br = band_rows if world > 1 else 8
        band = lr // br
        py = np.clip((rank + band * world) * br + (lr - band * br), 0, h - 1)
    ndc_x = ((px + 0.5) / w * 2.0 - 1.0) * fr["tan_half"] * fr["aspect"]
    ndc_y = (1.0 - (py + 0.5) / h * 2.0) * fr["tan_half"]
    d = fr["forward"] + ndc_x[..., None] * fr["right"] + ndc_y[..., None] * fr["up2"]
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
    return np.where(t_out > t_in, t_out - t_in, 0.0).mean(axis=-1)


def heavy_first(settings, band_rows: int = 8, rank: int = 0, world: int = 1, grid=None,
                row_range=None, empty_first: bool = False) -> np.ndarray:
    """int32 dispatch table: tile indices (ty * tiles_x + tx) by decreasing cost.

    ``empty_first``: tiles whose sampled rays all miss the cube go first
    instead of last. For an image in page-locked host memory (``render``)
    their pixels — a third of a centred frame — then cross PCIe while the
    heavy tiles march, instead of in one burst at the end of the kernel."""
    cost = tile_cost(settings, band_rows, rank, world, grid, row_range).reshape(-1)
    key = np.where(cost > 0.0, -cost, -np.inf) if empty_first else -cost
    return np.argsort(key, kind="stable").astype(np.int32)


class TileFeedback:
    """Heavy-first order from measured costs. K2 writes each tile's longest-ray
    sample count (``sbrc_render_params.tile_steps``); after the launch the
    tiles are sorted by it on the device, and the next frame of the same view
    dispatches in that order (the first frame uses the geometric estimate).
    Everything stays on the launching stream: no host round trip."""

    def __init__(self):
        self.grid = None
        self.order = None
        self.steps = None

    def prepare(self, grid, initial_order: torch.Tensor):
        """(order, steps) device tensors for a launch over ``grid``; zeroes steps."""
        grid = tuple(int(g) for g in grid)
        if grid != self.grid:
            self.grid = grid
            self.order = initial_order.clone()
            self.steps = torch.zeros(grid[0] * grid[1], dtype=torch.int32, device=initial_order.device)
        else:
            self.steps.zero_()
        return self.order, self.steps

    def update(self) -> None:
        """Sort the tiles just measured (call after the launch, same stream)."""
        if self.steps is not None:
            if self.steps.is_cuda:  # sbrc_tile_order: rank-by-count kernel on the launching stream
                from .device import current_stream_handle
                N.check(N.lib.sbrc_tile_order(self.steps.data_ptr(), self.steps.numel(), self.order.data_ptr(),
                                              current_stream_handle()), "sbrc_tile_order")
            else:  # host tensors (CPU tests of the ordering rule)
                idx = torch.argsort(self.steps, descending=True, stable=True)
                self.order.copy_(idx.to(torch.int32))
