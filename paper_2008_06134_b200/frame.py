"""Device-resident frame pipeline across the GPUs of one node.

A frame is K1 (attenuation build) + K2 (ray march) + image assembly, the
same work as ``bench.render_scene`` in the reference (bench.py:97-109) but
with every input resident in HBM. One process per GPU; ranks talk through
``torch.distributed`` (NCCL over NVLink/NVSwitch on a B200 node).

Partitioning:

- March: image space, in bands of ``band_rows`` rows dealt round-robin
  (band b -> rank b % world) so that every rank gets a similar share of the
  centred volume. Rays are independent (raycaster.py:447-448), so there is
  no exchange until the end: each rank writes its bands into a compact
  chunk and one ``all_gather_into_tensor`` + row permutation assembles the
  raster image on every rank.
- Build: either replicated (every rank runs the full K1; no collective) or
  row-sharded: rank r builds light rows [r*Hs, (r+1)*Hs) into a row-major
  [H][n][W] texel-quad buffer, whose row shards are contiguous, and one all-gather
  replicates the full buffer. Texels are independent in the reference build
  (lightbuffer.py:168-198), so the sharded build needs no halo; K2 reads the
  gathered buffer through strides, so no permutation pass is needed.
- Volume: replicated (uploaded or broadcast once per dataset).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .device import DeviceVolume, device_volume, f64_tensor, render_params, current_stream_handle
from .lightbuffer import build_into, check_frame


def band_layout(height: int, band_rows: int, world: int):
    """(rows_per_rank, perm): every rank's chunk has rows_per_rank rows, and
    raster row y of the image is row perm[y] of the gathered
    (world * rows_per_rank) stack."""
    bands = -(-height // band_rows)
    per_rank = -(-bands // world) * band_rows
    perm = np.empty(height, dtype=np.int64)
    for y in range(height):
        b, r = divmod(y, band_rows)
        owner, j = b % world, b // world
        perm[y] = owner * per_rank + j * band_rows + r
    return per_rank, perm


def shard_rows(height: int, world: int, rank: int) -> tuple[int, int, int]:
    """Light rows [begin, end) built by ``rank`` and the padded shard height."""
    hs = -(-height // world)
    begin = min(height, rank * hs)
    return begin, min(height, begin + hs), hs


def all_gather_into(out: torch.Tensor, chunk: torch.Tensor, group=None) -> None:
    """``out`` = concatenation of every rank's ``chunk`` along dim 0."""
    if out.device.type == "cuda" or dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, chunk, group=group)
    else:  # gloo (CPU tests)
        parts = list(out.view(-1, *chunk.shape).unbind(0))
        dist.all_gather(parts, chunk, group=group)


class FrameRenderer:
    """Build + march + assemble one frame of a fixed scene, all on device.

    ``build`` is "replicated" or "sharded" (row-sharded K1 + all-gather)."""

    def __init__(self, volume, tf, light_cam, spec, settings, *, group=None, build: str = "replicated",
                 band_rows: int = 8, compensation_n: float = 0.0, device=None):
        check_frame(light_cam, spec)
        if build not in ("replicated", "sharded"):
            raise ValueError(f"build must be 'replicated' or 'sharded', got {build!r}")
        if band_rows < 8 or band_rows % 8:
            raise ValueError("band_rows must be a positive multiple of 8")
        self.group = group
        self.distributed = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.distributed else 0
        self.world = dist.get_world_size(group) if self.distributed else 1
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dvol = volume if isinstance(volume, DeviceVolume) else device_volume(volume, self.dev)
        self.tf, self.settings, self.build_mode = tf, settings, build
        self.band_rows, self.comp = band_rows, compensation_n
        self.lut = f64_tensor(tf.resolve(settings.step), self.dev)
        self.counter = torch.zeros(1, dtype=torch.int64, device=self.dev)
        w, h = int(settings.viewport[0]), int(settings.viewport[1])
        self.width, self.height = w, h
        self.rows_local, perm = band_layout(h, band_rows, self.world)
        self.chunk = torch.zeros((self.rows_local, w, 4), dtype=torch.float32, device=self.dev)
        if self.world > 1:
            self.gathered = torch.empty((self.world * self.rows_local, w, 4), dtype=torch.float32, device=self.dev)
            self.perm = torch.from_numpy(perm).to(self.dev)
            self.image = torch.empty((h, w, 4), dtype=torch.float32, device=self.dev)
        else:
            self.image = self.chunk[:h]
        self.set_light(light_cam, spec)

    # -------------------------------------------------------------- light
    def prepare_light(self, light_cam, spec):
        """Device copies of a light frame's small inputs (alpha LUT at the slice
        spacing, plane offsets), so a moving light costs no allocation per frame."""
        check_frame(light_cam, spec)
        return (light_cam, spec, f64_tensor(self.tf.resolve(spec.spacing)[:, 3], self.dev),
                f64_tensor(spec.plane_offsets, self.dev))

    def use_light(self, prepared) -> None:
        """Switch to a prepared light frame; the buffer is reused when its shape is unchanged."""
        cam, spec, alpha, offsets = prepared
        shape = (int(spec.n_slices), int(cam.resolution[1]), int(cam.resolution[0]))
        if getattr(self, "_shape", None) != shape:
            self.set_light(cam, spec)
        self.cam, self.spec, self.alpha, self.offsets = cam, spec, alpha, offsets
        self._render_params = None

    def set_light(self, light_cam, spec) -> None:
        """(Re)allocate the attenuation buffer for a light frame (config 5 moves the light)."""
        check_frame(light_cam, spec)
        self.cam, self.spec = light_cam, spec
        self.alpha = f64_tensor(self.tf.resolve(spec.spacing)[:, 3], self.dev)
        self.offsets = f64_tensor(spec.plane_offsets, self.dev)
        n, h, w = int(spec.n_slices), int(light_cam.resolution[1]), int(light_cam.resolution[0])
        self._shape = (n, h, w)
        if self.build_mode == "replicated" or self.world == 1:
            self.storage = torch.empty((n, h, w, 4), dtype=torch.float32, device=self.dev)
            self.quads = self.storage
            self.shard = None
        else:
            b, e, hs = shard_rows(h, self.world, self.rank)
            # row-major [H][n][W] quads: a rank's rows are one contiguous chunk
            self.storage = torch.empty((self.world * hs, n, w, 4), dtype=torch.float32, device=self.dev)
            self.shard_rows = (b, e)
            self.shard = torch.empty((hs, n, w, 4), dtype=torch.float32, device=self.dev)
            self.quads = self.storage[:h].permute(1, 0, 2, 3)  # (n, H, W, 4) view
        self.intensity = self.quads[..., 0]
        self._render_params = None

    # -------------------------------------------------------------- stages
    def build(self) -> None:
        if self.shard is None:
            build_into(self.dvol, self.alpha, self.cam, self.spec, self.offsets, self.quads, self.comp)
            return
        b, e = self.shard_rows
        if e > b:
            view = self.shard[: e - b].permute(1, 0, 2, 3)  # (n, rows, W, 4), row stride n*W quads
            build_into(self.dvol, self.alpha, self.cam, self.spec, self.offsets, view, self.comp, b, e)
        all_gather_into(self.storage, self.shard, self.group)

    def march(self, count_samples: bool = True) -> None:
        if self._render_params is None:
            buf_modes = self.settings.shading_mode != "none"
            self._render_params = render_params(
                self.dvol, self.lut, self.settings, self.cam if buf_modes else None,
                self.spec if buf_modes else None, self.quads if buf_modes else None,
                self.cam.light_color, float(self.dvol.voxel_size.max()), self.chunk, self.counter,
                band_rows=self.band_rows, rank=self.rank, world=self.world)
        self._render_params.sample_count = self.counter.data_ptr() if count_samples else None
        N.check(N.lib.sbrc_render(self._render_params, current_stream_handle()), "sbrc_render")

    def assemble(self) -> torch.Tensor:
        if self.world > 1:
            all_gather_into(self.gathered, self.chunk, self.group)
            torch.index_select(self.gathered, 0, self.perm, out=self.image)
        return self.image

    def frame(self) -> torch.Tensor:
        self.build()
        self.march()
        return self.assemble()

    def reset_counter(self) -> None:
        self.counter.zero_()

    @property
    def buffer_bytes(self) -> int:
        return int(self.spec.n_slices) * int(self.cam.resolution[0]) * int(self.cam.resolution[1]) * 4
