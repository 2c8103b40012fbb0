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
  row-sharded: rank r builds light rows [r*Hs, (r+1)*Hs) of the plain float32
  stack into a row-major [H][n][W] buffer, whose row shards are contiguous,
  one all-gather replicates it (A bytes, not the 4A of texel quads), and each
  rank packs it into quads locally. Texels are independent in the reference
  build (lightbuffer.py:168-198), so the sharded build needs no halo.
- Volume: replicated (uploaded or broadcast once per dataset).
- Frustum-culled build (``build="frustum"``, contiguous partition,
  partition.py): each rank renders one contiguous, cost-balanced band of
  rows and builds only the texel-slices its band's lookups can read (K1
  clipped by the band's two eye planes); no exchange at all.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .device import (DeviceVolume, current_stream_handle, device_volume, f64_tensor, pack_quads, render_params,
                     tile_order_for)
from .lightbuffer import build_into, check_frame, lookup_reach
from . import partition as PT


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
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, chunk, group=group)
        return
    # gloo (tests): gather host copies
    host = chunk.cpu()
    parts = [torch.empty_like(host) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, host, group=group)
    out.copy_(torch.cat(parts).view_as(out))


class _DeviceBuffer:
    """An IPC-capable cudaMalloc allocation exposed to torch via __cuda_array_interface__."""

    def __init__(self, nbytes: int):
        ptr = C.c_void_p()
        N.check(N.lib.sbrc_ipc_alloc(nbytes, C.byref(ptr)), "sbrc_ipc_alloc")
        self.ptr, self.nbytes = ptr.value, nbytes
        self.__cuda_array_interface__ = {"shape": (nbytes // 4,), "typestr": "<f4", "data": (self.ptr, False),
                                         "version": 3, "strides": None}

    def handle(self) -> bytes:
        buf = (C.c_char * 64)()
        N.check(N.lib.sbrc_ipc_handle(self.ptr, buf), "sbrc_ipc_handle")
        return bytes(buf)

    def free(self) -> None:
        if self.ptr:
            N.lib.sbrc_ipc_free(self.ptr)
            self.ptr = None


def open_peer(handle: bytes) -> int:
    ptr = C.c_void_p()
    N.check(N.lib.sbrc_ipc_open((C.c_char * 64).from_buffer_copy(handle), C.byref(ptr)), "sbrc_ipc_open")
    return ptr.value


class FrameRenderer:
    """Build + march + assemble one frame of a fixed scene, all on device.

    ``build`` is "replicated" or "sharded" (row-sharded K1 + all-gather).
    ``assemble`` is "nccl" (compact chunks + all_gather_into_tensor + row
    permutation) or "p2p": the march kernel stores every finished pixel
    straight into each rank's raster image through CUDA-IPC peer mappings
    (NVLink), so the frame ends with a barrier instead of an all-gather. The
    p2p mode verifies itself against the NCCL path on the first frame and
    falls back to it (``assemble_mode``) if the images differ."""

    def __init__(self, volume, tf, light_cam, spec, settings, *, group=None, build: str = "replicated",
                 band_rows: int = 8, compensation_n: float = 0.0, device=None, assemble: str = "nccl",
                 heavy_first: bool | None = None, feedback: bool | None = None, sparse: bool = True,
                 partition: str | None = None):
        check_frame(light_cam, spec)
        if build not in ("replicated", "sharded", "frustum"):
            raise ValueError(f"build must be 'replicated', 'sharded' or 'frustum', got {build!r}")
        if partition is None:
            partition = "contiguous" if build == "frustum" else "bands"
        if partition not in ("bands", "contiguous"):
            raise ValueError(f"partition must be 'bands' or 'contiguous', got {partition!r}")
        if build == "frustum" and (partition != "contiguous" or not sparse):
            raise ValueError("the frustum-culled build needs the contiguous partition and sparse K1 writes")
        self.partition = partition
        self.march_kernel = 0  # K2 kernel choice (sbrc_render_params.march_kernel); see choose_march_kernel
        if band_rows < 8 or band_rows % 8:
            raise ValueError("band_rows must be a positive multiple of 8")
        self.group = group
        self.distributed = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.distributed else 0
        self.world = dist.get_world_size(group) if self.distributed else 1
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dvol = volume if isinstance(volume, DeviceVolume) else device_volume(volume, self.dev)
        self.tf, self.settings, self.build_mode = tf, settings, build
        # heavy-first dispatch (schedule.py) measured: +1% at 1 rank, +8% at 4, +14% at 8, -6% at 2
        self.heavy_first = heavy_first
        # heavy-first by the previous frame's measured tile costs (schedule.TileFeedback):
        # default with > 1 rank (rank shares at 2/4/8 ranks: 2.34/1.17/0.76 -> 1.63/0.90/0.62 ms
        # vs the geometric estimate); at 1 rank the geometric order keeps better locality
        from .schedule import TileFeedback
        if feedback is None:
            feedback = self.world > 1 and heavy_first is not False
        self.feedback = TileFeedback() if feedback else None
        self.band_rows, self.comp = band_rows, compensation_n
        # sparse K1: write only the quads this march's lookups can read (lightbuffer.lookup_reach)
        self.sparse = sparse
        # K2 params per (quads buffer, p2p raster parity); the structs own what they point to
        self._params: dict = {}
        self.lut_host = tf.resolve(settings.step)
        self.lut = f64_tensor(self.lut_host, self.dev)
        self.counter = torch.zeros(1, dtype=torch.int64, device=self.dev)
        w, h = int(settings.viewport[0]), int(settings.viewport[1])
        self.width, self.height = w, h
        self.ranges, self.row_range, self.clip = None, None, ()
        if partition == "contiguous":
            self.set_ranges(PT.balanced_ranges(PT.row_costs_geometric(settings), self.world), _init=True)
        else:
            self._layout(*band_layout(h, band_rows, self.world))
        self.set_light(light_cam, spec)
        if assemble not in ("nccl", "p2p"):
            raise ValueError(f"assemble must be 'nccl' or 'p2p', got {assemble!r}")
        self.assemble_mode = "nccl"
        self._peers: list[list[int]] = []
        self._parity = 0  # p2p raster buffer of the next frame
        if assemble == "p2p" and self.world > 1:
            self._setup_p2p()

    # -------------------------------------------------------------- partition
    def _layout(self, rows_local: int, perm) -> None:
        w, h = self.width, self.height
        self.rows_local = rows_local
        self.chunk = torch.zeros((rows_local, w, 4), dtype=torch.float32, device=self.dev)
        if self.world > 1:
            self.gathered = torch.empty((self.world * rows_local, w, 4), dtype=torch.float32, device=self.dev)
            self.perm = torch.from_numpy(perm).to(self.dev)
            self.image = torch.empty((h, w, 4), dtype=torch.float32, device=self.dev)
        else:
            self.image = self.chunk[:h]

    def set_ranges(self, ranges, _init: bool = False) -> None:
        """Contiguous partition: rank r renders rows [b_r, b_r + n_r) of ``ranges``
        (every rank passes the same list), and a frustum-culled build clips K1
        to that band."""
        if self.partition != "contiguous":
            raise ValueError("row ranges need the contiguous partition")
        ranges = [(int(b), int(n)) for b, n in ranges]
        if len(ranges) != self.world or ranges[0][0] != 0 or sum(n for _, n in ranges) != self.height or \
                any(n < 1 or ranges[i + 1][0] != b + n for i, (b, n) in enumerate(ranges[:-1])):
            raise ValueError(f"ranges must tile rows 0..{self.height} with one non-empty range per rank")
        self.ranges = ranges
        self.row_range = ranges[self.rank]
        rows = max(n for _, n in ranges)
        self._layout(rows, PT.row_permutation(ranges, self.height, rows))
        if not _init:
            self._update_clip()
            self._params.clear()
            self._complete = False
            if self.feedback is not None:
                self.feedback.grid = None

    def _update_clip(self) -> None:
        reach = self.reach
        if self.build_mode == "frustum" and reach is not None:
            b, n = self.row_range
            self.clip = PT.frustum_clip(self.settings, b, b + n, reach[0])
        else:
            self.clip = ()

    def rebalance(self, frame_ms: float) -> list:
        """Re-cut the contiguous bands by measured time: every rank passes the
        device time of its last frame (build + march, CUDA events); the times
        are exchanged (one small all-gather), spread over each band like the
        geometric row profile, cut into balanced ranges, and each boundary
        moves halfway there (partition.damped_ranges). Collective; returns
        the new ranges."""
        times = [float(frame_ms)]
        if self.world > 1:
            nccl = dist.get_backend(self.group) == "nccl"
            t = torch.zeros(self.world, dtype=torch.float64, device=self.dev if nccl else "cpu")
            t[self.rank] = float(frame_ms)
            dist.all_reduce(t, group=self.group)
            times = t.cpu().tolist()
        prof = PT.calibrated_profile(PT.row_costs_geometric(self.settings), self.ranges, times)
        self.set_ranges(PT.damped_ranges(self.ranges, PT.balanced_ranges(prof, self.world), self.height))
        return self.ranges

    def _frame_times(self, frames: int) -> list:
        """Every rank's device time of `frames` build + march frames (ms per
        frame), exchanged with one all-reduce."""
        stream = torch.cuda.current_stream(self.dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(frames):
            self.build()
            self.march(False)
        e1.record(stream)
        e1.synchronize()
        mine = e0.elapsed_time(e1) / frames
        if self.world == 1:
            return [mine]
        nccl = dist.get_backend(self.group) == "nccl"
        t = torch.zeros(self.world, dtype=torch.float64, device=self.dev if nccl else "cpu")
        t[self.rank] = mine
        dist.all_reduce(t, group=self.group)
        return t.cpu().tolist()

    def calibrate(self, iters: int = 10, frames: int = 3) -> list:
        """Contiguous partition: each round every rank picks its K2 kernel for
        its band (choose_march_kernel) and the bands are timed; the next cut
        steps from the best cut seen so far (its times spread over the bands
        like the geometric row profile, re-balanced, boundaries moved halfway:
        partition.calibrated_profile / balanced_ranges / damped_ranges), so
        timing noise cannot walk the cut away from a good one. Ends on the
        best cut and each rank's kernel for it. Collective; returns the cut."""
        shape = PT.row_costs_geometric(self.settings)
        best = None
        for _ in range(iters):
            self.choose_march_kernel()
            times = self._frame_times(frames)
            if best is None or max(times) < best[0]:
                best = (max(times), list(self.ranges), self.march_kernel, times)
            nxt = PT.damped_ranges(best[1], PT.balanced_ranges(PT.calibrated_profile(shape, best[1], best[3]),
                                                                self.world), self.height)
            if nxt == list(self.ranges):  # converged (every rank computes the same cut)
                break
            self.set_ranges(nxt)
        self.set_ranges(best[1])
        self.march_kernel = best[2]
        return self.ranges

    def choose_march_kernel(self, frames: int = 3) -> int:
        """Time this rank's march with the throughput and the latency K2
        kernel (CUDA events, after one warm-up each) and keep the faster —
        which one wins depends on the share's size and on its longest rays,
        so a contiguous band measures instead of trusting the size rule.
        Local (no collective); results are identical either way."""
        stream = torch.cuda.current_stream(self.dev)
        times = {}
        for k in (1, 2):
            self.march_kernel = k
            self._params.clear()
            self.build()
            self.march(False)  # warm-up (and a fresh heavy-first table for this grid)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(frames):
                self.march(False)
            e1.record(stream)
            e1.synchronize()
            times[k] = e0.elapsed_time(e1) / frames
        self.march_kernel = min(times, key=times.get)
        self._params.clear()
        if self.feedback is not None:
            self.feedback.grid = None
        return self.march_kernel

    # -------------------------------------------------------------- p2p
    def _setup_p2p(self) -> None:
        """Map every rank's two raster images (double buffer, selected by frame
        parity) into this process. Frame f's march stores into buffer f % 2 of
        every rank; the barrier that ends frame f+1 orders frame f+2's stores
        (the next writer of buffer f % 2) after every rank's reads of frame f
        that were issued before it called frame f+1, so a slow consumer never
        sees pixels of a later frame (the write-after-read race a single
        raster would have)."""
        h, w = self.height, self.width
        try:
            self._rasters = [_DeviceBuffer(h * w * 16), _DeviceBuffer(h * w * 16)]
            mine = b"".join(r.handle() for r in self._rasters)
        except RuntimeError:
            self._rasters, mine = [], b""
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=self.group)
        if not all(handles):  # every rank sees the same list: consistent fallback
            self._fallback()
            return
        rasters = [torch.as_tensor(r, device=self.dev).view(h, w, 4) for r in self._rasters]
        peers, opened = [[], []], []
        try:
            for r, hd in enumerate(handles):
                for b in range(2):
                    if r == self.rank:
                        peers[b].append(self._rasters[b].ptr)
                    else:
                        ptr = open_peer(hd[64 * b:64 * (b + 1)])
                        opened.append(ptr)
                        peers[b].append(ptr)
            ok = True
        except RuntimeError:
            ok = False
        self._opened = opened
        self._barrier = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # both decisions are collective and taken in the same order on every
        # rank, so a failure on one rank cannot desynchronise the collectives
        if not self._all_ok(ok):  # some rank could not map a peer image
            self._fallback()
            return
        ref = self.frame().clone()  # NCCL path
        self._peers = peers
        self._raster_t = rasters
        self.assemble_mode = "p2p"
        self._params.clear()
        same = bool(torch.equal(ref, self.frame())) and bool(torch.equal(ref, self.frame()))  # both buffers
        if not self._all_ok(same):
            self._fallback()

    def _all_ok(self, ok: bool) -> bool:
        nccl = dist.get_backend(self.group) == "nccl"
        flag = torch.tensor([0 if ok else 1], dtype=torch.int32, device=self.dev if nccl else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self.group)
        return int(flag.item()) == 0

    def _fallback(self) -> None:
        self._peers = []
        self.assemble_mode = "nccl"
        self._params.clear()

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
        self._update_clip()
        self._params.clear()
        self._complete = False

    def set_light(self, light_cam, spec) -> None:
        """(Re)allocate the attenuation buffer for a light frame (config 5 moves the light)."""
        check_frame(light_cam, spec)
        self.cam, self.spec = light_cam, spec
        self.alpha = f64_tensor(self.tf.resolve(spec.spacing)[:, 3], self.dev)
        self.offsets = f64_tensor(spec.plane_offsets, self.dev)
        n, h, w = int(spec.n_slices), int(light_cam.resolution[1]), int(light_cam.resolution[0])
        self._shape = (n, h, w)
        # the hard-shadow march reads one lookup per sample: half-size layer pairs
        # serve it faster than texel quads (profiles/r2_notes.md); the scattering modes keep quads
        pairs = self.settings.shading_mode == "sbrc_shadow" and self.build_mode != "sharded" and w >= 2
        self.storage = torch.empty((n, h, w, 2 if pairs else 4), dtype=torch.float32, device=self.dev)
        self.quads = self.storage
        if self.build_mode != "sharded" or self.world == 1:
            self.shard = None
        else:
            b, e, hs = shard_rows(h, self.world, self.rank)
            # row-major [H][n][W] plain stack: a rank's rows are one contiguous chunk;
            # the gathered stack is packed into quads locally (4x fewer bytes cross NVLink)
            self.plain = torch.empty((self.world * hs, n, w), dtype=torch.float32, device=self.dev)
            self.shard_rows = (b, e)
            self.shard = torch.empty((hs, n, w), dtype=torch.float32, device=self.dev)
        self._update_clip()
        self._params.clear()
        self._complete = False

    # -------------------------------------------------------------- stages
    @property
    def reach(self):
        """Lookup reach of this renderer's march (None: full K1 writes)."""
        if not self.sparse:
            return None
        return lookup_reach(self.settings, self.cam, self.spec, float(self.dvol.voxel_size.max()))

    @property
    def intensity(self) -> torch.Tensor:
        """(n, H, W) CUDA view of the current stack, complete: after a sparse
        build the unwritten quads are filled by a full K1 into the same
        storage first (identical values)."""
        if not self._complete:
            if self.shard is None:
                build_into(self.dvol, self.alpha, self.cam, self.spec, self.offsets, self.quads, self.comp)
            else:
                self.build()
            self._complete = True
        return self.quads[..., 0]

    @property
    def needs_buffer(self) -> bool:
        """Only the buffer modes read the attenuation stack (raycaster.py:395-411);
        none / phong / extinction frames run no K1 (bench.render_scene builds
        the buffer only for them too, bench.py:97-109)."""
        return self.settings.shading_mode in ("sbrc_shadow", "shell", "cone")

    def build_into_buffer(self, quads: torch.Tensor) -> None:
        """This rank's K1 (replicated or frustum-culled) into ``quads``."""
        if not self.needs_buffer:
            return
        build_into(self.dvol, self.alpha, self.cam, self.spec, self.offsets, quads, self.comp, sparse=self.reach,
                   clip=self.clip)

    def build(self) -> None:
        if not self.needs_buffer:
            return
        if self.shard is None:
            self.build_into_buffer(self.quads)
            self._complete = self.reach is None
            return
        self._complete = True
        b, e = self.shard_rows
        if e > b:
            view = self.shard[: e - b].permute(1, 0, 2)  # (n, rows, W), row stride n*W floats
            build_into(self.dvol, self.alpha, self.cam, self.spec, self.offsets, view, self.comp, b, e, plain=True)
        all_gather_into(self.plain, self.shard, self.group)
        h = int(self.cam.resolution[1])
        pack_quads(self.plain[:h].permute(1, 0, 2), self.quads)

    def march(self, count_samples: bool = True) -> None:
        p2p = self.assemble_mode == "p2p"
        key = (self.quads.data_ptr(), self._parity if p2p else 0)
        params = self._params.get(key)
        if params is None:
            buf_modes = self.settings.shading_mode in ("sbrc_shadow", "shell", "cone")
            params = render_params(
                self.dvol, self.lut, self.settings, self.cam if buf_modes else None,
                self.spec if buf_modes else None, self.quads if buf_modes else None,
                self.cam.light_color, float(self.dvol.voxel_size.max()), None if p2p else self.chunk, self.counter,
                band_rows=self.band_rows, rank=self.rank, world=self.world, voxel_size=self.dvol.voxel_size,
                peer_images=self._peers[key[1]] if p2p else (),
                heavy_first=(self.feedback is not None or self.world != 2) if self.heavy_first is None
                else self.heavy_first,
                lut_host=self.lut_host, feedback=self.feedback, row_range=self.row_range,
                march_kernel=self.march_kernel)
            self._params[key] = params
        elif self.feedback is not None and self.feedback.steps is not None:
            self.feedback.steps.zero_()
        params.sample_count = self.counter.data_ptr() if count_samples else None
        N.check(N.lib.sbrc_render(params, current_stream_handle()), "sbrc_render")
        if self.feedback is not None:
            self.feedback.update()

    def assemble(self) -> torch.Tensor:
        if self.world > 1:
            if self.assemble_mode == "p2p":
                # every rank's march has stored its pixels into every raster image;
                # the barrier (stream-ordered after the march) completes the frame
                if dist.get_backend(self.group) == "nccl":
                    dist.all_reduce(self._barrier, group=self.group)
                else:  # gloo (tests): host barrier after this rank's march completed
                    torch.cuda.current_stream(self.dev).synchronize()
                    dist.barrier(group=self.group)
                out = self._raster_t[self._parity]
                self._parity ^= 1
                return out
            all_gather_into(self.gathered, self.chunk, self.group)
            if self.gathered.is_cuda:
                N.check(N.lib.sbrc_permute_rows(self.gathered.data_ptr(), self.perm.data_ptr(), self.image.data_ptr(),
                                                self.height, self.width, current_stream_handle()), "sbrc_permute_rows")
            else:
                torch.index_select(self.gathered, 0, self.perm, out=self.image)
        return self.image

    def close(self) -> None:
        """Unmap the peer rasters, then free this rank's own (p2p mode).
        Collective: every rank first finishes its work and closes its
        mappings, and only after a barrier frees the rasters others mapped."""
        opened = getattr(self, "_opened", [])
        rasters = getattr(self, "_rasters", [])
        if not opened and not rasters:
            return
        torch.cuda.synchronize(self.dev)  # no march of this rank still stores to a peer
        for ptr in opened:
            N.lib.sbrc_ipc_close(ptr)
        self._opened = []
        if self.distributed and self.world > 1:
            dist.barrier(group=self.group)  # every importer has closed its handles
        for r in rasters:
            r.free()
        self._rasters = []
        self._peers = []

    def frame(self) -> torch.Tensor:
        self.build()
        self.march()
        return self.assemble()

    def reset_counter(self) -> None:
        self.counter.zero_()

    @property
    def buffer_bytes(self) -> int:
        return int(self.spec.n_slices) * int(self.cam.resolution[0]) * int(self.cam.resolution[1]) * 4


class FramePipeline:
    """Frames with the attenuation build of frame f+1 overlapping the march of
    frame f (replicated build): two texel-quad buffers, a build stream and the
    launching stream, ordered by events — build(f+1) waits until march(f-1)
    has released its buffer, march(f) waits for build(f). Every frame still
    runs its full build and march; the march leaves SMs idle in its tail (and
    throughout when one GPU's share of the image is small), which the next
    build fills."""

    def __init__(self, fr: FrameRenderer, build_priority: int = 0, build_after_march: bool = False):
        if fr.shard is not None:
            raise ValueError("pipelining needs the replicated build")
        self.fr = fr
        self.bufs = [fr.quads, torch.empty_like(fr.quads)]
        # build_priority: CUDA stream priority of the build stream (0 = default; higher-priority
        # launches get their blocks dispatched first when both kernels have blocks pending)
        self.build_stream = torch.cuda.Stream(fr.dev, priority=build_priority)
        # launch order of one step: the next frame's build before this march (its
        # blocks are dispatched first) or after it (it fills the march's tail)
        self.build_after_march = build_after_march
        self.built = [torch.cuda.Event(), torch.cuda.Event()]
        self.released = [torch.cuda.Event(), torch.cuda.Event()]
        self.f = 0
        self.pending = None  # buffer index whose build is in flight

    def _launch_build(self, i: int) -> None:
        fr = self.fr
        with torch.cuda.stream(self.build_stream):
            self.build_stream.wait_event(self.released[i])
            fr.build_into_buffer(self.bufs[i])
            self.built[i].record(self.build_stream)

    def step(self, count_samples: bool = False) -> torch.Tensor:
        fr, i = self.fr, self.f % 2
        if self.pending is None:
            self._launch_build(i)
        if not self.build_after_march:
            self._launch_build(1 - i)  # next frame's stack, overlapping this march
        self.pending = 1 - i
        main = torch.cuda.current_stream(fr.dev)
        main.wait_event(self.built[i])
        fr.quads = self.bufs[i]  # the renderer keeps one params struct per buffer
        fr._complete = fr.reach is None
        fr.march(count_samples)
        self.released[i].record(main)
        if self.build_after_march:
            self._launch_build(1 - i)
        img = fr.assemble()
        self.f += 1
        return img

    def drain(self) -> None:
        """Make the launching stream wait for the build in flight (end of a timed region)."""
        if self.pending is not None:
            torch.cuda.current_stream(self.fr.dev).wait_event(self.built[self.pending])
