"""Device residency: volume upload (K0), LUT upload and C-ABI parameter packing.

Volume (K0). The reference keeps a float32 (nz, ny, nx) array normalised at
load time (volume.py:141-151). A u8/u16 dataset crosses the bus in its raw
encoding (1 or 2 bytes per voxel) and is normalised once in HBM to the same
float32 values (``DeviceVolume.widened``, the default); kept raw, the kernels
renormalise at fetch with an IEEE float32 division, bit for bit the same. A
volume is uploaded once and cached by array identity, the way the reference
service keeps datasets resident (service.py:133-152); later calls with the
same array only re-use it.
"""

from __future__ import annotations

import math
import threading
import weakref
from collections import OrderedDict

import numpy as np
import torch

from . import _native as N
from .scene import camera_frame, ShellKernel, ConeKernel


def _require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2008_06134_b200 needs a CUDA device (sm_100a); there is no CPU path")
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def current_stream_handle() -> int:
    """cudaStream_t of the current stream on the current device."""
    if _RAW_STREAM is not None:
        return _RAW_STREAM(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


class DeviceVolume:
    """A VolumeDataset resident in HBM in its compact stored encoding."""

    def __init__(self, data: torch.Tensor, voxel_type: int, dims, box_lo, box_hi, source_type: int | None = None):
        self.data = data
        self.voxel_type = voxel_type
        self.source_type = voxel_type if source_type is None else source_type  # encoding of the dataset
        self.dims = tuple(int(d) for d in dims)
        self.box_lo = np.asarray(box_lo, dtype=np.float64)
        self.box_hi = np.asarray(box_hi, dtype=np.float64)
        self._value_min = None

    @property
    def value_min(self) -> float:
        """Smallest normalised voxel value (one reduction, cached; a speed hint
        for the zero-emission skip, never a correctness input)."""
        if self._value_min is None:
            d = self.data.reshape(-1)
            m = None
            for b in range(0, d.numel(), 1 << 26):  # slabs bound the temporaries
                c = d[b:b + (1 << 26)]
                if self.voxel_type == N.VOXEL_U16:
                    c = c.to(torch.int32) & 0xFFFF
                cm = c.min()
                m = cm if m is None else torch.minimum(m, cm)
            scale = {N.VOXEL_F32: 1.0, N.VOXEL_U8: 255.0, N.VOXEL_U16: 65535.0}[self.voxel_type]
            self._value_min = float(m) / scale
        return self._value_min

    @property
    def voxel_size(self) -> np.ndarray:
        """(box_hi - box_lo) / dims, as VolumeDataset.voxel_size (volume.py:119-122)."""
        return (self.box_hi - self.box_lo) / np.array(self.dims, dtype=np.float64)

    def widened(self) -> "DeviceVolume":
        """A float32 copy of a u8/u16 volume, normalised once with load_raw's IEEE
        float32 division (volume.py:143-146) — the same values the kernels
        compute at fetch, so results are identical."""
        if self.voxel_type == N.VOXEL_F32:
            return self
        f = torch.empty(self.data.numel(), dtype=torch.float32, device=self.data.device)
        N.check(N.lib.sbrc_widen_volume(self.data.data_ptr(), self.voxel_type, f.numel(), f.data_ptr(),
                                        current_stream_handle()), "sbrc_widen_volume")
        f = f.view(self.data.shape)
        out = DeviceVolume(f, N.VOXEL_F32, self.dims, self.box_lo, self.box_hi, source_type=self.voxel_type)
        out._value_min = self._value_min
        return out

    @property
    def nbytes(self) -> int:
        return self.data.numel() * self.data.element_size()

    @property
    def kernel_data(self) -> torch.Tensor:
        """The voxels in the layout the loaded library's kernels read: ``data``
        itself (linear), or — in a brick-layout A/B build (sbrc_volume_layout()
        == 1) — a bricked copy made once on the device."""
        if N.lib.sbrc_volume_layout() == 0:
            return self.data
        if getattr(self, "_bricked", None) is None:
            nx, ny, nz = self.dims
            out = torch.empty(int(N.lib.sbrc_brick_elems(nx, ny, nz)), dtype=self.data.dtype, device=self.data.device)
            N.check(N.lib.sbrc_brick_pack(self.data.data_ptr(), self.voxel_type, nx, ny, nz, out.data_ptr(),
                                          current_stream_handle()), "sbrc_brick_pack")
            self._bricked = out
        return self._bricked

    def struct(self) -> N.SbrcVolume:
        s = N.SbrcVolume()
        s.data = self.kernel_data.data_ptr()
        s.nx, s.ny, s.nz = self.dims
        s.voxel_type = self.voxel_type
        s.box_lo[:] = [float(x) for x in self.box_lo]
        s.box_ext[:] = [float(x) for x in (self.box_hi - self.box_lo)]
        return s

    @classmethod
    def from_dataset(cls, v, device=None, raw: np.ndarray | None = None, widen: bool = True) -> "DeviceVolume":
        """Upload ``v`` (a VolumeDataset, ours or the reference's).

        ``raw`` optionally supplies the u8/u16 voxels; otherwise, for a u8/u16
        dataset, they are recovered from ``v.data`` and kept only if they
        reproduce ``v.data`` exactly. The compact integers are what crosses
        the bus; with ``widen`` (default) they are normalised once to float32
        in HBM (faster fetches: config 4 march 24.0 -> 22.3 ms, config 2
        0.33 -> 0.25 ms; identical values), otherwise kept raw (1-2 B/voxel)."""
        dev = _require_cuda(device)
        data = np.ascontiguousarray(v.data, dtype=np.float32)
        kind, stored = N.VOXEL_F32, data
        scalar_type = getattr(v, "scalar_type", "f32")
        if raw is None:
            raw = getattr(v, "raw", None)
        if raw is None and scalar_type in ("u8", "u16"):
            raw = _recover_raw(data, scalar_type)
        if raw is not None:
            raw = np.ascontiguousarray(raw)
            kind = {np.dtype(np.uint8): N.VOXEL_U8, np.dtype(np.uint16): N.VOXEL_U16}[raw.dtype]
            stored = raw.view(np.int16) if raw.dtype == np.uint16 else raw
        t = torch.from_numpy(stored).to(dev)
        dv = cls(t, kind, v.dims, v.box_lo, v.box_hi)
        return dv.widened() if widen else dv


def _recover_raw(data: np.ndarray, scalar_type: str, slab: int = 1 << 24):
    """The u8/u16 integers behind a load_raw-normalised float32 grid, or None
    if they do not reproduce it exactly; processed in slabs (bounded memory)."""
    scale, dt = (255.0, np.uint8) if scalar_type == "u8" else (65535.0, np.uint16)
    flat = data.reshape(-1)
    out = np.empty(flat.shape, dtype=dt)
    s32 = np.float32(scale)
    for i in range(0, flat.size, slab):
        chunk = flat[i:i + slab]
        cand = np.rint(chunk.astype(np.float64) * scale)
        if cand.min() < 0 or cand.max() > scale:
            return None
        out[i:i + slab] = cand
        if not np.array_equal(out[i:i + slab].astype(np.float32) / s32, chunk):
            return None
    return out.reshape(data.shape)


_VOLUME_CACHE: dict[int, tuple[weakref.ref, DeviceVolume]] = {}


def device_volume(v, device=None) -> DeviceVolume:
    """Cached upload keyed by the identity of ``v.data``."""
    if isinstance(v, DeviceVolume):
        return v
    dv = getattr(v, "_device_volume", None)
    if isinstance(dv, DeviceVolume):
        return dv
    key = id(v.data)
    hit = _VOLUME_CACHE.get(key)
    if hit is not None and hit[0]() is v.data and hit[1].data.device == _require_cuda(device):
        return hit[1]
    dvol = DeviceVolume.from_dataset(v, device)
    try:
        ref = weakref.ref(v.data, lambda _r, k=key: _VOLUME_CACHE.pop(k, None))
        _VOLUME_CACHE[key] = (ref, dvol)
    except TypeError:
        pass
    return dvol


_VOXEL_TORCH = {N.VOXEL_F32: torch.float32, N.VOXEL_U8: torch.uint8, N.VOXEL_U16: torch.int16}


def broadcast_volume(dvol: "DeviceVolume | None", dims, voxel_type: int, box_lo, box_hi, device,
                     group=None, src: int = 0) -> "DeviceVolume":
    """Replicate rank ``src``'s device volume on every rank of ``group`` with one
    collective (NCCL over NVLink/NVSwitch: 512 MiB in about a millisecond,
    against a PCIe upload per rank) — SURVEY §8e's "volume replicated via one
    broadcast per dataset". Ranks other than ``src`` pass ``dvol=None`` and the
    dataset's dims / stored voxel type / box."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    if rank == src:
        if dvol is None:
            raise ValueError("the source rank must pass its DeviceVolume")
        t = dvol.data.contiguous()
    else:
        nx, ny, nz = (int(d) for d in dims)
        t = torch.empty((nz, ny, nx), dtype=_VOXEL_TORCH[voxel_type], device=device)
    # as raw bytes: NCCL (and gloo) have no 16-bit integer type, and a byte copy is exact for every encoding
    dist.broadcast(t.view(torch.uint8), src=dist.get_global_rank(group, src) if group is not None else src,
                   group=group)
    if rank == src:
        return dvol
    return DeviceVolume(t, voxel_type, dims, box_lo, box_hi)


class _PinnedRing:
    """Page-locked staging ring for the small per-frame uploads (LUTs, plane
    offsets): a host array is copied into the next free slot and sent with one
    asynchronous copy on the current stream. Slots are handed out in order;
    the ring wraps only once every copy of the previous lap has completed (at
    ~12 KiB per frame that is dozens of frames back), so a slot is never
    rewritten under a copy in flight. While a lap is still in flight (a host
    far ahead of the GPU) uploads take torch's pinned allocator instead of
    waiting. ``upload`` returns None then."""

    def __init__(self, nbytes: int = 1 << 20):
        self.size = nbytes
        self.off = 0
        self.buf = None
        self.host = None
        self.pending: list = []
        self.lock = threading.Lock()

    def upload(self, a: np.ndarray, device) -> torch.Tensor | None:
        nb = a.nbytes
        with self.lock:
            if self.buf is None:
                self.buf = torch.empty(self.size, dtype=torch.uint8, pin_memory=True)
                self.host = self.buf.numpy()
            start = (self.off + 255) & ~255
            if start + nb > self.size:
                # newest first: on one stream it completes last, so a lap in flight costs one query
                if not all(ev.query() for ev in reversed(self.pending)):
                    return None
                self.pending.clear()
                start = 0
            self.host[start:start + nb] = a.reshape(-1).view(np.uint8)
            dst = torch.empty(a.shape, dtype=torch.float64, device=device)
            dst.copy_(self.buf[start:start + nb].view(torch.float64).view(a.shape), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(dst.device))
            self.pending.append(ev)
            self.off = start + nb
        return dst


_STAGING = _PinnedRing()


def f64_tensor(arr, device) -> torch.Tensor:
    """float64 host array -> device, staged through pinned memory and copied
    asynchronously on the current stream (small arrays through the staging
    ring, larger ones through torch's caching host allocator)."""
    a = np.ascontiguousarray(arr, dtype=np.float64)
    if 0 < a.nbytes <= _STAGING.size // 8 and torch.device(device).type == "cuda":
        t = _STAGING.upload(a, device)
        if t is not None:
            return t
    if not a.flags.writeable:  # read-only cached arrays (scene.camera_frame): torch wants a writable buffer
        a = a.copy()
    host = torch.from_numpy(a)
    return host.pin_memory().to(device, non_blocking=True)


_CONST_CACHE: "OrderedDict" = None
_CONST_LOCK = threading.Lock()


def device_const(arr, device) -> torch.Tensor:
    """Device copy of a small float64 host array (LUTs, plane offsets), cached
    by value: a frame whose inputs did not change uploads nothing. The
    tensors are read-only inputs of the kernels; a caller keeps the one it
    got alive for as long as its launches need it."""
    global _CONST_CACHE
    a = np.ascontiguousarray(arr, dtype=np.float64)
    key = (str(device), a.shape, a.tobytes())
    with _CONST_LOCK:
        if _CONST_CACHE is None:
            _CONST_CACHE = OrderedDict()
        t = _CONST_CACHE.get(key)
        if t is not None:
            _CONST_CACHE.move_to_end(key)
            return t
    t = f64_tensor(a, device)
    with _CONST_LOCK:
        _CONST_CACHE[key] = t
        while len(_CONST_CACHE) > 256:
            _CONST_CACHE.popitem(last=False)
    return t


def device_consts(arrs, device) -> list:
    """Several small float64 host arrays as views of ONE device copy (one
    pinned staging buffer, one host-to-device copy), cached by value like
    ``device_const``."""
    parts = [np.ascontiguousarray(a, dtype=np.float64) for a in arrs]
    flat = np.concatenate([a.reshape(-1) for a in parts])
    t = device_const(flat, device)
    out, o = [], 0
    for a in parts:
        out.append(t[o:o + a.size].view(a.shape))
        o += a.size
    return out


_RESOLVED: dict = {}


def resolved_lut(tf, step: float) -> np.ndarray:
    """tf.resolve(step) (transfer.py:76-84), memoised by the LUT's bytes and the
    step: the float64 power of 256 entries is recomputed only when they change.
    The result is read-only."""
    lut = getattr(tf, "lut", None)
    if lut is None:
        return tf.resolve(step)
    key = (np.ascontiguousarray(lut).tobytes(), float(step), type(tf).resolve)
    out = _RESOLVED.get(key)
    if out is None:
        out = np.asarray(tf.resolve(step))
        out.setflags(write=False)
        if len(_RESOLVED) > 256:
            _RESOLVED.clear()
        _RESOLVED[key] = out
    return out


def drop_frame_constants() -> None:
    """Forget the value-cached device copies of the per-frame constants (LUTs,
    plane offsets), so the next call uploads them again — an end-to-end
    measurement whose every step pays its own host-to-device copies
    (bench.py e2e). The memoised LUT resolves (host arithmetic, a pure
    function of the LUT and step) are kept."""
    global _CONST_CACHE
    with _CONST_LOCK:
        _CONST_CACHE = None


def to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> new numpy array via a pinned buffer (fast D2H); the
    array owns the pinned block until it is garbage collected."""
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return out.numpy()


def light_frame(cam, spec, offsets_dev: torch.Tensor | None) -> N.SbrcLightFrame:
    """Pack LightCamera + SliceStackSpec (lightbuffer.py:37-86, slicing.py:22-33)."""
    lf = N.SbrcLightFrame()
    lf.width, lf.height = int(cam.resolution[0]), int(cam.resolution[1])
    lf.n_slices = int(spec.n_slices)
    lf.axis_u[:] = [float(x) for x in cam.axis_u]
    lf.axis_v[:] = [float(x) for x in cam.axis_v]
    lf.light_dir[:] = [float(x) for x in spec.light_dir]
    lf.u_range[:] = [float(cam.u_range[0]), float(cam.u_range[1])]
    lf.v_range[:] = [float(cam.v_range[0]), float(cam.v_range[1])]
    lf.d_min, lf.d_max = float(spec.d_min), float(spec.d_max)
    lf.plane_offsets = offsets_dev.data_ptr() if offsets_dev is not None else None
    return lf


def quad_strides(quads: torch.Tensor) -> tuple[int, int]:
    """(layer, row) strides in element units of an (n, H, W, 4) texel-quad view,
    or of an (n, H, W, 2) layer-pair view (sbrc quad_layout 1)."""
    c = quads.shape[3] if quads.dim() == 4 else 0
    if (quads.dtype != torch.float32 or quads.dim() != 4 or c not in (2, 4) or quads.stride(3) != 1
            or quads.stride(2) != c or quads.stride(0) % c or quads.stride(1) % c):
        raise ValueError("texel quads must be an (n, H, W, 4) (or layer pairs (n, H, W, 2)) float32 view "
                         "packed along W")
    return quads.stride(0) // c, quads.stride(1) // c


def quad_layout(quads: torch.Tensor) -> int:
    """0 = texel quads, 1 = layer pairs (sbrc_build_params.quad_layout)."""
    return 1 if quads.shape[-1] == 2 else 0


def build_params(dvol: DeviceVolume, cam, spec, alpha_lut_dev, offsets_dev, quads: torch.Tensor,
                 compensation_n: float, row_begin: int, row_end: int, sparse=None,
                 plain: bool = False, clip=()) -> N.SbrcBuildParams:
    """``quads`` is the (n, row_end-row_begin, W, 4) texel-quad view of the rows built;
    ``sparse`` = (reach_world, layers_below, layers_above) writes only the quads a
    march with that lookup reach can read (lightbuffer.lookup_reach), None all.
    ``plain``: ``quads`` is instead an (n, rows, W) float32 view that receives
    the plain stack (the row shard of a sharded build). ``clip``: the
    consumer's half-spaces (a, b, c, d), a.x + b.y + c.z + d >= 0, already
    widened by its lookup reach (partition.frustum_clip; needs ``sparse``)."""
    if plain:
        if quads.dtype != torch.float32 or quads.dim() != 3 or quads.stride(2) != 1:
            raise ValueError("a plain stack must be an (n, rows, W) float32 view with contiguous rows")
        qk, qy = quads.stride(0), quads.stride(1)
    else:
        qk, qy = quad_strides(quads)
    p = N.SbrcBuildParams()
    p.quad_layout = 0 if plain else quad_layout(quads)
    p.volume = dvol.struct()
    p.light = light_frame(cam, spec, offsets_dev)
    p.alpha_lut = alpha_lut_dev.data_ptr()
    p.compensation_n = float(compensation_n)
    p.row_begin, p.row_end = int(row_begin), int(row_end)
    p.quads, p.quad_layer_stride, p.quad_row_stride = quads.data_ptr(), qk, qy
    p.output_plain = int(bool(plain))
    if sparse is not None:
        p.write_sparse = 1
        p.write_reach, p.write_below, p.write_above = float(sparse[0]), int(sparse[1]), int(sparse[2])
    if clip:
        if sparse is None:
            raise ValueError("a clipped (frustum-culled) build is a sparse build: pass the lookup reach")
        if len(clip) > N.MAX_CLIP:
            raise ValueError(f"at most {N.MAX_CLIP} clip half-spaces")
        p.n_clip = len(clip)
        for i, h in enumerate(clip):
            p.clip[i][:] = [float(x) for x in h]
    return p


def pack_quads(plain: torch.Tensor, quads: torch.Tensor | None = None) -> torch.Tensor:
    """Texel quads of a plain (n, H, W) float32 CUDA stack (any layer/row strides)."""
    if plain.dtype != torch.float32 or plain.dim() != 3 or plain.stride(2) != 1:
        raise ValueError("intensity must be an (n, H, W) float32 tensor with contiguous rows")
    n, h, w = plain.shape
    if quads is None:
        quads = torch.empty((n, h, w, 4), dtype=torch.float32, device=plain.device)
    qk, qy = quad_strides(quads)
    N.check(N.lib.sbrc_pack_quads(plain.data_ptr(), plain.stride(0), plain.stride(1), n, h, w,
                                  quads.data_ptr(), qk, qy, current_stream_handle()), "sbrc_pack_quads")
    return quads


def clear_entries(lut: np.ndarray) -> int:
    """Length of the LUT's leading run of entries with zero (premultiplied)
    emission: a sample whose LUT coordinate clip(s,0,1)*255 is at most
    run - 1 adds exactly nothing to the pixel (raycaster.py:436)."""
    nz = np.flatnonzero(np.any(np.asarray(lut)[:, :3] != 0.0, axis=1))
    return int(nz[0]) if nz.size else len(lut)


def skip_clear_hint(dvol: DeviceVolume, lut: np.ndarray) -> bool:
    """Use the zero-emission skip when the volume reaches into that run
    (some voxel's value maps there). Results are identical either way."""
    run = clear_entries(lut)
    return run >= 1 and dvol.value_min * 255.0 <= run - 1


def render_params(dvol: DeviceVolume, lut_dev: torch.Tensor, settings, buffer_cam, buffer_spec,
                  quads_dev: torch.Tensor | None, light_color, voxel_size_max: float,
                  image: torch.Tensor, counter: torch.Tensor | None,
                  band_rows: int = 8, rank: int = 0, world: int = 1, voxel_size=None,
                  peer_images=(), heavy_first: bool = False,
                  lut_host: np.ndarray | None = None, feedback=None, row_range=None,
                  march_kernel: int = 0) -> N.SbrcRenderParams:
    """Pack RenderSettings + buffer into the K2 params (raycaster.py:443-469).
    ``lut_host`` (the resolved LUT on the host) enables the skip_clear hint.
    ``row_range`` = (row_begin, row_count): a contiguous share of the image
    rows instead of the (band_rows, rank, world) bands."""
    mode = settings.shading_mode
    if mode not in N.SHADE:
        raise ValueError(f"unknown shading mode {mode!r}")
    if settings.lookup_mode not in N.LOOKUP:
        raise ValueError(f"unknown lookup mode {settings.lookup_mode!r}")
    p = N.SbrcRenderParams()
    p.volume = dvol.struct()
    p.lut_rgba = lut_dev.data_ptr()
    w, h = int(settings.viewport[0]), int(settings.viewport[1])
    p.width, p.height = w, h
    p.shading = N.SHADE[mode]
    p.lookup = N.LOOKUP[settings.lookup_mode]
    cam = settings.camera
    fr = camera_frame(cam, settings.viewport)
    p.eye[:] = [float(x) for x in cam.position]
    p.forward[:] = [float(x) for x in fr["forward"]]
    p.right[:] = [float(x) for x in fr["right"]]
    p.up2[:] = [float(x) for x in fr["up2"]]
    p.tan_half, p.aspect = fr["tan_half"], fr["aspect"]
    p.step = float(settings.step)
    p.et_alpha = float(settings.early_termination_alpha)
    if mode in ("sbrc_shadow", "shell", "cone"):
        p.light = light_frame(buffer_cam, buffer_spec, None)
        if quads_dev is not None:
            p.quads = quads_dev.data_ptr()
            p.quad_layer_stride, p.quad_row_stride = quad_strides(quads_dev)
            p.quad_layout = quad_layout(quads_dev)
        p.light_color[:] = [float(c) for c in np.asarray(light_color, dtype=np.float64)]
        p.ambient_floor = float(settings.ambient_floor)
    if mode in ("phong", "extinction"):
        p.scene_light_dir[:] = [float(x) for x in np.asarray(settings.light.direction, dtype=np.float64)]
        ph = settings.phong
        p.phong[:] = [float(ph.ambient), float(ph.diffuse), float(ph.specular), float(ph.shininess)]
        p.voxel_size[:] = [float(x) for x in voxel_size]
        p.ambient_floor = float(settings.ambient_floor)
    if mode == "shell":
        k = settings.shell_kernel or ShellKernel.default(float(voxel_size_max))
        if len(k.radii) > N.MAX_SHELLS or len(k.radii) != len(k.weights) or not k.radii:
            raise ValueError(f"shell kernel must have 1..{N.MAX_SHELLS} radii with matching weights")
        p.shell_count = len(k.radii)
        for i, (r, wt) in enumerate(zip(k.radii, k.weights)):
            p.shell_radius[i], p.shell_weight[i] = float(r), float(wt)
    if mode == "cone":
        k = settings.cone_kernel or ConeKernel()
        if not 1 <= len(k.angles) <= N.MAX_ANGLES:
            raise ValueError(f"cone kernel must have 1..{N.MAX_ANGLES} angles")
        p.cone_axis_samples = int(k.axis_samples)
        p.cone_angle_count = len(k.angles)
        p.cone_ring = float(k.ring_radius_per_step)
        for i, th in enumerate(k.angles):
            p.cone_cos[i], p.cone_sin[i] = math.cos(th), math.sin(th)
    if lut_host is not None and mode != "none":
        p.skip_clear = int(skip_clear_hint(dvol, lut_host))
    p.band_rows, p.rank, p.world = int(band_rows), int(rank), int(world)
    if row_range is not None:
        p.row_begin, p.row_count = int(row_range[0]), int(row_range[1])
    p.march_kernel = int(march_kernel)
    p.image = image.data_ptr() if image is not None else None
    if len(peer_images) > N.MAX_PEERS:
        raise ValueError(f"at most {N.MAX_PEERS} peer images")
    for i, ptr in enumerate(peer_images):
        p.peer_images[i] = int(ptr)
    p.n_peers = len(peer_images)
    p.sample_count = counter.data_ptr() if counter is not None else None
    # The struct holds raw device addresses: it keeps the tensors behind them
    # alive for as long as a caller caches it (FrameRenderer, FramePipeline).
    keep = [dvol.data, dvol.kernel_data, lut_dev, quads_dev, image, counter]
    if heavy_first:  # dispatch table over the exact grid sbrc_render will launch
        grid = N.render_grid(p)
        order = tile_order_for(settings, band_rows, rank, world, lut_dev.device, grid, row_range,
                               empty_first=image is not None and image.device.type == "cpu")
        if feedback is not None:  # measured order of the previous frame (schedule.TileFeedback)
            order, steps = feedback.prepare(grid, order)
            p.tile_steps = steps.data_ptr()
            keep.append(steps)
        p.tile_order, p.n_tiles = order.data_ptr(), int(order.numel())
        keep.append(order)
    p._keep = keep
    return p


_ORDER_CACHE: dict = {}


def tile_order_for(settings, band_rows: int, rank: int, world: int, device, grid=None,
                   row_range=None, empty_first: bool = False) -> torch.Tensor:
    """Device copy of the heavy-first dispatch table (schedule.heavy_first) over
    ``grid`` (tiles_x, tiles_y, tile_w, tile_h; default the block grid), cached per view."""
    from .schedule import heavy_first
    cam = settings.camera
    key = (tuple(np.asarray(cam.position, np.float64)), tuple(np.asarray(cam.target, np.float64)),
           tuple(np.asarray(cam.up, np.float64)), float(cam.fov_deg), tuple(settings.viewport), band_rows, rank,
           world, str(device), None if grid is None else tuple(grid), None if row_range is None else tuple(row_range),
           bool(empty_first))
    t = _ORDER_CACHE.get(key)
    if t is None:
        # dropping the cache is safe: cached render params own their table (render_params._keep)
        if len(_ORDER_CACHE) > 64:
            _ORDER_CACHE.clear()
        t = torch.from_numpy(heavy_first(settings, band_rows, rank, world, grid, row_range, empty_first)).to(device)
        _ORDER_CACHE[key] = t
    return t
