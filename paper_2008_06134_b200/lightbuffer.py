"""Drop-in ``build_attenuation_buffer`` on the GPU (K1).

Same signature, validation and result semantics as the reference
``slicecast.lightbuffer.build_attenuation_buffer`` (lightbuffer.py:144-199):
layer k of the (n, H, W) float32 intensity stack is the light arriving at
slice k, i.e. the product of (1 - alpha) over slices 0..k-1 at that texel.
The stack stays in HBM (``intensity_device``); ``intensity`` copies it to a
numpy array on first access for callers that expect the reference type.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .device import (_require_cuda, build_params, current_stream_handle, device_consts, device_volume, f64_tensor,
                     pack_quads, resolved_lut, to_host)


class AttenuationBuffer:
    """Layered light-space intensity stack plus its light frame (lightbuffer.py:107-131).

    On the device the stack is held as texel quads (include/sbrc.h): an
    (n, H, W, 4) float32 view whose component 0 is ``intensity``. A buffer
    made from a plain stack (numpy, as the reference returns, or an
    (n, H, W) CUDA tensor) is packed into quads on first device use.

    A buffer from ``build_attenuation_buffer`` is built *sparse*: K1 writes
    only the quads a march can read with the default shell / cone / shadow
    lookups (``sparse`` = their reach, see ``lookup_reach``). ``render``
    uses it as is when its own reach fits; every other consumer (the
    ``intensity`` stack, point lookups, wider kernels) first completes it
    with a full build into the same storage (identical values).
    """

    def __init__(self, camera, spec, compensation_n: float = 0.0, intensity=None, *, quads=None,
                 sparse=None, rebuild=None):
        self.camera = camera
        self.spec = spec
        self.compensation_n = compensation_n
        self._host = None
        self._plain_dev = None
        self.quads: torch.Tensor | None = quads
        self.sparse = sparse          # (reach_world, layers_below, layers_above) of a sparse build, or None
        self._rebuild = rebuild       # full build into self.quads (completes a sparse buffer)
        if isinstance(intensity, torch.Tensor):
            self._plain_dev = intensity
        elif intensity is not None:
            self._host = np.asarray(intensity, dtype=np.float32)

    @property
    def intensity(self) -> np.ndarray:
        """(n, H, W) float32 numpy stack, as the reference returns it."""
        if self._host is None:
            self._host = to_host(self.intensity_device.contiguous())
        return self._host

    @intensity.setter
    def intensity(self, value):
        self._host = None if value is None else np.asarray(value, dtype=np.float32)
        self._plain_dev, self.quads = None, None

    def complete(self) -> None:
        """Write every quad of a sparse buffer (a full K1 into the same storage)."""
        if self.sparse is not None:
            self._rebuild()
            self.sparse = None

    def quads_for(self, need, device=None) -> torch.Tensor:
        """Device quads for a march whose lookups reach ``need`` (lookup_reach)."""
        if self.sparse is not None and not covers(self.sparse, need):
            self.complete()
        if self.quads is None:
            return self.device_quads(device)
        return self.quads

    @property
    def intensity_device(self) -> torch.Tensor:
        """(n, H, W) CUDA view of the stack (component 0 of the quads)."""
        if self.quads is not None:
            self.complete()
            return self.quads[..., 0]
        if self._plain_dev is not None:
            return self._plain_dev
        return self.device_quads()[..., 0]

    def device_quads(self, device=None) -> torch.Tensor:
        """The complete quad stack on the device."""
        self.complete()
        if self.quads is None:
            plain = self._plain_dev
            if plain is None:
                if self._host is None:
                    raise ValueError("attenuation buffer has no intensity")
                plain = torch.from_numpy(np.ascontiguousarray(self._host)).to(_require_cuda(device))
            self.quads = pack_quads(plain)
        return self.quads

    @property
    def shadow_matrix(self) -> np.ndarray:
        return self.camera.shadow_matrix

    @property
    def light_color(self) -> np.ndarray:
        return self.camera.light_color

    @property
    def layers(self) -> np.ndarray:
        return (self.intensity[..., None] * self.light_color).astype(np.float32)

    def layer(self, k: int) -> np.ndarray:
        return (self.intensity[k][..., None] * self.light_color).astype(np.float32)


def lookup_reach(settings, cam, spec, voxel_size_max: float):
    """(reach_world, layers_below, layers_above) the march's light lookups can
    reach from a sample inside the cube, or None for modes without a buffer.

    Lateral reach: the scattering kernel's extent in the light plane plus two
    texel diagonals (bilinear footprint); layers: the kernel's extent along
    the light (the cone steps toward the light, raycaster.py:266-300; the
    shell spans +-r, :239-250) plus one layer for the linear blend and one
    of margin."""
    mode = settings.shading_mode
    if mode not in ("sbrc_shadow", "shell", "cone"):
        return None
    w, h = int(cam.resolution[0]), int(cam.resolution[1])
    texel = max((cam.u_range[1] - cam.u_range[0]) / w, (cam.v_range[1] - cam.v_range[0]) / h)
    spacing = float(spec.spacing)
    lat, below, above = 0.0, 1, 1
    if mode == "shell":
        radii = settings.shell_kernel.radii if settings.shell_kernel is not None else (3.0 * voxel_size_max,)
        r = float(max(radii))
        lat = r
        below = above = int(math.ceil(r / spacing)) + 1
    elif mode == "cone":
        k = settings.cone_kernel
        a = 2 if k is None else int(k.axis_samples)
        ring = 0.5 if k is None else float(k.ring_radius_per_step)
        lat = ring * a * spacing
        below, above = a + 1, 1
    return (lat + 2.0 * math.sqrt(2.0) * texel, below + 1, above + 1)


_REACH: dict = {}


def default_reach(cam, spec, voxel_size_max: float):
    """Reach covering the default kernels of every buffer mode (the sparse
    build of ``build_attenuation_buffer``, whose consumer is not known yet);
    memoised by the quantities it depends on."""
    key = (tuple(int(r) for r in cam.resolution), tuple(float(u) for u in cam.u_range),
           tuple(float(v) for v in cam.v_range), float(spec.spacing), float(voxel_size_max))
    out = _REACH.get(key)
    if out is None:
        from types import SimpleNamespace
        reaches = [lookup_reach(SimpleNamespace(shading_mode=m, shell_kernel=None, cone_kernel=None), cam, spec,
                                voxel_size_max) for m in ("sbrc_shadow", "shell", "cone")]
        out = tuple(max(r[i] for r in reaches) for i in range(3))
        if len(_REACH) > 256:
            _REACH.clear()
        _REACH[key] = out
    return out


def covers(have, need) -> bool:
    return need is None or (have[0] >= need[0] and have[1] >= need[1] and have[2] >= need[2])


def check_frame(cam, spec) -> None:
    """lightbuffer.py:155-156: camera and stack must agree on the light direction."""
    a, b = cam.light_dir, spec.light_dir  # (3,) each; the norm of the difference, as numpy computes it
    if len(a) != len(b) or math.sqrt(sum((float(x) - float(y)) ** 2 for x, y in zip(a, b))) > 1e-9:
        raise ValueError("light camera and slice stack disagree on light direction")


def build_into(dvol, alpha_lut_dev, cam, spec, offsets_dev, quads: torch.Tensor, compensation_n=0.0,
               row_begin: int = 0, row_end: int | None = None, stream: int | None = None, sparse=None,
               plain: bool = False, clip=()) -> None:
    """Enqueue K1 for light rows [row_begin, row_end) into ``quads``, the
    (n, row_end - row_begin, W, 4) texel-quad view of those rows (only the
    quads within ``sparse`` reach when given)."""
    h = int(cam.resolution[1])
    row_end = h if row_end is None else row_end
    p = build_params(dvol, cam, spec, alpha_lut_dev, offsets_dev, quads, compensation_n, row_begin, row_end,
                     sparse, plain, clip)
    N.check(N.lib.sbrc_build(p, current_stream_handle() if stream is None else stream), "sbrc_build")


def build_attenuation_buffer(v, tf, cam, spec, compensation_n: float = 0.0, device=None) -> AttenuationBuffer:
    """GPU attenuation build; drop-in for lightbuffer.py:144-199."""
    check_frame(cam, spec)
    dev = _require_cuda(device)
    w, h = int(cam.resolution[0]), int(cam.resolution[1])
    n = int(spec.n_slices)
    dvol = device_volume(v, dev)
    # alpha LUT at the slice spacing (:159-160) and the plane offsets: one upload
    alpha, offsets = device_consts((resolved_lut(tf, spec.spacing)[:, 3], spec.plane_offsets), dev)
    quads = torch.empty((n, h, w, 4), dtype=torch.float32, device=dev)
    reach = default_reach(cam, spec, float(dvol.voxel_size.max()))
    build_into(dvol, alpha, cam, spec, offsets, quads, compensation_n, sparse=reach)

    def rebuild():
        build_into(dvol, alpha, cam, spec, offsets, quads, compensation_n)

    return AttenuationBuffer(camera=cam, spec=spec, compensation_n=compensation_n, quads=quads, sparse=reach,
                             rebuild=rebuild)
