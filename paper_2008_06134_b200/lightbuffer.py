"""Drop-in ``build_attenuation_buffer`` on the GPU (K1).

Same signature, validation and result semantics as the reference
``slicecast.lightbuffer.build_attenuation_buffer`` (lightbuffer.py:144-199):
layer k of the (n, H, W) float32 intensity stack is the light arriving at
slice k, i.e. the product of (1 - alpha) over slices 0..k-1 at that texel.
The stack stays in HBM (``intensity_device``); ``intensity`` copies it to a
numpy array on first access for callers that expect the reference type.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .device import _require_cuda, build_params, current_stream_handle, device_volume, f64_tensor, pack_quads, to_host


class AttenuationBuffer:
    """Layered light-space intensity stack plus its light frame (lightbuffer.py:107-131).

    On the device the stack is held as texel quads (include/sbrc.h): an
    (n, H, W, 4) float32 view whose component 0 is ``intensity``. A buffer
    made from a plain stack (numpy, as the reference returns, or an
    (n, H, W) CUDA tensor) is packed into quads on first device use.
    """

    def __init__(self, camera, spec, compensation_n: float = 0.0, intensity=None, *, quads=None):
        self.camera = camera
        self.spec = spec
        self.compensation_n = compensation_n
        self._host = None
        self._plain_dev = None
        self.quads: torch.Tensor | None = quads
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

    @property
    def intensity_device(self) -> torch.Tensor:
        """(n, H, W) CUDA view of the stack (component 0 of the quads)."""
        if self.quads is not None:
            return self.quads[..., 0]
        if self._plain_dev is not None:
            return self._plain_dev
        return self.device_quads()[..., 0]

    def device_quads(self, device=None) -> torch.Tensor:
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


def check_frame(cam, spec) -> None:
    """lightbuffer.py:155-156: camera and stack must agree on the light direction."""
    if float(np.linalg.norm(np.asarray(cam.light_dir) - np.asarray(spec.light_dir))) > 1e-9:
        raise ValueError("light camera and slice stack disagree on light direction")


def build_into(dvol, alpha_lut_dev, cam, spec, offsets_dev, quads: torch.Tensor, compensation_n=0.0,
               row_begin: int = 0, row_end: int | None = None, stream: int | None = None) -> None:
    """Enqueue K1 for light rows [row_begin, row_end) into ``quads``, the
    (n, row_end - row_begin, W, 4) texel-quad view of those rows."""
    h = int(cam.resolution[1])
    row_end = h if row_end is None else row_end
    p = build_params(dvol, cam, spec, alpha_lut_dev, offsets_dev, quads, compensation_n, row_begin, row_end)
    N.check(N.lib.sbrc_build(p, current_stream_handle() if stream is None else stream), "sbrc_build")


def build_attenuation_buffer(v, tf, cam, spec, compensation_n: float = 0.0, device=None) -> AttenuationBuffer:
    """GPU attenuation build; drop-in for lightbuffer.py:144-199."""
    check_frame(cam, spec)
    dev = _require_cuda(device)
    w, h = int(cam.resolution[0]), int(cam.resolution[1])
    n = int(spec.n_slices)
    dvol = device_volume(v, dev)
    alpha = f64_tensor(tf.resolve(spec.spacing)[:, 3], dev)   # :159-160
    offsets = f64_tensor(spec.plane_offsets, dev)
    quads = torch.empty((n, h, w, 4), dtype=torch.float32, device=dev)
    build_into(dvol, alpha, cam, spec, offsets, quads, compensation_n)
    return AttenuationBuffer(camera=cam, spec=spec, compensation_n=compensation_n, quads=quads)
