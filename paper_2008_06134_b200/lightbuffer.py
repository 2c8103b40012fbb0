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
from .device import _require_cuda, build_params, current_stream_handle, device_volume, f64_tensor


class AttenuationBuffer:
    """Layered light-space intensity stack plus its light frame (lightbuffer.py:107-131)."""

    def __init__(self, camera, spec, compensation_n: float = 0.0, intensity=None):
        self.camera = camera
        self.spec = spec
        self.compensation_n = compensation_n
        self._host = None
        self.intensity_device: torch.Tensor | None = None
        if isinstance(intensity, torch.Tensor):
            self.intensity_device = intensity
        elif intensity is not None:
            self._host = np.asarray(intensity, dtype=np.float32)

    @property
    def intensity(self) -> np.ndarray:
        if self._host is None and self.intensity_device is not None:
            self._host = self.intensity_device.cpu().numpy()
        return self._host

    @intensity.setter
    def intensity(self, value):
        self._host = None if value is None else np.asarray(value, dtype=np.float32)
        self.intensity_device = None

    def device_intensity(self, device=None) -> torch.Tensor:
        if self.intensity_device is None:
            if self._host is None:
                raise ValueError("attenuation buffer has no intensity")
            self.intensity_device = torch.from_numpy(np.ascontiguousarray(self._host)).to(_require_cuda(device))
        return self.intensity_device

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


def build_into(dvol, alpha_lut_dev, cam, spec, offsets_dev, out: torch.Tensor, compensation_n=0.0,
               row_begin: int = 0, row_end: int | None = None, stream: int | None = None) -> None:
    """Enqueue K1 for light rows [row_begin, row_end) into ``out`` ((n, rows, W) view-compatible)."""
    h = int(cam.resolution[1])
    row_end = h if row_end is None else row_end
    p = build_params(dvol, cam, spec, alpha_lut_dev, offsets_dev, out, compensation_n, row_begin, row_end)
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
    out = torch.empty((n, h, w), dtype=torch.float32, device=dev)
    build_into(dvol, alpha, cam, spec, offsets, out, compensation_n)
    return AttenuationBuffer(camera=cam, spec=spec, compensation_n=compensation_n, intensity=out)
