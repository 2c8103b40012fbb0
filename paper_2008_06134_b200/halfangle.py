"""Half-angle slicing baseline on the GPU (halfangle.py:48-142).

The comparison point of the paper: slices perpendicular to
the half vector between view and light, and per slice two dependent passes —
an eye pass compositing the slice into the float64 accumulation image,
modulated by the light transmittance accumulated so far, and a light pass
attenuating that transmittance. The pass count is 2n, so its cost grows with
the slice count, unlike the buffer-based ray caster.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .device import _require_cuda, current_stream_handle, device_volume, f64_tensor, to_host
from .scene import LightCamera, camera_frame, make_slice_stack, normalize


def half_vector(view_dir, light_dir):
    """(half, order) (halfangle.py:35-45)."""
    view_dir = np.asarray(view_dir, dtype=np.float64)
    light_dir = np.asarray(light_dir, dtype=np.float64)
    if float(np.dot(view_dir, light_dir)) >= 0.0:
        s, order = view_dir + light_dir, "front_to_back"
    else:
        s, order = -view_dir + light_dir, "back_to_front"
    if float(np.linalg.norm(s)) < 1e-9:
        return light_dir.copy(), "back_to_front"
    return normalize(s), order


def render_half_angle(v, tf, settings, n_slices: int, light_resolution=None, light_trace: list | None = None,
                      device=None):
    """(image (H, W, 4) float32 numpy, pass_count = 2n) — drop-in for halfangle.py:48-142.
    ``light_trace`` (a list) receives the light transmittance after every slice."""
    img, passes = render_half_angle_device(v, tf, settings, n_slices, light_resolution, light_trace, device)
    return to_host(img), passes


def render_half_angle_device(v, tf, settings, n_slices: int, light_resolution=None, light_trace: list | None = None,
                             device=None):
    """As render_half_angle, returning the (H, W, 4) CUDA image (no host copy)."""
    if n_slices < 1:
        raise ValueError("n_slices must be >= 1")
    dev = _require_cuda(device)
    light, cam = settings.light, settings.camera
    w, h = int(settings.viewport[0]), int(settings.viewport[1])
    lw, lh = (int(x) for x in (light_resolution or settings.viewport))
    view_dir = normalize(cam.target - cam.position)
    half, order = half_vector(view_dir, light.direction)
    stack = make_slice_stack(half, n_slices)
    lcam = LightCamera.fit(light.direction, light.color, (lw, lh))
    fr = camera_frame(cam, settings.viewport)
    dvol = device_volume(v, dev)
    lut = f64_tensor(tf.lut, dev)
    offs = f64_tensor(stack.plane_offsets, dev)
    eye_acc = torch.empty(h * w * 4, dtype=torch.float64, device=dev)
    light_acc = torch.empty(lh * lw, dtype=torch.float64, device=dev)
    image = torch.empty((h, w, 4), dtype=torch.float32, device=dev)
    p = N.SbrcHalfAngleParams()
    p.volume = dvol.struct()
    p.lut, p.plane_offsets = lut.data_ptr(), offs.data_ptr()
    p.width, p.height, p.light_width, p.light_height = w, h, lw, lh
    p.n_slices, p.front_to_back = int(n_slices), int(order == "front_to_back")
    p.eye[:] = [float(x) for x in cam.position]
    p.forward[:], p.right[:], p.up2[:] = ([float(x) for x in fr[k]] for k in ("forward", "right", "up2"))
    p.tan_half, p.aspect = fr["tan_half"], fr["aspect"]
    p.half[:] = [float(x) for x in half]
    p.delta = float(stack.spacing)
    p.light_dir[:] = [float(x) for x in light.direction]
    p.axis_u[:], p.axis_v[:] = [float(x) for x in lcam.axis_u], [float(x) for x in lcam.axis_v]
    p.u_range[:], p.v_range[:] = list(lcam.u_range), list(lcam.v_range)
    p.hl = float(np.dot(half, light.direction))          # :81
    p.h_dot_u = float(np.dot(half, lcam.axis_u))          # :82
    p.h_dot_v = float(np.dot(half, lcam.axis_v))          # :83
    p.h_dot_e = float(np.dot(half, cam.position))         # :88
    p.eye_accum, p.light_accum, p.image = eye_acc.data_ptr(), light_acc.data_ptr(), image.data_ptr()
    count = C.c_int(0)
    stream = current_stream_handle()
    if light_trace is None:
        N.check(N.lib.sbrc_half_angle(C.byref(p), 0, n_slices, 1, 1, C.byref(count), stream), "sbrc_half_angle")
        total = count.value
    else:
        total = 0
        for k in range(n_slices):
            N.check(N.lib.sbrc_half_angle(C.byref(p), k, k + 1, int(k == 0), int(k == n_slices - 1),
                                          C.byref(count), stream), "sbrc_half_angle")
            total += count.value
            light_trace.append(to_host(light_acc).reshape(lh, lw).copy())
    return image, total
