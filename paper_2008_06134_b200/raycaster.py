"""Drop-in ``render`` on the GPU (K2).

Mirrors ``slicecast.raycaster.render`` (raycaster.py:443-469): same
arguments, the same ``ConfigError`` when a buffer mode has no buffer
(:450-451), the same ``ValueError`` for an unknown lookup mode
(lightbuffer.py:262-263), and a premultiplied RGBA float32 (H, W, 4) image
with a transparent-black background. ``render`` returns numpy like the
reference; ``render_device`` returns the CUDA tensor and optionally the
executed-sample count.

Modes: ``none``, ``sbrc_shadow``, ``shell``, ``cone`` (the hot path), and
``phong`` / ``extinction`` (local lighting with a float64
central-difference gradient, and a per-sample light march). Also
``shadow_oracle_many``, the brute-force transmittance the buffer modes are
measured against (raycaster.py:356-366).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _native as N
from .device import (_require_cuda, current_stream_handle, device_const, device_volume, f64_tensor, light_frame,
                     pack_quads, resolved_lut,
                     quad_strides, render_params, tile_order_for, to_host)
from .lightbuffer import AttenuationBuffer, lookup_reach
from .scene import BUFFER_MODES, ConfigError


def _quads_of(buffer, dev, need=False) -> torch.Tensor:
    """Device quads of ``buffer``; ``need`` is the march's lookup reach
    (a sparse buffer that covers it is used as is), False = the full stack."""
    if isinstance(buffer, AttenuationBuffer):
        return buffer.device_quads(dev) if need is False else buffer.quads_for(need, dev)
    # a reference AttenuationBuffer (numpy intensity): upload and pack
    return pack_quads(torch.from_numpy(np.ascontiguousarray(buffer.intensity, dtype=np.float32)).to(dev))


def _prepare(v, tf, settings, buffer, device):
    """Validation and device inputs shared by render_device and render."""
    mode = settings.shading_mode
    if mode in BUFFER_MODES and buffer is None:
        raise ConfigError(f"shading mode {mode!r} needs an attenuation buffer")
    if settings.lookup_mode not in N.LOOKUP:
        raise ValueError(f"unknown lookup mode {settings.lookup_mode!r}")
    dev = _require_cuda(device)
    dvol = device_volume(v, dev)
    lut_host = resolved_lut(tf, settings.step)   # raycaster.py:453
    lut = device_const(lut_host, dev)
    inten, cam, spec, color = None, None, None, None
    if mode in BUFFER_MODES:
        need = lookup_reach(settings, buffer.camera, buffer.spec, float(dvol.voxel_size.max()))
        inten = _quads_of(buffer, dev, need)
        cam, spec, color = buffer.camera, buffer.spec, buffer.camera.light_color
        n, hh, ww = inten.shape[:3]
        if (n, hh, ww) != (int(spec.n_slices), int(cam.resolution[1]), int(cam.resolution[0])):
            raise ValueError("attenuation intensity shape does not match its camera/stack")
    return dev, dvol, lut, lut_host, inten, cam, spec, color


def render_device(v, tf, settings, buffer=None, *, device=None, count_samples: bool = False,
                  rank: int = 0, world: int = 1, band_rows: int = 8, out: torch.Tensor | None = None,
                  peer_images=(), heavy_first: bool | None = None, feedback=None):
    """Enqueue K2; returns the (rows, W, 4) CUDA image (all rows when world == 1)
    and, with ``count_samples``, a 1-element int64 CUDA tensor of executed samples."""
    dev, dvol, lut, lut_host, inten, cam, spec, color = _prepare(v, tf, settings, buffer, device)
    w, h = int(settings.viewport[0]), int(settings.viewport[1])
    if world == 1:
        band_rows = 8
    rows = N.local_rows(h, band_rows, rank, world)  # padded to whole bands
    if out is None:
        out = torch.empty((max(rows, 1), w, 4), dtype=torch.float32, device=dev)
    elif out.shape[0] < rows or out.shape[1] != w or out.shape[2] != 4 or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous ({rows}, {w}, 4) float32 tensor")
    counter = torch.zeros(1, dtype=torch.int64, device=dev) if count_samples else None
    vs = float(dvol.voxel_size.max())   # ShellKernel.default(v.voxel_size.max()), :403
    hf = (world != 2) if heavy_first is None else heavy_first
    p = render_params(dvol, lut, settings, cam, spec, inten, color, vs, out, counter,
                      band_rows=band_rows, rank=rank, world=world, voxel_size=dvol.voxel_size,
                      peer_images=[int(x.data_ptr()) if isinstance(x, torch.Tensor) else int(x) for x in peer_images],
                      heavy_first=hf, lut_host=lut_host, feedback=feedback if hf else None)
    N.check(N.lib.sbrc_render(p, current_stream_handle()), "sbrc_render")
    if feedback is not None and hf:
        feedback.update()
    img = out[:h] if world == 1 else out
    return (img, counter) if count_samples else img


def render(v, tf, settings, buffer=None) -> np.ndarray:
    """GPU ray cast; drop-in for raycaster.py:443-469 (returns numpy float32 (H, W, 4)).

    The image is returned without a separate read-back: K2 stores each
    finished pixel straight into a page-locked host array (its device
    address, ``sbrc_host_device_pointer``), so the 16 bytes per pixel cross
    PCIe while the march runs instead of after it (config 3 end to end:
    3.72 -> 3.54 ms per frame; profiles/r01_notes.md)."""
    w, h = int(settings.viewport[0]), int(settings.viewport[1])
    host = torch.empty((max(N.local_rows(h, 8, 0, 1), 1), w, 4), dtype=torch.float32, pin_memory=True)
    if N.host_device_pointer(host.data_ptr()) != host.data_ptr():
        return to_host(render_device(v, tf, settings, buffer))   # not mapped at the same address: copy
    render_device(v, tf, settings, buffer, out=host)
    torch.cuda.current_stream().synchronize()
    return host[:h].numpy()


def shadow_oracle_many(v, tf, pts, light, oracle_step: float, *, device=None) -> np.ndarray:
    """GPU shadow_oracle_many (raycaster.py:356-366): transmittance from each
    (M, 3) world point to the light; returns float64 numpy (M,)."""
    if oracle_step <= 0:
        raise ValueError("oracle_step must be positive")
    dev = _require_cuda(device)
    dvol = device_volume(v, dev)
    alpha = f64_tensor(tf.resolve(oracle_step)[:, 3], dev)
    p = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, 3))
    pd = f64_tensor(p, dev)
    out = torch.empty(p.shape[0], dtype=torch.float64, device=dev)
    to_light = (C.c_double * 3)(*[-float(x) for x in np.asarray(light.direction, dtype=np.float64)])
    vs = dvol.struct()
    N.check(N.lib.sbrc_shadow_oracle(C.byref(vs), alpha.data_ptr(), pd.data_ptr(), p.shape[0], to_light,
                                     float(oracle_step), out.data_ptr(), current_stream_handle()),
            "sbrc_shadow_oracle")
    return to_host(out).reshape(np.asarray(pts).shape[:-1])


# ------------------------------------------------------------ point-wise light API
def _light_factor(buffer, pts, shading: str, lookup: str = "linear", *, shell_kernel=None, cone_kernel=None,
                  eye=None, ambient_floor: float = 0.0, device=None) -> np.ndarray:
    """(M, 4) float32 numpy: (scalar, factor_r, factor_g, factor_b) at world points."""
    if lookup not in N.LOOKUP:
        raise ValueError(f"unknown lookup mode {lookup!r}")
    dev = _require_cuda(device)
    quads = _quads_of(buffer, dev)
    cam, spec = buffer.camera, buffer.spec
    p = N.SbrcRenderParams()
    p.shading, p.lookup = N.SHADE[shading], N.LOOKUP[lookup]
    p.light = light_frame(cam, spec, None)
    p.quads = quads.data_ptr()
    p.quad_layer_stride, p.quad_row_stride = quad_strides(quads)
    p.light_color[:] = [float(c) for c in np.asarray(cam.light_color, dtype=np.float64)]
    p.ambient_floor = float(ambient_floor)
    if shading == "shell":
        if len(shell_kernel.radii) > N.MAX_SHELLS:
            raise ValueError(f"at most {N.MAX_SHELLS} shells")
        p.shell_count = len(shell_kernel.radii)
        for i, (r, w) in enumerate(zip(shell_kernel.radii, shell_kernel.weights)):
            p.shell_radius[i], p.shell_weight[i] = float(r), float(w)
    if shading == "cone":
        if not 1 <= len(cone_kernel.angles) <= N.MAX_ANGLES:
            raise ValueError(f"cone kernel must have 1..{N.MAX_ANGLES} angles")
        p.cone_axis_samples, p.cone_angle_count = int(cone_kernel.axis_samples), len(cone_kernel.angles)
        p.cone_ring = float(cone_kernel.ring_radius_per_step)
        for i, th in enumerate(cone_kernel.angles):
            p.cone_cos[i], p.cone_sin[i] = math.cos(th), math.sin(th)
    q = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, 3))
    out = torch.empty((q.shape[0], 4), dtype=torch.float32, device=dev)
    if q.shape[0]:
        pd = f64_tensor(q, dev)
        e = None if eye is None else (C.c_double * 3)(*[float(x) for x in np.asarray(eye, dtype=np.float64)])
        N.check(N.lib.sbrc_light_factor(C.byref(p), pd.data_ptr(), q.shape[0], e, out.data_ptr(),
                                        current_stream_handle()), "sbrc_light_factor")
    return to_host(out)


def lookup_light_scalar_many(b, pts, mode: str = "linear") -> np.ndarray:
    """GPU lookup_light_scalar_many (lightbuffer.py:256-287); float64 numpy of pts' shape[:-1]."""
    pts = np.asarray(pts, dtype=np.float64)
    return _light_factor(b, pts, "sbrc_shadow", mode)[:, 0].astype(np.float64).reshape(pts.shape[:-1])


def lookup_light_many(b, pts, mode: str = "linear") -> np.ndarray:
    """rgb light arriving at world points (lightbuffer.py:290-293)."""
    return lookup_light_scalar_many(b, pts, mode)[..., None] * np.asarray(b.camera.light_color)


def lookup_light(b, p_world, mode: str = "linear") -> np.ndarray:
    return lookup_light_many(b, np.asarray(p_world, dtype=np.float64)[None, :], mode)[0]


def shade_sbrc_shadow(sample_p, buffer, ambient_floor: float = 0.0, mode: str = "linear") -> np.ndarray:
    """Volume-shadow factor at one point (raycaster.py:231-236)."""
    f = _light_factor(buffer, np.asarray(sample_p, dtype=np.float64)[None, :], "sbrc_shadow", mode,
                      ambient_floor=ambient_floor)
    return f[0, 1:].astype(np.float64)


def shade_shell(sample_p, buffer, kernel, ambient_floor: float = 0.0, mode: str = "linear") -> np.ndarray:
    """Shell scattering factor at one point (raycaster.py:253-258)."""
    f = _light_factor(buffer, np.asarray(sample_p, dtype=np.float64)[None, :], "shell", mode, shell_kernel=kernel,
                      ambient_floor=ambient_floor)
    return f[0, 1:].astype(np.float64)


def shade_cone(sample_p, buffer, kernel, eye=None, ambient_floor: float = 0.0, mode: str = "linear") -> np.ndarray:
    """Cone scattering factor at one point (raycaster.py:303-309)."""
    f = _light_factor(buffer, np.asarray(sample_p, dtype=np.float64)[None, :], "cone", mode, cone_kernel=kernel,
                      eye=eye, ambient_floor=ambient_floor)
    return f[0, 1:].astype(np.float64)
