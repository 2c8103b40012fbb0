"""ORACLE — CPU restatement of the reference's scene setup. TEST INFRASTRUCTURE ONLY.

The inputs of the benchmark configurations built without the product
package, so that the reference arm of ``bench.py`` (``--impl reference``)
and the oracle checks never load the CUDA library. Plain objects carrying
the reference's attribute names (duck types for ``oracle.slicecast_oracle``):

- ``preset`` / ``TF``         transfer.py:33-51 (256-entry LUT of a piecewise-linear
                              ramp), presets transfer.py:103-126
- ``light_camera``            lightbuffer.py:56-81 (LightCamera.fit) with
                              geometry.py:23-43 (normalize, plane_basis)
- ``slice_stack``             slicing.py:52-64 (make_slice_stack)
- ``render_settings``         raycaster.py:37-150 (Camera, Light, RenderSettings defaults)
- ``blob_field``              datasets.py:31-42 (make_sphere_blobs), evaluated in
                              z-slabs (same per-voxel float64 formula)
- ``perforated_block``        datasets.py:53-70
- ``raw_roundtrip``           datasets.py:83-89 (save_raw u8/u16 encoding) +
                              volume.py:141-151 (load_raw normalisation)
- ``volume``                  volume.py:61-122 (VolumeDataset box fit)

Pinned: ``tests/test_oracle_golden.py`` checks these against the reference's
own objects stored in the golden fixtures (LUTs, light frames, slice stacks,
the config-1 volume hash).
"""

from __future__ import annotations

import math
from types import SimpleNamespace

import numpy as np

LUT_SIZE = 256

PRESETS = {
    "linear": [(0.0, (0.0, 0.0, 0.0, 0.0)), (1.0, (1.0, 1.0, 1.0, 1.0))],
    "soft-gray": [(0.0, (0.0, 0.0, 0.0, 0.0)), (0.3, (0.4, 0.4, 0.4, 0.05)), (1.0, (0.95, 0.95, 0.95, 0.6))],
    "hot": [(0.0, (0.0, 0.0, 0.0, 0.0)), (0.33, (0.8, 0.1, 0.0, 0.15)), (0.66, (1.0, 0.6, 0.0, 0.45)),
            (1.0, (1.0, 1.0, 0.9, 0.9))],
    "bone": [(0.0, (0.0, 0.0, 0.0, 0.0)), (0.35, (0.25, 0.25, 0.3, 0.02)), (0.6, (0.85, 0.8, 0.75, 0.35)),
             (1.0, (1.0, 1.0, 0.98, 0.95))],
}

_CORNERS = np.array([(i & 1, (i >> 1) & 1, (i >> 2) & 1) for i in range(8)], dtype=np.float64)


def _normalize(v) -> np.ndarray:
    a = np.asarray(v, dtype=np.float64)
    return a / float(np.linalg.norm(a))


def _plane_basis(direction):
    w = _normalize(direction)
    hint = np.array([0.0, 1.0, 0.0])
    if abs(float(np.dot(hint, w))) > 1.0 - 1e-9:
        hint = np.array([0.0, 0.0, 1.0])
    u = _normalize(np.cross(hint, w))
    return u, _normalize(np.cross(w, u))


def preset(name: str) -> SimpleNamespace:
    """A transfer function with the reference's ``lut`` (256, 4) float64."""
    pts = PRESETS[name]
    xs = [x for x, _ in pts]
    cols = np.array([c for _, c in pts], dtype=np.float64)
    grid = np.linspace(0.0, 1.0, LUT_SIZE)
    return SimpleNamespace(lut=np.stack([np.interp(grid, xs, cols[:, ch]) for ch in range(4)], axis=1),
                           control_points=pts)


def _ortho(l, r, b, t, n, f) -> np.ndarray:
    """lightbuffer.py:26-34."""
    m = np.eye(4)
    m[0, 0], m[0, 3] = 2.0 / (r - l), -(r + l) / (r - l)
    m[1, 1], m[1, 3] = 2.0 / (t - b), -(t + b) / (t - b)
    m[2, 2], m[2, 3] = 2.0 / (f - n), -(f + n) / (f - n)
    return m


def light_camera(light_dir, light_color=(1.0, 1.0, 1.0), resolution=(256, 256)) -> SimpleNamespace:
    ld = _normalize(light_dir)
    au, av = _plane_basis(ld)
    pu, pv, pd = _CORNERS @ au, _CORNERS @ av, _CORNERS @ ld
    view = np.eye(4)
    view[0, :3], view[1, :3], view[2, :3] = au, av, -ld
    proj = _ortho(pu.min(), pu.max(), pv.min(), pv.max(), -pd.max(), -pd.min())
    return SimpleNamespace(light_dir=ld, light_color=np.asarray(light_color, dtype=np.float64),
                           resolution=(int(resolution[0]), int(resolution[1])), axis_u=au, axis_v=av,
                           u_range=(float(pu.min()), float(pu.max())), v_range=(float(pv.min()), float(pv.max())),
                           view_matrix=view, proj_matrix=proj, shadow_matrix=proj @ view)


def slice_stack(light_dir, n_slices: int) -> SimpleNamespace:
    ld = _normalize(light_dir)
    proj = _CORNERS @ ld
    lo, hi = float(proj.min()), float(proj.max())
    width = (hi - lo) / n_slices
    return SimpleNamespace(light_dir=ld, n_slices=int(n_slices), d_min=lo, d_max=hi, spacing=width,
                           plane_offsets=lo + (np.arange(n_slices, dtype=np.float64) + 0.5) * width)


def render_settings(position, target, viewport, step, mode, light_dir, light_color=(1.0, 1.0, 1.0),
                    up=(0.0, 1.0, 0.0), fov_deg=45.0, et=0.99, floor=0.0, lookup="linear") -> SimpleNamespace:
    """RenderSettings with the default shell/cone kernels (None) and phong parameters."""
    camera = SimpleNamespace(position=np.asarray(position, np.float64), target=np.asarray(target, np.float64),
                             up=np.asarray(up, np.float64), fov_deg=float(fov_deg))
    light = SimpleNamespace(direction=_normalize(light_dir), color=np.asarray(light_color, np.float64))
    phong = SimpleNamespace(ambient=0.1, diffuse=0.7, specular=0.2, shininess=32.0)
    return SimpleNamespace(camera=camera, light=light, viewport=tuple(viewport), step=float(step),
                           shading_mode=mode, early_termination_alpha=float(et), ambient_floor=float(floor),
                           shell_kernel=None, cone_kernel=None, phong=phong, lookup_mode=lookup, threads=1)


def volume(data: np.ndarray, spacing=(1.0, 1.0, 1.0), scalar_type: str = "f32") -> SimpleNamespace:
    """VolumeDataset (volume.py:61-122): longest axis fitted to [0, 1], centred."""
    data = np.asarray(data, dtype=np.float32)
    nz, ny, nx = data.shape
    dims = (nx, ny, nz)
    ext = np.asarray(dims, dtype=np.float64) * np.asarray(spacing, dtype=np.float64)
    frac = ext / ext.max()
    lo = (1.0 - frac) / 2.0
    return SimpleNamespace(dims=dims, spacing=tuple(spacing), scalar_type=scalar_type, data=data,
                           box_lo=lo, box_hi=lo + frac, voxel_size=frac / np.asarray(dims, dtype=np.float64))


def _axes(n: int) -> np.ndarray:
    return (np.arange(n) + 0.5) / n


def blob_params(seed: int, n_blobs: int = 5):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_blobs):
        centre = rng.uniform(0.2, 0.8, size=3)
        sigma = rng.uniform(0.08, 0.2)
        amp = rng.uniform(0.5, 1.0)
        out.append((centre, sigma, amp))
    return out


def blob_field(d: int, seed: int, n_blobs: int = 5) -> np.ndarray:
    """make_sphere_blobs((d,)*3, seed) as float32 (d, d, d), in z-slabs of <= 2^24 voxels."""
    out = np.empty((d, d, d), dtype=np.float32)
    ax = _axes(d)
    params = blob_params(seed, n_blobs)
    step = max(1, min(d, (1 << 24) // (d * d)))
    for z0 in range(0, d, step):
        z1 = min(d, z0 + step)
        zz, yy, xx = np.meshgrid(ax[z0:z1], ax, ax, indexing="ij")
        acc = np.zeros_like(xx)
        for c, s, a in params:
            acc += a * np.exp(-((xx - c[0]) ** 2 + (yy - c[1]) ** 2 + (zz - c[2]) ** 2) / (2.0 * s * s))
        out[z0:z1] = np.clip(acc, 0.0, 1.0)
    return out


def perforated_block(d: int, seed: int, n_holes: int = 6) -> np.ndarray:
    rng = np.random.default_rng(seed)
    ax = _axes(d)
    zz, yy, xx = np.meshgrid(ax, ax, ax, indexing="ij")
    field = np.where((xx > 0.15) & (xx < 0.85) & (yy > 0.15) & (yy < 0.85) & (zz > 0.15) & (zz < 0.85), 0.8, 0.0)
    coords = (xx, yy, zz)
    for _ in range(n_holes):
        axis = int(rng.integers(0, 3))
        a, b = [i for i in range(3) if i != axis]
        ca, cb = rng.uniform(0.25, 0.75, size=2)
        radius = rng.uniform(0.04, 0.1)
        field[(coords[a] - ca) ** 2 + (coords[b] - cb) ** 2 < radius * radius] = 0.0
    return field.astype(np.float32)


def raw_roundtrip(data: np.ndarray, scalar_type: str) -> tuple[np.ndarray, np.ndarray]:
    """(raw integers, normalised float32): save_raw's encoding then load_raw's division."""
    scale, dt = (255.0, "<u1") if scalar_type == "u8" else (65535.0, "<u2")
    raw = (np.clip(data, 0.0, 1.0) * scale + 0.5).astype(dt)
    return raw, raw.astype(np.float32) / scale


def orbit_light(az_deg: float, el_deg: float):
    """frontend/src/orbit.ts:28-35: the direction the light travels."""
    el, az = math.radians(el_deg), math.radians(az_deg)
    return (-math.cos(el) * math.sin(az), -math.sin(el), math.cos(el) * math.cos(az))
