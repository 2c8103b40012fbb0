"""Host-side parameter types mirroring the reference package's public API.

These are the objects a caller of ``slicecast`` builds before calling the hot
path: the volume, transfer function, light camera, slice stack, eye camera,
light, render settings and scattering kernels. Field names, defaults,
validation and exception types follow the reference so that code written
against ``slicecast`` runs unchanged, and the shims in ``lightbuffer.py`` /
``raycaster.py`` also accept the reference's own objects (duck typing).

All setup arithmetic is float64 numpy, evaluated the way the reference
evaluates it (the device kernels consume these numbers bit for bit):

- geometry: ``normalize`` / ``plane_basis`` / cube vertices — geometry.py:12-43
- ``VolumeDataset`` and its unit-cube box fit — volume.py:61-122
- ``TransferFunction`` LUT and ``resolve(step)`` — transfer.py:33-84, presets :103-126
- ``LightCamera.fit`` — lightbuffer.py:37-86
- ``SliceStackSpec`` / ``make_slice_stack`` — slicing.py:22-64
- ``Camera``, ``Light``, ``ShellKernel``, ``ConeKernel``, ``RenderSettings`` —
  raycaster.py:37-150
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


class ConfigError(ValueError):
    """Inconsistent or incomplete scene/render configuration (errors.py:4-5)."""


class DescriptorError(ValueError):
    """Volume metadata inconsistent with its voxels (volume.py:19-20)."""


# ----------------------------------------------------------------- geometry
def _corner(i: int) -> tuple[int, int, int]:
    return (i & 1, (i >> 1) & 1, (i >> 2) & 1)


#: The 8 unit-cube corners; corner i = (bit0, bit1, bit2) (geometry.py:12-14).
CUBE_CORNERS = np.array([_corner(i) for i in range(8)], dtype=np.float64)


def normalize(vec) -> np.ndarray:
    """v / |v| in float64; a zero vector is a ValueError (geometry.py:23-28)."""
    arr = np.asarray(vec, dtype=np.float64)
    length = float(np.linalg.norm(arr))
    if length == 0.0:
        raise ValueError("cannot normalize a zero vector")
    return arr / length


def plane_basis(direction) -> tuple[np.ndarray, np.ndarray]:
    """Orthonormal (u, v) perpendicular to ``direction`` (geometry.py:31-43).

    Up hint +y, or +z when the direction is within 1e-9 of parallel to +y.
    """
    w = normalize(direction)
    hint = np.array([0.0, 1.0, 0.0])
    if abs(float(np.dot(hint, w))) > 1.0 - 1e-9:
        hint = np.array([0.0, 0.0, 1.0])
    u = normalize(np.cross(hint, w))
    return u, normalize(np.cross(w, u))


# ------------------------------------------------------------------- volume
@dataclass
class VolumeDataset:
    """Normalised scalar grid in the unit cube (volume.py:61-122).

    ``data`` is (nz, ny, nx) float32 in [0, 1]; voxel (x, y, z) is flat index
    x + nx*(y + ny*z). ``box_lo``/``box_hi`` fit the physical extent into the
    cube with the longest axis spanning [0, 1].
    """

    dims: tuple[int, int, int]
    spacing: tuple[float, float, float]
    scalar_type: str
    data: np.ndarray
    value_range: tuple[float, float]
    box_lo: np.ndarray = field(default=None)  # type: ignore[assignment]
    box_hi: np.ndarray = field(default=None)  # type: ignore[assignment]

    def __post_init__(self):
        nx, ny, nz = self.dims
        if min(self.dims) < 2:
            raise DescriptorError(f"dims must all be >= 2, got {self.dims}")
        if tuple(self.data.shape) != (nz, ny, nx):
            raise DescriptorError(f"data shape {self.data.shape} does not match dims {self.dims}")
        if self.box_lo is None:
            ext = np.asarray(self.dims, dtype=np.float64) * np.asarray(self.spacing, dtype=np.float64)
            frac = ext / ext.max()
            self.box_lo = (1.0 - frac) / 2.0
            self.box_hi = self.box_lo + frac

    @classmethod
    def from_array(cls, values, spacing=(1.0, 1.0, 1.0), scalar_type: str = "f32") -> "VolumeDataset":
        arr = np.asarray(values, dtype=np.float32)
        nz, ny, nx = arr.shape
        return cls(dims=(nx, ny, nz), spacing=spacing, scalar_type=scalar_type, data=arr,
                   value_range=(float(arr.min()), float(arr.max())))

    @classmethod
    def from_raw_array(cls, raw: np.ndarray, spacing=(1.0, 1.0, 1.0)) -> "VolumeDataset":
        """Normalise a raw u8/u16/f32 (nz, ny, nx) grid as load_raw does (volume.py:141-151)."""
        raw = np.asarray(raw)
        flat = raw.reshape(-1)
        lo, hi = float(flat.min()), float(flat.max())
        if raw.dtype == np.uint8:
            kind, data = "u8", flat.astype(np.float32) / 255.0
        elif raw.dtype == np.uint16:
            kind, data = "u16", flat.astype(np.float32) / 65535.0
        elif raw.dtype == np.float32:
            kind = "f32"
            data = ((flat - lo) / (hi - lo)).astype(np.float32) if hi > lo else np.zeros(flat.shape, np.float32)
        else:
            raise ValueError(f"unsupported raw dtype {raw.dtype}")
        nz, ny, nx = raw.shape
        ds = cls(dims=(nx, ny, nz), spacing=tuple(spacing), scalar_type=kind,
                 data=data.reshape(raw.shape), value_range=(lo, hi))
        if kind in ("u8", "u16"):
            ds.raw = raw  # the stored integers: the device copy keeps these (1-2 B per voxel)
        return ds

    @property
    def voxel_size(self) -> np.ndarray:
        return (self.box_hi - self.box_lo) / np.array(self.dims, dtype=np.float64)


# --------------------------------------------------------- transfer function
LUT_SIZE = 256
OPACITY_REF_STEP = 1.0 / 256.0

PRESETS: dict[str, list] = {
    "linear": [(0.0, (0.0, 0.0, 0.0, 0.0)), (1.0, (1.0, 1.0, 1.0, 1.0))],
    "soft-gray": [(0.0, (0.0, 0.0, 0.0, 0.0)), (0.3, (0.4, 0.4, 0.4, 0.05)),
                  (1.0, (0.95, 0.95, 0.95, 0.6))],
    "hot": [(0.0, (0.0, 0.0, 0.0, 0.0)), (0.33, (0.8, 0.1, 0.0, 0.15)),
            (0.66, (1.0, 0.6, 0.0, 0.45)), (1.0, (1.0, 1.0, 0.9, 0.9))],
    "bone": [(0.0, (0.0, 0.0, 0.0, 0.0)), (0.35, (0.25, 0.25, 0.3, 0.02)),
             (0.6, (0.85, 0.8, 0.75, 0.35)), (1.0, (1.0, 1.0, 0.98, 0.95))],
}


class TransferFunction:
    """Piecewise-linear RGBA ramp sampled into a 256-entry LUT (transfer.py:33-84)."""

    def __init__(self, control_points):
        if len(control_points) < 2:
            raise ValueError("need at least two control points")
        xs = [float(x) for x, _ in control_points]
        if xs[0] != 0.0 or xs[-1] != 1.0:
            raise ValueError("control points must start at 0.0 and end at 1.0")
        if any(b <= a for a, b in zip(xs, xs[1:])):
            raise ValueError("control point scalars must be strictly increasing")
        colors = np.array([c for _, c in control_points], dtype=np.float64)
        if colors.shape[1] != 4 or colors.min() < 0.0 or colors.max() > 1.0:
            raise ValueError("rgba components must lie in [0,1]")
        self.control_points = [(x, tuple(map(float, c))) for x, c in control_points]
        grid = np.linspace(0.0, 1.0, LUT_SIZE)
        self.lut = np.stack([np.interp(grid, xs, colors[:, ch]) for ch in range(4)], axis=1)

    def resolve(self, step: float) -> np.ndarray:
        """Opacity corrected to ``step`` (a' = 1-(1-a)^(step/ref)), colours
        premultiplied by a' (transfer.py:76-84)."""
        return resolve_lut(self.lut, step)


def resolve_lut(lut: np.ndarray, step: float) -> np.ndarray:
    corrected = 1.0 - np.power(1.0 - lut[:, 3], step / OPACITY_REF_STEP)
    out = np.empty_like(lut)
    out[:, :3] = lut[:, :3] * corrected[:, None]
    out[:, 3] = corrected
    return out


def preset(name: str) -> TransferFunction:
    if name not in PRESETS:
        raise ValueError(f"unknown transfer-function preset {name!r}")
    return TransferFunction(PRESETS[name])


# ------------------------------------------------------- light-space framing
@dataclass(frozen=True)
class SliceStackSpec:
    """n bin-centred planes perpendicular to the light (slicing.py:22-33)."""

    light_dir: np.ndarray
    n_slices: int
    d_min: float
    d_max: float
    plane_offsets: np.ndarray

    @property
    def spacing(self) -> float:
        return (self.d_max - self.d_min) / self.n_slices


def make_slice_stack(light_dir, n_slices: int) -> SliceStackSpec:
    """Split [min, max] of L.corner into n bins, one plane per bin centre (slicing.py:52-64)."""
    if n_slices < 1:
        raise ValueError(f"n_slices must be >= 1, got {n_slices}")
    ld = normalize(light_dir)
    proj = CUBE_CORNERS @ ld
    lo, hi = float(proj.min()), float(proj.max())
    width = (hi - lo) / n_slices
    centres = lo + (np.arange(n_slices, dtype=np.float64) + 0.5) * width
    return SliceStackSpec(light_dir=ld, n_slices=n_slices, d_min=lo, d_max=hi, plane_offsets=centres)


def _ortho(l, r, b, t, n, f) -> np.ndarray:
    m = np.eye(4)
    m[0, 0], m[0, 3] = 2.0 / (r - l), -(r + l) / (r - l)
    m[1, 1], m[1, 3] = 2.0 / (t - b), -(t + b) / (t - b)
    m[2, 2], m[2, 3] = 2.0 / (f - n), -(f + n) / (f - n)
    return m


@dataclass(frozen=True)
class LightCamera:
    """Orthographic light view fitted to the cube footprint (lightbuffer.py:37-86)."""

    light_dir: np.ndarray
    light_color: np.ndarray
    resolution: tuple[int, int]
    axis_u: np.ndarray
    axis_v: np.ndarray
    u_range: tuple[float, float]
    v_range: tuple[float, float]
    view_matrix: np.ndarray
    proj_matrix: np.ndarray

    @classmethod
    def fit(cls, light_dir, light_color=(1.0, 1.0, 1.0), resolution=(256, 256)) -> "LightCamera":
        w, h = int(resolution[0]), int(resolution[1])
        if w < 1 or h < 1:
            raise ValueError(f"resolution must be positive, got {resolution}")
        ld = normalize(light_dir)
        au, av = plane_basis(ld)
        pu, pv, pd = CUBE_CORNERS @ au, CUBE_CORNERS @ av, CUBE_CORNERS @ ld
        view = np.eye(4)
        view[0, :3], view[1, :3], view[2, :3] = au, av, -ld
        proj = _ortho(pu.min(), pu.max(), pv.min(), pv.max(), -pd.max(), -pd.min())
        return cls(light_dir=ld, light_color=np.asarray(light_color, dtype=np.float64),
                   resolution=(w, h), axis_u=au, axis_v=av,
                   u_range=(float(pu.min()), float(pu.max())),
                   v_range=(float(pv.min()), float(pv.max())),
                   view_matrix=view, proj_matrix=proj)

    @property
    def shadow_matrix(self) -> np.ndarray:
        return self.proj_matrix @ self.view_matrix


# ----------------------------------------------------------- eye and shading
@dataclass(frozen=True)
class Camera:
    """Pinhole camera, one ray per pixel, row 0 at the top (raycaster.py:37-68)."""

    position: np.ndarray
    target: np.ndarray
    up: np.ndarray = field(default_factory=lambda: np.array([0.0, 1.0, 0.0]))
    fov_deg: float = 45.0

    def __post_init__(self):
        for name in ("position", "target", "up"):
            object.__setattr__(self, name, np.asarray(getattr(self, name), dtype=np.float64))
        if float(np.linalg.norm(self.target - self.position)) < 1e-12:
            raise ValueError("camera position and target coincide")


_FRAME_CACHE: dict = {}


def camera_frame(cam, viewport) -> dict:
    """The float64 quantities Camera.rays derives before the per-pixel work
    (raycaster.py:55-60), computed with the same numpy calls. Cached per
    camera/viewport: the numpy calls cost ~0.1 ms per frame on the host."""
    w, h = int(viewport[0]), int(viewport[1])
    key = (*(float(x) for x in cam.position), *(float(x) for x in cam.target), *(float(x) for x in cam.up),
           float(cam.fov_deg), w, h)
    fr = _FRAME_CACHE.get(key)
    if fr is None:
        forward = normalize(cam.target - cam.position)
        right = normalize(np.cross(forward, cam.up))
        up2 = np.cross(right, forward)
        for arr in (forward, right, up2):  # shared by every caller of this view: read-only
            arr.setflags(write=False)
        fr = dict(forward=forward, right=right, up2=up2,
                  tan_half=math.tan(math.radians(cam.fov_deg) / 2.0), aspect=w / h)
        if len(_FRAME_CACHE) > 256:
            _FRAME_CACHE.clear()
        _FRAME_CACHE[key] = fr
    return dict(fr)


@dataclass(frozen=True)
class Light:
    """Directional light; ``direction`` is the way light travels (raycaster.py:71-80)."""

    direction: np.ndarray
    color: np.ndarray = field(default_factory=lambda: np.ones(3))

    def __post_init__(self):
        object.__setattr__(self, "direction", normalize(self.direction))
        object.__setattr__(self, "color", np.asarray(self.color, dtype=np.float64))


@dataclass(frozen=True)
class PhongParams:
    ambient: float = 0.1
    diffuse: float = 0.7
    specular: float = 0.2
    shininess: float = 32.0


@dataclass(frozen=True)
class ShellKernel:
    """Concentric cuboid shells, six axis taps each (raycaster.py:91-109)."""

    radii: tuple
    weights: tuple

    def __post_init__(self):
        if any(b <= a for a, b in zip(self.radii, self.radii[1:])):
            raise ValueError("shell radii must be strictly increasing")
        if any(w < 0 for w in self.weights) or abs(sum(self.weights) - 1.0) > 1e-9:
            raise ValueError("shell weights must be non-negative and sum to 1")

    @classmethod
    def default(cls, voxel_size: float) -> "ShellKernel":
        h = voxel_size
        return cls(radii=(h, 2 * h, 3 * h), weights=(0.5, 0.3, 0.2))


@dataclass(frozen=True)
class ConeKernel:
    """Rings stepping toward the light; 2 steps x 4 angles by default (raycaster.py:112-124)."""

    axis_samples: int = 2
    angles: tuple = (0.0, math.pi / 2, math.pi, 3 * math.pi / 2)
    ring_radius_per_step: float = 0.5

    def __post_init__(self):
        if self.axis_samples < 1:
            raise ValueError("axis_samples must be >= 1")
        if self.ring_radius_per_step < 0:
            raise ValueError("ring radius growth must be >= 0")


BUFFER_MODES = ("sbrc_shadow", "shell", "cone")
SHADING_MODES = ("none", "phong") + BUFFER_MODES + ("extinction",)
#: every reference shading mode runs on the GPU
GPU_MODES = SHADING_MODES


@dataclass(frozen=True)
class RenderSettings:
    """Render parameters and their validation (raycaster.py:127-150)."""

    camera: Camera
    light: Light
    viewport: tuple = (512, 512)
    step: float = 1.0 / 256.0
    shading_mode: str = "none"
    early_termination_alpha: float = 0.99
    ambient_floor: float = 0.0
    shell_kernel: ShellKernel | None = None
    cone_kernel: ConeKernel | None = None
    phong: PhongParams = PhongParams()
    lookup_mode: str = "linear"
    threads: int = 1

    def __post_init__(self):
        if self.step <= 0:
            raise ValueError("step must be positive")
        if self.viewport[0] < 1 or self.viewport[1] < 1:
            raise ValueError("viewport dimensions must be >= 1")
        if not 0.0 < self.early_termination_alpha <= 1.0:
            raise ValueError("early_termination_alpha must be in (0, 1]")
        if self.shading_mode not in SHADING_MODES:
            raise ValueError(f"unknown shading mode {self.shading_mode!r}")
