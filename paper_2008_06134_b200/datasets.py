"""Synthetic input volumes of the benchmark configurations.

Same formulas and random streams as the reference generators
(datasets.py:24-70): cell-centred coordinates (i + 0.5)/n, gaussian blobs
from ``default_rng(seed)``, the perforated block with random bores, and the
u8/u16 quantisation of ``save_raw`` (datasets.py:83-89). The numpy versions
reproduce the reference arrays bit for bit (pinned by a sha256 in
tests/golden); ``sphere_blobs_device`` evaluates the same formula on the
GPU in float64 z-slabs for the 512^3 / 1024^3 benchmark volumes, which
would take tens of seconds and ~56 GiB of host memory in numpy.
"""

from __future__ import annotations

import numpy as np

from .scene import VolumeDataset


def _axes(dims):
    nx, ny, nz = dims
    return ((np.arange(nx) + 0.5) / nx, (np.arange(ny) + 0.5) / ny, (np.arange(nz) + 0.5) / nz)


def _blob_params(seed: int, n_blobs: int):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_blobs):
        centre = rng.uniform(0.2, 0.8, size=3)
        sigma = rng.uniform(0.08, 0.2)
        amp = rng.uniform(0.5, 1.0)
        out.append((centre, sigma, amp))
    return out


def sphere_blobs_field(dims=(64, 64, 64), seed: int = 0, n_blobs: int = 5) -> np.ndarray:
    """Clipped sum of gaussian blobs as float32 (nz, ny, nx) (datasets.py:31-42)."""
    x, y, z = _axes(dims)
    zz, yy, xx = np.meshgrid(z, y, x, indexing="ij")
    acc = np.zeros_like(xx)
    for centre, sigma, amp in _blob_params(seed, n_blobs):
        r2 = (xx - centre[0]) ** 2 + (yy - centre[1]) ** 2 + (zz - centre[2]) ** 2
        acc += amp * np.exp(-r2 / (2.0 * sigma * sigma))
    return np.clip(acc, 0.0, 1.0).astype(np.float32)


def make_sphere_blobs(dims=(64, 64, 64), seed: int = 0, n_blobs: int = 5) -> VolumeDataset:
    return VolumeDataset.from_array(sphere_blobs_field(dims, seed, n_blobs))


def make_perforated_block(dims=(64, 64, 64), seed: int = 0, n_holes: int = 6) -> VolumeDataset:
    """Solid 0.8 block with cylindrical bores (datasets.py:53-70)."""
    rng = np.random.default_rng(seed)
    x, y, z = _axes(dims)
    zz, yy, xx = np.meshgrid(z, y, x, indexing="ij")
    inside = (xx > 0.15) & (xx < 0.85) & (yy > 0.15) & (yy < 0.85) & (zz > 0.15) & (zz < 0.85)
    field = np.where(inside, 0.8, 0.0)
    coords = (xx, yy, zz)
    for _ in range(n_holes):
        axis = int(rng.integers(0, 3))
        a, b = [i for i in range(3) if i != axis]
        ca, cb = rng.uniform(0.25, 0.75, size=2)
        radius = rng.uniform(0.04, 0.1)
        field[(coords[a] - ca) ** 2 + (coords[b] - cb) ** 2 < radius * radius] = 0.0
    return VolumeDataset.from_array(field)


def make_slab(dims=(32, 32, 32), axis: int = 2, lo: float = 0.4, hi: float = 0.6, value: float = 1.0):
    """Constant slab along one axis (datasets.py:45-50)."""
    c = np.meshgrid(*reversed(_axes(dims)), indexing="ij")[2 - axis]
    return VolumeDataset.from_array(np.where((c >= lo) & (c <= hi), value, 0.0))


def quantize(data: np.ndarray, scalar_type: str) -> np.ndarray:
    """save_raw's encoding (datasets.py:88-89): (clip(v)*max + 0.5) truncated."""
    if scalar_type == "u8":
        return (np.clip(data, 0.0, 1.0) * 255.0 + 0.5).astype("<u1")
    if scalar_type == "u16":
        return (np.clip(data, 0.0, 1.0) * 65535.0 + 0.5).astype("<u2")
    raise ValueError(f"unsupported scalar_type {scalar_type!r}")


def raw_roundtrip(v: VolumeDataset, scalar_type: str) -> VolumeDataset:
    """save_raw + load_raw in memory: the CT-like integer dataset of config 2/4."""
    return VolumeDataset.from_raw_array(quantize(v.data, scalar_type), spacing=v.spacing)


def sphere_blobs_device(dims=(512, 512, 512), seed: int = 7, n_blobs: int = 5, device="cuda",
                        quantize_to: str | None = None, slab: int = 64):
    """The sphere-blob field evaluated on the GPU in float64 z-slabs.

    Returns a (nz, ny, nx) CUDA tensor: float32 normalised values, or the
    raw u16/u8 encoding when ``quantize_to`` is given (config 4)."""
    import torch

    nx, ny, nz = dims
    dev = torch.device(device)
    params = _blob_params(seed, n_blobs)
    xs = (torch.arange(nx, dtype=torch.float64, device=dev) + 0.5) / nx
    ys = (torch.arange(ny, dtype=torch.float64, device=dev) + 0.5) / ny
    if quantize_to is None:
        out = torch.empty((nz, ny, nx), dtype=torch.float32, device=dev)
    else:
        out = torch.empty((nz, ny, nx), dtype=torch.int16 if quantize_to == "u16" else torch.uint8, device=dev)
    for z0 in range(0, nz, slab):
        z1 = min(nz, z0 + slab)
        zs = (torch.arange(z0, z1, dtype=torch.float64, device=dev) + 0.5) / nz
        acc = torch.zeros((z1 - z0, ny, nx), dtype=torch.float64, device=dev)
        for centre, sigma, amp in params:
            r2 = ((xs - centre[0]) ** 2)[None, None, :] + ((ys - centre[1]) ** 2)[None, :, None] \
                + ((zs - centre[2]) ** 2)[:, None, None]
            acc += amp * torch.exp(-r2 / (2.0 * sigma * sigma))
        acc.clamp_(0.0, 1.0)
        if quantize_to is None:
            out[z0:z1] = acc.to(torch.float32)
        else:
            scale = 65535.0 if quantize_to == "u16" else 255.0
            q = (acc * scale + 0.5).floor()
            out[z0:z1] = q.to(torch.int32).to(out.dtype) if quantize_to == "u16" else q.to(torch.uint8)
    return out
