"""`.raw` volumes with a JSON sidecar descriptor, streamed into HBM.

Same file format, validation and exception types as the reference
(volume.py:19-58 descriptor, :125-158 load_raw; datasets.py:83-97 save_raw):
a tightly packed little-endian (nz, ny, nx) grid of u8, u16 or f32 next to
``{"dims": [nx, ny, nz], "scalar_type": ..., "spacing": [...]}``.

``load_raw_device`` reads the file in chunks through two pinned host buffers
and copies each chunk to the device asynchronously while the next is read.
u8/u16 cross the bus compact and are normalised once to float32 in HBM
(or kept raw with ``widen=False``; the kernels then normalise at fetch,
bit-identically); f32 is min-max normalised on the device with numpy's
float32 arithmetic (``sbrc_normalize_f32``). Nothing of the volume is kept
on the host.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .device import DeviceVolume, _require_cuda, current_stream_handle
from .scene import DescriptorError, VolumeDataset


class FormatError(ValueError):
    """Unsupported raw scalar encoding (volume.py:23-24)."""


_DTYPES = {"u8": np.dtype("<u1"), "u16": np.dtype("<u2"), "f32": np.dtype("<f4")}


@dataclass(frozen=True)
class VolumeDescriptor:
    """Sidecar metadata of a .raw file (volume.py:34-58)."""

    dims: tuple
    scalar_type: str
    spacing: tuple = (1.0, 1.0, 1.0)

    @classmethod
    def from_json(cls, path) -> "VolumeDescriptor":
        raw = json.loads(Path(path).read_text())
        try:
            dims = tuple(int(d) for d in raw["dims"])
            scalar_type = str(raw["scalar_type"])
        except (KeyError, TypeError, ValueError) as exc:
            raise DescriptorError(f"malformed descriptor {path}: {exc}") from exc
        spacing = tuple(float(s) for s in raw.get("spacing", (1.0, 1.0, 1.0)))
        if len(dims) != 3 or len(spacing) != 3:
            raise DescriptorError(f"descriptor {path}: dims and spacing must be 3-vectors")
        return cls(dims=dims, scalar_type=scalar_type, spacing=spacing)

    def to_json(self) -> str:
        return json.dumps({"dims": list(self.dims), "scalar_type": self.scalar_type, "spacing": list(self.spacing)})


def _checked(path, meta: VolumeDescriptor) -> tuple[np.dtype, int]:
    dtype = _DTYPES.get(meta.scalar_type)
    if dtype is None:
        raise FormatError(f"unsupported scalar_type {meta.scalar_type!r}")
    nx, ny, nz = meta.dims
    expected = nx * ny * nz * dtype.itemsize
    size = os.path.getsize(path)
    if size != expected:
        raise DescriptorError(f"{path}: file is {size} bytes, descriptor implies {expected}")
    return dtype, expected


def load_raw(path, meta: VolumeDescriptor) -> VolumeDataset:
    """Host load with the reference's normalisation (volume.py:125-158)."""
    _checked(path, meta)
    flat = np.frombuffer(Path(path).read_bytes(), dtype=_DTYPES[meta.scalar_type])
    nx, ny, nz = meta.dims
    ds = VolumeDataset.from_raw_array(flat.reshape(nz, ny, nx), spacing=meta.spacing)
    return ds


def save_raw(v: VolumeDataset, raw_path, scalar_type: str = "u8") -> Path:
    """Write v.data as .raw plus the JSON descriptor (datasets.py:83-97)."""
    raw_path = Path(raw_path)
    if scalar_type == "u8":
        payload = (np.clip(v.data, 0.0, 1.0) * 255.0 + 0.5).astype("<u1")
    elif scalar_type == "u16":
        payload = (np.clip(v.data, 0.0, 1.0) * 65535.0 + 0.5).astype("<u2")
    elif scalar_type == "f32":
        payload = v.data.astype("<f4")
    else:
        raise ValueError(f"unsupported scalar_type {scalar_type!r}")
    raw_path.write_bytes(payload.tobytes())
    raw_path.with_suffix(".json").write_text(VolumeDescriptor(v.dims, scalar_type, tuple(v.spacing)).to_json())
    return raw_path


def load_raw_device(path, meta: VolumeDescriptor | None = None, device=None,
                    chunk_bytes: int = 64 << 20, widen: bool = True) -> DeviceVolume:
    """Stream a .raw file into HBM (see module docstring). ``meta`` defaults to
    the sidecar ``<path>.json``; ``widen`` normalises u8/u16 to float32 once
    in HBM (DeviceVolume.widened)."""
    path = Path(path)
    meta = meta or VolumeDescriptor.from_json(path.with_suffix(".json"))
    dtype, total = _checked(path, meta)
    dev = _require_cuda(device)
    nx, ny, nz = meta.dims
    out = torch.empty(total, dtype=torch.uint8, device=dev)
    chunk = max(dtype.itemsize, chunk_bytes - chunk_bytes % dtype.itemsize)
    stage = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    done = [None, None]
    stream = torch.cuda.current_stream(dev)
    with open(path, "rb", buffering=0) as fh:
        off, i = 0, 0
        while off < total:
            buf = stage[i % 2]
            if done[i % 2] is not None:
                done[i % 2].synchronize()  # the copy that last used this buffer has finished
            n = fh.readinto(memoryview(buf.numpy())[: min(chunk, total - off)])
            if not n:
                raise DescriptorError(f"{path}: short read at byte {off}")
            out[off:off + n].copy_(buf[:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            done[i % 2] = ev
            off += n
            i += 1
    # unit-cube box fit from dims and spacing (volume.py:86-90)
    ext = np.asarray(meta.dims, dtype=np.float64) * np.asarray(meta.spacing, dtype=np.float64)
    frac = ext / ext.max()
    box_lo = (1.0 - frac) / 2.0
    box_hi = box_lo + frac
    if meta.scalar_type == "u8":
        dv = DeviceVolume(out, N.VOXEL_U8, meta.dims, box_lo, box_hi)
        return dv.widened() if widen else dv
    if meta.scalar_type == "u16":
        dv = DeviceVolume(out.view(torch.int16), N.VOXEL_U16, meta.dims, box_lo, box_hi)
        return dv.widened() if widen else dv
    data = out.view(torch.float32)
    lo, hi = (float(x) for x in torch.aminmax(data))
    if hi > lo:
        N.check(N.lib.sbrc_normalize_f32(data.data_ptr(), data.numel(), lo, float(np.float32(hi - lo)),
                                         current_stream_handle()), "sbrc_normalize_f32")
    else:
        data.zero_()
    return DeviceVolume(data, N.VOXEL_F32, meta.dims, box_lo, box_hi)
