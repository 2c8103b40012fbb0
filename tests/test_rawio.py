"""`.raw` + JSON descriptor datasets (volume.py:19-158, datasets.py:83-97) and
their streamed upload to HBM."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC


def _blobs(dims=(20, 16, 12), seed=3, spacing=(1.0, 1.0, 1.0)):
    from paper_2008_06134_b200.datasets import make_sphere_blobs
    from paper_2008_06134_b200.scene import VolumeDataset
    return VolumeDataset.from_array(make_sphere_blobs(dims, seed=seed).data, spacing=spacing)


@pytest.mark.parametrize("kind", ["u8", "u16", "f32"])
def test_save_load_round_trip(tmp_path, kind):
    from paper_2008_06134_b200 import rawio
    v = _blobs(spacing=(1.0, 1.25, 0.8))
    if kind == "f32":  # an un-normalised f32 file exercises the min-max branch
        v = type(v).from_array(v.data * 3.0 - 1.0, spacing=v.spacing)
    p = rawio.save_raw(v, tmp_path / "vol.raw", kind)
    meta = rawio.VolumeDescriptor.from_json(p.with_suffix(".json"))
    assert meta.dims == v.dims and meta.scalar_type == kind and meta.spacing == tuple(v.spacing)
    back = rawio.load_raw(p, meta)
    assert back.scalar_type == kind and back.data.dtype == np.float32
    assert np.allclose(back.box_lo, v.box_lo) and np.allclose(back.box_hi, v.box_hi)
    if kind == "f32":
        lo, hi = float(v.data.min()), float(v.data.max())
        assert np.array_equal(back.data, ((v.data - lo) / (hi - lo)).astype(np.float32))


def test_descriptor_errors(tmp_path):
    from paper_2008_06134_b200 import rawio
    from paper_2008_06134_b200.scene import DescriptorError
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"dims": [2, 2]}))
    with pytest.raises(DescriptorError):
        rawio.VolumeDescriptor.from_json(bad)
    bad.write_text(json.dumps({"scalar_type": "u8"}))
    with pytest.raises(DescriptorError):
        rawio.VolumeDescriptor.from_json(bad)
    raw = tmp_path / "v.raw"
    raw.write_bytes(b"\0" * 7)
    with pytest.raises(DescriptorError):
        rawio.load_raw(raw, rawio.VolumeDescriptor((2, 2, 2), "u8"))
    with pytest.raises(rawio.FormatError):
        rawio.load_raw(raw, rawio.VolumeDescriptor((2, 2, 2), "f16"))
    assert issubclass(rawio.FormatError, ValueError) and issubclass(DescriptorError, ValueError)


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not present")
@pytest.mark.parametrize("kind", ["u8", "u16", "f32"])
def test_load_raw_matches_reference(tmp_path, kind):
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    from slicecast import volume as rv
    from paper_2008_06134_b200 import rawio
    v = _blobs(spacing=(1.0, 1.25, 0.8))
    if kind == "f32":
        v = type(v).from_array(v.data * 3.0 - 1.0, spacing=v.spacing)
    p = rawio.save_raw(v, tmp_path / "vol.raw", kind)
    ours = rawio.load_raw(p, rawio.VolumeDescriptor.from_json(p.with_suffix(".json")))
    ref = rv.load_raw(p, rv.VolumeDescriptor.from_json(p.with_suffix(".json")))
    assert np.array_equal(ours.data, ref.data) and ours.value_range == ref.value_range
    assert np.array_equal(ours.box_lo, ref.box_lo) and np.array_equal(ours.box_hi, ref.box_hi)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["u8", "u16", "f32"])
def test_streamed_upload_matches_host_load(tmp_path, kind):
    """load_raw_device == load_raw on the host, bit for bit, and renders identically."""
    import torch
    import paper_2008_06134_b200 as sb
    from paper_2008_06134_b200 import rawio
    v = _blobs(dims=(40, 36, 30), spacing=(1.0, 1.1, 0.9))
    if kind == "f32":
        v = type(v).from_array(v.data * 3.0 - 1.0, spacing=v.spacing)
    p = rawio.save_raw(v, tmp_path / "vol.raw", kind)
    host = rawio.load_raw(p, rawio.VolumeDescriptor.from_json(p.with_suffix(".json")))
    dev = rawio.load_raw_device(p, chunk_bytes=4096, widen=False)  # many chunks through the double buffer
    assert np.array_equal(dev.box_lo, host.box_lo) and np.array_equal(dev.box_hi, host.box_hi)
    if kind == "f32":
        assert np.array_equal(dev.data.cpu().numpy(), host.data.reshape(-1))
    tf = sb.preset("hot")
    ld = (0.3, -0.5, 0.8)
    cam = sb.LightCamera.fit(ld, (1, 1, 1), (24, 24))
    spec = sb.make_slice_stack(ld, 16)
    a = sb.build_attenuation_buffer(host, tf, cam, spec)
    b = sb.build_attenuation_buffer(dev, tf, cam, spec)
    assert np.array_equal(a.intensity, b.intensity)
    s = sb.RenderSettings(camera=sb.Camera(position=(0.5, 0.5, -1.6), target=(0.5, 0.5, 0.5)),
                          light=sb.Light(direction=ld), viewport=(20, 20), step=1 / 64, shading_mode="cone")
    assert np.array_equal(sb.render(host, tf, s, a), sb.render(dev, tf, s, b))
    wide = rawio.load_raw_device(p, chunk_bytes=1 << 16)
    assert wide.voxel_type == 0 and np.array_equal(wide.data.cpu().numpy(), host.data.reshape(-1))
