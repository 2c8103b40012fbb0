"""Sparse K1 writes (sbrc_build_params.write_sparse): the march never reads
a quad the sparse build skipped. Needs a B200.

The stack is pre-filled with NaN, built sparse for the march's lookup reach
(lightbuffer.lookup_reach), and every shading mode is rendered from it: the
image must equal, bit for bit, the image rendered from a fully written
stack (a NaN read anywhere would propagate into a pixel). Written quads
must equal the full build's.
"""

from __future__ import annotations

import sys

import numpy as np
import pytest

from conftest import GOLDEN_CASES, ROOT, load_golden, scene_from_golden

pytestmark = pytest.mark.gpu
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def sb():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    import paper_2008_06134_b200 as sb
    return sb


def _sparse_vs_full(sb, dvol, tf, cam, spec, settings, comp=0.0):
    import torch
    from paper_2008_06134_b200.device import f64_tensor
    from paper_2008_06134_b200.lightbuffer import AttenuationBuffer, build_into, lookup_reach
    dev = dvol.data.device
    alpha = f64_tensor(tf.resolve(spec.spacing)[:, 3], dev)
    offsets = f64_tensor(spec.plane_offsets, dev)
    n, h, w = int(spec.n_slices), int(cam.resolution[1]), int(cam.resolution[0])
    full = torch.empty((n, h, w, 4), dtype=torch.float32, device=dev)
    build_into(dvol, alpha, cam, spec, offsets, full, comp)
    reach = lookup_reach(settings, cam, spec, float(dvol.voxel_size.max()))
    sparse = torch.full((n, h, w, 4), float("nan"), dtype=torch.float32, device=dev)
    build_into(dvol, alpha, cam, spec, offsets, sparse, comp, sparse=reach)
    written = ~torch.isnan(sparse[..., 0])
    assert torch.equal(sparse[written], full[written])
    a = sb.render_device(dvol, tf, settings, AttenuationBuffer(cam, spec, comp, quads=full))
    b = sb.render_device(dvol, tf, settings, AttenuationBuffer(cam, spec, comp, quads=sparse, sparse=reach))
    torch.cuda.synchronize()
    assert not bool(torch.isnan(b).any())
    assert torch.equal(a, b)
    return float(written.float().mean())


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_sparse_build_golden_cases(sb, case):
    from paper_2008_06134_b200.device import device_volume
    g = load_golden(case)
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    dvol = device_volume(v)
    for mode, lookup in g["meta"]["modes"]:
        if mode in ("sbrc_shadow", "shell", "cone"):
            _sparse_vs_full(sb, dvol, tf, cam, spec, settings_for(mode, lookup), g["meta"]["comp"])


def test_sparse_build_config3_all_modes(sb):
    import torch
    import bench
    cfg = bench.CONFIGS[3]
    dvol, _ = bench.device_volume_for(cfg, torch.device("cuda"))
    fracs = {}
    for mode in ("cone", "shell", "sbrc_shadow"):
        tf, cam, spec, settings = bench.scene_objects(cfg, mode)
        fracs[mode] = _sparse_vs_full(sb, dvol, tf, cam, spec, settings)
    print(f"[sparse] config 3 fraction of quads written: {fracs}")
    assert fracs["cone"] < 0.6  # the build skips most of the stack


def test_sparse_build_orbit_light_large_buffer(sb):
    """A config-5 point with a moving light: 256 slices at 1024^2, azimuth 135."""
    import torch
    import bench
    from paper_2008_06134_b200 import scene
    cfg = bench.CONFIGS[5]
    dvol, _ = bench.device_volume_for(cfg, torch.device("cuda"))
    tf, _, _, settings = bench.scene_objects(cfg, "cone")
    ld = bench.orbit_light(135.0, 30.0)
    cam = scene.LightCamera.fit(ld, (1, 1, 1), (1024, 1024))
    spec = scene.make_slice_stack(ld, 256)
    _sparse_vs_full(sb, dvol, tf, cam, spec, settings)


def test_public_build_is_sparse_and_completes(sb):
    """build_attenuation_buffer builds sparse for the default kernels; render
    uses it as is, ``intensity`` completes it (golden stack, bit for bit)."""
    g = load_golden("blob32")
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    buf = sb.build_attenuation_buffer(v, tf, cam, spec)
    assert buf.sparse is not None
    img = sb.render(v, tf, settings_for("cone"), buf)
    assert buf.sparse is not None  # the cone march fits the default reach: no completion
    assert float(np.abs(img - g["image_cone_linear"]).max()) <= 1e-4
    assert np.array_equal(buf.intensity, g["intensity"])
    assert buf.sparse is None
