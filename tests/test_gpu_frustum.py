"""Contiguous partition + frustum-culled attenuation build (partition.py,
``FrameRenderer(build="frustum")``). Needs a B200.

Every rank builds only the texel-slices its own band of image rows can
read (K1 clipped by the band's two eye planes, ``sbrc_build_params.clip``)
and marches its rows (``sbrc_render_params.row_begin/row_count``). The
ranks are emulated one after the other on this GPU. Contract: each rank's
rows are bit-identical to the single-GPU frame, and the march never reads a
quad the clipped build skipped (the buffer is filled with NaN first: one
such read would poison a pixel).
"""

from __future__ import annotations

import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden, scene_from_golden

pytestmark = pytest.mark.gpu
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    return torch


def _rank(fr_cls, scene, world, rank, ranges, **kw):
    v, tf, cam, spec, settings = scene
    fr = fr_cls(v, tf, cam, spec, settings, build="frustum", **kw)
    fr.rank, fr.world = rank, world
    fr.set_ranges(ranges)
    return fr


def _check_ranks(torch, scene, world, ref, ranges=None, poison=True):
    from paper_2008_06134_b200 import partition as PT
    from paper_2008_06134_b200.frame import FrameRenderer
    settings = scene[4]
    if ranges is None:
        ranges = PT.balanced_ranges(PT.row_costs_geometric(settings), world)
    for r in range(world):
        fr = _rank(FrameRenderer, scene, world, r, ranges)
        assert len(fr.clip) == 2
        if poison:
            fr.quads.fill_(float("nan"))
        fr.build()
        fr.march()
        b, n = fr.row_range
        got = fr.chunk[:n]
        assert not bool(torch.isnan(got).any()), (world, r, "read a quad the clipped build skipped")
        assert torch.equal(got, ref[b:b + n]), (world, r, ranges)
    return ranges


@pytest.mark.parametrize("mode", ["cone", "shell", "sbrc_shadow"])
def test_frustum_ranks_identical_golden(torch, mode):
    """blob32 golden scene: 2, 3 and 4 contiguous ranks, each with its own
    clipped build, reassemble the single-GPU image bit for bit."""
    import paper_2008_06134_b200 as sb
    g = load_golden("blob32")
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    s = settings_for(mode)
    ref = sb.render_device(v, tf, s, sb.build_attenuation_buffer(v, tf, cam, spec))
    for world in (2, 3, 4):
        _check_ranks(torch, (v, tf, cam, spec, s), world, ref)


def test_frustum_clip_skips_work(torch):
    """The clipped build really writes less than the (sparse) full build: a
    16-row middle band leaves part of the stack unwritten (NaN), yet its rows
    match. (On this 32^3 scene the lookups' reach spans much of the stack;
    at config 3 a middle band of 8 builds ~40-65% of the texel-slices,
    scripts/frustum_check.py.)"""
    import paper_2008_06134_b200 as sb
    from paper_2008_06134_b200 import partition as PT
    from paper_2008_06134_b200.frame import FrameRenderer
    g = load_golden("blob32")
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    s = settings_for("cone")
    ref = sb.render_device(v, tf, s, sb.build_attenuation_buffer(v, tf, cam, spec))
    h = s.viewport[1]
    ranges = [(0, h // 2 - 8), (h // 2 - 8, 16), (h // 2 + 8, h // 2 - 8)]
    fr = _rank(FrameRenderer, (v, tf, cam, spec, s), 3, 1, ranges)
    fr.quads.fill_(float("nan"))
    fr.build()
    written = float((~torch.isnan(fr.quads[..., 0])).float().mean())
    fr.march()
    assert torch.equal(fr.chunk[:16], ref[h // 2 - 8:h // 2 + 8])
    full = FrameRenderer(v, tf, cam, spec, s)
    full.quads.fill_(float("nan"))
    full.build()
    written_full = float((~torch.isnan(full.quads[..., 0])).float().mean())
    print(f"[frustum] quads written: band {written:.3f} vs sparse full {written_full:.3f}")
    assert written < written_full


def test_frustum_eye_inside_and_edges(torch):
    """Eye inside the cube (samples on both sides of the eye plane) and
    one-group bands at the image edges."""
    import paper_2008_06134_b200 as sb
    from paper_2008_06134_b200 import scene
    g = load_golden("blob32")
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    base = settings_for("cone")
    s = scene.RenderSettings(camera=scene.Camera(position=(0.45, 0.55, 0.4), target=(0.6, 0.4, 1.0), fov_deg=70.0),
                             light=base.light, viewport=(48, 40), step=base.step, shading_mode="cone")
    ref = sb.render_device(v, tf, s, sb.build_attenuation_buffer(v, tf, cam, spec))
    _check_ranks(torch, (v, tf, cam, spec, s), 3, ref)
    _check_ranks(torch, (v, tf, cam, spec, s), 3, ref, ranges=[(0, 8), (8, 24), (32, 8)])


def test_frustum_rebalance_and_pipeline(torch):
    """A re-cut from measured per-rank times (partition.calibrated_profile +
    damped_ranges, FrameRenderer.rebalance's math) keeps the image, and so
    does the pipelined frame (next clipped build overlapping the march)."""
    import paper_2008_06134_b200 as sb
    from paper_2008_06134_b200 import partition as PT
    from paper_2008_06134_b200.frame import FramePipeline, FrameRenderer
    g = load_golden("config1")
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    s = settings_for("shell")
    ref = sb.render_device(v, tf, s, sb.build_attenuation_buffer(v, tf, cam, spec))
    world = 4
    shape = PT.row_costs_geometric(s)
    ranges = PT.balanced_ranges(shape, world)
    times = []
    for r in range(world):
        fr = _rank(FrameRenderer, (v, tf, cam, spec, s), world, r, ranges)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fr.build()
        fr.march()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    new = PT.damped_ranges(ranges, PT.balanced_ranges(PT.calibrated_profile(shape, ranges, times), world),
                           s.viewport[1])
    assert sum(n for _, n in new) == s.viewport[1] and all(n > 0 for _, n in new)
    for r in range(world):
        fr = _rank(FrameRenderer, (v, tf, cam, spec, s), world, r, new, feedback=True)
        fr.assemble = lambda fr=fr: fr.chunk
        pipe = FramePipeline(fr)
        for _ in range(3):
            pipe.step()
        pipe.drain()
        torch.cuda.synchronize()
        b, n = fr.row_range
        assert torch.equal(fr.chunk[:n], ref[b:b + n]), (r, new)


def test_frustum_config3_full_size(torch):
    """Config 3 (512^3 -> 1024^2, cone, 256 slices @512^2) cut for 8 ranks:
    an edge band and the two middle bands, bit-identical rows."""
    import bench
    from paper_2008_06134_b200 import partition as PT
    from paper_2008_06134_b200.frame import FrameRenderer
    cfg = bench.CONFIGS[3]
    tf, cam, spec, settings = bench.scene_objects(cfg, "cone")
    dvol, _ = bench.device_volume_for(cfg, torch.device("cuda"))
    ref = FrameRenderer(dvol, tf, cam, spec, settings).frame().clone()
    ranges = PT.balanced_ranges(PT.row_costs_geometric(settings), 8)
    for r in (0, 3, 4):
        fr = _rank(FrameRenderer, (dvol, tf, cam, spec, settings), 8, r, ranges)
        fr.quads.fill_(float("nan"))
        fr.build()
        fr.march()
        b, n = fr.row_range
        assert torch.equal(fr.chunk[:n], ref[b:b + n]), (r, ranges)
        del fr


@pytest.mark.parametrize("mode", ["cone", "shell", "sbrc_shadow"])
def test_forced_march_kernel_identical(torch, mode):
    """sbrc_render_params.march_kernel (throughput / latency K2, and the
    measured choice of FrameRenderer.choose_march_kernel) never changes the
    image."""
    import paper_2008_06134_b200 as sb
    from paper_2008_06134_b200.frame import FrameRenderer
    g = load_golden("config1")
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    s = settings_for(mode)
    ref = sb.render_device(v, tf, s, sb.build_attenuation_buffer(v, tf, cam, spec))
    fr = FrameRenderer(v, tf, cam, spec, s)
    for k in (1, 2, 0):
        fr.march_kernel = k
        fr._params.clear()
        assert torch.equal(fr.frame(), ref), k
    assert fr.choose_march_kernel() in (1, 2)
    assert torch.equal(fr.frame(), ref)
