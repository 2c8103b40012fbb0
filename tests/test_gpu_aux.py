"""The small native kernels around the path (no eager PyTorch on the
per-frame path): K0 widening, the measured heavy-first order, the NCCL
assembly's row permutation. Needs a B200."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    return torch


def test_widen_volume_every_value(torch):
    """sbrc_widen_volume equals numpy's float32 load_raw normalisation
    (volume.py:143-146) for every u8 and u16 value, ragged lengths included."""
    from paper_2008_06134_b200 import _native as N
    from paper_2008_06134_b200.device import current_stream_handle
    for vt, dt, scale in ((N.VOXEL_U8, np.uint8, 255.0), (N.VOXEL_U16, np.uint16, 65535.0)):
        vals = np.arange(np.iinfo(dt).max + 1, dtype=dt)
        for n in (len(vals), len(vals) - 3):
            host = vals[:n]
            src = torch.from_numpy(host.view(np.int8 if dt == np.uint8 else np.int16).copy()).cuda()
            out = torch.empty(n, dtype=torch.float32, device="cuda")
            N.check(N.lib.sbrc_widen_volume(src.data_ptr(), vt, n, out.data_ptr(), current_stream_handle()), "widen")
            want = host.astype(np.float32) / np.float32(scale)
            assert np.array_equal(out.cpu().numpy(), want), (vt, n)


def test_tile_order_matches_stable_argsort(torch):
    from paper_2008_06134_b200 import _native as N
    from paper_2008_06134_b200.device import current_stream_handle
    rng = np.random.default_rng(3)
    for n in (1, 7, 256, 257, 5000, 16384):
        steps = torch.from_numpy(rng.integers(0, 40, n).astype(np.int32)).cuda()  # many ties
        order = torch.full((n,), -1, dtype=torch.int32, device="cuda")
        N.check(N.lib.sbrc_tile_order(steps.data_ptr(), n, order.data_ptr(), current_stream_handle()), "order")
        want = torch.argsort(steps, descending=True, stable=True).to(torch.int32)
        assert torch.equal(order, want), n


def test_permute_rows_matches_index_select(torch):
    from paper_2008_06134_b200 import _native as N
    from paper_2008_06134_b200.device import current_stream_handle
    from paper_2008_06134_b200.frame import band_layout
    h, w = 1031, 37
    rows, perm = band_layout(h, 16, 3)
    src = torch.randn((3 * rows, w, 4), device="cuda")
    p = torch.from_numpy(perm).cuda()
    dst = torch.empty((h, w, 4), device="cuda")
    N.check(N.lib.sbrc_permute_rows(src.data_ptr(), p.data_ptr(), dst.data_ptr(), h, w, current_stream_handle()),
            "permute")
    assert torch.equal(dst, torch.index_select(src, 0, p))


@pytest.mark.parametrize("case", ["blob32", "block48_u8", "config1"])
def test_layer_pair_shadow_frames_identical(torch, case):
    """FrameRenderer stores the stack as layer pairs (quad_layout 1) for the
    one-lookup sbrc_shadow march; its frames equal the texel-quad path's bit
    for bit (render_device + build_attenuation_buffer), and its intensity
    view equals the reference's stack."""
    from conftest import load_golden, scene_from_golden
    import paper_2008_06134_b200 as sb
    from paper_2008_06134_b200.frame import FramePipeline, FrameRenderer
    g = load_golden(case)
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    s = settings_for("sbrc_shadow")
    ref = sb.render_device(v, tf, s, sb.build_attenuation_buffer(v, tf, cam, spec))
    fr = FrameRenderer(v, tf, cam, spec, s)
    assert fr.quads.shape[-1] == 2
    assert torch.equal(fr.frame(), ref)
    pipe = FramePipeline(fr)
    for _ in range(3):
        out = pipe.step()
    pipe.drain()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    assert np.array_equal(fr.intensity.cpu().numpy(), g["intensity"])


def test_pinned_staging_ring_wraps(torch):
    """device.f64_tensor's staging ring: uploads across several wrap-arounds
    (each lap waits for the previous lap's copies) all arrive intact, and
    device_consts views split one upload correctly."""
    from paper_2008_06134_b200 import device as D
    ring = D._PinnedRing(nbytes=64 * 1024)
    rng = np.random.default_rng(5)
    sent, fallbacks = [], 0
    for i in range(300):  # ~ 300 * 2-4 KiB = several laps of 64 KiB
        a = rng.random(int(rng.integers(1, 512)))
        t = ring.upload(a, "cuda")
        if t is None:  # previous lap still in flight: the caller falls back
            fallbacks += 1
            torch.cuda.synchronize()
            t = ring.upload(a, "cuda")
        sent.append((a, t))
    torch.cuda.synchronize()
    for a, t in sent:
        assert np.array_equal(t.cpu().numpy(), a)
    D.drop_frame_constants()
    x, y = rng.random(256), rng.random(37)
    tx, ty = D.device_consts((x, y), "cuda")
    assert np.array_equal(tx.cpu().numpy(), x) and np.array_equal(ty.cpu().numpy(), y)
    assert ty.data_ptr() == tx.data_ptr() + 256 * 8
