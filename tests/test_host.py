"""Host-side logic without a GPU: parameter types mirror the reference bit for
bit, the synthetic generators reproduce the reference arrays, the device
entry points refuse to run without CUDA (no CPU fallback), and the
multi-rank image assembly / sharded-build gather work over gloo."""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC, load_golden

HAVE_REF = os.path.isdir(REFERENCE_SRC)


def _ref():
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import slicecast
    return slicecast


@pytest.mark.skipif(not HAVE_REF, reason="reference not present")
@pytest.mark.parametrize("ld", [(0.3, -0.5, 0.8), (0, 1, 0), (0, -1, 1e-12), (0.41, 0.2, -0.7), (1, 1, 1)])
def test_light_frame_identical_to_reference(ld):
    sc = _ref()
    from paper_2008_06134_b200 import scene
    a = scene.LightCamera.fit(ld, (0.9, 0.8, 0.7), (40, 36))
    b = sc.LightCamera.fit(ld, (0.9, 0.8, 0.7), (40, 36))
    for f in ("light_dir", "light_color", "axis_u", "axis_v", "view_matrix", "proj_matrix"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.u_range == b.u_range and a.v_range == b.v_range and a.resolution == b.resolution
    sa, sb_ = scene.make_slice_stack(ld, 37), sc.make_slice_stack(ld, 37)
    assert np.array_equal(sa.plane_offsets, sb_.plane_offsets)
    assert (sa.d_min, sa.d_max, sa.spacing) == (sb_.d_min, sb_.d_max, sb_.spacing)


@pytest.mark.skipif(not HAVE_REF, reason="reference not present")
def test_tf_and_volume_identical_to_reference():
    sc = _ref()
    from slicecast import datasets as rd
    from paper_2008_06134_b200 import scene, datasets
    for name in ("linear", "soft-gray", "hot", "bone"):
        a, b = scene.preset(name), sc.preset(name)
        assert np.array_equal(a.lut, b.lut)
        for step in (1 / 64, 1 / 512, 0.013):
            assert np.array_equal(a.resolve(step), b.resolve(step))
    va, vb = datasets.make_sphere_blobs((20, 24, 16), seed=3), rd.make_sphere_blobs((20, 24, 16), seed=3)
    assert np.array_equal(va.data, vb.data) and np.array_equal(va.box_lo, vb.box_lo)
    pa, pb = datasets.make_perforated_block((24, 24, 24), seed=3), rd.make_perforated_block((24, 24, 24), seed=3)
    assert np.array_equal(pa.data, pb.data)
    sa, sb_ = datasets.make_slab((16, 16, 16), axis=1, lo=0.3, hi=0.5), rd.make_slab((16, 16, 16), axis=1, lo=0.3, hi=0.5)
    assert np.array_equal(sa.data, sb_.data)
    an = scene.VolumeDataset.from_array(va.data, spacing=(1.0, 1.2, 0.9))
    bn = sc.VolumeDataset.from_array(vb.data, spacing=(1.0, 1.2, 0.9))
    assert np.array_equal(an.box_lo, bn.box_lo) and np.array_equal(an.box_hi, bn.box_hi)
    assert np.array_equal(an.voxel_size, bn.voxel_size)


@pytest.mark.skipif(not HAVE_REF, reason="reference not present")
def test_camera_frame_identical_to_reference():
    """Ray basis on the host matches Camera.rays' intermediates (raycaster.py:55-60)."""
    sc = _ref()
    from paper_2008_06134_b200 import scene
    from oracle import slicecast_oracle as O
    cam = sc.Camera(position=(1.9, 1.3, -0.9), target=(0.5, 0.5, 0.5), fov_deg=50.0)
    fr = scene.camera_frame(cam, (23, 17))
    w, h = 23, 17
    xs = ((np.arange(w) + 0.5) / w * 2.0 - 1.0) * fr["tan_half"] * fr["aspect"]
    ys = (1.0 - (np.arange(h) + 0.5) / h * 2.0) * fr["tan_half"]
    d = fr["forward"] + xs[None, :, None] * fr["right"] + ys[:, None, None] * fr["up2"]
    d = d / np.linalg.norm(d, axis=-1, keepdims=True)
    assert np.array_equal(d, cam.rays((w, h)))


def test_config1_volume_regenerates_reference_bits():
    from paper_2008_06134_b200.datasets import sphere_blobs_field
    g = load_golden("config1")
    data = sphere_blobs_field((64, 64, 64), seed=7)
    assert hashlib.sha256(data.tobytes()).hexdigest() == str(g["volume_sha256"])


def test_raw_roundtrip_matches_load_raw():
    """u8/u16 quantisation + normalisation equals the reference's save_raw/load_raw."""
    from paper_2008_06134_b200 import datasets
    g = load_golden("block48_u8")
    blk = datasets.make_perforated_block((48, 48, 48), seed=3)
    assert np.array_equal(datasets.raw_roundtrip(blk, "u8").data, g["volume"])
    g16 = load_golden("aniso_u16")
    from paper_2008_06134_b200.scene import VolumeDataset
    bl = datasets.make_sphere_blobs((24, 28, 20), seed=5)
    bl = VolumeDataset.from_array(bl.data, spacing=(1.0, 1.2, 0.9))
    assert np.array_equal(datasets.raw_roundtrip(bl, "u16").data, g16["volume"])


def test_validation_mirrors_reference():
    from paper_2008_06134_b200 import scene
    cam = scene.Camera(position=(0.5, 0.5, -1.6), target=(0.5, 0.5, 0.5))
    light = scene.Light(direction=(0, 0, 1))
    for bad in (dict(step=0.0), dict(viewport=(0, 4)), dict(early_termination_alpha=0.0), dict(shading_mode="x")):
        with pytest.raises(ValueError):
            scene.RenderSettings(camera=cam, light=light, **bad)
    with pytest.raises(ValueError):
        scene.LightCamera.fit((0, 0, 1), resolution=(0, 8))
    with pytest.raises(ValueError):
        scene.make_slice_stack((0, 0, 1), 0)
    with pytest.raises(ValueError):
        scene.ShellKernel(radii=(0.2, 0.1), weights=(0.5, 0.5))
    with pytest.raises(ValueError):
        scene.ConeKernel(axis_samples=0)
    with pytest.raises(ValueError):
        scene.Camera(position=(1, 1, 1), target=(1, 1, 1))
    with pytest.raises(ValueError):
        scene.normalize((0, 0, 0))
    assert issubclass(scene.ConfigError, ValueError)


def test_check_frame_light_direction():
    """lightbuffer.check_frame (lightbuffer.py:155-156): a light camera and a
    slice stack of different light directions are refused."""
    from paper_2008_06134_b200 import scene
    from paper_2008_06134_b200.lightbuffer import check_frame
    cam = scene.LightCamera.fit((0.3, -0.5, 0.8), (1, 1, 1), (8, 8))
    check_frame(cam, scene.make_slice_stack((0.3, -0.5, 0.8), 4))
    check_frame(cam, scene.make_slice_stack((0.6, -1.0, 1.6), 4))  # normalised: the same direction
    with pytest.raises(ValueError):
        check_frame(cam, scene.make_slice_stack((0.3, -0.5, 0.81), 4))


def test_no_cpu_fallback():
    """Without CUDA the product path raises instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_2008_06134_b200 as sb
    v = sb.VolumeDataset.from_array(np.zeros((4, 4, 4), np.float32))
    cam = sb.LightCamera.fit((0, 0, 1), (1, 1, 1), (4, 4))
    with pytest.raises(RuntimeError, match="CUDA"):
        sb.build_attenuation_buffer(v, sb.preset("hot"), cam, sb.make_slice_stack((0, 0, 1), 4))


# ------------------------------------------------------------------ multi-rank (gloo)
def _worker(rank, world, port, h, w, br, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2008_06134_b200.frame import band_layout, all_gather_into, shard_rows
    import paper_2008_06134_b200._native as N
    # march partition: rank-local rows -> global rows exactly as the kernel maps them
    rows, perm = band_layout(h, br, world)
    chunk = torch.zeros((rows, w, 4))
    for lr in range(N.local_rows(h, br, rank, world)):
        band, r = divmod(lr, br)
        y = (rank + band * world) * br + r
        if y < h:
            chunk[lr] = torch.arange(w * 4, dtype=torch.float32).view(w, 4) + 1000.0 * y
    gathered = torch.empty((world * rows, w, 4))
    all_gather_into(gathered, chunk)
    image = gathered[torch.from_numpy(perm)]
    expect = torch.arange(w * 4, dtype=torch.float32).view(1, w, 4) + 1000.0 * torch.arange(h).view(h, 1, 1)
    ok_img = bool(torch.equal(image, expect))
    # sharded build: row shards of an [H][n][W] buffer gather into the full buffer
    n, hl, wl = 5, 13, 6
    b, e, hs = shard_rows(hl, world, rank)
    shard = torch.zeros((hs, n, wl))
    for y in range(b, e):
        shard[y - b] = torch.arange(n * wl, dtype=torch.float32).view(n, wl) + 100.0 * y
    store = torch.empty((world * hs, n, wl))
    all_gather_into(store, shard)
    inten = store[:hl].permute(1, 0, 2)
    want = torch.arange(n * wl, dtype=torch.float32).view(n, 1, wl) + 100.0 * torch.arange(hl).view(1, hl, 1)
    ok_buf = bool(torch.equal(inten, want))
    q.put((rank, ok_img, ok_buf))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,h,br", [(2, 30, 8), (3, 1031, 16)])
def test_multirank_assembly_gloo(world, h, br):
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, h, 7, br, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok_img and ok_buf for _, ok_img, ok_buf in res), res


def test_skip_clear_hint():
    """Leading zero-emission run of a LUT and the volume-minimum test that
    selects the skip kernels (a speed hint only)."""
    from paper_2008_06134_b200 import device
    from paper_2008_06134_b200.scene import TransferFunction, preset
    assert device.clear_entries(preset("hot").lut) == 1
    assert device.clear_entries(np.zeros((256, 4))) == 256
    lut = np.ones((256, 4))
    assert device.clear_entries(lut) == 0
    tf = TransferFunction([(0.0, (0, 0, 0, 0)), (0.5, (1, 1, 1, 0)), (1.0, (1, 1, 1, 1))])
    run = device.clear_entries(tf.resolve(1 / 256))  # premultiplied (transfer.py:78-82)
    assert 120 <= run <= 129

    class V:
        value_min = 0.0
    assert device.skip_clear_hint(V, preset("hot").lut)
    V.value_min = 0.001
    assert not device.skip_clear_hint(V, preset("hot").lut)   # no voxel reaches the run
    assert device.skip_clear_hint(V, tf.resolve(1 / 256))
    assert not device.skip_clear_hint(V, lut)


def test_tile_feedback_order():
    """schedule.TileFeedback: the measured order lists tiles by decreasing
    longest-ray sample count (stable for ties), is kept across frames of
    the same grid and reset when the grid changes (device-agnostic logic,
    run here on CPU tensors)."""
    import torch
    from paper_2008_06134_b200.schedule import TileFeedback
    fb = TileFeedback()
    init = torch.arange(6, dtype=torch.int32)
    order, steps = fb.prepare((3, 2, 16, 8), init)
    assert torch.equal(order, init) and int(steps.sum()) == 0
    steps.copy_(torch.tensor([5, 9, 0, 9, 2, 7], dtype=torch.int32))
    fb.update()
    assert fb.order.tolist() == [1, 3, 5, 0, 4, 2]
    order2, steps2 = fb.prepare((3, 2, 16, 8), init)
    assert order2 is fb.order and int(steps2.sum()) == 0          # same grid: order kept, costs zeroed
    order3, _ = fb.prepare((2, 2, 32, 8), torch.arange(4, dtype=torch.int32))
    assert order3.tolist() == [0, 1, 2, 3]                          # new grid: fresh initial order


def test_heavy_first_empty_first_order():
    """schedule.heavy_first: a permutation of the tiles by decreasing estimated
    cost; with ``empty_first`` (render() into page-locked host memory) the
    zero-cost tiles lead, in index order, and the rest keep the heavy-first
    order."""
    from paper_2008_06134_b200 import scene
    from paper_2008_06134_b200.schedule import heavy_first, tile_cost
    s = scene.RenderSettings(camera=scene.Camera(position=(0.5, 0.5, -1.6), target=(0.5, 0.5, 0.5), fov_deg=45.0),
                             light=scene.Light(direction=(0.3, -0.5, 0.8)), viewport=(96, 80), shading_mode="none")
    grid = (6, 10, 16, 8)
    cost = tile_cost(s, grid=grid).reshape(-1)
    assert (cost == 0).any() and (cost > 0).any()
    base = heavy_first(s, grid=grid)
    ef = heavy_first(s, grid=grid, empty_first=True)
    assert sorted(base.tolist()) == sorted(ef.tolist()) == list(range(60))
    assert np.all(np.diff(cost[base]) <= 0)
    n0 = int((cost == 0).sum())
    assert ef[:n0].tolist() == sorted(np.flatnonzero(cost == 0).tolist())
    assert ef[n0:].tolist() == [t for t in base.tolist() if cost[t] > 0]


@pytest.mark.parametrize("light,res,n", [((0.3, -0.5, 0.8), 48, 24), ((0.0, 0.0, 1.0), 16, 8), ((1.0, 1.0, 1.0), 33, 17)])
def test_covered_texel_slices_matches_brute_force(light, res, n):
    """bench.covered_texel_slices (the K1 algorithmic-byte count: an analytic
    slab count per texel line) matches the number of texel-slice points the
    oracle's build tests as inside the cube (lightbuffer.py:182-183) to 0.5%
    (points within rounding of a cube face may go either way)."""
    import sys
    from conftest import ROOT
    sys.path.insert(0, ROOT)
    import bench
    from paper_2008_06134_b200 import scene
    cam = scene.LightCamera.fit(light, (1, 1, 1), (res, res))
    spec = scene.make_slice_stack(light, n)
    w, h = cam.resolution
    (u0, u1), (v0, v1) = cam.u_range, cam.v_range
    ug, vg = np.meshgrid(u0 + (np.arange(w) + 0.5) / w * (u1 - u0), v0 + (np.arange(h) + 0.5) / h * (v1 - v0))
    plane = ug[..., None] * np.asarray(cam.axis_u) + vg[..., None] * np.asarray(cam.axis_v)
    count = 0
    for k in range(n):
        p = plane + float(spec.plane_offsets[k]) * np.asarray(spec.light_dir)
        count += int(np.all((p >= 0.0) & (p <= 1.0), axis=-1).sum())
    got = bench.covered_texel_slices(cam, spec)
    assert abs(got - count) <= 0.005 * count, (got, count)


def test_reference_arm_runs_without_the_product_package():
    """bench.py --impl reference (the driver's reference arm) on config 1: one
    JSON line from the numpy port on the host cores, exit 0, nothing of the
    product package (or its CUDA library) imported, the same config keys as
    the GPU arm, and an e2e entry with no device copies."""
    import json
    import subprocess
    from conftest import ROOT
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "1",
                          "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "frames/s"
    assert d["product_package_loaded"] is False
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert {"workload", "image", "n_slices", "slice_res", "shading_mode"} <= set(d["config"])
