"""Host logic of the contiguous partition and the frustum-culled build
(partition.py): balanced cuts, the eye-plane half-spaces, the gather
permutation, and the collective re-cut over gloo (world 2 and 3)."""

from __future__ import annotations

import itertools
import os
import random

import numpy as np
import pytest


def _opt_max(g, world):
    """Brute-force min-max contiguous cut of group costs g into world parts."""
    best = None
    for cut in itertools.combinations(range(1, len(g)), world - 1):
        edges = (0,) + cut + (len(g),)
        m = max(sum(g[edges[i]:edges[i + 1]]) for i in range(world))
        best = m if best is None else min(best, m)
    return best


@pytest.mark.parametrize("seed", range(6))
def test_balanced_ranges_optimal(seed):
    from paper_2008_06134_b200 import partition as PT
    rng = np.random.default_rng(seed)
    groups = int(rng.integers(4, 11))
    costs = np.repeat(rng.random(groups) * (rng.random(groups) > 0.3), 8)  # some empty groups
    h = 8 * groups - int(rng.integers(0, 8))  # ragged last group
    costs = costs[:h]
    for world in range(1, min(groups, 5) + 1):
        r = PT.balanced_ranges(costs, world)
        assert len(r) == world and r[0][0] == 0 and sum(n for _, n in r) == h
        assert all(n >= 1 for _, n in r) and all(b % 8 == 0 for b, _ in r)
        assert all(r[i + 1][0] == r[i][0] + r[i][1] for i in range(world - 1))
        g = [float(costs[i:i + 8].sum()) for i in range(0, h, 8)]
        got = max(float(costs[b:b + n].sum()) for b, n in r)
        assert got <= _opt_max(g, world) * (1 + 1e-6) + 1e-9, (world, r)


def test_balanced_ranges_errors():
    from paper_2008_06134_b200 import partition as PT
    with pytest.raises(ValueError):
        PT.balanced_ranges(np.ones(16), 3)  # 2 groups of 8 rows for 3 ranks
    assert PT.balanced_ranges(np.zeros(64), 8) == [(8 * i, 8) for i in range(8)]


def _settings(pos=(0.5, 0.5, -1.6), target=(0.5, 0.5, 0.5), fov=45.0, viewport=(96, 80)):
    from paper_2008_06134_b200 import scene
    return scene.RenderSettings(camera=scene.Camera(position=pos, target=target, fov_deg=fov),
                                light=scene.Light(direction=(0.3, -0.5, 0.8)), viewport=viewport,
                                shading_mode="cone")


@pytest.mark.parametrize("pos,target,fov", [((0.5, 0.5, -1.6), (0.5, 0.5, 0.5), 45.0),
                                            ((1.7, 1.2, 0.3), (0.4, 0.5, 0.6), 60.0),
                                            ((0.45, 0.55, 0.4), (0.6, 0.4, 1.0), 70.0)])
def test_frustum_clip_contains_band_rays(pos, target, fov):
    """Every sample of the band's rays (Camera.rays, raycaster.py:53-68, any
    t > 0) satisfies both half-spaces; samples of rows two or more rows
    outside the band violate one; points within ``reach`` of a band sample
    satisfy the widened half-spaces."""
    from oracle import slicecast_oracle as O
    from paper_2008_06134_b200 import partition as PT
    s = _settings(pos, target, fov)
    cam = s.camera
    dirs = O.camera_rays(np.asarray(cam.position, float), np.asarray(cam.target, float),
                         np.asarray(cam.up, float), cam.fov_deg, s.viewport)
    eye = np.asarray(cam.position, float)
    rng = np.random.default_rng(1)
    r0, r1 = 24, 40
    planes = np.array(PT.frustum_clip(s, r0, r1, 0.0))
    t = rng.random((dirs.shape[0], dirs.shape[1], 1)) * 3.0 + 1e-3
    pts = eye + t * dirs
    val = pts @ planes[:, :3].T + planes[:, 3]  # (H, W, 2)
    inside = val.min(axis=-1)
    assert (inside[r0:r1] >= -1e-12).all()
    assert (inside[:r0 - 1] < 0).all() and (inside[r1 + 1:] < 0).all()
    reach = 0.01
    wide = np.array(PT.frustum_clip(s, r0, r1, reach))
    jitter = rng.normal(size=pts[r0:r1].shape)
    jitter *= reach * rng.random(pts[r0:r1].shape[:2] + (1,)) / np.linalg.norm(jitter, axis=-1, keepdims=True)
    near = pts[r0:r1] + jitter
    assert ((near @ wide[:, :3].T + wide[:, 3]).min(axis=-1) >= 0).all()


def test_calibrated_profile_and_damped_ranges():
    """A band's profile integrates to its measured time; damped re-cuts move
    boundaries halfway, stay aligned and non-empty, and converge when times
    follow the profile."""
    from paper_2008_06134_b200 import partition as PT
    shape = np.exp(-((np.arange(160) - 90.0) / 30.0) ** 2)
    ranges = [(0, 40), (40, 40), (80, 40), (120, 40)]
    prof = PT.calibrated_profile(shape, ranges, [1.0, 2.0, 3.0, 4.0])
    assert np.allclose([prof[b:b + n].sum() for b, n in ranges], [1.0, 2.0, 3.0, 4.0])
    d = PT.damped_ranges(ranges, [(0, 8), (8, 8), (16, 8), (24, 136)], 160)
    assert d == [(0, 24), (24, 24), (48, 24), (72, 88)]
    truth = shape + 0.05 * shape.mean()
    for _ in range(12):
        times = [truth[b:b + n].sum() for b, n in ranges]
        ranges = PT.damped_ranges(ranges, PT.balanced_ranges(PT.calibrated_profile(shape, ranges, times), 4), 160)
    times = [truth[b:b + n].sum() for b, n in ranges]
    assert max(times) <= 1.35 * (sum(times) / 4)


def test_row_permutation_and_measured_costs():
    from paper_2008_06134_b200 import partition as PT
    ranges = [(0, 16), (16, 8), (24, 13)]
    perm = PT.row_permutation(ranges, 37, 16)
    stack = np.full((3 * 16,), -1)
    for r, (b, n) in enumerate(ranges):
        stack[r * 16:r * 16 + n] = np.arange(b, b + n)
    assert (stack[perm] == np.arange(37)).all()
    steps = np.array([[3, 5], [0, 2]], dtype=np.int32).reshape(-1)  # 2 x 2 tiles of 8 rows
    prof = PT.row_costs_measured(steps, (2, 2, 16, 8), 16, 40)
    assert (prof[:16] == 0).all() and np.allclose(prof[16:24], 1.0) and np.allclose(prof[24:32], 0.25)
    assert (prof[32:] == 0).all()


def _recut_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2008_06134_b200 import partition as PT
    h = 96
    true_cost = np.exp(-((np.arange(h) - 50.0) / 15.0) ** 2)
    ranges = PT.balanced_ranges(np.ones(h), world)  # first cut: uniform guess
    b, n = ranges[rank]
    # this rank "measures" its own rows only (FrameRenderer.rebalance's profile)
    prof = np.zeros(h)
    prof[b:b + n] = true_cost[b:b + n]
    t = torch.from_numpy(prof)
    dist.all_reduce(t)
    new = PT.balanced_ranges(t.numpy(), world)
    q.put((rank, new, PT.balanced_ranges(true_cost, world)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_recut_collective_gloo(world):
    """Every rank measures only its own band; one all-reduce gives all ranks
    the same full profile and so the same new cut (the one of the true costs)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_recut_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    cuts = {tuple(map(tuple, new)) for _, new, _ in res}
    assert len(cuts) == 1
    assert list(cuts)[0] == tuple(map(tuple, res[0][2]))


def _bcast_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2008_06134_b200 import _native as N
    from paper_2008_06134_b200.device import DeviceVolume, broadcast_volume
    dims = (6, 5, 4)
    src = None
    if rank == 0:
        t = (torch.arange(4 * 5 * 6, dtype=torch.int32) * 517 % 65536).to(torch.int16).view(4, 5, 6)
        src = DeviceVolume(t, N.VOXEL_U16, dims, np.zeros(3), np.ones(3))
    got = broadcast_volume(src, dims, N.VOXEL_U16, np.zeros(3), np.ones(3), "cpu")
    want = (torch.arange(4 * 5 * 6, dtype=torch.int32) * 517 % 65536).to(torch.int16).view(4, 5, 6)
    q.put((rank, bool(torch.equal(got.data, want)), got.voxel_type, got.dims))
    dist.destroy_process_group()


def test_broadcast_volume_gloo():
    """device.broadcast_volume: every rank ends with rank 0's voxels, type and dims."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_bcast_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok and vt == 2 and dims == (6, 5, 4) for _, ok, vt, dims in res), res
