"""The real peer-memory path of the fused image assembly, on one GPU: two
processes (gloo for the host-side collectives) exchange CUDA-IPC handles of
their raster images, map each other's, and render one frame each through
FrameRenderer(assemble="p2p"), whose start-up self-check compares against
the gather path. No kernel waits on another process's kernel."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from conftest import load_golden, scene_from_golden
        from paper_2008_06134_b200.frame import FrameRenderer
        g = load_golden("blob32")
        v, tf, cam, spec, settings_for = scene_from_golden(g)
        fr = FrameRenderer(v, tf, cam, spec, settings_for("cone"), assemble="p2p")
        mode = fr.assemble_mode
        img = fr.frame().cpu().numpy()
        err = float(np.abs(img - g["image_cone_linear"]).max())
        # pipelined frames (next build overlapping this march) give the same image
        from paper_2008_06134_b200.frame import FramePipeline
        pipe = FramePipeline(fr)
        for _ in range(3):
            out = pipe.step()
        pipe.drain()
        err = max(err, float(np.abs(out.cpu().numpy() - g["image_cone_linear"]).max()))
        fr.close()
        q.put((rank, mode, err, None))
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, None, None, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_p2p_assembly_two_processes_one_gpu():
    import multiprocessing as mp
    import random
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(e is None for *_, e in res), res
    assert all(mode == "p2p" for _, mode, _, _ in res), res
    assert all(err <= 1e-4 for _, _, err, _ in res), res


def _worker_frames(rank, world, port, q, frames):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import time
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from conftest import load_golden, scene_from_golden
        import paper_2008_06134_b200 as sb
        from paper_2008_06134_b200 import scene
        from paper_2008_06134_b200.frame import FrameRenderer
        from oracle.scenes import orbit_light
        g = load_golden("blob32")
        v, tf, cam, spec, settings_for = scene_from_golden(g)
        st = settings_for("cone")
        lights = [orbit_light(360.0 * f / frames, 30.0) for f in range(frames)]
        frames_in = [(scene.LightCamera.fit(ld, (1, 1, 1), cam.resolution), scene.make_slice_stack(ld, spec.n_slices))
                     for ld in lights]
        expected = []  # single-process frames of the same lights
        for c, s in frames_in:
            expected.append(sb.render_device(v, tf, st, sb.build_attenuation_buffer(v, tf, c, s)).clone())
        fr = FrameRenderer(v, tf, cam, spec, st, assemble="p2p")
        prepared = [fr.prepare_light(c, s) for c, s in frames_in]
        bad = []
        for f in range(frames):
            fr.use_light(prepared[f])
            img = fr.frame()
            if rank == 1:
                time.sleep(0.05)  # slow consumer: rank 0 is already marching frame f+1
            if not torch.equal(img, expected[f]):
                bad.append(f)
        mode = fr.assemble_mode
        fr.close()
        q.put((rank, mode, bad, None))
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, None, None, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_p2p_assembly_every_frame_with_slow_consumer():
    """12 frames with a different (orbit) light each; rank 1 reads every frame
    late. The double-buffered rasters must give each rank exactly the
    single-process image of every frame."""
    import multiprocessing as mp
    import random
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_worker_frames, args=(r, 2, port, q, 12)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(e is None for *_, e in res), res
    assert all(mode == "p2p" for _, mode, _, _ in res), res
    assert all(bad == [] for _, _, bad, _ in res), res
