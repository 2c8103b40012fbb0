"""Single-GPU emulation of the contiguous partition with frustum-culled builds
(partition.py): for N = 1, 2, 4, 8 ranks of config 3, every rank's share is
run on this GPU one after the other — its clipped K1, its march, serial and
with the next frame's build overlapping the march — after two calibration
frames that re-cut the bands by the measured tile costs. Each rank's rows are
compared bit for bit with the single-GPU frame. Prints one JSON line.

    python scripts/frustum_check.py [config]
"""
import gc
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2008_06134_b200 import partition as PT  # noqa: E402
from paper_2008_06134_b200.frame import FramePipeline, FrameRenderer  # noqa: E402


def timed(fn, k=20):
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(k):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def rank_renderer(dvol, scene, world, rank, ranges, build="frustum"):
    tf, cam, spec, settings = scene
    fr = FrameRenderer(dvol, tf, cam, spec, settings, device=dvol.data.device, build=build,
                       partition="contiguous", feedback=True)
    fr.rank, fr.world = rank, world
    fr.set_ranges(ranges)
    fr.assemble = lambda: fr.chunk  # no collectives in the emulation: the rank's rows stay in its chunk
    return fr


def main():
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cfg = bench.CONFIGS[cfg_id]
    dev = torch.device("cuda")
    scene = bench.scene_objects(cfg, cfg["mode"])
    tf, cam, spec, settings = scene
    dvol, _ = bench.device_volume_for(cfg, dev)
    dvol = dvol.widened()
    ref_fr = FrameRenderer(dvol, tf, cam, spec, settings, device=dev)
    ref = ref_fr.frame().clone()
    full_build = timed(lambda: ref_fr.build())
    del ref_fr
    out = {"config": cfg_id, "full_build_ms": full_build}
    for world in (1, 2, 4, 8):
        shape = PT.row_costs_geometric(settings)
        ranges = PT.balanced_ranges(shape, world)
        history = []
        kernels = [0] * world
        best = None
        for _ in range(10 if world > 1 else 0):  # FrameRenderer.calibrate's search, ranks one after the other
            times = []
            for r in range(world):
                fr = rank_renderer(dvol, scene, world, r, ranges)
                kernels[r] = fr.choose_march_kernel()
                times.append(timed(lambda: (fr.build(), fr.march(False)), k=5))
                del fr
                gc.collect()
            history.append({"ranges": ranges, "max_ms": max(times), "times": times, "kernels": list(kernels)})
            if best is None or max(times) < best["max_ms"]:
                best = history[-1]
            nxt = PT.damped_ranges(best["ranges"], PT.balanced_ranges(
                PT.calibrated_profile(shape, best["ranges"], best["times"]), world), settings.viewport[1])
            if nxt == ranges:
                break
            ranges = nxt
        if best is not None:  # the best cut seen, with the kernels each rank chose for it
            ranges, kernels = best["ranges"], best["kernels"]
        ranks = []
        same = True
        for r in range(world):
            fr = rank_renderer(dvol, scene, world, r, ranges)
            fr.march_kernel = kernels[r]
            b, n = fr.row_range
            fr.build()
            fr.march(False)
            same &= bool(torch.equal(fr.chunk[:n], ref[b:b + n]))
            t_build = timed(fr.build)
            t_march = timed(lambda: fr.march(False))
            t_serial = timed(lambda: (fr.build(), fr.march(False)))
            pipe = FramePipeline(fr)
            t_pipe = timed(lambda: pipe.step())
            pipe.drain()
            torch.cuda.synchronize()
            pipe_hi = FramePipeline(fr, build_after_march=True)  # next build launched after the march (A/B)
            t_pipe_hi = timed(lambda: pipe_hi.step())
            pipe_hi.drain()
            torch.cuda.synchronize()
            del pipe_hi
            same &= bool(torch.equal(fr.chunk[:n], ref[b:b + n]))
            ranks.append({"rows": [b, n], "march_kernel": kernels[r], "build_ms": t_build, "march_ms": t_march,
                          "serial_ms": t_serial, "pipelined_ms": t_pipe, "pipelined_build_after_ms": t_pipe_hi})
            del pipe, fr
            gc.collect()
            torch.cuda.empty_cache()
        out[world] = {"ranges": ranges, "identical": same, "calibration": history,
                      "max_build_ms": max(x["build_ms"] for x in ranks),
                      "max_march_ms": max(x["march_ms"] for x in ranks),
                      "max_serial_ms": max(x["serial_ms"] for x in ranks),
                      "max_pipelined_ms": max(x["pipelined_ms"] for x in ranks),
                      "max_pipelined_build_after_ms": max(x["pipelined_build_after_ms"] for x in ranks), "ranks": ranks}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
