"""A small workload that exercises every kernel, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_run.py

Config-1-sized scene (64^3 blobs, 32 slices at 128^2): K1 full, sparse and
plain-output builds; K2 in every shading mode and lookup at 128^2 (the
latency kernels with 4-lane ray groups and partial-mask shuffles) and at
256^2 (throughput kernels), with heavy-first tables and measured tile costs;
K2 of a 2-rank split storing into two peer rasters (the fused-assembly store
path, both "ranks" in this process); the point-wise light factor, GPU
shadow oracle, half-angle baseline and raw-volume normalisation.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import paper_2008_06134_b200 as sb
    from paper_2008_06134_b200 import scene
    from paper_2008_06134_b200.datasets import make_sphere_blobs, raw_roundtrip
    from paper_2008_06134_b200.device import device_volume, f64_tensor, pack_quads
    from paper_2008_06134_b200.lightbuffer import build_into, lookup_reach
    from paper_2008_06134_b200.schedule import TileFeedback
    from paper_2008_06134_b200.halfangle import render_half_angle_device

    v = make_sphere_blobs((64, 64, 64), seed=7)
    tf = sb.preset("hot")
    ld = (0.3, -0.5, 0.8)
    cam = sb.LightCamera.fit(ld, (1, 1, 1), (128, 128))
    spec = sb.make_slice_stack(ld, 32)
    dev = torch.device("cuda")
    dvol = device_volume(v, dev)
    alpha = f64_tensor(tf.resolve(spec.spacing)[:, 3], dev)
    offs = f64_tensor(spec.plane_offsets, dev)
    buf = sb.build_attenuation_buffer(v, tf, cam, spec)  # sparse
    plain = torch.empty((32, 128, 128), dtype=torch.float32, device=dev)
    build_into(dvol, alpha, cam, spec, offs, plain, 0.0, plain=True)
    pack_quads(plain)
    camera = sb.Camera(position=(0.5, 0.5, -1.6), target=(0.5, 0.5, 0.5))
    for vp in ((128, 128), (256, 256)):
        for mode in ("none", "sbrc_shadow", "shell", "cone", "phong", "extinction"):
            for lookup in (("linear", "nearest") if mode in ("sbrc_shadow", "cone") else ("linear",)):
                st = sb.RenderSettings(camera=camera, light=sb.Light(direction=ld), viewport=vp, step=1 / 128,
                                       shading_mode=mode, lookup_mode=lookup)
                sb.render_device(v, tf, st, buf if mode in ("sbrc_shadow", "shell", "cone") else None,
                                 count_samples=True, heavy_first=True, feedback=TileFeedback())
    # fused assembly: two "ranks" of a 2-way split storing into two full rasters
    st = sb.RenderSettings(camera=camera, light=sb.Light(direction=ld), viewport=(128, 128), step=1 / 128,
                           shading_mode="cone")
    rasters = [torch.zeros((128, 128, 4), dtype=torch.float32, device=dev) for _ in range(2)]
    for r in range(2):
        sb.render_device(v, tf, st, buf, rank=r, world=2, band_rows=8, peer_images=rasters)
    # u8 raw volume (fetch-time normalisation) and the normalisation kernel
    vb = raw_roundtrip(make_sphere_blobs((40, 40, 40), seed=3), "u8")
    from paper_2008_06134_b200.device import DeviceVolume
    draw = DeviceVolume.from_dataset(vb, dev, widen=False)
    draw.widened()
    sb.render_device(draw, tf, st, sb.build_attenuation_buffer(draw, tf, cam, spec))
    # point API, shadow oracle, half-angle
    pts = np.random.default_rng(0).uniform(0, 1, size=(500, 3))
    sb.lookup_light_scalar_many(buf, pts)
    sb.shade_cone(pts[0], buf, scene.ConeKernel(), eye=(0.5, 0.5, -1.6))
    sb.shadow_oracle_many(v, tf, pts, sb.Light(direction=ld), 1 / 64)
    render_half_angle_device(v, tf, st, 16, light_resolution=(64, 64))
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
