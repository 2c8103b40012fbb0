"""Host time of each step of the public build + render calls (config 3 cone),
microseconds per call over many iterations (GPU work drained in between)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2008_06134_b200 as sb  # noqa: E402
from paper_2008_06134_b200 import device as D, lightbuffer as LB  # noqa: E402


def per_call(fn, n=2000):
    for _ in range(20):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    cfg = bench.CONFIGS[3]
    tf, cam, spec, settings = bench.scene_objects(cfg, "cone")
    v = bench.host_volume(cfg)
    dev = torch.device("cuda", 0)
    dvol = D.device_volume(v, dev)
    alpha = D.device_const(D.resolved_lut(tf, spec.spacing)[:, 3], dev)
    offsets = D.device_const(spec.plane_offsets, dev)
    quads = torch.empty((spec.n_slices, cam.resolution[1], cam.resolution[0], 4), device=dev)
    reach = LB.default_reach(cam, spec, float(dvol.voxel_size.max()))
    out = {
        "check_frame": per_call(lambda: LB.check_frame(cam, spec)),
        "require_cuda": per_call(lambda: D._require_cuda(None)),
        "device_volume": per_call(lambda: D.device_volume(v, dev)),
        "resolved_lut+device_const": per_call(lambda: D.device_const(D.resolved_lut(tf, spec.spacing)[:, 3], dev)),
        "device_const(offsets)": per_call(lambda: D.device_const(spec.plane_offsets, dev)),
        "torch.empty(quads)": per_call(lambda: torch.empty((spec.n_slices, cam.resolution[1], cam.resolution[0], 4), device=dev)),
        "default_reach": per_call(lambda: LB.default_reach(cam, spec, float(dvol.voxel_size.max()))),
        "build_params": per_call(lambda: D.build_params(dvol, cam, spec, alpha, offsets, quads, 0.0, 0, cam.resolution[1], reach)),
        "current_stream_handle": per_call(D.current_stream_handle),
    }
    torch.cuda.synchronize()
    out["build_attenuation_buffer(total, async)"] = per_call(lambda: sb.build_attenuation_buffer(v, tf, cam, spec), 200)
    torch.cuda.synchronize()
    buf = sb.build_attenuation_buffer(v, tf, cam, spec)
    host = torch.empty((1024, 1024, 4), pin_memory=True)
    out["render_device(host out, async)"] = per_call(lambda: sb.render_device(v, tf, settings, buf, out=host), 100)
    torch.cuda.synchronize()
    print(json.dumps({k: round(x, 2) for k, x in out.items()}))


if __name__ == "__main__" and "--uploads" not in sys.argv:
    main()


def uploads():
    """Host time of the public build call with and without the per-step
    constant uploads (device value cache dropped before each call)."""
    cfg = bench.CONFIGS[3]
    tf, cam, spec, settings = bench.scene_objects(cfg, "cone")
    v = bench.host_volume(cfg)
    dev = torch.device("cuda", 0)
    out = {}
    for name, drop in (("cached", False), ("upload", True), ("cached2", False), ("upload2", True)):
        def call():
            if drop:
                D.drop_frame_constants()
            sb.build_attenuation_buffer(v, tf, cam, spec)
        out[name] = per_call(call, 300)
        torch.cuda.synchronize()
    out["f64_tensor(4 KB)"] = per_call(lambda: D.f64_tensor(spec.plane_offsets, dev))
    a = spec.plane_offsets
    out["pageable .to(non_blocking)"] = per_call(lambda: torch.from_numpy(a).to(dev, non_blocking=True))
    out["pin_memory only"] = per_call(lambda: torch.from_numpy(a).pin_memory())
    torch.cuda.synchronize()
    print(json.dumps({k: round(x, 2) for k, x in out.items()}))


if __name__ == "__main__" and "--uploads" in sys.argv:
    uploads()
