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


if __name__ == "__main__" and not {"--uploads", "--lines", "--ring"} & set(sys.argv):
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


def lines():
    """Per-line host time of build_attenuation_buffer (its body restated with timers)."""
    import numpy as np
    from paper_2008_06134_b200 import _native as N
    cfg = bench.CONFIGS[3]
    tf, cam, spec, settings = bench.scene_objects(cfg, "cone")
    v = bench.host_volume(cfg)
    dev0 = torch.device("cuda", 0)
    acc = {}
    pc = time.perf_counter

    def tick(name, t):
        acc[name] = acc.get(name, 0.0) + (pc() - t)
        return pc()

    n_it = 300
    for it in range(n_it + 20):
        if it == 20:
            acc.clear()
            torch.cuda.synchronize()
        D.drop_frame_constants()
        t = pc()
        LB.check_frame(cam, spec); t = tick("check_frame", t)
        dev = D._require_cuda(None); t = tick("require_cuda", t)
        w, h, n = int(cam.resolution[0]), int(cam.resolution[1]), int(spec.n_slices)
        dvol = D.device_volume(v, dev); t = tick("device_volume", t)
        lut = D.resolved_lut(tf, spec.spacing)[:, 3]; t = tick("resolved_lut", t)
        alpha, offsets = D.device_consts((lut, spec.plane_offsets), dev); t = tick("device_consts(upload)", t)
        quads = torch.empty((n, h, w, 4), dtype=torch.float32, device=dev); t = tick("torch.empty", t)
        reach = LB.default_reach(cam, spec, float(dvol.voxel_size.max())); t = tick("default_reach", t)
        p = D.build_params(dvol, cam, spec, alpha, offsets, quads, 0.0, 0, h, reach); t = tick("build_params", t)
        sh = D.current_stream_handle(); t = tick("stream_handle", t)
        st = N.lib.sbrc_build(p, sh); t = tick("sbrc_build (launch)", t)
        buf = LB.AttenuationBuffer(camera=cam, spec=spec, quads=quads, sparse=reach, rebuild=lambda: None)
        t = tick("AttenuationBuffer", t)
        del buf, quads
        t = tick("free", t)
        if "--sync" in sys.argv:  # as in the e2e frame: the host waits for the GPU every iteration
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    print(json.dumps({k: round(x / n_it * 1e6, 2) for k, x in acc.items()}))


if __name__ == "__main__" and "--lines" in sys.argv:
    lines()


def ring_parts():
    """Host time of the pieces of one staging-ring upload (synchronous loop)."""
    import numpy as np
    dev = torch.device("cuda", 0)
    a = np.random.default_rng(0).random(512)
    buf = torch.empty(1 << 20, dtype=torch.uint8, pin_memory=True)
    host = buf.numpy()
    acc = {}
    pc = time.perf_counter

    def tick(name, t):
        acc[name] = acc.get(name, 0.0) + (pc() - t)
        return pc()
    n_it = 500
    for it in range(n_it + 20):
        if it == 20:
            acc.clear()
        t = pc()
        host[0:4096] = a.reshape(-1).view(np.uint8); t = tick("memcpy to pinned", t)
        src = buf[0:4096].view(torch.float64).view(a.shape); t = tick("pinned view", t)
        dst = torch.empty(a.shape, dtype=torch.float64, device=dev); t = tick("torch.empty(cuda)", t)
        dst.copy_(src, non_blocking=True); t = tick("copy_ async", t)
        ev = torch.cuda.Event(); t = tick("Event()", t)
        ev.record(torch.cuda.current_stream(dst.device)); t = tick("record", t)
        key = a.tobytes(); t = tick("tobytes key", t)
        flat = np.concatenate([a, a[:256]]); t = tick("concatenate", t)
        torch.cuda.synchronize(); t = tick("sync", t)
    print(json.dumps({k: round(x / n_it * 1e6, 2) for k, x in acc.items()}))


if __name__ == "__main__" and "--ring" in sys.argv:
    ring_parts()
