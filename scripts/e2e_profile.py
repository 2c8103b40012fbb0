"""Where the end-to-end (numpy in / numpy out) frame time goes, config 3:
host time of each public call, GPU-idle gaps, and the image read-back."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2008_06134_b200 as sb  # noqa: E402
from paper_2008_06134_b200.device import to_host  # noqa: E402


def main():
    cfg = bench.CONFIGS[3]
    dev = torch.device("cuda")
    tf, cam, spec, settings = bench.scene_objects(cfg, "cone")
    host_vol = bench.host_volume(cfg)
    for _ in range(3):
        buf = sb.build_attenuation_buffer(host_vol, tf, cam, spec)
        img = sb.render(host_vol, tf, settings, buf)
    torch.cuda.synchronize()
    n = 20
    t_build = t_render_launch = t_d2h = 0.0
    t0 = time.perf_counter()
    for _ in range(n):
        a = time.perf_counter()
        buf = sb.build_attenuation_buffer(host_vol, tf, cam, spec)
        b = time.perf_counter()
        out = sb.render_device(host_vol, tf, settings, buf)
        c = time.perf_counter()
        img = to_host(out)
        d = time.perf_counter()
        t_build += b - a
        t_render_launch += c - b
        t_d2h += d - c
    total = (time.perf_counter() - t0) / n
    # pure D2H of a 16 MiB image from a resident tensor
    x = torch.empty((1024, 1024, 4), device=dev)
    torch.cuda.synchronize()
    e = time.perf_counter()
    for _ in range(n):
        to_host(x)
    d2h = (time.perf_counter() - e) / n
    print(json.dumps({"frame_ms": total * 1e3, "build_call_ms": t_build / n * 1e3,
                      "render_launch_call_ms": t_render_launch / n * 1e3,
                      "to_host_incl_wait_ms": t_d2h / n * 1e3, "pure_d2h_16MiB_ms": d2h * 1e3}))


if __name__ == "__main__":
    main()
