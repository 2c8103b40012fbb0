"""K2 time (CUDA events) with the image in HBM vs in page-locked host memory
(render()'s direct read-back), and the host time of the public calls,
config 3 cone."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2008_06134_b200 as sb  # noqa: E402


def main():
    cfg = bench.CONFIGS[3]
    tf, cam, spec, settings = bench.scene_objects(cfg, "cone")
    host_vol = bench.host_volume(cfg)
    buf = sb.build_attenuation_buffer(host_vol, tf, cam, spec)
    dev_img = torch.empty((1024, 1024, 4), device="cuda")
    host_img = torch.empty((1024, 1024, 4), pin_memory=True)
    out = {}
    from paper_2008_06134_b200 import device as D, schedule as S
    hf = S.heavy_first

    def order(empty_first):  # A/B of the host-image tile order (empty tiles first vs last)
        def patched(settings, band_rows=8, rank=0, world=1, grid=None, row_range=None, ef=False):
            return hf(settings, band_rows, rank, world, grid, row_range, empty_first and ef)
        S.heavy_first = patched
        D._ORDER_CACHE.clear()
    runs = (("hbm", dev_img, True), ("host_empty_last", host_img, False), ("host", host_img, True),
            ("hbm2", dev_img, True), ("host_empty_last2", host_img, False), ("host2", host_img, True))
    for name, img, ef in runs:
        order(ef)
        for _ in range(3):
            sb.render_device(host_vol, tf, settings, buf, out=img)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            sb.render_device(host_vol, tf, settings, buf, out=img)
        e1.record()
        torch.cuda.synchronize()
        out[name + "_march_ms"] = e0.elapsed_time(e1) / 20
    # host time of the calls (GPU busy, so launches are asynchronous)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        b = sb.build_attenuation_buffer(host_vol, tf, cam, spec)
    t1 = time.perf_counter()
    for _ in range(20):
        sb.render_device(host_vol, tf, settings, buf, out=host_img)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    out["build_call_host_ms"] = (t1 - t0) / 20 * 1e3
    out["render_call_host_ms"] = (t2 - t1) / 20 * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
