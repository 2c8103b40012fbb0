"""Where the end-to-end frame time goes (config 3, public API, numpy in/out):
host time of build_attenuation_buffer and render per call, GPU time of the
frame (events around both), and the wall time per frame."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import paper_2008_06134_b200 as sb
    cfg = bench.CONFIGS[3]
    tf, cam, spec, settings = bench.scene_objects(cfg, "cone")
    host_vol = bench.host_volume(cfg)
    s = torch.cuda.current_stream()
    rows = []
    for i in range(40):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        w0 = time.perf_counter()
        e0.record(s)
        buf = sb.build_attenuation_buffer(host_vol, tf, cam, spec)
        e1.record(s)
        w1 = time.perf_counter()
        sb.render(host_vol, tf, settings, buf)
        e2.record(s)
        w2 = time.perf_counter()
        torch.cuda.synchronize()
        if i >= 10:
            rows.append((w1 - w0, w2 - w1, w2 - w0, e0.elapsed_time(e1), e1.elapsed_time(e2)))
    med = [statistics.median(r[i] for r in rows) for i in range(5)]
    print(json.dumps({"host_build_ms": med[0] * 1e3, "render_call_ms": med[1] * 1e3, "frame_wall_ms": med[2] * 1e3,
                      "gpu_build_span_ms": med[3], "gpu_render_span_ms": med[4]}))


if __name__ == "__main__":
    main()
