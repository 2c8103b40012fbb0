"""Critical path of the config-3 march: time thin rank shares (8 rows of the
image, world = 128) at several ranks — with ~2 warps per SM the kernel time
is close to its longest ray's latency — next to the full frame."""
import json
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2008_06134_b200 as sb  # noqa: E402


def main():
    cfg = bench.CONFIGS[3]
    dev = torch.device("cuda")
    tf, cam, spec, settings = bench.scene_objects(cfg, "cone")
    dvol, _ = bench.device_volume_for(cfg, dev)
    buf = sb.build_attenuation_buffer(dvol, tf, cam, spec)
    out = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for world, ranks in ((1, [0]), (8, [0, 4]), (32, [0, 16]), (128, [0, 32, 64])):
        for r in ranks:
            for _ in range(3):
                sb.render_device(dvol, tf, settings, buf, rank=r, world=world, band_rows=8)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                img, n = sb.render_device(dvol, tf, settings, buf, rank=r, world=world, band_rows=8, count_samples=True)
            e1.record()
            torch.cuda.synchronize()
            out[f"{world}/{r}"] = {"ms": e0.elapsed_time(e1) / 10, "samples": int(n.item()) // 10 * 10 // 10}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
