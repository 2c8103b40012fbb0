"""Time one rank's share of the config-3 march (rank 0 of `world`) on one GPU,
vs the full frame divided by `world`: the single-GPU view of strong-scaling
efficiency for the march (tail effects at small per-rank work)."""
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
    band = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    hf = {"hf": True, "nohf": False}.get(sys.argv[2]) if len(sys.argv) > 2 else None  # None: library default
    fb = len(sys.argv) > 3 and sys.argv[3] == "fb"  # measured (feedback) heavy-first order
    from paper_2008_06134_b200.schedule import TileFeedback
    out = {}
    for world in (1, 2, 4, 8):
        br = band if band > 0 else -(-(settings.viewport[1] // world) // 8) * 8  # 0: contiguous blocks
        for r in range(3):
            sb.render_device(dvol, tf, settings, buf, rank=0, world=world, band_rows=br, heavy_first=hf)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ranks = range(world)
        times = []
        for rank in ranks:  # every rank's share, one after the other
            feed = TileFeedback() if fb else None
            if fb:  # one frame to measure the tiles
                sb.render_device(dvol, tf, settings, buf, rank=rank, world=world, band_rows=br, heavy_first=hf,
                                 feedback=feed)
            e0.record()
            for _ in range(5):
                sb.render_device(dvol, tf, settings, buf, rank=rank, world=world, band_rows=br, heavy_first=hf,
                                 feedback=feed)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 5)
        out[world] = {"max_rank_ms": max(times), "mean_rank_ms": sum(times) / len(times), "band_rows": br}
    full = out[1]["max_rank_ms"]
    for w, d in out.items():
        d["efficiency"] = full / (w * d["max_rank_ms"])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
