"""K1 alone on config 3 (or --config N): sparse build for the cone march, and
full build; CUDA events over 20 launches after 3 warm-ups."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2008_06134_b200 import _native as N
    from paper_2008_06134_b200.frame import FrameRenderer
    from paper_2008_06134_b200.lightbuffer import build_into
    args = sys.argv[1:]
    cfg_id = int(args[args.index("--config") + 1]) if "--config" in args else 3
    cfg = bench.CONFIGS[cfg_id]
    dev = torch.device("cuda", 0)
    tf, cam, spec, settings = bench.scene_objects(cfg, cfg["mode"])
    dvol, _ = bench.device_volume_for(cfg, dev)
    fr = FrameRenderer(dvol.widened(), tf, cam, spec, settings, device=dev)
    s = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(20):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 20

    sparse = timed(fr.build)
    full = timed(lambda: build_into(fr.dvol, fr.alpha, fr.cam, fr.spec, fr.offsets, fr.quads, fr.comp))
    import hashlib
    fr.quads.zero_()
    build_into(fr.dvol, fr.alpha, fr.cam, fr.spec, fr.offsets, fr.quads, fr.comp)
    torch.cuda.synchronize()
    digest = hashlib.sha256(fr.quads.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"lib": os.path.basename(N.LIB_PATH), "config": cfg_id, "k1_sparse_ms": sparse,
                      "k1_full_ms": full, "quads_sha": digest}))


if __name__ == "__main__":
    main()
