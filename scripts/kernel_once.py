"""Launch the config-3 kernels a few times (for ncu captures): build x3, march x3.

    python scripts/kernel_once.py [--config 3] [--mode cone]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2008_06134_b200.frame import FrameRenderer
    args = sys.argv[1:]
    cfg_id = int(args[args.index("--config") + 1]) if "--config" in args else 3
    cfg = bench.CONFIGS[cfg_id]
    mode = args[args.index("--mode") + 1] if "--mode" in args else cfg["mode"]
    dev = torch.device("cuda", 0)
    tf, cam, spec, settings = bench.scene_objects(cfg, mode)
    dvol, _ = bench.device_volume_for(cfg, dev)
    fr = FrameRenderer(dvol.widened(), tf, cam, spec, settings, device=dev)
    for _ in range(3):
        fr.build()
    for _ in range(3):
        fr.march(count_samples=False)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
