"""Render one frame of a config through FrameRenderer and print the sha256 of
the image (A/B builds must produce the same bits):
    SBRC_LIB=... python scripts/image_hash.py [config] [mode]"""
import hashlib
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
    cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    cfg = bench.CONFIGS[cfg_id]
    mode = sys.argv[2] if len(sys.argv) > 2 else cfg["mode"]
    tf, cam, spec, settings = bench.scene_objects(cfg, mode)
    dvol, _ = bench.device_volume_for(cfg, torch.device("cuda"))
    img = FrameRenderer(dvol.widened(), tf, cam, spec, settings).frame()
    torch.cuda.synchronize()
    print(json.dumps({"lib": os.path.basename(N.LIB_PATH), "config": cfg_id, "mode": mode,
                      "image_sha": hashlib.sha256(img.cpu().numpy().tobytes()).hexdigest()[:16]}))


if __name__ == "__main__":
    main()
