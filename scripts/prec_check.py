"""A/B a K2 precision variant against the exact library on one config-3 frame.

    SBRC_LIB=<variant .so> python scripts/prec_check.py TAG [--save REF.npy] [--ref REF.npy] [--mode cone]

Times the march (CUDA events, 20 launches after 3 warm-ups) and, with
``--ref``, compares the frame against the exact library's frame saved by an
earlier ``--save`` run: max |d|, count over 1e-3 / 1e-4, and the executed
sample count (equal when every early-termination decision matches).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2008_06134_b200.frame import FrameRenderer
    tag = sys.argv[1]
    args = sys.argv[2:]
    mode = args[args.index("--mode") + 1] if "--mode" in args else "cone"
    cfg_id = int(args[args.index("--config") + 1]) if "--config" in args else 3
    cfg = bench.CONFIGS[cfg_id]
    dev = torch.device("cuda", 0)
    tf, cam, spec, settings = bench.scene_objects(cfg, mode)
    dvol, _ = bench.device_volume_for(cfg, dev)
    fr = FrameRenderer(dvol.widened(), tf, cam, spec, settings, device=dev)
    fr.reset_counter()
    img = fr.frame()
    torch.cuda.synchronize()
    samples = int(fr.counter.item())
    s = torch.cuda.current_stream()
    for _ in range(3):
        fr.march(count_samples=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(20):
        fr.march(count_samples=False)
    e1.record(s)
    torch.cuda.synchronize()
    out = {"tag": tag, "mode": mode, "config": cfg_id, "march_ms": e0.elapsed_time(e1) / 20, "samples": samples}
    fr.reset_counter()
    fr.march()
    img = fr.assemble().cpu().numpy()
    if "--save" in args:
        p = args[args.index("--save") + 1]
        np.save(p, img)
        with open(p + ".json", "w") as f:
            json.dump({"samples": samples}, f)
    if "--ref" in args:
        p = args[args.index("--ref") + 1]
        ref = np.load(p)
        d = np.abs(img.astype(np.float64) - ref)
        out.update(max_abs=float(d.max()), over_1e3=int((d > 1e-3).sum()), over_1e4=int((d > 1e-4).sum()),
                   ref_samples=json.load(open(p + ".json"))["samples"])
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
