"""Full-frame parity on the GPU box: EVERY pixel of a config's GPU frame
against the oracle (numpy port of the reference), the oracle's march
parallelised over row bands on all host cores, reading the GPU-built
attenuation stack (itself checked bit-exact on sampled light rows here and
in every bench run). Test infrastructure, like the bench's CPU legs.

    python scripts/full_parity.py [config ...] [--mode M]    (default: 1 2 3; 5 = one orbit-light frame)

Prints one JSON line per (config, mode): max-abs, PSNR, pixels over 1e-3 /
1e-4, whether the image is bit-identical, executed samples GPU vs oracle.
"""
import json
import math
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from oracle import slicecast_oracle as O
    from paper_2008_06134_b200.frame import FrameRenderer
    args = [x for x in sys.argv[1:] if not x.startswith("--")]
    mode_arg = sys.argv[sys.argv.index("--mode") + 1] if "--mode" in sys.argv else None
    configs = [int(x) for x in args if x.isdigit()] or [1, 2, 3]
    workers = len(os.sched_getaffinity(0))
    dev = torch.device("cuda", 0)
    for cid in configs:
        cfg = bench.CONFIGS[cid]
        mode = mode_arg or cfg["mode"]
        tf, cam, spec, settings = bench.scene_objects(cfg, mode)
        if cid == 5:  # one moving-light frame of the sweep: orbit light az 135, el 30 (orbit.ts:28-35)
            from paper_2008_06134_b200 import scene
            ld = bench.orbit_light(135.0, 30.0)
            cam = scene.LightCamera.fit(ld, (1.0, 1.0, 1.0), (cfg["res"], cfg["res"]))
            spec = scene.make_slice_stack(ld, cfg["n"])
        dvol, _ = bench.device_volume_for(cfg, dev)
        dvol = dvol.widened()
        fr = FrameRenderer(dvol, tf, cam, spec, settings, device=dev)
        fr.reset_counter()
        img = fr.frame().cpu().numpy()
        torch.cuda.synchronize()
        gpu_samples = int(fr.counter.item())
        inten = fr.intensity.contiguous().cpu().numpy() if fr.needs_buffer else None
        # the oracle reads the same voxels (the device volume, float32)
        from paper_2008_06134_b200.scene import VolumeDataset
        host = VolumeDataset.from_array(dvol.data.cpu().numpy())
        rows_chk = np.arange(3, cfg["res"], max(1, cfg["res"] // 16))
        build_exact = None
        if inten is not None:
            want_rows = O.build_intensity(host, tf.lut, cam, spec, rows=rows_chk)
            build_exact = bool(np.array_equal(inten[:, rows_chk], want_rows))
        bench.set_cpu_context(host, tf, cam, spec, settings, inten)
        t0 = time.perf_counter()
        rows = np.arange(cfg["image"])
        cols = np.arange(cfg["image"])
        with mp.get_context("fork").Pool(workers) as pool:
            parts = pool.map(bench._cpu_march_part, [(r, cols) for r in np.array_split(rows, 4 * workers) if len(r)])
        cpu_s = time.perf_counter() - t0
        want = np.concatenate([im for _, _, im in parts], axis=0)
        oracle_samples = int(sum(n for _, n, _ in parts))
        d = np.abs(img.astype(np.float64) - want.astype(np.float64))
        mse = float((d ** 2).mean())
        print(json.dumps({
            "config": cid, "mode": mode, "pixels": int(img.shape[0] * img.shape[1]),
            "max_abs": float(d.max()), "psnr": float("inf") if mse == 0 else 10 * math.log10(1.0 / mse),
            "over_1e_3": int((d.max(axis=-1) > 1e-3).sum()), "over_1e_4": int((d.max(axis=-1) > 1e-4).sum()),
            "bit_identical": bool(np.array_equal(img, want)), "gpu_samples": gpu_samples,
            "oracle_samples": oracle_samples, "build_rows_checked": int(len(rows_chk)) if inten is not None else 0,
            "build_rows_bit_exact": build_exact, "oracle_cpu_s": cpu_s, "cpu_workers": workers}), flush=True)
        fr.close()
        del fr, dvol, host
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
