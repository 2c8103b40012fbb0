"""Bounds evidence without compute-sanitizer (closed on this GPU pool).

    python paper_2008_06134_b200/build.py -DSBRC_CHECKED=1 --out=$PWD/paper_2008_06134_b200/_sbrc_checked.so
    SBRC_LIB=$PWD/paper_2008_06134_b200/_sbrc_checked.so python scripts/checked_run.py

Runs scripts/sanitize_run.py's workload (every kernel, every mode, ray
groups, peer-raster stores, sparse/plain builds) plus config-2/3 frames, the
8 contiguous ranks of config 3 with frustum-culled builds, on the checked
library and prints the violation counters by kind; all must be 0. Built
with -DSBRC_BUILD_TMA=1 too, the TMA-staged K1's shared-memory box reads
are checked as well (kind "volume").
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

KINDS = ("volume", "quad_read", "quad_write", "image", "peer_image", "tile_table", "lut_index", "plane_offset")


def main():
    import torch
    from paper_2008_06134_b200 import _native as N
    counts = (C.c_uint * 8)()
    st = N.lib.sbrc_debug_violations(C.byref(counts), 1)
    if st != 0:
        raise SystemExit(f"library is not a checked build (status {st}); set SBRC_LIB to _sbrc_checked.so")
    import sanitize_run
    sanitize_run.main()
    import bench
    from paper_2008_06134_b200.frame import FrameRenderer
    for cfg_id in (2, 3):
        cfg = bench.CONFIGS[cfg_id]
        tf, cam, spec, settings = bench.scene_objects(cfg, cfg["mode"])
        dvol, _ = bench.device_volume_for(cfg, torch.device("cuda"))
        fr = FrameRenderer(dvol, tf, cam, spec, settings)
        fr.frame()
        fr.intensity  # full build too
    from paper_2008_06134_b200 import partition as PT
    cfg = bench.CONFIGS[3]
    tf, cam, spec, settings = bench.scene_objects(cfg, cfg["mode"])
    dvol, _ = bench.device_volume_for(cfg, torch.device("cuda"))
    ranges = PT.balanced_ranges(PT.row_costs_geometric(settings), 8)
    for r in range(8):  # contiguous bands, clipped K1 + row-range K2
        fr = FrameRenderer(dvol, tf, cam, spec, settings, build="frustum")
        fr.rank, fr.world = r, 8
        fr.set_ranges(ranges)
        fr.build()
        fr.march()
        del fr
    torch.cuda.synchronize()
    N.check(N.lib.sbrc_debug_violations(C.byref(counts), 0), "sbrc_debug_violations")
    out = dict(zip(KINDS, list(counts)))
    print(json.dumps({"lib": N.LIB_PATH, "violations": out, "clean": not any(counts)}))


if __name__ == "__main__":
    main()
