"""Single-GPU check of frame pipelining: serial (build; march) vs pipelined,
for the full frame (N=1) and for one rank's share at N=8 (rank 0 of 8)."""
import gc
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2008_06134_b200.frame import FramePipeline, FrameRenderer  # noqa: E402


class FakeRank(FrameRenderer):
    """FrameRenderer that marches rank r's bands of a `world`-way split (no collectives)."""

    def __init__(self, *a, rank=0, world=1, **k):
        super().__init__(*a, **k)
        self.rank, self.world = rank, world
        from paper_2008_06134_b200.frame import band_layout
        self.rows_local, _ = band_layout(self.height, self.band_rows, world)
        self.chunk = torch.zeros((self.rows_local, self.width, 4), dtype=torch.float32, device=self.dev)
        self._params.clear()

    def assemble(self):
        return self.chunk


def timed(fn, k=20):
    s = torch.cuda.current_stream()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(k):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


def main():
    cfg = bench.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
    dev = torch.device("cuda")
    tf, cam, spec, settings = bench.scene_objects(cfg, cfg["mode"])
    dvol, _ = bench.device_volume_for(cfg, dev)
    dvol = dvol.widened()
    out = {}
    for world in (1, 2, 4, 8):
        fr = FakeRank(dvol, tf, cam, spec, settings, device=dev, rank=0, world=world, feedback=world > 1)
        serial = timed(lambda: (fr.build(), fr.march(False)))
        ref = fr.chunk.clone()
        pipe = FramePipeline(fr)

        def step():
            pipe.step()
            pipe.drain()  # (per-frame drain keeps the timing honest: every build counted)
        piped_drain = timed(step)
        pipe2 = FramePipeline(FakeRank(dvol, tf, cam, spec, settings, device=dev, rank=0, world=world,
                                       feedback=world > 1))
        piped = timed(lambda: pipe2.step())
        same = bool(torch.equal(pipe2.fr.chunk, ref))
        out[world] = {"serial_ms": serial, "pipelined_ms": piped, "pipelined_drain_each_ms": piped_drain,
                      "identical": same}
        del fr, pipe, pipe2, ref
        gc.collect()
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
