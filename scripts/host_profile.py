"""cProfile of the public-API frame (build_attenuation_buffer + render, config 3):
where the host time of each call goes."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2008_06134_b200 as sb  # noqa: E402


def main():
    cfg = bench.CONFIGS[3]
    tf, cam, spec, settings = bench.scene_objects(cfg, "cone")
    host_vol = bench.host_volume(cfg)

    def step():
        buf = sb.build_attenuation_buffer(host_vol, tf, cam, spec)
        return sb.render(host_vol, tf, settings, buf)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        step()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(30)
    st.sort_stats("cumulative").print_stats(40)


if __name__ == "__main__":
    main()
