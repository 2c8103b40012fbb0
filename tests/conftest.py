"""Shared fixtures: golden-case loaders and the `gpu` marker.

`-m "not gpu"` runs here (no GPU): the oracle against the reference's golden
vectors, host-side logic, the C-ABI library's exports, and the multi-rank
assembly over gloo. `-m gpu` runs on a B200: the CUDA path against the
golden vectors and the oracle.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def load_golden(name: str) -> dict:
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)
    out = {k: z[k] for k in z.files}
    out["meta"] = json.loads(str(out["meta"]))
    return out


GOLDEN_CASES = ("blob32", "blob32_color", "block48_u8", "aniso_u16", "config1")


def scene_from_golden(g: dict):
    """Rebuild the inputs of a golden case with this package's host types.

    Returns (volume, tf, light_cam, spec, settings_for(mode, lookup))."""
    from paper_2008_06134_b200 import scene
    from paper_2008_06134_b200.datasets import sphere_blobs_field
    import hashlib

    m = g["meta"]
    if "volume" in g:
        data = g["volume"]
    else:  # config 1: regenerate and pin by the reference's sha256
        data = sphere_blobs_field(tuple(m["dims"]), seed=7)
        assert hashlib.sha256(data.tobytes()).hexdigest() == str(g["volume_sha256"])
    v = scene.VolumeDataset.from_array(data, spacing=tuple(m["spacing"]), scalar_type=m["scalar_type"])
    tf = scene.preset(m["tf"])
    cam = scene.LightCamera.fit(m["light_dir"], m["light_color"], tuple(m["res"]))
    spec = scene.make_slice_stack(m["light_dir"], m["n"])
    camera = scene.Camera(position=m["cam_pos"], target=m["cam_target"], fov_deg=m["fov"])
    light = scene.Light(direction=m["light_dir"], color=m["light_color"])
    sk = scene.ShellKernel(radii=tuple(m["shell"][0]), weights=tuple(m["shell"][1])) if m.get("shell") else None
    ck = (scene.ConeKernel(axis_samples=m["cone"][0], angles=tuple(m["cone"][1]),
                           ring_radius_per_step=m["cone"][2]) if m.get("cone") else None)

    def settings_for(mode: str, lookup: str = "linear"):
        return scene.RenderSettings(camera=camera, light=light, viewport=tuple(m["viewport"]), step=m["step"],
                                    shading_mode=mode, early_termination_alpha=m["et"],
                                    ambient_floor=m["floor"], shell_kernel=sk, cone_kernel=ck,
                                    lookup_mode=lookup)

    return v, tf, cam, spec, settings_for


def parity_stats(got: np.ndarray, want: np.ndarray) -> dict:
    """max-abs, PSNR (peak 1), count over 1e-3 and worst location."""
    d = np.abs(got.astype(np.float64) - want.astype(np.float64))
    mse = float(np.mean(d * d))
    return dict(max_abs=float(d.max()) if d.size else 0.0,
                psnr=float("inf") if mse == 0 else 10 * np.log10(1.0 / mse),
                over=int((d > 1e-3).sum()),
                worst=tuple(int(i) for i in np.unravel_index(np.argmax(d), d.shape)) if d.size else ())
