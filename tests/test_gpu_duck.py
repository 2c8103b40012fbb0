"""Reference-shaped objects on the GPU path (INTEGRATION.md §1 duck typing).

``tests/golden/reference_api.json`` lists, per reference type, the public
attribute names of the reference's own objects (written by make_golden.py
from the unmodified ``slicecast``). Here every input is rebuilt as a plain
object with exactly those names and nothing else (``__slots__``), with values
from the oracle's scene port — no class of this package is involved — and
passed to ``build_attenuation_buffer`` / ``render``. Methods the hot path
has no business calling raise. Results must equal the reference's golden
outputs: the attenuation stack bit for bit, images within 1e-4 (``none``
bit for bit).
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu

API = json.load(open(os.path.join(GOLDEN, "reference_api.json")))


def _not_on_path(name):
    def stub(*a, **k):
        raise AssertionError(f"the GPU hot path called {name}(), which it must not need")
    return stub


def strict(kind: str, **values):
    """An object carrying exactly the reference type's public names."""
    names = tuple(API[kind])
    extra = set(values) - set(names)
    assert not extra, f"{kind} has no attribute(s) {extra} in the reference"
    cls = type(f"Ref{kind}", (), {"__slots__": names})
    obj = cls()
    for n in names:
        setattr(obj, n, values[n] if n in values else _not_on_path(f"{kind}.{n}"))
    return obj


def _inputs(g):
    from oracle import scenes as S
    from oracle import slicecast_oracle as O
    m = g["meta"]
    sv = S.volume(g["volume"], spacing=tuple(m["spacing"]), scalar_type=m["scalar_type"])
    v = strict("VolumeDataset", dims=sv.dims, spacing=sv.spacing, scalar_type=sv.scalar_type, data=sv.data,
               value_range=(float(sv.data.min()), float(sv.data.max())), box_lo=sv.box_lo, box_hi=sv.box_hi,
               voxel_size=sv.voxel_size)
    st = S.preset(m["tf"])
    tf = strict("TransferFunction", lut=st.lut, control_points=st.control_points,
                resolve=lambda step, lut=st.lut: O.resolve(lut, step))
    sc = S.light_camera(m["light_dir"], m["light_color"], tuple(m["res"]))
    cam = strict("LightCamera", **{k: getattr(sc, k) for k in ("axis_u", "axis_v", "light_color", "light_dir",
                                                              "proj_matrix", "resolution", "shadow_matrix",
                                                              "u_range", "v_range", "view_matrix")})
    ss = S.slice_stack(m["light_dir"], m["n"])
    spec = strict("SliceStackSpec", d_max=ss.d_max, d_min=ss.d_min, light_dir=ss.light_dir, n_slices=ss.n_slices,
                  plane_offsets=ss.plane_offsets, spacing=ss.spacing)
    camera = strict("Camera", position=np.asarray(m["cam_pos"], np.float64),
                    target=np.asarray(m["cam_target"], np.float64), up=np.array([0.0, 1.0, 0.0]),
                    fov_deg=float(m["fov"]))
    ld = np.asarray(m["light_dir"], np.float64)
    light = strict("Light", direction=ld / np.linalg.norm(ld), color=np.asarray(m["light_color"], np.float64))
    phong = strict("PhongParams", ambient=0.1, diffuse=0.7, specular=0.2, shininess=32.0)

    def settings(mode, lookup):
        return strict("RenderSettings", ambient_floor=float(m["floor"]), camera=camera, cone_kernel=None,
                      early_termination_alpha=float(m["et"]), light=light, lookup_mode=lookup, phong=phong,
                      shading_mode=mode, shell_kernel=None, step=float(m["step"]), threads=1,
                      viewport=tuple(m["viewport"]))

    return v, tf, cam, spec, settings


@pytest.mark.parametrize("case", ["blob32", "block48_u8"])
def test_reference_shaped_objects(case):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    import paper_2008_06134_b200 as sb
    g = load_golden(case)
    v, tf, cam, spec, settings = _inputs(g)
    buf = sb.build_attenuation_buffer(v, tf, cam, spec)
    assert np.array_equal(buf.intensity, g["intensity"])
    # a reference AttenuationBuffer: numpy intensity plus its light frame
    ref_buf = strict("AttenuationBuffer", camera=cam, spec=spec, compensation_n=0.0, intensity=g["intensity"],
                     light_color=cam.light_color, shadow_matrix=cam.shadow_matrix,
                     layers=(g["intensity"][..., None] * cam.light_color).astype(np.float32))
    for mode, lookup in g["meta"]["modes"]:
        want = g[f"image_{mode}_{lookup}"]
        for b in (ref_buf, buf):
            img = sb.render(v, tf, settings(mode, lookup), b)
            assert img.shape == want.shape and img.dtype == np.float32
            err = float(np.abs(img - want).max())
            assert (err == 0.0) if mode == "none" else (err <= 1e-4), (case, mode, lookup, err)
