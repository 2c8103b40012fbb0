"""The oracle (oracle/slicecast_oracle.py) against the reference's own outputs.

The golden files were written by tests/golden/make_golden.py, which runs the
unmodified reference. The oracle restates the same float64 arithmetic, so
every comparison here is bit-exact (np.array_equal), except where BLAS
matrix products are involved (light uv), which are compared at 1e-15.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden, scene_from_golden
from oracle import slicecast_oracle as O


class _Vol:
    def __init__(self, data, spacing=(1.0, 1.0, 1.0)):
        from paper_2008_06134_b200.scene import VolumeDataset
        self.__dict__.update(vars(VolumeDataset.from_array(data, spacing=spacing)))

    @property
    def voxel_size(self):
        return (self.box_hi - self.box_lo) / np.array(self.dims, dtype=np.float64)


@pytest.fixture(scope="module")
def prim():
    return load_golden("primitives")


def test_trilinear_bit_exact(prim):
    v = _Vol(prim["volume"])
    assert np.array_equal(O.trilinear(v, prim["pts"]), prim["trilinear"])


def test_lut_bit_exact(prim):
    lut = O.resolve(prim["tf_lut"], 1.0 / 300.0)
    assert np.array_equal(lut, prim["lut_step"])
    assert np.array_equal(O.lut_blend(lut, prim["s"]), prim["lut_vals"])


def test_rays_and_box_bit_exact(prim):
    m = prim["meta"]
    rays = O.camera_rays(m["cam_pos"], (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), m["fov"], tuple(m["viewport"]))
    assert np.array_equal(rays, prim["rays"])
    t_in, t_out, hit = O.box_hit(np.broadcast_to(np.array(m["cam_pos"]), rays.shape), rays)
    assert np.array_equal(t_in, prim["t_in"]) and np.array_equal(t_out, prim["t_out"])
    assert np.array_equal(hit, prim["hit"])


def _prim_buffer(prim):
    from paper_2008_06134_b200 import scene
    m = prim["meta"]
    cam = scene.LightCamera.fit(m["light_dir"], (1, 1, 1), tuple(m["res"]))
    spec = scene.make_slice_stack(m["light_dir"], m["n"])
    return cam, spec


def test_build_small_bit_exact(prim):
    cam, spec = _prim_buffer(prim)
    v = _Vol(prim["volume"])
    assert np.array_equal(O.build_intensity(v, prim["tf_lut"], cam, spec), prim["intensity"])


def test_lookups_match(prim):
    cam, spec = _prim_buffer(prim)
    inten = prim["intensity"]
    probe = prim["probe"]
    np.testing.assert_allclose(O.light_uv(cam, probe), prim["uv"], rtol=0, atol=1e-15)
    assert np.array_equal(O.lookup_scalar(inten, cam, spec, probe, "linear"), prim["look_lin"])
    assert np.array_equal(O.lookup_scalar(inten, cam, spec, probe, "nearest"), prim["look_near"])
    sh = O.shell_scalar(inten, cam, spec, probe, (0.05, 0.1, 0.15000000000000002), (0.5, 0.3, 0.2))
    assert np.array_equal(sh, prim["shell"])
    angles = (0.0, math.pi / 2, math.pi, 3 * math.pi / 2)
    cone = O.cone_scalar(inten, cam, spec, probe, 2, angles, 0.5, np.array([0.5, 0.5, -1.6]))
    assert np.array_equal(cone, prim["cone"])
    cone2 = O.cone_scalar(inten, cam, spec, probe, 2, angles, 0.5, None)
    assert np.array_equal(cone2, prim["cone_noeye"])


def test_lookup_rejects_unknown_mode(prim):
    cam, spec = _prim_buffer(prim)
    with pytest.raises(ValueError):
        O.lookup_scalar(prim["intensity"], cam, spec, prim["probe"], "cubic")


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_case_build_bit_exact(case):
    g = load_golden(case)
    v, tf, cam, spec, _ = scene_from_golden(g)
    got = O.build_intensity(v, tf.lut, cam, spec, g["meta"]["comp"])
    assert np.array_equal(got, g["intensity"])


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_case_render_bit_exact(case):
    g = load_golden(case)
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    from paper_2008_06134_b200.lightbuffer import AttenuationBuffer
    buf = AttenuationBuffer(cam, spec, g["meta"]["comp"], g["intensity"])
    for mode, lookup in g["meta"]["modes"]:
        if case == "config1" and mode == "shell":
            continue  # ~7 s on one core; covered by the GPU test against the same golden
        img = O.render_image(v, tf.lut, settings_for(mode, lookup), buf)
        assert np.array_equal(img, g[f"image_{mode}_{lookup}"]), (case, mode, lookup)


def _extra_scene(g, aniso=False):
    from paper_2008_06134_b200 import scene
    m = g["meta"]
    data = g["volume_aniso"] if aniso else g["volume"]
    v = scene.VolumeDataset.from_array(data, spacing=tuple(m["spacing_aniso"]) if aniso else (1.0, 1.0, 1.0))
    tf = scene.preset(m["tf"])
    cam = scene.Camera(position=m["cam_pos"], target=(0.5, 0.5, 0.5), fov_deg=m["fov"])
    light = scene.Light(direction=m["light_dir"])

    def settings(mode):
        return scene.RenderSettings(camera=cam, light=light, viewport=tuple(m["viewport"]), step=m["step"],
                                    shading_mode=mode, ambient_floor=m["floor"],
                                    phong=scene.PhongParams(*m["phong"]))
    return v, tf, light, settings


def test_extra_modes_bit_exact():
    """phong / extinction images, gradient and shadow_oracle_many vs the reference."""
    g = load_golden("extra_modes")
    for aniso in (False, True):
        tag = "_aniso" if aniso else ""
        v, tf, light, settings = _extra_scene(g, aniso)
        for mode in ("phong", "extinction"):
            assert np.array_equal(O.render_image(v, tf.lut, settings(mode)), g[f"image_{mode}{tag}"]), (mode, tag)
        want = g["oracle_aniso" if aniso else "oracle"]
        assert np.array_equal(O.shadow_oracle(v, tf.lut, g["probe"], light.direction, g["meta"]["oracle_step"]), want)
    v, *_ = _extra_scene(g, True)
    assert np.array_equal(O.gradient(v, g["probe"]), g["grad"])


def _has_scene(g, tag):
    from paper_2008_06134_b200 import scene
    m = g["meta"]
    c = m["cases"][tag]
    v = scene.VolumeDataset.from_array(g["volume"])
    cam = scene.Camera(position=c["pos"], target=(0.5, 0.5, 0.5), fov_deg=45.0)
    s = scene.RenderSettings(camera=cam, light=scene.Light(direction=c["light"]), viewport=tuple(m["viewport"]),
                             step=1 / 64)
    return v, scene.preset(m["tf"]), s, m, c


@pytest.mark.parametrize("tag", ["f2b", "b2f"])
def test_half_angle_oracle(tag):
    """render_half_angle in both slice orders vs the reference (1e-12: BLAS dots)."""
    g = load_golden("half_angle")
    v, tf, s, m, c = _has_scene(g, tag)
    img, passes = O.half_angle(v, tf.lut, s, m["n"], tuple(m["light_res"]))
    assert passes == c["passes"] == 2 * m["n"]
    np.testing.assert_allclose(img, g[f"image_{tag}"], rtol=0, atol=1e-6)


# ------------------------------------------------------------ config 5 (moving light) and the scene port
def test_scene_port_matches_reference_objects(prim):
    """oracle/scenes.py (used by bench.py's reference arm instead of the product
    package) reproduces the reference's LUT, light frame and slice stack."""
    from oracle import scenes as S
    from paper_2008_06134_b200 import scene
    for name in S.PRESETS:
        assert np.array_equal(S.preset(name).lut, scene.preset(name).lut)
    g = load_golden("config1")
    assert __import__("hashlib").sha256(S.blob_field(64, 7).tobytes()).hexdigest() == str(g["volume_sha256"])
    m = g["meta"]
    cam = S.light_camera(m["light_dir"], m["light_color"], tuple(m["res"]))
    spec = S.slice_stack(m["light_dir"], m["n"])
    v = S.volume(S.blob_field(64, 7))
    inten = O.build_intensity(v, S.preset(m["tf"]).lut, cam, spec)
    assert np.array_equal(inten, g["intensity"])
    blk = load_golden("block48_u8")
    raw, f = S.raw_roundtrip(S.perforated_block(48, 3), "u8")
    assert np.array_equal(f, blk["volume"])


def test_orbit_light_cases_bit_exact():
    """BASELINE config 5's orbit lights (orbit.ts:28-35): the oracle's build and
    cone render equal the reference's at three azimuths."""
    from oracle import scenes as S
    g = load_golden("orbit32")
    m = g["meta"]
    v = S.volume(g["volume"])
    tf = S.preset(m["tf"])
    for az in m["azimuths"]:
        ld = S.orbit_light(az, m["elevation"])
        assert np.array_equal(np.asarray(ld), g[f"light_{int(az)}"])
        cam = S.light_camera(ld, (1, 1, 1), tuple(m["res"]))
        spec = S.slice_stack(ld, m["n"])
        inten = O.build_intensity(v, tf.lut, cam, spec)
        assert np.array_equal(inten, g[f"intensity_{int(az)}"])
        st = S.render_settings(m["cam_pos"], m["cam_target"], m["viewport"], m["step"], "cone", ld,
                               fov_deg=m["fov"])
        from types import SimpleNamespace
        buf = SimpleNamespace(intensity=inten, camera=cam, spec=spec)
        img = O.render_image(v, tf.lut, st, buf)
        assert np.array_equal(img, g[f"image_{int(az)}"])
