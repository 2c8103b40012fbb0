"""Point-wise light API on the GPU: lookup_light*, shade_sbrc_shadow/shell/cone.

The reference's own shading-factor and lookup unit tests
(tests/test_raycaster.py:248-323, tests/test_lightbuffer.py:159-213)
re-expressed against the CUDA lookup code, plus the reference's values at
300 random probes (tests/golden/primitives.npz).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sb():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    import paper_2008_06134_b200 as sb
    return sb


def synthetic_buffer(sb, intensity, light_dir=(0, 0, 1), light_color=(1, 1, 1)):
    """tests/test_raycaster.py:51-56: a hand-made (n, H, W) stack on the default frame."""
    n, h, w = intensity.shape
    spec = sb.make_slice_stack(light_dir, n)
    cam = sb.LightCamera.fit(light_dir, light_color, (w, h))
    return sb.AttenuationBuffer(cam, spec, 0.0, np.asarray(intensity, dtype=np.float32))


def texel_field(sb, n=8, res=32, fn=None):
    """tests/test_raycaster.py:59-68: intensity[k, iy, ix] = fn(x, y, z_plane_k) for a +z light."""
    spec = sb.make_slice_stack((0, 0, 1), n)
    xs = (np.arange(res) + 0.5) / res
    out = np.empty((n, res, res))
    for k in range(n):
        out[k] = fn(xs[None, :], xs[:, None], float(spec.plane_offsets[k]))
    return out


def test_probes_match_reference(sb):
    g = load_golden("primitives")
    m = g["meta"]
    cam = sb.LightCamera.fit(m["light_dir"], (1, 1, 1), tuple(m["res"]))
    spec = sb.make_slice_stack(m["light_dir"], m["n"])
    buf = sb.AttenuationBuffer(cam, spec, 0.0, g["intensity"])
    probe = g["probe"]
    np.testing.assert_allclose(sb.lookup_light_scalar_many(buf, probe, "linear"), g["look_lin"], atol=2e-6)
    near = sb.lookup_light_scalar_many(buf, probe, "nearest")
    assert np.sum(np.abs(near - g["look_near"]) > 2e-6) == 0
    from paper_2008_06134_b200.raycaster import _light_factor
    sh = _light_factor(buf, probe, "shell", shell_kernel=sb.ShellKernel.default(0.05))[:, 0]
    np.testing.assert_allclose(sh, g["shell"], atol=2e-6)
    cone = _light_factor(buf, probe, "cone", cone_kernel=sb.ConeKernel(), eye=(0.5, 0.5, -1.6))[:, 0]
    np.testing.assert_allclose(cone, g["cone"], atol=2e-6)
    cone2 = _light_factor(buf, probe, "cone", cone_kernel=sb.ConeKernel(), eye=None)[:, 0]
    np.testing.assert_allclose(cone2, g["cone_noeye"], atol=2e-6)


# ------------------------------------------------ tests/test_raycaster.py:248-323
def test_sbrc_empty_volume_factor_one(sb):
    buf = synthetic_buffer(sb, np.ones((8, 16, 16)))
    assert np.allclose(sb.shade_sbrc_shadow((0.5, 0.5, 0.5), buf), 1.0, atol=1e-9)


def test_sbrc_behind_opaque_slab_floor(sb):
    inten = np.ones((8, 16, 16))
    inten[4:] = 0.0
    buf = synthetic_buffer(sb, inten)
    assert np.allclose(sb.shade_sbrc_shadow((0.5, 0.5, 0.9), buf, ambient_floor=0.07), 0.07)


def test_shell_constant_field_matches_sbrc(sb):
    buf = synthetic_buffer(sb, np.full((8, 16, 16), 0.37))
    k = sb.ShellKernel(radii=(0.05, 0.1), weights=(0.6, 0.4))
    p = (0.5, 0.5, 0.5)
    assert np.allclose(sb.shade_shell(p, buf, k), sb.shade_sbrc_shadow(p, buf), atol=1e-6)


def test_shell_hard_edge_half(sb):
    field = texel_field(sb, fn=lambda x, y, z: np.where(x + y + z < 1.5, 1.0, 0.0))
    buf = synthetic_buffer(sb, field)
    assert np.allclose(sb.shade_shell((0.5, 0.5, 0.5), buf, sb.ShellKernel(radii=(0.25,), weights=(1.0,))), 0.5,
                       atol=1e-6)


def test_shell_linear_gradient_cancels(sb):
    field = texel_field(sb, fn=lambda x, y, z: 0.2 + 0.3 * x + 0.25 * y + 0.2 * z)
    buf = synthetic_buffer(sb, field)
    p = (0.5, 0.5, 0.5)
    center = sb.lookup_light_scalar_many(buf, np.array([p]))[0]
    f = sb.shade_shell(p, buf, sb.ShellKernel(radii=(0.1, 0.25), weights=(0.7, 0.3)))
    assert np.allclose(f, center, atol=1e-6)


def test_cone_constant_field_matches_sbrc(sb):
    buf = synthetic_buffer(sb, np.full((8, 16, 16), 0.42))
    p = (0.5, 0.5, 0.5)
    assert np.allclose(sb.shade_cone(p, buf, sb.ConeKernel(), eye=(0.5, 0.5, -2.0)), sb.shade_sbrc_shadow(p, buf),
                       atol=1e-6)


def test_cone_zero_radius_collapses_to_axis(sb):
    field = texel_field(sb, fn=lambda x, y, z: 0.1 + 0.8 * z)
    buf = synthetic_buffer(sb, field)
    k = sb.ConeKernel(axis_samples=2, ring_radius_per_step=0.0)
    p = np.array([0.5, 0.5, 0.7])
    f = sb.shade_cone(p, buf, k)[0]
    sp = buf.spec.spacing
    axis_pts = np.array([p - sp * np.array([0, 0, 1.0]), p - 2 * sp * np.array([0, 0, 1.0])])
    assert f == pytest.approx(sb.lookup_light_scalar_many(buf, axis_pts).mean(), rel=1e-6)


def test_cone_brackets_hard_shadow_near_edge(sb):
    from paper_2008_06134_b200.datasets import make_slab
    v = make_slab((32, 32, 32), axis=2, lo=0.3, hi=0.5, value=1.0)
    d = (0, 0, 1)
    buf = sb.build_attenuation_buffer(v, sb.preset("linear"), sb.LightCamera.fit(d, (1, 1, 1), (64, 64)),
                                      sb.make_slice_stack(d, 32))
    rng = np.random.default_rng(4)
    for _ in range(20):
        p = np.array([rng.uniform(0.1, 0.9), rng.uniform(0.1, 0.9), rng.uniform(0.55, 0.9)])
        hard = sb.shade_sbrc_shadow(p, buf)[0]
        soft = sb.shade_cone(p, buf, sb.ConeKernel(), eye=(0.5, 0.5, -2.0))[0]
        assert hard - 1e-6 <= soft <= 1.0 + 1e-6


# ------------------------------------------------ tests/test_lightbuffer.py:159-213
def _homogeneous(sb, n_slices=16, per_slice_alpha=0.5, res=(32, 32)):
    spec = sb.make_slice_stack((0, 0, 1), n_slices)
    expo = spec.spacing / (1.0 / 256.0)
    a_tf = 1.0 - (1.0 - per_slice_alpha) ** (1.0 / expo)
    tf = sb.TransferFunction([(0.0, (1, 1, 1, a_tf)), (1.0, (1, 1, 1, a_tf))])
    v = sb.VolumeDataset.from_array(np.ones((8, 8, 8), dtype=np.float32))
    cam = sb.LightCamera.fit((0, 0, 1), (1.0, 1.0, 1.0), res)
    return sb.build_attenuation_buffer(v, tf, cam, spec), spec


def test_lookup_transparent_returns_light_color(sb):
    v = sb.VolumeDataset.from_array(np.zeros((8, 8, 8), dtype=np.float32))
    tf = sb.TransferFunction([(0.0, (0, 0, 0, 0)), (1.0, (0.5, 0.5, 0.5, 0.0))])
    cam = sb.LightCamera.fit((0, 0, 1), (0.5, 1.0, 0.25), (16, 16))
    buf = sb.build_attenuation_buffer(v, tf, cam, sb.make_slice_stack((0, 0, 1), 8))
    pts = np.random.default_rng(2).random((20, 3))
    assert np.allclose(sb.lookup_light_many(buf, pts), [0.5, 1.0, 0.25], atol=1e-7)


def test_lookup_on_planes_and_between(sb):
    buf, spec = _homogeneous(sb)
    for k in (0, 3, 10, 15):
        p = np.array([(0.5, 0.5, float(spec.plane_offsets[k]))])
        near = sb.lookup_light_scalar_many(buf, p, "nearest")[0]
        lin = sb.lookup_light_scalar_many(buf, p, "linear")[0]
        assert near == pytest.approx(0.5 ** k, rel=1e-5) and lin == pytest.approx(near, rel=1e-5)
    k = 6
    z = 0.5 * (spec.plane_offsets[k] + spec.plane_offsets[k + 1])
    val = sb.lookup_light_scalar_many(buf, np.array([(0.5, 0.5, z)]), "linear")[0]
    assert val == pytest.approx(0.5 * (0.5 ** k + 0.5 ** (k + 1)), rel=1e-5)
    assert np.allclose(sb.lookup_light(buf, (0.5, 0.5, 0.0)), 1.0, atol=1e-6)   # before slice 0
    assert np.allclose(sb.lookup_light(buf, (3.0, 0.5, 0.9)), 1.0)              # outside the footprint
    with pytest.raises(ValueError):
        sb.lookup_light(buf, (0.5, 0.5, 0.5), mode="cubic")


def test_lookup_energy_bound(sb):
    from paper_2008_06134_b200.datasets import make_sphere_blobs
    v = make_sphere_blobs((32, 32, 32), seed=7)
    d = (0.3, 0.3, 0.9)
    buf = sb.build_attenuation_buffer(v, sb.preset("linear"), sb.LightCamera.fit(d, (1, 1, 1), (32, 32)),
                                      sb.make_slice_stack(d, 16))
    vals = sb.lookup_light_many(buf, np.random.default_rng(4).uniform(-0.2, 1.2, size=(200, 3)))
    assert np.all(vals <= 1.0 + 1e-6) and np.all(vals >= 0.0)
