"""BASELINE config 5: the moving-light sweep (512^3 blobs -> 1024^2, cone),
the attenuation buffer rebuilt for every light. Needs a B200.

Lights follow the viewer's orbit (frontend/src/orbit.ts:28-35: elevation
30 deg, azimuth 360 f / 16), and the buffer is rebuilt per light
(lightbuffer.py:144-199) through ``FrameRenderer.use_light`` exactly as
``bench.py --config 5`` drives it. For corner points of the sweep —
(n, slice res) = (32, 256^2), (256, 512^2) and the largest (512, 2048^2; 32 GiB
of texel quads, close to the 32-bit quad-offset limit) — every frame is
checked against the oracle: light rows of the stack bit-exact, stratified
pixels of the cone image within 1e-4 (the oracle's march reading the
GPU-built stack, itself bit-exact on the checked rows).
"""

from __future__ import annotations

import sys

import numpy as np
import pytest

from conftest import ROOT, parity_stats

pytestmark = pytest.mark.gpu
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def world5():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    import bench
    from paper_2008_06134_b200.frame import FrameRenderer
    from paper_2008_06134_b200.scene import VolumeDataset
    cfg = bench.CONFIGS[5]
    tf, cam, spec, settings = bench.scene_objects(cfg, cfg["mode"])
    dvol, _ = bench.device_volume_for(cfg, torch.device("cuda"))
    host = VolumeDataset.from_array(dvol.data.cpu().numpy())  # the same voxels on both sides
    fr = FrameRenderer(dvol, tf, cam, spec, settings)
    return cfg, tf, fr, host


@pytest.mark.parametrize("n,res", [(32, 256), (256, 512), (512, 2048)])
def test_orbit_sweep_point(world5, n, res):
    import torch
    from types import SimpleNamespace
    import bench
    from oracle import slicecast_oracle as O
    from paper_2008_06134_b200 import scene
    cfg, tf, fr, host = world5
    rows = np.array([res // 4, res // 2, (3 * res) // 4])
    pix = np.arange(32, 1024, 128)  # 8 x 8 stratified pixels of the 1024^2 frame
    for az in (0.0, 135.0, 270.0):
        ld = bench.orbit_light(az, 30.0)
        fr.use_light(fr.prepare_light(scene.LightCamera.fit(ld, (1, 1, 1), (res, res)), scene.make_slice_stack(ld, n)))
        img = fr.frame()
        torch.cuda.synchronize()
        inten = fr.intensity
        assert bool((inten[0] == 1.0).all()) and float(inten.min()) >= 0.0
        assert bool((inten[1:] <= inten[:-1]).all())  # transmittance never grows along the light
        want = O.build_intensity(host, tf.lut, fr.cam, fr.spec, rows=rows)
        assert np.array_equal(inten[:, rows].contiguous().cpu().numpy(), want), (n, res, az)
        buf = SimpleNamespace(camera=fr.cam, spec=fr.spec, compensation_n=0.0,
                              intensity=inten.contiguous().cpu().numpy())
        want_img = O.render_image(host, tf.lut, fr.settings, buf, rows=pix, cols=pix)
        st = parity_stats(img.cpu().numpy()[np.ix_(pix, pix)], want_img)
        print(f"[config5] n={n} res={res} az={az}: max_abs={st['max_abs']:.2e} psnr={st['psnr']:.1f}")
        assert st["max_abs"] <= 1e-4, (n, res, az, st)
        del buf
