"""Callers of the hot path: the device buffer cache (service.py:98-130 semantics)
and the CSV bench harness (bench.py:26-146 schema)."""

from __future__ import annotations

import hashlib
import os
import sys
import threading
import time

import numpy as np
import pytest

from conftest import REFERENCE_SRC, load_golden, scene_from_golden


def test_cache_hit_miss_and_lru():
    from paper_2008_06134_b200.harness import BufferCache
    c = BufferCache(max_entries=2)
    calls = []
    mk = lambda k: (lambda: calls.append(k) or f"buf-{k}")
    assert c.get_or_build("a", mk("a")) == ("buf-a", False)
    assert c.get_or_build("a", mk("a")) == ("buf-a", True)
    c.get_or_build("b", mk("b"))
    c.get_or_build("a", mk("a"))          # refresh a
    c.get_or_build("c", mk("c"))          # evicts b (least recent)
    assert c.get_or_build("a", mk("a"))[1] is True
    assert c.get_or_build("b", mk("b"))[1] is False
    assert calls == ["a", "b", "c", "b"]


def test_cache_concurrent_build_once_and_failure_releases():
    from paper_2008_06134_b200.harness import BufferCache
    c = BufferCache()
    n = {"builds": 0}

    def slow():
        n["builds"] += 1
        time.sleep(0.2)
        return "v"

    res = []
    ts = [threading.Thread(target=lambda: res.append(c.get_or_build("k", slow))) for _ in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert n["builds"] == 1 and sorted(h for _, h in res) == [False] + [True] * 5

    def boom():
        raise RuntimeError("build failed")

    with pytest.raises(RuntimeError):
        c.get_or_build("bad", boom)
    assert c.get_or_build("bad", lambda: "ok") == ("ok", False)  # waiters released, retry builds


def test_buffer_key_rounds_light_direction():
    from paper_2008_06134_b200.harness import buffer_key
    from paper_2008_06134_b200 import scene
    tf = scene.preset("hot")
    a = buffer_key("ds", tf, (0.3, -0.5, 0.8), (1, 1, 1), 64, (128, 128))
    b = buffer_key("ds", tf, (0.3 + 1e-15, -0.5, 0.8), (1, 1, 1), 64, (128, 128))
    c = buffer_key("ds", tf, (0.3, -0.5, 0.8), (1, 1, 1), 65, (128, 128))
    assert a == b and a != c


def test_csv_schema_round_trip():
    from paper_2008_06134_b200.harness import BenchRecord, CSV_FIELDS, csv_text, parse_row
    import csv as _csv
    import io
    recs = [BenchRecord("cone", 64, (128, 96), 1 / 256, 1.25, 3.5, 1, "ab"),
            BenchRecord("none", 8, (16, 16), 1 / 64, 0.0, 0.125, 1, "cd")]
    text = csv_text(recs)
    rows = list(_csv.DictReader(io.StringIO(text)))
    assert tuple(rows[0].keys()) == CSV_FIELDS
    back = [parse_row(r) for r in rows]
    assert back[0].buffer_resolution == (128, 96) and back[0].total_ms == pytest.approx(4.75)
    with pytest.raises(ValueError):
        BenchRecord("cone", 1, (1, 1), 0.1, -1.0, 0.0, 1)


@pytest.mark.skipif(not os.path.isdir(REFERENCE_SRC), reason="reference not present")
def test_csv_schema_matches_reference():
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    from slicecast import bench as rb
    from paper_2008_06134_b200.harness import CSV_FIELDS, METHOD_MODES
    from slicecast.config import METHOD_MODES as REF_MODES
    assert CSV_FIELDS == rb.CSV_FIELDS
    assert METHOD_MODES == REF_MODES


@pytest.mark.gpu
def test_sweep_on_gpu_and_none_hash_equals_reference():
    """The `none` image is bit-identical, so its sha256 equals the reference image's."""
    import torch
    assert torch.cuda.is_available()
    from paper_2008_06134_b200.harness import run_sweep, csv_text
    g = load_golden("blob32")
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    s = settings_for("none")
    recs = run_sweep(v, tf, s, ["none", "sbrc", "cone"], [8, 24], [16, 40], repeats=2)
    assert len(recs) == 12 and all(r.render_ms > 0 for r in recs)
    assert all(r.build_ms == 0.0 for r in recs if r.method == "none")
    assert all(r.build_ms > 0.0 for r in recs if r.method != "none")
    want = hashlib.sha256(np.ascontiguousarray(g["image_none_linear"]).tobytes()).hexdigest()
    assert all(r.image_sha256 == want for r in recs if r.method == "none")
    assert csv_text(recs).count("\n") == 13


@pytest.mark.gpu
def test_cached_build_skips_rebuild():
    import torch
    from paper_2008_06134_b200.harness import BufferCache, cached_build
    from paper_2008_06134_b200 import scene
    g = load_golden("blob32")
    v, tf, cam, spec, settings_for = scene_from_golden(g)
    cache = BufferCache(max_entries=2, max_bytes=1 << 30)
    light = scene.Light(direction=g["meta"]["light_dir"])
    b1, hit1 = cached_build(cache, "blob32", v, tf, light, 24, (40, 36))
    b2, hit2 = cached_build(cache, "blob32", v, tf, light, 24, (40, 36))
    assert (hit1, hit2) == (False, True) and b1 is b2
    assert np.array_equal(b1.intensity, g["intensity"])
    assert cache.bytes == 24 * 36 * 40 * 16


@pytest.mark.gpu
def test_acceptance_c4_trend_on_gpu():
    """Acceptance C4 (reference tests/test_acceptance.py:148-165) with
    device timing: SBRC render(256)/render(64) <= 1.5 and the half-angle total
    grows >= 2.5x (pass count 2n)."""
    from paper_2008_06134_b200.harness import run_sweep
    from paper_2008_06134_b200.datasets import make_sphere_blobs
    from paper_2008_06134_b200 import scene
    v = make_sphere_blobs((128, 128, 128), seed=7)
    tf = scene.preset("hot")
    s = scene.RenderSettings(camera=scene.Camera(position=(0.5, 0.5, -1.6), target=(0.5, 0.5, 0.5)),
                             light=scene.Light(direction=(0.3, -0.5, 0.8)), viewport=(256, 256), step=1 / 256)
    recs = {(r.method, r.n_slices): r for r in run_sweep(v, tf, s, ["sbrc", "has"], [64, 256], [256], repeats=5)}
    for r in recs.values():
        print(f"[c4] {r.method} n={r.n_slices} build {r.build_ms:.3f} render {r.render_ms:.3f} ms")
    sbrc_ratio = recs[("sbrc", 256)].render_ms / recs[("sbrc", 64)].render_ms
    has_ratio = recs[("has", 256)].total_ms / recs[("has", 64)].total_ms
    print(f"[c4] sbrc render ratio {sbrc_ratio:.2f}, has total ratio {has_ratio:.2f}, "
          f"passes {recs[('has', 64)].pass_count}->{recs[('has', 256)].pass_count}")
    assert sbrc_ratio <= 1.5 and has_ratio >= 2.5
    assert recs[("has", 256)].pass_count == 512
