"""Callers of the hot path: a device-resident buffer cache and a benchmark sweep.

- ``BufferCache`` mirrors the reference service's bounded LRU with an atomic
  get-or-build per key (service.py:98-130) and its key (dataset, TF, light
  direction rounded to 12 digits, light colour, slice count, resolution,
  compensation; service.py:231-239). Entries are ``AttenuationBuffer``s whose
  stacks stay in HBM, so a camera-only change costs no build
  (service.py:246-248: build_ms = 0 on a hit). A byte budget bounds the HBM
  the cache may hold (a 1024-slice 1024^2 stack is 16 GiB of texel quads).
- ``run_sweep`` / ``write_csv`` reproduce ``slicecast.bench`` (bench.py:26-146):
  every (method, n_slices, resolution), ``repeats`` timed runs after one
  discarded warm-up whose image is hashed, the same CSV columns. Times are
  device times (CUDA events around the build and the render enqueue).
"""

from __future__ import annotations

import csv
import hashlib
import io
import itertools
import json
import threading
from collections import OrderedDict
from concurrent.futures import Future
from dataclasses import dataclass

import numpy as np
import torch

from .lightbuffer import AttenuationBuffer, build_attenuation_buffer
from .raycaster import render_device
from .scene import BUFFER_MODES, LightCamera, RenderSettings, make_slice_stack

#: bench/CLI method names -> shading modes (config.py:18-25); "has" = half-angle slicing (halfangle.py)
METHOD_MODES = {"none": "none", "phong": "phong", "sbrc": "sbrc_shadow", "shell": "shell", "cone": "cone",
                "extinction": "extinction"}

CSV_FIELDS = ("method", "n_slices", "buffer_resolution", "sample_step", "build_ms", "render_ms", "total_ms",
              "pass_count", "image_sha256")


def tf_key(tf) -> str:
    cp = getattr(tf, "control_points", None)
    if cp is not None:
        return json.dumps([[x, list(c)] for x, c in cp])
    return hashlib.sha256(np.ascontiguousarray(tf.lut).tobytes()).hexdigest()


def buffer_key(dataset_id, tf, light_dir, light_color, n_slices: int, resolution, compensation_n: float = 0.0):
    """service.py:231-239."""
    return (dataset_id, tf_key(tf), tuple(np.round(np.asarray(light_dir, dtype=np.float64), 12)),
            tuple(float(c) for c in light_color), int(n_slices), tuple(int(r) for r in resolution),
            float(compensation_n))


def _buffer_bytes(buf) -> int:
    q = getattr(buf, "quads", None)
    return 0 if q is None else q.numel() * q.element_size()


class _Slot:
    """One cache key: a future for the buffer, and the CUDA event recorded on
    the building stream right after K1 was enqueued (None off-GPU)."""

    __slots__ = ("future", "ready", "nbytes")

    def __init__(self):
        self.future: Future = Future()
        self.ready = None
        self.nbytes = 0


class BufferCache:
    """LRU of HBM-resident attenuation buffers, bounded by entry count and bytes.

    Same contract as the service's cache (service.py:98-130): ``get_or_build``
    returns ``(buffer, hit)`` and concurrent requests for one key build once.
    The mechanism is device-aware: a key maps to a slot holding a future.
    The first requester becomes the builder — it enqueues K1 on its stream
    and records a CUDA event after it, then resolves the future without
    waiting for the GPU. Every other requester (another thread, or a later
    call) takes the buffer from the future and makes *its* current stream
    wait on that event, so readiness is ordered on the device and no host
    thread blocks on a build that is merely in flight. A builder that raises
    resolves the future with the exception: concurrent waiters re-raise it,
    and the slot is dropped so the next request builds again. In-flight
    slots are never evicted."""

    def __init__(self, max_entries: int = 8, max_bytes: int | None = None):
        self.max_entries = max_entries
        self.max_bytes = max_bytes
        self._slots: OrderedDict = OrderedDict()
        self._lock = threading.Lock()

    def __len__(self) -> int:
        with self._lock:
            return sum(1 for s in self._slots.values() if s.future.done() and s.future.exception() is None)

    @property
    def bytes(self) -> int:
        with self._lock:
            return sum(s.nbytes for s in self._slots.values())

    def get_or_build(self, key, builder):
        with self._lock:
            slot = self._slots.get(key)
            mine = slot is None
            if mine:
                slot = self._slots[key] = _Slot()
            else:
                self._slots.move_to_end(key)
        if not mine:
            value = slot.future.result()  # the builder's exception propagates to waiters
            if slot.ready is not None:
                torch.cuda.current_stream().wait_event(slot.ready)
            return value, True
        try:
            value = builder()
        except BaseException as exc:
            with self._lock:
                if self._slots.get(key) is slot:
                    del self._slots[key]
            slot.future.set_exception(exc)
            raise
        if torch.cuda.is_available() and getattr(value, "quads", None) is not None:
            slot.ready = torch.cuda.Event()
            slot.ready.record(torch.cuda.current_stream(value.quads.device))
        slot.nbytes = _buffer_bytes(value)
        slot.future.set_result(value)
        with self._lock:
            self._shrink()
        return value, False

    def _shrink(self) -> None:
        """Drop least-recently used finished slots until both bounds hold
        (the newest entry always stays)."""
        def over():
            n = len(self._slots)
            return n > self.max_entries or (self.max_bytes is not None and n > 1 and
                                            sum(s.nbytes for s in self._slots.values()) > self.max_bytes)
        for key in list(self._slots):
            if not over():
                break
            if self._slots[key].future.done() and key != next(reversed(self._slots)):
                del self._slots[key]

    def clear(self) -> None:
        with self._lock:
            for key in [k for k, s in self._slots.items() if s.future.done()]:
                del self._slots[key]


def cached_build(cache: BufferCache, dataset_id, v, tf, light, n_slices: int, resolution,
                 compensation_n: float = 0.0) -> tuple[AttenuationBuffer, bool]:
    """The service's build path (service.py:241-248) over the device cache."""
    key = buffer_key(dataset_id, tf, light.direction, light.color, n_slices, resolution, compensation_n)

    def _build():
        cam = LightCamera.fit(light.direction, light.color, resolution)
        stack = make_slice_stack(light.direction, n_slices)
        return build_attenuation_buffer(v, tf, cam, stack, compensation_n)

    return cache.get_or_build(key, _build)


# ------------------------------------------------------------------ bench sweep
def _res_text(r) -> str:
    return f"{int(r[0])}x{int(r[1])}"


def _res_parse(text: str) -> tuple:
    w, h = text.split("x")
    return int(w), int(h)


def _ms(x) -> str:
    return f"{float(x):.3f}"


#: The reference's CSV schema (bench.py:26-36) as (column, render, parse):
#: timings with three decimals, the resolution as "WxH", the step as repr.
_SCHEMA = (
    ("method", str, str),
    ("n_slices", int, int),
    ("buffer_resolution", _res_text, _res_parse),
    ("sample_step", repr, float),
    ("build_ms", _ms, float),
    ("render_ms", _ms, float),
    ("total_ms", _ms, None),  # derived: build + render
    ("pass_count", int, int),
    ("image_sha256", str, str),
)
assert tuple(c for c, _, _ in _SCHEMA) == CSV_FIELDS


@dataclass
class BenchRecord:
    """One sweep point; ``total_ms`` is derived. Negative timings are a
    ValueError, as in the reference's record (bench.py:49-51)."""

    method: str
    n_slices: int
    buffer_resolution: tuple
    sample_step: float
    build_ms: float
    render_ms: float
    pass_count: int
    image_sha256: str = ""

    def __post_init__(self):
        if min(self.build_ms, self.render_ms) < 0:
            raise ValueError("timings must be >= 0")

    @property
    def total_ms(self) -> float:
        return self.build_ms + self.render_ms

    def as_row(self) -> dict:
        return {col: out(getattr(self, col)) for col, out, _ in _SCHEMA}


def parse_row(row: dict) -> BenchRecord:
    """Inverse of ``BenchRecord.as_row`` (the CSV round trip)."""
    return BenchRecord(**{col: parse(row[col]) for col, _, parse in _SCHEMA if parse is not None})


def image_sha256(img) -> str:
    """Hash of the float32 (H, W, 4) image bytes, as the reference computes it (bench.py:112-113)."""
    arr = img.cpu().numpy() if isinstance(img, torch.Tensor) else np.asarray(img)
    return hashlib.sha256(np.ascontiguousarray(arr, dtype=np.float32).tobytes()).hexdigest()


METHODS = tuple(METHOD_MODES) + ("has",)


def render_scene(v, tf, settings, method: str, n_slices: int, resolution, compensation_n: float = 0.0):
    """bench.render_scene (bench.py:87-109) on the device: (image, build_ms, render_ms, pass_count)."""
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r} (choose from {METHODS})")
    if method == "has":  # half-angle slicing: all of its cost is render (bench.py:90-95)
        from .halfangle import render_half_angle_device
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        img, passes = render_half_angle_device(v, tf, settings, n_slices, light_resolution=resolution)
        e1.record(stream)
        e1.synchronize()
        return img, 0.0, e0.elapsed_time(e1), passes
    mode = METHOD_MODES[method]
    s = RenderSettings(camera=settings.camera, light=settings.light, viewport=settings.viewport,
                       step=settings.step, shading_mode=mode,
                       early_termination_alpha=settings.early_termination_alpha,
                       ambient_floor=settings.ambient_floor, shell_kernel=settings.shell_kernel,
                       cone_kernel=settings.cone_kernel, phong=settings.phong, lookup_mode=settings.lookup_mode)
    stream = torch.cuda.current_stream()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    buf = None
    e0.record(stream)
    if mode in BUFFER_MODES:
        light = settings.light
        cam = LightCamera.fit(light.direction, light.color, resolution)
        stack = make_slice_stack(light.direction, n_slices)
        buf = build_attenuation_buffer(v, tf, cam, stack, compensation_n)
    e1.record(stream)
    img = render_device(v, tf, s, buf)
    e2.record(stream)
    e2.synchronize()
    build_ms = e0.elapsed_time(e1) if buf is not None else 0.0
    return img, build_ms, e1.elapsed_time(e2), 1


def _measure_point(v, tf, settings, method: str, n: int, res: tuple, repeats: int) -> BenchRecord:
    """One sweep point: the first run only provides the image hash (warm-up),
    the next ``repeats`` runs are averaged."""
    runs = [render_scene(v, tf, settings, method, n, res) for _ in range(repeats + 1)]
    timed = np.array([(b, r) for _, b, r, _ in runs[1:]], dtype=np.float64)
    return BenchRecord(method=method, n_slices=n, buffer_resolution=res, sample_step=settings.step,
                       build_ms=float(timed[:, 0].mean()), render_ms=float(timed[:, 1].mean()),
                       pass_count=runs[-1][3], image_sha256=image_sha256(runs[0][0]))


def run_sweep(v, tf, settings, methods, slices, resolutions, repeats: int = 3) -> list[BenchRecord]:
    """The reference sweep (bench.py:116-146) with device timing: every
    (method, n_slices, resolution) in that nesting order."""
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    grid = itertools.product(methods, slices, [(r, r) if isinstance(r, int) else tuple(r) for r in resolutions])
    return [_measure_point(v, tf, settings, m, n, res, repeats) for m, n, res in grid]


def write_csv(records, fh_or_path) -> None:
    own = isinstance(fh_or_path, (str, bytes)) or hasattr(fh_or_path, "__fspath__")
    fh = open(fh_or_path, "w", newline="") if own else fh_or_path
    try:
        w = csv.DictWriter(fh, fieldnames=CSV_FIELDS)
        w.writeheader()
        for rec in records:
            w.writerow(rec.as_row())
    finally:
        if own:
            fh.close()


def csv_text(records) -> str:
    buf = io.StringIO()
    write_csv(records, buf)
    return buf.getvalue()
