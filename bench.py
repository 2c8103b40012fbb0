#!/usr/bin/env python
"""Benchmark: frames/s + Gsamples/s of slice-based ray casting on B200.

Default workload = BASELINE.json config 3: a 512^3 float32 sphere-blob volume
(seed 7, TF "hot") rendered to 1024^2 with cone scattering from a 256-slice
attenuation buffer at 512^2, step 1/512. One step = one frame = K1
(attenuation build, the light is rebuilt every frame) + K2 (ray march) +
image assembly (NCCL all-gather when N > 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--build replicated|sharded]
    python bench.py --impl reference ...   # the reference CPU path (oracle port), all host cores

Prints ONE JSON line on rank 0. Timing: CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks; inputs (512 MiB volume,
256 MiB buffer) are larger than L2, so no explicit flush is needed.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/s + Gsamples/s, 512³ vol→1024² image, 256 light slices, 1–8 GPU"
LIGHT = (0.3, -0.5, 0.8)
EYE, TARGET = (0.5, 0.5, -1.6), (0.5, 0.5, 0.5)

CONFIGS = {
    1: dict(name="64^3 f32 sphere blobs -> 128^2, 32 slices @128^2, shell", dims=64, volume="blobs", seed=7,
            tf="hot", n=32, res=128, image=128, step=1 / 256, mode="shell"),
    2: dict(name="256^3 u8 perforated block -> 512^2, 128 slices @512^2, sbrc_shadow", dims=256, volume="block_u8",
            seed=3, tf="bone", n=128, res=512, image=512, step=1 / 256, mode="sbrc_shadow"),
    3: dict(name="512^3 f32 sphere blobs -> 1024^2, 256 slices @512^2, cone", dims=512, volume="blobs", seed=7,
            tf="hot", n=256, res=512, image=1024, step=1 / 512, mode="cone"),
    4: dict(name="1024^3 u16 sphere blobs -> 2048^2, 512 slices @1024^2, cone", dims=1024, volume="blobs_u16",
            seed=7, tf="hot", n=512, res=1024, image=2048, step=1 / 1024, mode="cone"),
    5: dict(name="512^3 f32 sphere blobs -> 1024^2, cone, moving light (az = 360*f/16, el = 30), "
                 "slices {32..512} x slice res {256^2..2048^2}, buffer rebuilt every frame", dims=512,
            volume="blobs", seed=7, tf="hot", n=256, res=512, image=1024, step=1 / 512, mode="cone",
            sweep_n=(32, 64, 128, 256, 512), sweep_res=(256, 512, 1024, 2048), frames=16),
}


def orbit_light(az_deg: float, el_deg: float):
    """frontend/src/orbit.ts:28-35: direction the light travels."""
    el, az = math.radians(el_deg), math.radians(az_deg)
    return (-math.cos(el) * math.sin(az), -math.sin(el), math.cos(el) * math.cos(az))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--mode", default=None, help="override shading mode")
    ap.add_argument("--build", choices=("replicated", "sharded", "frustum"), default="frustum",
                    help="N > 1: full K1 per rank, row-sharded K1 + all-gather, or frustum-culled K1 per "
                         "contiguous rank band (partition.py)")
    ap.add_argument("--assemble", choices=("p2p", "nccl"), default="p2p",
                    help="N>1 image assembly: fused peer-memory stores from the march kernel (self-checked, "
                         "falls back to NCCL) or NCCL all-gather")
    ap.add_argument("--tile-order", choices=("auto", "heavy", "natural", "measured"), default="auto",
                    help="K2 dispatch order: heavy-first by ray length, natural, or heavy-first by the previous "
                         "frame's measured tile costs; auto = measured with > 1 rank, ray length at 1")
    ap.add_argument("--raw-voxels", action="store_true",
                    help="u8/u16 volumes: keep the integers in HBM (default: normalised to float32 once)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="disable overlapping the next frame's build with this frame's march")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-frame", action="store_true",
                    help="reference arm: skip the unextrapolated config-2 frame; ours: skip the config-2 GPU frame")
    a = ap.parse_args()
    a.warmup = max(a.warmup, 3)
    return a


# --------------------------------------------------------------- scene inputs
def scene_objects(cfg, mode):
    from paper_2008_06134_b200 import scene
    tf = scene.preset(cfg["tf"])
    cam = scene.LightCamera.fit(LIGHT, (1.0, 1.0, 1.0), (cfg["res"], cfg["res"]))
    spec = scene.make_slice_stack(LIGHT, cfg["n"])
    settings = scene.RenderSettings(camera=scene.Camera(position=EYE, target=TARGET), light=scene.Light(direction=LIGHT),
                                    viewport=(cfg["image"], cfg["image"]), step=cfg["step"], shading_mode=mode)
    return tf, cam, spec, settings


def host_volume(cfg):
    """The config's volume as a host VolumeDataset (numpy; bit-identical to the reference generators)."""
    from paper_2008_06134_b200 import datasets
    d = cfg["dims"]
    if cfg["volume"] == "block_u8":
        return datasets.raw_roundtrip(datasets.make_perforated_block((d, d, d), seed=cfg["seed"]), "u8")
    field = np.empty((d, d, d), dtype=np.float32)
    step = max(1, min(d, (1 << 24) // (d * d)))
    for z0 in range(0, d, step):  # z-slabs bound host memory; per-voxel formula unchanged
        field[z0:z0 + step] = _blob_slab(d, cfg["seed"], z0, min(d, z0 + step))
    from paper_2008_06134_b200.scene import VolumeDataset
    if cfg["volume"] == "blobs_u16":
        return datasets.raw_roundtrip(VolumeDataset.from_array(field), "u16")
    return VolumeDataset.from_array(field)


def _blob_slab(d, seed, z0, z1):
    from paper_2008_06134_b200.datasets import _blob_params
    ax = (np.arange(d) + 0.5) / d
    zs = (np.arange(z0, z1) + 0.5) / d
    zz, yy, xx = np.meshgrid(zs, ax, ax, indexing="ij")
    acc = np.zeros_like(xx)
    for c, s, a in _blob_params(seed, 5):
        acc += a * np.exp(-((xx - c[0]) ** 2 + (yy - c[1]) ** 2 + (zz - c[2]) ** 2) / (2.0 * s * s))
    return np.clip(acc, 0.0, 1.0).astype(np.float32)


def device_volume_for(cfg, dev):
    """Generate the config's volume directly in HBM (float64 formula on the GPU)."""
    import torch
    from paper_2008_06134_b200 import datasets
    from paper_2008_06134_b200.device import DeviceVolume
    d = cfg["dims"]
    if cfg["volume"] == "block_u8":
        v = host_volume(cfg)
        return DeviceVolume.from_dataset(v, dev, widen=False), v
    q = "u16" if cfg["volume"] == "blobs_u16" else None
    t = datasets.sphere_blobs_device((d, d, d), seed=cfg["seed"], device=dev, quantize_to=q)
    kind = 2 if q else 0
    one = np.ones(3)
    return DeviceVolume(t, kind, (d, d, d), np.zeros(3), one), None


VOLUME_TYPE = {"blobs": ("f32", 4), "block_u8": ("u8", 1), "blobs_u16": ("u16", 2)}


def workload_config(a, cfg, mode, world):
    """The ``config`` object of the JSON line: the workload only, identical in
    both arms (implementation choices go to ``setup``)."""
    vt, vb = VOLUME_TYPE[cfg["volume"]]
    V, A = cfg["dims"] ** 3 * vb, 4 * cfg["n"] * cfg["res"] ** 2
    return {"workload": f"config {a.config}: {cfg['name']}", "volume": f"{cfg['dims']}^3 {vt}",
            "image": [cfg["image"], cfg["image"]], "n_slices": cfg["n"], "slice_res": [cfg["res"], cfg["res"]],
            "step": cfg["step"], "shading_mode": mode, "parallelism": f"image-tiles x{world}",
            "l2": "inputs larger than L2 (volume %d MiB, buffer %d MiB)" % (V >> 20, A >> 20)}


def host_cpu():
    """CPU model and the cores this process may use (the reference arm's host)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"model": model, "logical_cpus": os.cpu_count(), "usable_cores": cores}


def algorithmic_bytes(cfg, voxel_bytes, world):
    """K1 = V + A (sharded: V + A/G); K2 = V + A + I/G (buffer modes)."""
    V = cfg["dims"] ** 3 * voxel_bytes
    A = 4 * cfg["n"] * cfg["res"] ** 2
    I = 16 * cfg["image"] ** 2
    return V, A, I


def covered_texel_slices(cam, spec) -> int:
    """Texel-slice points of the stack inside the unit cube (the ones K1
    trilinearly samples, lightbuffer.py:182-191): per texel line base + o*L,
    the slab test gives the covered offset interval, counted in slices."""
    w, h = int(cam.resolution[0]), int(cam.resolution[1])
    au, av, L = (np.asarray(x, dtype=np.float64) for x in (cam.axis_u, cam.axis_v, cam.light_dir))
    x = cam.u_range[0] + (np.arange(w) + 0.5) / w * (cam.u_range[1] - cam.u_range[0])
    y = cam.v_range[0] + (np.arange(h) + 0.5) / h * (cam.v_range[1] - cam.v_range[0])
    lo = np.full((h, w), -np.inf)
    hi = np.full((h, w), np.inf)
    for c in range(3):
        base = x[None, :] * au[c] + y[:, None] * av[c]
        if abs(L[c]) < 1e-12:
            out = (base < 0.0) | (base > 1.0)
            lo[out], hi[out] = np.inf, -np.inf
            continue
        a, b = (0.0 - base) / L[c], (1.0 - base) / L[c]
        lo, hi = np.maximum(lo, np.minimum(a, b)), np.minimum(hi, np.maximum(a, b))
    n = int(spec.n_slices)
    sp = (spec.d_max - spec.d_min) / n
    k0 = np.ceil((lo - spec.d_min) / sp - 0.5)
    k1 = np.floor((hi - spec.d_min) / sp - 0.5)
    return int(np.where(hi > lo, np.clip(np.minimum(k1, n - 1) - np.maximum(k0, 0) + 1, 0, None), 0).sum())


def k1_volume_bytes(V, voxel_bytes, covered) -> int:
    """K1's compulsory volume bytes: the whole volume, or — when the stack
    samples fewer cells than there are voxels (small n / slice res) — the 8
    corner voxels of every covered texel-slice, whichever is smaller."""
    return min(V, 8 * voxel_bytes * covered)


# --------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock, power and throttle reasons sampled during the timed region.

    Two samplers run side by side: NVML polled every ~2 ms from a thread
    (tens of samples even in a 50 ms region) and ``nvidia-smi -lms 50`` as a
    backup; the summary uses NVML rows when it got any, else the nvidia-smi
    rows. ``mark()`` brackets the timed region and only samples inside it
    (or the nearest one after its start) are summarised."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.thread = None
        self.rows = []
        self.t0 = self.t1 = None
        self.errors = []

    def _nvml_loop(self, nv, h, bits):
        try:
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception as exc:  # noqa: BLE001
            self.errors.append(f"nvml max clock: {exc!r}")
            return
        reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                rs = reasons(h)
                self.rows.append((time.time(), float(sm), float(mx), pw,
                                  [nm for nm, b in zip(self.NAMES, bits) if rs & b]))
            except Exception as exc:  # noqa: BLE001 - a failed poll is just a missing sample
                if len(self.errors) < 3:
                    self.errors.append(f"nvml poll: {exc!r}")
            self.stop.wait(0.002)

    def __enter__(self):
        import threading
        self.stop = threading.Event()
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(int(self.index))
            bits = tuple(getattr(nv, a, b) for a, b in (
                ("nvmlClocksEventReasonHwSlowdown", 0x8), ("nvmlClocksEventReasonHwThermalSlowdown", 0x40),
                ("nvmlClocksEventReasonSwThermalSlowdown", 0x20), ("nvmlClocksEventReasonSwPowerCap", 0x4)))
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h, bits), daemon=True)
            self.thread.start()
        except Exception as exc:  # noqa: BLE001 - the nvidia-smi sampler still runs
            self.errors.append(f"nvml init: {exc!r}")
            self.thread = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError as exc:
            self.errors.append(f"nvidia-smi: {exc!r}")
            self.proc = None
        time.sleep(0.4)
        return self

    def mark(self, which):
        setattr(self, which, time.time())

    def __exit__(self, *exc):
        time.sleep(0.12)  # one more nvidia-smi period after the region
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=5)
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def _smi_rows(self):
        import datetime as _dt
        if self.proc is None:
            return []
        self.f.flush()
        self.f.seek(0)
        rows = []
        for line in self.f.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                ts = _dt.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(parts[1]), float(parts[2]), float(parts[3]),
                             [nm for nm, val in zip(self.NAMES, parts[4:8]) if val.lower() == "active"]))
            except ValueError:
                continue
        return rows

    def summary(self):
        rows, source = list(self.rows), "nvml"
        if not rows:
            rows, source = self._smi_rows(), "nvidia-smi"
        if not rows:
            return {"sm_mhz": None, "reasons": None, "samples": 0, "errors": self.errors}
        inside = [r for r in rows if self.t0 is not None and self.t0 <= r[0] <= (self.t1 or r[0])]
        if not inside:  # timed region shorter than the sampling period: nearest sample after start
            after = [r for r in rows if self.t0 is None or r[0] >= self.t0]
            inside = after[:1] or rows[-1:]
        reasons = sorted({nm for r in inside for nm in r[4]})
        return {"sm_mhz": statistics.median(r[1] for r in inside), "sm_max_mhz": inside[0][2],
                "power_w_max": max(r[3] for r in inside), "reasons": reasons, "samples": len(inside),
                "window_s": (self.t1 - self.t0) if (self.t0 and self.t1) else None, "source": source,
                **({"errors": self.errors} if self.errors else {})}


# --------------------------------------------------------------- CPU sample
def cpu_sample_plan(cfg, workers: int = 1):
    """Bounded, stratified sample of one frame for the CPU path: every 16th light
    row for the build, full-width image rows for the march — every 16th on one
    core, and on `workers` cores enough rows for 16 per worker. The oracle's
    numpy march has a fixed cost per call and per step, so each worker must get
    as many rays per call as on a whole frame for the extrapolation by row
    count to match a measured full frame (a sparse 85x85 pixel grid overstated
    the CPU frame ~6x, 4 rows per worker ~1.7x: r4f-r4h)."""
    res, img = cfg["res"], cfg["image"]
    bstride = 16 if workers <= 1 else max(1, res // (16 * workers))
    b_rows = np.arange(bstride // 2, res, bstride) if res >= 32 else np.arange(res)
    stride = 16 if workers <= 1 else max(1, img // (16 * workers))
    p_rows = np.arange(stride // 2, img, stride) if img >= 256 else np.arange(img)
    return b_rows, p_rows


_CPU_CTX: dict = {}


def set_cpu_context(vol, tf, cam, spec, settings, intensity):
    """State the CPU workers read (set before forking a pool). The buffer is a
    plain object with the reference AttenuationBuffer's fields."""
    from types import SimpleNamespace
    _CPU_CTX.update(vol=vol, tf=tf, cam=cam, spec=spec, settings=settings,
                    buffer=None if intensity is None else SimpleNamespace(camera=cam, spec=spec, compensation_n=0.0,
                                                                          intensity=intensity))


def _cpu_build_part(args):
    rows, = args
    from oracle import slicecast_oracle as O
    g = _CPU_CTX
    t = time.perf_counter()
    out = O.build_intensity(g["vol"], g["tf"].lut, g["cam"], g["spec"], 0.0, rows=rows)
    return time.perf_counter() - t, out


def _cpu_march_part(args):
    rows, cols = args
    from oracle import slicecast_oracle as O
    g = _CPU_CTX
    t = time.perf_counter()
    img, n = O.render_image(g["vol"], g["tf"].lut, g["settings"], g["buffer"], rows=rows, cols=cols,
                            return_samples=True)
    return time.perf_counter() - t, n, img


def cpu_frame_sample(cfg, workers=1, pool=None):
    """Time the oracle on the bounded sample of one frame; extrapolate to the
    full frame. Returns (frame_seconds, detail, (build_rows_out, march_pixels_out))."""
    b_rows, p_rows = cpu_sample_plan(cfg, workers if pool is not None else 1)
    t0 = time.perf_counter()
    if pool is None:
        built = [_cpu_build_part((b_rows,))[1]]
    else:
        bparts = [b_rows[i::workers] for i in range(workers) if len(b_rows[i::workers])]
        built = [o for _, o in pool.map(_cpu_build_part, [(c,) for c in bparts])]
        border = np.argsort(np.concatenate([np.arange(len(b_rows))[i::workers] for i in range(workers)
                                            if len(b_rows[i::workers])]), kind="stable")
        built = [np.concatenate(built, axis=1)[:, border]]
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    cols = np.arange(cfg["image"])
    if pool is None:
        parts = [_cpu_march_part((p_rows, cols))]
    else:
        # rows dealt round-robin: every worker gets rows from the whole image (balanced cost)
        parts = list(pool.map(_cpu_march_part, [(p_rows[i::workers], cols) for i in range(workers)
                                                if len(p_rows[i::workers])]))
    t_march = time.perf_counter() - t0
    samples = sum(n for _, n, _ in parts)
    full_build = t_build * cfg["res"] / len(b_rows)
    full_march = t_march * cfg["image"] / len(p_rows)
    detail = dict(build_rows=int(len(b_rows)), march_pixels=int(len(p_rows) * cfg["image"]), march_samples=int(samples),
                  build_fraction=len(b_rows) / cfg["res"], march_fraction=len(p_rows) / cfg["image"],
                  t_build_s=t_build, t_march_s=t_march, build_s_extrapolated=full_build,
                  march_s_extrapolated=full_march, extrapolated=True)
    march = np.concatenate([im for _, _, im in parts], axis=0)
    if pool is not None:  # back to p_rows order (rows were dealt round-robin)
        order = np.concatenate([np.arange(len(p_rows))[i::workers] for i in range(workers)
                                if len(p_rows[i::workers])])
        march = march[np.argsort(order, kind="stable")]
    outputs = (np.concatenate(built, axis=1), march)
    return full_build + full_march, detail, outputs


def cpu_sample_text(cfg, workers: int = 1):
    b_rows, p_rows = cpu_sample_plan(cfg, workers)
    return (f"oracle (numpy port of the reference) on a stratified sample of one frame: build on "
            f"{len(b_rows)}/{cfg['res']} light rows, march on {len(p_rows)} full-width rows ({len(p_rows)}x{cfg['image']}) of "
            f"{cfg['image']}x{cfg['image']} pixels; frame time extrapolated by row/pixel count")


# --------------------------------------------------------------- reference arm
def oracle_scene(cfg, mode):
    """The config's inputs built by the oracle's scene port (no product code)."""
    from oracle import scenes as S
    tf = S.preset(cfg["tf"])
    cam = S.light_camera(LIGHT, (1.0, 1.0, 1.0), (cfg["res"], cfg["res"]))
    spec = S.slice_stack(LIGHT, cfg["n"])
    settings = S.render_settings(EYE, TARGET, (cfg["image"], cfg["image"]), cfg["step"], mode, LIGHT)
    d = cfg["dims"]
    if cfg["volume"] == "block_u8":
        _, f = S.raw_roundtrip(S.perforated_block(d, cfg["seed"]), "u8")
        vol = S.volume(f, scalar_type="u8")
    elif cfg["volume"] == "blobs_u16":
        _, f = S.raw_roundtrip(S.blob_field(d, cfg["seed"]), "u16")
        vol = S.volume(f, scalar_type="u16")
    else:
        vol = S.volume(S.blob_field(d, cfg["seed"]))
    return vol, tf, cam, spec, settings


def _full_build(pool, workers, res):
    parts = pool.map(_cpu_build_part, [(c,) for c in np.array_split(np.arange(res), workers) if len(c)])
    return np.concatenate([o for _, o in parts], axis=1)


def reference_full_frame(workers, ctx, cfg_id: int = 2, mode: str | None = None, scene=None):
    """One complete, unextrapolated frame of the reference CPU path (build on
    all light rows, march on every pixel, 4 row bands per core for balance)
    on all host cores. ``scene`` reuses already generated oracle inputs."""
    cfg = CONFIGS[cfg_id]
    vol, tf, cam, spec, settings = scene if scene is not None else oracle_scene(cfg, mode or cfg["mode"])
    set_cpu_context(vol, tf, cam, spec, settings, None)
    with ctx.Pool(workers) as pool:
        t0 = time.perf_counter()
        inten = _full_build(pool, workers, cfg["res"])
        t_build = time.perf_counter() - t0
        set_cpu_context(vol, tf, cam, spec, settings, inten)
    with ctx.Pool(workers) as pool:  # forked after the stack exists
        t0 = time.perf_counter()
        rows = np.arange(cfg["image"])
        parts = pool.map(_cpu_march_part, [(r, rows) for r in np.array_split(rows, 4 * workers) if len(r)])
        t_march = time.perf_counter() - t0
    frame = t_build + t_march
    return {"config": f"config {cfg_id}: {cfg['name']}", "fps": 1.0 / frame, "frame_s": frame, "build_s": t_build,
            "march_s": t_march, "samples": int(sum(n for _, n, _ in parts)), "cores": workers,
            "extrapolated": False}


def run_reference(a, cfg, mode):
    """The reference's CPU path (the oracle port: the reference is Python, so
    nothing compiles into oracle/_ref) on all host cores, rank 0 only. Imports
    nothing from the product package."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    import multiprocessing as mp
    vol, tf, cam, spec, settings = oracle_scene(cfg, mode)
    host = host_cpu()
    workers = host["usable_cores"]
    ctx = mp.get_context("fork")
    inten = None
    if mode in ("sbrc_shadow", "shell", "cone"):  # the march reads the full stack: built once, untimed
        set_cpu_context(vol, tf, cam, spec, settings, None)
        with ctx.Pool(workers) as pool:
            inten = _full_build(pool, workers, cfg["res"])
    set_cpu_context(vol, tf, cam, spec, settings, inten)
    with ctx.Pool(workers) as pool:
        for _ in range(a.warmup):
            cpu_frame_sample(cfg, workers, pool)
        times, walls = [], []
        detail = None
        for _ in range(a.steps):
            w0 = time.perf_counter()
            ft, detail, _ = cpu_frame_sample(cfg, workers, pool)
            walls.append(time.perf_counter() - w0)
            times.append(ft)
    frame_s = statistics.median(times)
    fps = 1.0 / frame_s
    full = None if a.no_full_frame else reference_full_frame(workers, ctx)
    # the benchmarked workload itself, complete and unextrapolated (config 3: ~20 s on 16 cores)
    full_cfg = None if (a.no_full_frame or a.config not in (1, 3)) else \
        reference_full_frame(workers, ctx, a.config, mode, scene=(vol, tf, cam, spec, settings))
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": frame_s * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(a, cfg, mode, world),
        "setup": {"cpu": host, "processes": workers, "path": "oracle/slicecast_oracle.py (numpy restatement "
                  "of slicecast, bit-identical on the golden fixtures), fork pool over light rows / image rows"},
        "extrapolated": True,
        "sample_ms_per_step": statistics.median(walls) * 1e3,
        "gsamples_per_s": detail["march_samples"] / max(detail["t_march_s"], 1e-12) / 1e9,
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": workers, "kind": "port",
                         "sample": cpu_sample_text(cfg, workers), "cpu_model": host["model"], "detail": detail},
        "full_frame_config2": full,
        "full_frame": full_cfg,
        "product_package_loaded": any(m.split(".")[0] == "paper_2008_06134_b200" for m in sys.modules),
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm
def run_ours(a, cfg, mode):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SBRC_BENCH_SAME_GPU=1 + SBRC_BENCH_BACKEND=gloo: every rank on cuda:0 — a
    # control-flow check of the multi-rank bench on a one-GPU box (NCCL needs
    # distinct GPUs); timings of such a run mean nothing.
    if os.environ.get("SBRC_BENCH_SAME_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("SBRC_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    import paper_2008_06134_b200 as sb
    from paper_2008_06134_b200.frame import FramePipeline, FrameRenderer

    tf, cam, spec, settings = scene_objects(cfg, mode)
    t0 = time.perf_counter()
    bcast_ms = None
    if world > 1:
        # rank 0 makes the dataset, one broadcast replicates it, timed on its own
        from paper_2008_06134_b200.device import broadcast_volume
        dvol, host_vol = device_volume_for(cfg, dev) if rank == 0 else (None, None)
        d = cfg["dims"]
        vt = {"blobs": 0, "block_u8": 1, "blobs_u16": 2}[cfg["volume"]]
        torch.cuda.synchronize()
        dist.barrier()
        tb = time.perf_counter()
        dvol = broadcast_volume(dvol, (d, d, d), vt, np.zeros(3), np.ones(3), dev)
        torch.cuda.synchronize()
        bcast_ms = (time.perf_counter() - tb) * 1e3
    else:
        dvol, host_vol = device_volume_for(cfg, dev)
    if not a.raw_voxels:
        dvol = dvol.widened()
    torch.cuda.synchronize()
    vol_gen_s = time.perf_counter() - t0
    fr = FrameRenderer(dvol, tf, cam, spec, settings, build=a.build if world > 1 else "replicated",
                       band_rows=8, device=dev, assemble=a.assemble,
                       heavy_first={"auto": None, "heavy": True, "natural": False, "measured": True}[a.tile_order],
                       feedback={"auto": None, "heavy": False, "natural": False, "measured": True}[a.tile_order])
    stream = torch.cuda.current_stream()

    # samples per frame (deterministic): one counted frame
    fr.reset_counter()
    fr.frame()
    torch.cuda.synchronize()
    samples = int(fr.counter.item())
    if world > 1:
        t = torch.tensor([samples], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        samples = int(t.item())

    if world > 1 and a.build == "frustum":
        # contiguous bands cut from measured per-rank frame times, each rank's K2 kernel measured too
        fr.calibrate()
        fr.frame()
    pipelined = (world == 1 or a.build in ("replicated", "frustum")) and not a.no_pipeline
    pipe = FramePipeline(fr) if pipelined else None

    def one_step(ev=None):
        if pipe is not None:  # build(f+1) on the build stream overlaps march(f)
            pipe.step()
            return
        if ev is not None:
            ev[0].record(stream)
        fr.build()
        if ev is not None:
            ev[1].record(stream)
        fr.march(count_samples=False)
        if ev is not None:
            ev[2].record(stream)
        fr.assemble()
        if ev is not None:
            ev[3].record(stream)

    for _ in range(a.warmup):
        one_step()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(a.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        clocks.mark("t0")
        start.record(stream)
        for i in range(a.steps):
            one_step(evs[i])
        if pipe is not None:
            pipe.drain()  # the build launched by the last step is inside the timed region
        end.record(stream)
        torch.cuda.synchronize()
        clocks.mark("t1")
    if world > 1:
        dist.barrier()
    total_ms = start.elapsed_time(end)
    if pipe is None:
        k1 = [e[0].elapsed_time(e[1]) for e in evs]
        k2 = [e[1].elapsed_time(e[2]) for e in evs]
        asm = [e[2].elapsed_time(e[3]) for e in evs]
    else:  # overlapped kernels: per-kernel times from a short serial run after the timed region
        ser = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(5)]
        fr.quads = pipe.bufs[0]
        for e in ser:
            e[0].record(stream)
            fr.build()
            e[1].record(stream)
            fr.march(count_samples=False)
            e[2].record(stream)
            fr.assemble()
            e[3].record(stream)
        torch.cuda.synchronize()
        k1 = [e[0].elapsed_time(e[1]) for e in ser]
        k2 = [e[1].elapsed_time(e[2]) for e in ser]
        asm = [e[2].elapsed_time(e[3]) for e in ser]
    stats = torch.tensor([total_ms, sum(k1) / len(k1), sum(k2) / len(k2), sum(asm) / len(asm)],
                         dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    total_ms, k1_ms, k2_ms, asm_ms = stats.tolist()
    ms_per_step = total_ms / a.steps
    fps = 1000.0 / ms_per_step

    # ---- end to end through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        e2e = e2e_public(a, cfg, tf, cam, spec, settings, dvol, host_vol, fr, world, dev)

    # ---- roofline of the dominant kernel
    vbytes = {0: 4, 1: 1, 2: 2}[dvol.source_type]  # algorithmic V counts the source bytes per voxel
    V, A, I = algorithmic_bytes(cfg, vbytes, world)
    k1_bytes = k1_volume_bytes(V, vbytes, covered_texel_slices(cam, spec)) + \
        (A if (world == 1 or a.build != "sharded") else A // world)
    k2_bytes = (V + A + I // world) if mode != "none" else (V + I // world)
    peaks = load_peaks()
    dominant = "march" if k2_ms >= k1_ms else "build"
    d_bytes, d_ms = (k2_bytes, k2_ms) if dominant == "march" else (k1_bytes, k1_ms)
    achieved = d_bytes / (d_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "peak_source": peaks["source"],
                "algorithmic_bytes": d_bytes, "kernel_ms": d_ms,
                "traffic": load_traffic(a.config, mode, dominant)}
    if fr.needs_buffer:
        roofline_k1 = {"bound": "hbm", "kernel": "build", "achieved": k1_bytes / (k1_ms * 1e-3) / 1e9,
                       "peak": peaks["hbm_gbs"], "unit": "GB/s", "algorithmic_bytes": k1_bytes, "kernel_ms": k1_ms,
                       "traffic": load_traffic(a.config, mode, "build")}
        roofline_k1["frac"] = roofline_k1["achieved"] / peaks["hbm_gbs"]
    else:  # none / phong / extinction read no attenuation stack: no K1 in the frame
        roofline_k1 = None
    # Secondary view of K2: the bytes its gathers pull through L1/L2 per sample
    # (8 voxels + 2 16-byte texel quads per light lookup) against the SM-side
    # L1 data bandwidth (128 B/clk/SM at the max SM clock). The march is bound
    # there (and by load latency), not by HBM (DRAM ~2% busy, L1 hit ~95%).
    lookups = {"none": 0, "sbrc_shadow": 1, "shell": 18, "cone": 8, "phong": 0, "extinction": 0}.get(mode, 0)
    gathered = samples * (8 * vbytes + 32 * lookups)
    l1_peak = 148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e9
    l1 = {"bound": "l1", "kernel": "march", "achieved": gathered / (k2_ms * 1e-3) / 1e9, "peak": l1_peak,
          "unit": "GB/s", "bytes_per_sample": 8 * vbytes + 32 * lookups}
    l1["frac"] = l1["achieved"] / l1_peak

    cpu, parity = None, None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        inten = fr.intensity.contiguous().cpu().numpy() if mode in ("sbrc_shadow", "shell", "cone") else None
        image = fr.assemble().cpu().numpy()
        cpu, parity = cpu_baseline_leg(cfg, tf, cam, spec, settings, dvol, host_vol, inten, image)
    full2 = None
    if rank == 0 and world == 1 and not a.no_full_frame and a.config != 2:
        full2 = gpu_full_frame_config2(dev)

    if rank == 0:
        line = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
            "config": workload_config(a, cfg, mode, world),
            "setup": {"build": a.build if world > 1 else "single",
                      "row_ranges": fr.ranges if fr.partition == "contiguous" else None,
                      "march_kernel": {0: "by size", 1: "throughput", 2: "latency"}[fr.march_kernel],
                      "assemble": fr.assemble_mode if world > 1 else "none",
                      "frame_pipelining": "build(f+1) overlaps march(f)" if pipelined else "off",
                      "tile_order": "measured (previous frame)" if fr.feedback is not None else
                      ("ray length" if (fr.world != 2 if fr.heavy_first is None else fr.heavy_first) else "natural"),
                      "volume_in_hbm": "float32" if dvol.voxel_type == 0 else "raw"},
            "gsamples_per_s": samples / (k2_ms * 1e-3) / 1e9,
            "samples_per_frame": samples,
            "march_only_fps": 1000.0 / (k2_ms + asm_ms),
            "kernels": {"build_ms": k1_ms, "march_ms": k2_ms, "assemble_ms": asm_ms,
                        "build_gbs": k1_bytes / (k1_ms * 1e-3) / 1e9 if fr.needs_buffer else None,
                        "march_gbs": k2_bytes / (k2_ms * 1e-3) / 1e9,
                        "build_gtexel_slices_s": cfg["n"] * cfg["res"] ** 2 / (k1_ms * 1e-3) / 1e9
                        if fr.needs_buffer else None},
            "roofline": roofline,
            "roofline_build": roofline_k1,
            "roofline_l1": l1,
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_full_frame_config2": full2,
            # per frame: K1 (if the mode reads a buffer) + K2, plus the measured
            # heavy-first sort (sbrc_tile_order) and the NCCL assembly's row permutation at N > 1
            "gpu_launches": a.steps * (int(fr.needs_buffer) + 1 + int(fr.feedback is not None)
                                       + int(world > 1 and fr.assemble_mode == "nccl")),
            "clocks": clocks.summary(),
            "volume_gen_s": vol_gen_s,
            "volume_broadcast_ms": bcast_ms,
        }
        print(json.dumps(line), flush=True)
    fr.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_public(a, cfg, tf, cam, spec, settings, dvol, host_vol, fr, world, dev):
    """Same frame through the public API with host buffers: LUTs and slice
    offsets copied host->device every step, the image read back to host
    (at N=1 ``render`` has K2 store the pixels into a page-locked host array
    over PCIe during the march: the same 16 bytes per pixel cross to the host).
    The volume is uploaded once (device cache keyed by the host array, as the
    reference service keeps datasets resident) and that upload is reported
    separately."""
    import torch
    import paper_2008_06134_b200 as sb
    if host_vol is None:
        from paper_2008_06134_b200.scene import VolumeDataset
        raw = dvol.data.cpu().numpy()
        if dvol.voxel_type == 0:
            host_vol = VolumeDataset.from_array(raw)
        else:
            host_vol = VolumeDataset.from_raw_array(raw.view(np.uint16) if dvol.voxel_type == 2 else raw)
    t0 = time.perf_counter()
    if world == 1:
        from paper_2008_06134_b200.device import device_volume
        device_volume(host_vol, dev)
        torch.cuda.synchronize()
    upload_s = time.perf_counter() - t0
    n = int(spec.n_slices)
    h2d = 256 * 4 * 8 + 256 * 8 + n * 8
    d2h = cfg["image"] ** 2 * 16

    host_img = None
    if world > 1:  # page-locked landing buffer for the assembled image (one async D2H per frame)
        host_img = torch.empty((cfg["image"], cfg["image"], 4), dtype=torch.float32).pin_memory()

    from paper_2008_06134_b200.device import drop_frame_constants

    def step():
        if world == 1:
            # every step uploads its own constants (resolved LUTs, slice offsets):
            # the value cache that would skip unchanged ones is dropped first
            drop_frame_constants()
            buf = sb.build_attenuation_buffer(host_vol, tf, cam, spec)
            img = sb.render(host_vol, tf, settings, buf)
        else:
            # this step's constants, host -> device from page-locked memory
            for dst, src in ((fr.lut, tf.resolve(settings.step)), (fr.alpha, tf.resolve(spec.spacing)[:, 3]),
                             (fr.offsets, spec.plane_offsets)):
                dst.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64)).pin_memory(),
                          non_blocking=True)
            host_img.copy_(fr.frame(), non_blocking=True)
            torch.cuda.current_stream().synchronize()
            img = host_img.numpy()
        return img

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    k = max(3, a.steps // 2)
    for _ in range(k):
        step()
    torch.cuda.synchronize()
    el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    sec = el.item() / k
    return {"value": 1.0 / sec, "unit": "frames/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": sec * 1e3, "steps": k, "volume_upload_s_once": upload_s,
            "path": "paper_2008_06134_b200.build_attenuation_buffer + render (numpy in, numpy out; "
                    "the resolved LUTs and slice offsets uploaded every step; K2 stores the image into "
                    "pinned host memory)"
            if world == 1 else "FrameRenderer (host LUTs in, host image out)"}


def cpu_baseline_leg(cfg, tf, cam, spec, settings, dvol, host_vol, intensity, image):
    """The oracle port, single thread, on the bounded sample of this workload,
    and the parity of this run's GPU frame against it: the sampled light rows
    of the stack (bit-exact expected) and the sampled pixels of the image
    (north_star tolerance 1e-3; the tests assert 1e-4). The sampled march reads
    the GPU-built stack, which the row check shows is the oracle's."""
    from paper_2008_06134_b200.scene import VolumeDataset
    if host_vol is None:
        raw = dvol.data.cpu().numpy()
        host_vol = VolumeDataset.from_array(raw) if dvol.voxel_type == 0 else \
            VolumeDataset.from_raw_array(raw.view(np.uint16) if dvol.voxel_type == 2 else raw)
    set_cpu_context(host_vol, tf, cam, spec, settings, intensity)
    frame_s, detail, (rows_cpu, pix_cpu) = cpu_frame_sample(cfg)
    b_rows, p_rows = cpu_sample_plan(cfg)
    parity = {"rows": int(len(b_rows)), "pixels": int(len(p_rows) * cfg["image"]), "tolerance": 1e-3}
    if intensity is not None:
        got = intensity[:, b_rows]
        parity["build_rows_bit_exact"] = bool(np.array_equal(got, rows_cpu))
        parity["build_max_abs"] = float(np.abs(got.astype(np.float64) - rows_cpu).max())
    got = image[p_rows].astype(np.float64)
    d = np.abs(got - pix_cpu.astype(np.float64))
    mse = float(np.mean(d * d))
    parity.update(max_abs=float(d.max()), psnr=float("inf") if mse == 0 else 10.0 * math.log10(1.0 / mse),
                  over_1e_3=int((d > 1e-3).sum()), over_1e_4=int((d > 1e-4).sum()))
    cpu = {"value": 1.0 / frame_s, "unit": "frames/s", "cores": 1, "kind": "port", "sample": cpu_sample_text(cfg),
           "cpu_model": host_cpu()["model"], "detail": detail}
    return cpu, parity


def gpu_full_frame_config2(dev, frames: int = 20):
    """Config 2 (256^3 u8 block -> 512^2, 128 slices, sbrc_shadow) on this GPU:
    the same complete frame the reference arm times unextrapolated
    (``full_frame_config2``), device-timed over ``frames`` frames."""
    import torch
    from paper_2008_06134_b200.frame import FrameRenderer
    cfg = CONFIGS[2]
    tf, cam, spec, settings = scene_objects(cfg, cfg["mode"])
    dvol, _ = device_volume_for(cfg, dev)
    fr = FrameRenderer(dvol.widened(), tf, cam, spec, settings, device=dev)
    for _ in range(3):
        fr.frame()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(frames):
        fr.build()
        fr.march(count_samples=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / frames
    fr.close()
    return {"config": f"config 2: {cfg['name']}", "fps": 1000.0 / ms, "ms_per_frame": ms, "frames": frames,
            "timing": "CUDA events, build + march per frame, no pipelining"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


def load_traffic(config, mode, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(f"config{config}/{mode}/{kernel}")
        return None if e is None else e["bytes"]
    except (OSError, ValueError):
        return None


def run_sweep(a, cfg, mode):
    """Config 5: moving light, buffer rebuilt every frame, over slices x slice resolution."""
    import torch
    from paper_2008_06134_b200 import scene
    from paper_2008_06134_b200.frame import FrameRenderer
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tf, cam, spec, settings = scene_objects(cfg, mode)
    dvol, _ = device_volume_for(cfg, dev)
    fr = FrameRenderer(dvol, tf, cam, spec, settings, device=dev)
    host_vol = None
    if not a.no_cpu_baseline:
        from paper_2008_06134_b200.scene import VolumeDataset
        host_vol = VolumeDataset.from_array(dvol.data.cpu().numpy())
    stream = torch.cuda.current_stream()
    rows = []
    frames = cfg["frames"]
    peak = load_peaks()["hbm_gbs"]
    for n in cfg["sweep_n"]:
        for res in cfg["sweep_res"]:
            lights = [orbit_light(360.0 * f / frames, 30.0) for f in range(frames)]
            prepared = [fr.prepare_light(scene.LightCamera.fit(ld, (1, 1, 1), (res, res)),
                                         scene.make_slice_stack(ld, n)) for ld in lights]
            for f in range(max(a.warmup, 3)):
                fr.use_light(prepared[f % frames])
                fr.frame()
            torch.cuda.synchronize()
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(frames)]
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(stream)
            for f in range(frames):
                fr.use_light(prepared[f])
                ev[f][0].record(stream)
                fr.build()
                ev[f][1].record(stream)
                fr.march(count_samples=False)
                fr.assemble()
                ev[f][2].record(stream)
            end.record(stream)
            torch.cuda.synchronize()
            ms = start.elapsed_time(end) / frames
            b = sum(e[0].elapsed_time(e[1]) for e in ev) / frames
            m = sum(e[1].elapsed_time(e[2]) for e in ev) / frames
            V = cfg["dims"] ** 3 * 4
            A = 4 * n * res * res
            I = 16 * cfg["image"] ** 2
            cov = sum(covered_texel_slices(c, s_) for c, s_, _, _ in prepared[::4]) // len(prepared[::4])
            K1 = k1_volume_bytes(V, 4, cov) + A
            rows.append({"n_slices": n, "slice_res": res, "fps": 1000.0 / ms, "ms_per_frame": ms,
                         "build_ms": b, "march_ms": m,
                         "build_gtexel_slices_s": n * res * res / (b * 1e-3) / 1e9,
                         "covered_texel_slices": cov,
                         "roofline_build": {"algorithmic_bytes": K1, "achieved_gbs": K1 / (b * 1e-3) / 1e9,
                                            "frac": K1 / (b * 1e-3) / 1e9 / peak},
                         "roofline_march": {"algorithmic_bytes": V + A + I,
                                            "achieved_gbs": (V + A + I) / (m * 1e-3) / 1e9,
                                            "frac": (V + A + I) / (m * 1e-3) / 1e9 / peak}})
            if not a.no_cpu_baseline:
                rows[-1]["parity"] = sweep_point_parity(cfg, fr, tf, host_vol)
            fr.set_light(cam, spec)  # release the large buffer before the next shape
            torch.cuda.empty_cache()
    head = next(r for r in rows if r["n_slices"] == 256 and r["slice_res"] == 512)
    line = {"metric": METRIC, "value": head["fps"], "unit": "frames/s", "n_gpus": 1, "steps": frames,
            "warmup": max(a.warmup, 3), "ms_per_step": head["ms_per_frame"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(a, cfg, mode, 1), value_at="n=256, res=512"),
            "sweep": rows, "gpu_launches": 2 * frames * len(rows)}
    print(json.dumps(line), flush=True)
    return 0


def sweep_point_parity(cfg, fr, tf, host_vol, pixels: int = 8):
    """Oracle check of the last frame of a sweep point (its orbit light): two
    light rows of the stack (bit-exact expected) and, when the stack is small
    enough to copy to the host, a pixels x pixels grid of the image."""
    from oracle import slicecast_oracle as O
    from types import SimpleNamespace
    cam, spec = fr.cam, fr.spec
    res = int(cam.resolution[1])
    b_rows = np.array([res // 3, (2 * res) // 3])
    want = O.build_intensity(host_vol, tf.lut, cam, spec, rows=b_rows)
    got = fr.intensity[:, b_rows].contiguous().cpu().numpy()
    out = {"build_rows": b_rows.tolist(), "build_rows_bit_exact": bool(np.array_equal(got, want))}
    if int(spec.n_slices) * res * res <= (1 << 26):
        img = fr.frame().cpu().numpy()
        buf = SimpleNamespace(camera=cam, spec=spec, compensation_n=0.0,
                              intensity=fr.intensity.contiguous().cpu().numpy())
        pix = np.linspace(cfg["image"] // (2 * pixels), cfg["image"] - 1, pixels).astype(int)
        want_img = O.render_image(host_vol, tf.lut, fr.settings, buf, rows=pix, cols=pix)
        d = np.abs(img[np.ix_(pix, pix)].astype(np.float64) - want_img)
        out.update(pixels=int(pixels * pixels), max_abs=float(d.max()), over_1e_3=int((d > 1e-3).sum()))
    return out


def main():
    a = parse()
    cfg = CONFIGS[a.config]
    mode = a.mode or cfg["mode"]
    if a.impl == "reference":
        return run_reference(a, cfg, mode)
    if a.config == 5:
        # the sweep is a single-GPU measurement: under torchrun rank 0 runs it, the others exit
        if int(os.environ.get("RANK", "0")) != 0:
            return 0
        return run_sweep(a, cfg, mode)
    return run_ours(a, cfg, mode)


if __name__ == "__main__":
    sys.exit(main())
