"""ORACLE — CPU restatement of the reference hot path. TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and the ``--impl reference`` arm) may import this
module, and only as the checker / the timed CPU baseline — never as part of
the product path (the package ``paper_2008_06134_b200`` has no CPU path).

What it restates: the numpy implementation in the reference package
``slicecast`` (/root/reference/pkg/src/slicecast, arXiv 2008.06134), with
the same float64 operation order so that results agree bit for bit:

- ``trilinear``          volume.py:161-194  (sample_trilinear_many)
- ``lut_blend``          transfer.py:93-100 (lut_interp_many), lightbuffer.py:188-192
- ``resolve``            transfer.py:76-84  (TransferFunction.resolve)
- ``build_intensity``    lightbuffer.py:134-199 (build_attenuation_buffer, Alg. 1)
- ``light_uv``           lightbuffer.py:202-212 (world_to_light_uv_many)
- ``lookup_scalar``      lightbuffer.py:238-287 (lookup_light_scalar_many)
- ``shell_scalar``       raycaster.py:239-250
- ``cone_scalar``        raycaster.py:261-300
- ``light_factor``       raycaster.py:197-201
- ``camera_rays``        raycaster.py:53-68
- ``box_hit``            geometry.py:46-67
- ``march``              raycaster.py:415-440 (_march_rays) with _make_shader :376-412
- ``render_image``       raycaster.py:443-469
- ``gradient``           volume.py:201-220 (gradient_many)
- ``phong_scalar``       raycaster.py:204-220
- ``light_march``        raycaster.py:312-353 (_extinction_scalar, _shadow_oracle_scalar)
- ``shadow_oracle``      raycaster.py:356-366 (shadow_oracle_many)
- ``half_angle``         halfangle.py:35-142 (render_half_angle)

Deliberate restatement choices (semantics-neutral):
the build evaluates every texel of each slice instead of the polygon's
±1-texel bounding window, since texels outside the window are never
covered. Inputs are duck-typed: objects with the reference's attribute
names (``dims``, ``data``, ``box_lo``, ``camera.axis_u``, ...).

Parity pinned: ``tests/test_oracle_golden.py`` compares every function here
with outputs of the reference itself, stored in ``tests/golden/*.npz`` by
``tests/golden/make_golden.py`` (which imports /root/reference in the build
container).
"""

from __future__ import annotations

import math

import numpy as np

LUT_SIZE = 256
OPACITY_REF_STEP = 1.0 / 256.0


# ------------------------------------------------------------ primitives
def _unit(vec) -> np.ndarray:
    arr = np.asarray(vec, dtype=np.float64)
    return arr / float(np.linalg.norm(arr))


def _light_plane_u(direction) -> np.ndarray:
    """First axis of geometry.plane_basis (geometry.py:31-43)."""
    w = _unit(direction)
    hint = np.array([0.0, 1.0, 0.0])
    if abs(float(np.dot(hint, w))) > 1.0 - 1e-9:
        hint = np.array([0.0, 0.0, 1.0])
    return _unit(np.cross(hint, w))


def resolve(lut: np.ndarray, step: float) -> np.ndarray:
    """Opacity correction + premultiplication of a (256, 4) LUT (transfer.py:76-84)."""
    a = 1.0 - np.power(1.0 - lut[:, 3], step / OPACITY_REF_STEP)
    res = np.empty_like(lut)
    res[:, :3] = lut[:, :3] * a[:, None]
    res[:, 3] = a
    return res


def _lerp(a, b, w):
    return a * (1 - w) + b * w


def trilinear(vol, pts) -> np.ndarray:
    """Clamp-to-edge cell-centred trilinear; 0 outside [0,1]^3 (volume.py:161-194)."""
    pts = np.asarray(pts, dtype=np.float64)
    q = pts.reshape(-1, 3)
    res = np.zeros(q.shape[0], dtype=np.float64)
    ok = np.all((q >= 0.0) & (q <= 1.0), axis=1)
    if ok.any():
        dims = np.array(vol.dims, dtype=np.float64)
        local = (q[ok] - vol.box_lo) / (vol.box_hi - vol.box_lo)
        np.clip(local, 0.0, 1.0, out=local)
        g = local * dims - 0.5
        lo = np.floor(g).astype(np.intp)
        frac = g - lo
        top = np.array(vol.dims, dtype=np.intp) - 1
        a = np.clip(lo, 0, top)
        b = np.clip(lo + 1, 0, top)
        grid = vol.data
        wx, wy, wz = frac[:, 0], frac[:, 1], frac[:, 2]
        # data is (nz, ny, nx): index [z, y, x]
        row00 = _lerp(grid[a[:, 2], a[:, 1], a[:, 0]], grid[a[:, 2], a[:, 1], b[:, 0]], wx)
        row10 = _lerp(grid[a[:, 2], b[:, 1], a[:, 0]], grid[a[:, 2], b[:, 1], b[:, 0]], wx)
        row01 = _lerp(grid[b[:, 2], a[:, 1], a[:, 0]], grid[b[:, 2], a[:, 1], b[:, 0]], wx)
        row11 = _lerp(grid[b[:, 2], b[:, 1], a[:, 0]], grid[b[:, 2], b[:, 1], b[:, 0]], wx)
        res[ok] = _lerp(_lerp(row00, row10, wy), _lerp(row01, row11, wy), wz)
    return res.reshape(pts.shape[:-1])


def lut_blend(table: np.ndarray, s: np.ndarray) -> np.ndarray:
    """Linear LUT interpolation at clamped scalars (transfer.py:93-100).

    ``table`` is (256,) or (256, k). The builder's variant
    (lightbuffer.py:188-192) truncates instead of flooring, which is the
    same for the non-negative clamped index."""
    t = np.clip(s, 0.0, 1.0) * (LUT_SIZE - 1)
    i0 = np.floor(t).astype(np.intp)
    i1 = np.minimum(i0 + 1, LUT_SIZE - 1)
    f = t - i0
    if table.ndim == 2:
        f = f[..., None]
    return table[i0] * (1.0 - f) + table[i1] * f


# ------------------------------------------------------------ K1: the build
def build_intensity(vol, tf_lut: np.ndarray, cam, spec, compensation_n: float = 0.0,
                    rows=None) -> np.ndarray:
    """(n, H, W) float32 incoming intensity per slice (lightbuffer.py:144-199).

    ``tf_lut`` is the raw (256, 4) TransferFunction.lut; it is resolved to
    the slice spacing here (:159-160). ``rows`` optionally restricts the
    build to a subset of light-texel rows (texels are independent), giving
    (n, len(rows), W) — used for bounded CPU baselines."""
    alpha = np.ascontiguousarray(resolve(tf_lut, spec.spacing)[:, 3])
    w, h = cam.resolution
    (u0, u1), (v0, v1) = cam.u_range, cam.v_range
    ucol = u0 + (np.arange(w, dtype=np.float64) + 0.5) / w * (u1 - u0)
    vrow = v0 + (np.arange(h, dtype=np.float64) + 0.5) / h * (v1 - v0)
    if rows is not None:
        vrow = vrow[np.asarray(rows)]
        h = vrow.shape[0]
    ug, vg = np.meshgrid(ucol, vrow)
    plane = ug[..., None] * cam.axis_u + vg[..., None] * cam.axis_v
    light = spec.light_dir
    trans = np.ones((h, w), dtype=np.float64)
    out = np.empty((spec.n_slices, h, w), dtype=np.float32)
    for k in range(spec.n_slices):
        out[k] = trans
        p = plane + float(spec.plane_offsets[k]) * light
        hit = np.all((p >= 0.0) & (p <= 1.0), axis=-1)
        if not hit.any():
            continue
        a = lut_blend(alpha, trilinear(vol, p[hit]))
        if compensation_n > 0.0:
            layer = out[k]
            layer[hit] = layer[hit] * np.power(1.0 + a, compensation_n)
        trans[hit] *= 1.0 - a
    return out


# ------------------------------------------------------------ light lookups
def light_uv(cam, pts: np.ndarray) -> np.ndarray:
    """Shadow-matrix projection to [0,1]^2 light uv (lightbuffer.py:202-212)."""
    m = cam.shadow_matrix
    clip = pts @ m[:3, :3].T + m[:3, 3]
    ww = pts @ m[3, :3] + m[3, 3]
    return (clip[:, :2] / ww[:, None] + 1.0) / 2.0


def _stack_bilinear(stack: np.ndarray, k: np.ndarray, uv: np.ndarray) -> np.ndarray:
    """Clamp-to-edge bilinear in per-point layers (lightbuffer.py:238-253)."""
    h, w = stack.shape[1:]
    tx = uv[:, 0] * w - 0.5
    ty = uv[:, 1] * h - 0.5
    xi = np.floor(tx).astype(np.intp)
    yi = np.floor(ty).astype(np.intp)
    fx, fy = tx - xi, ty - yi
    xa, xb = np.clip(xi, 0, w - 1), np.clip(xi + 1, 0, w - 1)
    ya, yb = np.clip(yi, 0, h - 1), np.clip(yi + 1, 0, h - 1)
    top = stack[k, ya, xa] * (1 - fx) + stack[k, ya, xb] * fx
    bot = stack[k, yb, xa] * (1 - fx) + stack[k, yb, xb] * fx
    return top * (1 - fy) + bot * fy


def lookup_scalar(intensity: np.ndarray, cam, spec, pts, mode: str = "linear") -> np.ndarray:
    """Light factor relative to light_color at world points (lightbuffer.py:256-287)."""
    if mode not in ("nearest", "linear"):
        raise ValueError(f"unknown lookup mode {mode!r}")
    pts = np.asarray(pts, dtype=np.float64)
    q = pts.reshape(-1, 3)
    uv = light_uv(cam, q)
    ok = np.all((uv >= 0.0) & (uv <= 1.0), axis=1)
    res = np.ones(q.shape[0], dtype=np.float64)
    if ok.any():
        n = spec.n_slices
        idx = n * (q[ok] @ spec.light_dir - spec.d_min) / (spec.d_max - spec.d_min)
        if mode == "nearest":
            k = np.clip(np.floor(np.clip(idx, 0.0, n - 1.0)), 0, n - 1).astype(np.intp)
            res[ok] = _stack_bilinear(intensity, k, uv[ok])
        else:
            li = np.clip(idx - 0.5, 0.0, n - 1.0)
            k0 = np.minimum(np.floor(li).astype(np.intp), n - 1)
            k1 = np.minimum(k0 + 1, n - 1)
            f = li - k0
            res[ok] = (_stack_bilinear(intensity, k0, uv[ok]) * (1.0 - f)
                       + _stack_bilinear(intensity, k1, uv[ok]) * f)
    return res.reshape(pts.shape[:-1])


def shell_scalar(intensity, cam, spec, pts, radii, weights, mode="linear") -> np.ndarray:
    """Weighted mean of 6 axis taps per shell (raycaster.py:239-250)."""
    total = np.zeros(pts.shape[0], dtype=np.float64)
    for r, wgt in zip(radii, weights):
        ring = np.zeros(pts.shape[0], dtype=np.float64)
        for axis in range(3):
            for sgn in (1.0, -1.0):
                tap = pts.copy()
                tap[:, axis] += sgn * r
                ring += lookup_scalar(intensity, cam, spec, tap, mode)
        total += wgt * ring / 6.0
    return total


def cone_scalar(intensity, cam, spec, pts, axis_samples, angles, ring_per_step, eye,
                mode="linear") -> np.ndarray:
    """Mean of ring taps on a cone opening toward the light (raycaster.py:266-300)."""
    l = spec.light_dir
    m = pts.shape[0]
    fb = _light_plane_u(l)
    if eye is None:
        basis = np.tile(fb, (m, 1))
    else:
        e = eye - pts
        basis = e - (e @ l)[:, None] * l
        nrm = np.linalg.norm(basis, axis=-1)
        good = nrm > 1e-12
        basis[good] /= nrm[good][:, None]
        basis[~good] = fb
    total = np.zeros(m, dtype=np.float64)
    taps = 0
    for i in range(1, axis_samples + 1):
        dist = i * spec.spacing
        centre = pts + dist * (-l)
        radius = ring_per_step * dist
        for th in angles:
            c, s = math.cos(th), math.sin(th)
            rot = basis * c + np.cross(l, basis) * s + l * (basis @ l)[:, None] * (1.0 - c)
            perp = rot - (rot @ l)[:, None] * l
            pn = np.linalg.norm(perp, axis=-1)
            pn = np.where(pn > 1e-12, pn, 1.0)
            total += lookup_scalar(intensity, cam, spec, centre + radius * perp / pn[:, None], mode)
            taps += 1
    return total / taps


def light_factor(scalar: np.ndarray, color: np.ndarray, floor: float) -> np.ndarray:
    """max(s*c, floor)/c per channel, 1 where c == 0 (raycaster.py:197-201)."""
    rgb = np.maximum(scalar[..., None] * color, floor)
    safe = np.where(color > 0.0, color, 1.0)
    return np.where(color > 0.0, rgb / safe, 1.0)


# ------------------------------------------------------------ K2: the march
def camera_rays(position, target, up, fov_deg, viewport) -> np.ndarray:
    """(H, W, 3) unit directions, row 0 on top (raycaster.py:53-68)."""
    w, h = viewport
    fwd = _unit(np.asarray(target, np.float64) - np.asarray(position, np.float64))
    right = _unit(np.cross(fwd, np.asarray(up, np.float64)))
    up2 = np.cross(right, fwd)
    th = math.tan(math.radians(fov_deg) / 2.0)
    xs = ((np.arange(w) + 0.5) / w * 2.0 - 1.0) * th * (w / h)
    ys = (1.0 - (np.arange(h) + 0.5) / h * 2.0) * th
    d = fwd + xs[None, :, None] * right + ys[:, None, None] * up2
    return d / np.linalg.norm(d, axis=-1, keepdims=True)


def box_hit(origins: np.ndarray, dirs: np.ndarray):
    """Slab test against [0,1]^3 -> (t_enter, t_exit, hit) (geometry.py:46-67)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / dirs
        ta = (0.0 - origins) * inv
        tb = (1.0 - origins) * inv
    flat = dirs == 0.0
    inside = (origins >= 0.0) & (origins <= 1.0)
    ta = np.where(flat, np.where(inside, -np.inf, np.inf), ta)
    tb = np.where(flat, np.where(inside, np.inf, -np.inf), tb)
    t_in = np.maximum(np.minimum(ta, tb).max(axis=-1), 0.0)
    t_out = np.maximum(ta, tb).min(axis=-1)
    return t_in, t_out, t_out > t_in


ALPHA_MAX = 1.0 - 1e-6


def gradient(vol, pts) -> np.ndarray:
    """Central differences, probes clamped to the cube, divided by the actual
    probe separation (volume.py:201-220)."""
    q = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    h = (vol.box_hi - vol.box_lo) / np.array(vol.dims, dtype=np.float64)
    g = np.empty_like(q)
    for a in range(3):
        d = np.zeros(3)
        d[a] = h[a]
        up = np.clip(q + d, 0.0, 1.0)
        dn = np.clip(q - d, 0.0, 1.0)
        sep = up[:, a] - dn[:, a]
        sep = np.where(sep == 0.0, 1.0, sep)
        g[:, a] = (trilinear(vol, up) - trilinear(vol, dn)) / sep
    return g.reshape(np.asarray(pts).shape)


def phong_scalar(vol, pts, light_dir, eye, ambient, diffuse, specular, shininess) -> np.ndarray:
    """ambient + diffuse*max(0,N.L) + specular*max(0,R.V)^n (raycaster.py:204-220)."""
    g = gradient(vol, pts)
    mag = np.linalg.norm(g, axis=-1)
    lit = mag > 1e-12
    res = np.full(pts.shape[0], ambient, dtype=np.float64)
    if lit.any():
        nrm = -g[lit] / mag[lit][:, None]
        tl = -np.asarray(light_dir, dtype=np.float64)
        ndl = np.maximum(0.0, nrm @ tl)
        view = eye - pts[lit]
        view /= np.linalg.norm(view, axis=-1, keepdims=True)
        refl = 2.0 * ndl[:, None] * nrm - tl
        rdv = np.maximum(0.0, np.sum(refl * view, axis=-1))
        res[lit] += diffuse * ndl + specular * np.power(rdv, shininess)
    return res


def light_march(vol, alpha_lut, pts, to_light, step, extinction: bool) -> np.ndarray:
    """March from each point toward the light: sum of -log1p(-a) (extinction,
    raycaster.py:312-332) or the product of (1 - a) (oracle, :335-353), with
    a = min(lut(trilinear), ALPHA_MAX)."""
    m = pts.shape[0]
    t_in, t_out, hit = box_hit(pts, np.broadcast_to(to_light, (m, 3)))
    acc = np.zeros(m) if extinction else np.ones(m)
    live = np.flatnonzero(hit)
    t = t_in[live] + 0.5 * step
    t_end = t_out[live]
    while live.size:
        keep = t < t_end
        live, t, t_end = live[keep], t[keep], t_end[keep]
        if not live.size:
            break
        a = lut_blend(alpha_lut[:, None], trilinear(vol, pts[live] + t[:, None] * to_light))[:, 0]
        if extinction:
            acc[live] += -np.log1p(-np.minimum(a, ALPHA_MAX))
        else:
            acc[live] *= 1.0 - np.minimum(a, ALPHA_MAX)
        t = t + step
    return acc


def shadow_oracle(vol, tf_lut, pts, light_dir, oracle_step) -> np.ndarray:
    """Brute-force transmittance to the light (raycaster.py:356-366)."""
    alpha = resolve(tf_lut, oracle_step)[:, 3]
    p = np.asarray(pts, dtype=np.float64)
    return light_march(vol, alpha, p.reshape(-1, 3), -np.asarray(light_dir, dtype=np.float64), oracle_step,
                       False).reshape(p.shape[:-1])


def make_shader(vol, settings, buffer, alpha_lut_step=None):
    """pts (M,3) -> rgb factor (M,3) (raycaster.py:376-412)."""
    mode = settings.shading_mode
    if mode == "none":
        return lambda p: np.ones((p.shape[0], 3), dtype=np.float64)
    if mode == "phong":
        ph = settings.phong
        eye = np.asarray(settings.camera.position, dtype=np.float64)
        ld = settings.light.direction
        return lambda p: np.repeat(phong_scalar(vol, p, ld, eye, ph.ambient, ph.diffuse, ph.specular,
                                                ph.shininess)[:, None], 3, axis=1)
    if mode == "extinction":
        tl = -np.asarray(settings.light.direction, dtype=np.float64)
        fl = settings.ambient_floor
        return lambda p: np.repeat(np.maximum(np.exp(-light_march(vol, alpha_lut_step, p, tl, settings.step, True)),
                                              fl)[:, None], 3, axis=1)
    if mode not in ("sbrc_shadow", "shell", "cone"):
        raise ValueError(f"unknown shading mode {mode!r}")
    inten = np.asarray(buffer.intensity)
    cam, spec = buffer.camera, buffer.spec
    color = np.asarray(buffer.camera.light_color, dtype=np.float64)
    floor = settings.ambient_floor
    lk = settings.lookup_mode
    if mode == "sbrc_shadow":
        return lambda p: light_factor(lookup_scalar(inten, cam, spec, p, lk), color, floor)
    if mode == "shell":
        sk = settings.shell_kernel
        if sk is None:
            h = float(vol.voxel_size.max())
            radii, weights = (h, 2 * h, 3 * h), (0.5, 0.3, 0.2)
        else:
            radii, weights = sk.radii, sk.weights
        return lambda p: light_factor(shell_scalar(inten, cam, spec, p, radii, weights, lk), color, floor)
    ck = settings.cone_kernel
    axis_samples = 2 if ck is None else ck.axis_samples
    angles = (0.0, math.pi / 2, math.pi, 3 * math.pi / 2) if ck is None else ck.angles
    ring = 0.5 if ck is None else ck.ring_radius_per_step
    eye = np.asarray(settings.camera.position, dtype=np.float64)
    return lambda p: light_factor(cone_scalar(inten, cam, spec, p, axis_samples, angles, ring, eye, lk),
                                  color, floor)


def march(vol, lut: np.ndarray, step: float, thresh: float, shader, origin, dirs):
    """Front-to-back wavefront march of (N,3) rays -> ((N,4) rgba, samples)
    (raycaster.py:415-440)."""
    n = dirs.shape[0]
    rgb = np.zeros((n, 3), dtype=np.float64)
    alpha = np.zeros(n, dtype=np.float64)
    t_in, t_out, hit = box_hit(np.broadcast_to(origin, (n, 3)), dirs)
    live = np.flatnonzero(hit)
    t = t_in[live] + 0.5 * step
    t_end = t_out[live]
    samples = 0
    while live.size:
        keep = (t < t_end) & (alpha[live] < thresh)
        live, t, t_end = live[keep], t[keep], t_end[keep]
        if not live.size:
            break
        p = origin + t[:, None] * dirs[live]
        rgba = lut_blend(lut, trilinear(vol, p))
        fac = shader(p)
        one_m = (1.0 - alpha[live])[:, None]
        rgb[live] += one_m * rgba[:, :3] * fac
        alpha[live] += one_m[:, 0] * rgba[:, 3]
        samples += live.size
        t = t + step
    return np.concatenate([rgb, alpha[:, None]], axis=1), samples


def render_image(vol, tf_lut: np.ndarray, settings, buffer=None, rows=None, cols=None,
                 return_samples: bool = False):
    """(H, W, 4) float32 premultiplied image (raycaster.py:443-469).

    ``rows``/``cols`` optionally restrict the march to a pixel subset (used
    for bounded CPU baselines on large frames); the result is then
    (len(rows), len(cols), 4)."""
    mode = settings.shading_mode
    if mode in ("sbrc_shadow", "shell", "cone") and buffer is None:
        raise ValueError(f"shading mode {mode!r} needs an attenuation buffer")
    w, h = settings.viewport
    lut = resolve(tf_lut, settings.step)
    cam = settings.camera
    dirs = camera_rays(cam.position, cam.target, cam.up, cam.fov_deg, settings.viewport)
    if rows is not None:
        dirs = dirs[np.asarray(rows)]
    if cols is not None:
        dirs = dirs[:, np.asarray(cols)]
    hh, ww = dirs.shape[:2]
    flat, samples = march(vol, lut, settings.step, settings.early_termination_alpha,
                          make_shader(vol, settings, buffer, np.ascontiguousarray(lut[:, 3])),
                          np.asarray(cam.position, np.float64), dirs.reshape(-1, 3))
    img = flat.reshape(hh, ww, 4).astype(np.float32)
    return (img, samples) if return_samples else img


# ------------------------------------------------------------ half-angle baseline
def _plane_uv_axes(direction):
    w = _unit(direction)
    hint = np.array([0.0, 1.0, 0.0])
    if abs(float(np.dot(hint, w))) > 1.0 - 1e-9:
        hint = np.array([0.0, 0.0, 1.0])
    u = _unit(np.cross(hint, w))
    return u, _unit(np.cross(w, u))


def half_angle(vol, tf_lut, settings, n_slices, light_resolution=None):
    """(image, passes): eye and light pass per slice (halfangle.py:48-142)."""
    light, cam = settings.light, settings.camera
    w, h = settings.viewport
    lw, lh = light_resolution or settings.viewport
    view = _unit(np.asarray(cam.target, np.float64) - np.asarray(cam.position, np.float64))
    ld = np.asarray(light.direction, np.float64)
    if float(np.dot(view, ld)) >= 0.0:
        s, f2b = view + ld, True
    else:
        s, f2b = -view + ld, False
    half = ld.copy() if float(np.linalg.norm(s)) < 1e-9 else _unit(s)
    if float(np.linalg.norm(s)) < 1e-9:
        f2b = False
    corners = np.array([[(i >> a) & 1 for a in range(3)] for i in range(8)], dtype=np.float64)
    proj = corners @ half
    dlo, dhi = float(proj.min()), float(proj.max())
    delta = (dhi - dlo) / n_slices
    offsets = dlo + (np.arange(n_slices, dtype=np.float64) + 0.5) * delta
    au, av = _plane_uv_axes(ld)
    pu, pv = corners @ au, corners @ av
    u0, u1, v0, v1 = float(pu.min()), float(pu.max()), float(pv.min()), float(pv.max())
    uc = u0 + (np.arange(lw, dtype=np.float64) + 0.5) / lw * (u1 - u0)
    vc = v0 + (np.arange(lh, dtype=np.float64) + 0.5) / lh * (v1 - v0)
    ug, vg = np.meshgrid(uc, vc)
    lbase = ug[..., None] * au + vg[..., None] * av
    hl, hu, hv = float(np.dot(half, ld)), float(np.dot(half, au)), float(np.dot(half, av))
    eye = np.asarray(cam.position, np.float64)
    dirs = camera_rays(cam.position, cam.target, cam.up, cam.fov_deg, settings.viewport).reshape(-1, 3)
    hd = dirs @ half
    he = float(np.dot(half, eye))
    acc = np.zeros((h * w, 4))
    trans = np.ones((lh, lw))
    lut = tf_lut
    passes = 0
    for k in range(n_slices):
        off = float(offsets[k])
        with np.errstate(divide="ignore", invalid="ignore"):
            t = (off - he) / hd
        pts = eye + t[:, None] * dirs
        ok = (hd != 0) & (t > 0) & np.all((pts >= 0.0) & (pts <= 1.0), axis=1)
        if ok.any():
            p = pts[ok]
            rgba = lut_blend(lut, trilinear(vol, p))
            a = 1.0 - np.power(1.0 - rgba[:, 3], delta / (OPACITY_REF_STEP * np.abs(hd[ok])))
            uv = np.stack([(p @ au - u0) / (u1 - u0), (p @ av - v0) / (v1 - v0)], axis=1)
            tx, ty = uv[:, 0] * lw - 0.5, uv[:, 1] * lh - 0.5
            xi, yi = np.floor(tx).astype(np.intp), np.floor(ty).astype(np.intp)
            fx, fy = tx - xi, ty - yi
            xa, xb = np.clip(xi, 0, lw - 1), np.clip(xi + 1, 0, lw - 1)
            ya, yb = np.clip(yi, 0, lh - 1), np.clip(yi + 1, 0, lh - 1)
            shade = ((trans[ya, xa] * (1 - fx) + trans[ya, xb] * fx) * (1 - fy)
                     + (trans[yb, xa] * (1 - fx) + trans[yb, xb] * fx) * fy)
            src = rgba[:, :3] * (a * shade)[:, None]
            if f2b:
                one_m = (1.0 - acc[ok, 3])[:, None]
                acc[ok, :3] += one_m * src
                acc[ok, 3] += one_m[:, 0] * a
            else:
                acc[ok, :3] = (1.0 - a)[:, None] * acc[ok, :3] + src
                acc[ok, 3] = a + (1.0 - a) * acc[ok, 3]
        passes += 1
        tl = (off - ug * hu - vg * hv) / hl
        lp = lbase + tl[..., None] * ld
        cov = np.all((lp >= 0.0) & (lp <= 1.0), axis=-1)
        if cov.any():
            rgba = lut_blend(lut, trilinear(vol, lp[cov]))
            a = 1.0 - np.power(1.0 - rgba[:, 3], delta / (OPACITY_REF_STEP * hl))
            trans[cov] *= 1.0 - a
        passes += 1
    return acc.reshape(h, w, 4).astype(np.float32), passes
