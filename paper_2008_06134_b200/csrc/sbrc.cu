// sbrc.cu — B200 (sm_100a) kernels for slice-based ray casting with volume
// illumination (arXiv 2008.06134), behind the C ABI in include/sbrc.h.
//
//   K1 build_kernel  <- slicecast.lightbuffer.build_attenuation_buffer
//                       (/root/reference/pkg/src/slicecast/lightbuffer.py:144-199)
//   K2 march_kernel  <- slicecast.raycaster.render / _march_rays / _make_shader
//                       (raycaster.py:376-469) with lookup_light_scalar_many
//                       (lightbuffer.py:256-287), _shell_scalar (:239-250),
//                       _cone_scalar (:266-300), _factor_from_intensity (:197-201)
//
// Numerics. Everything that decides WHICH samples exist —
// cube coverage of a texel-slice point, ray entry/exit, the float64 march
// counter `t += step`, the inside-cube test, trilinear reconstruction, the
// TF lookup and the alpha accumulation that drives early termination — is
// float64 with numpy's operation order and no FMA contraction (explicit
// __dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn), so it is bit-identical to the
// reference. The light factor (buffer lookups for sbrc/shell/cone) is a
// continuous function of position and runs in fp32; it only scales colour.
// No hardware texture filtering: its 8-bit weights would break 1e-3.

#include "../../include/sbrc.h"

#include <cuda_runtime.h>
#include <stdint.h>

namespace {

// ---------------------------------------------------------------- float64
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dclip01(double x) { return fmin(fmax(x, 0.0), 1.0); }
__device__ __forceinline__ bool in01(double x) { return x >= 0.0 && x <= 1.0; }

// ---------------------------------------------------------------- volume
// Voxel fetch with load_raw's normalisation (volume.py:143-149): u8/u16 are
// kept raw in HBM and normalised at fetch by an IEEE float32 division,
// which is bit-identical to numpy's float32 `astype(float32) / 255.0`.
template <int VT> struct Voxel;
template <> struct Voxel<SBRC_VOXEL_F32> {
  static __device__ __forceinline__ double get(const void* d, size_t i) {
    return (double)__ldg(reinterpret_cast<const float*>(d) + i);
  }
};
template <> struct Voxel<SBRC_VOXEL_U8> {
  static __device__ __forceinline__ double get(const void* d, size_t i) {
    return (double)__fdiv_rn((float)__ldg(reinterpret_cast<const unsigned char*>(d) + i), 255.0f);
  }
};
template <> struct Voxel<SBRC_VOXEL_U16> {
  static __device__ __forceinline__ double get(const void* d, size_t i) {
    return (double)__fdiv_rn((float)__ldg(reinterpret_cast<const unsigned short*>(d) + i), 65535.0f);
  }
};

// Cell-centred trilinear reconstruction, clamp-to-edge, 0 outside the unit
// cube: sample_trilinear_many (volume.py:161-194), same op order.
template <int VT>
__device__ __forceinline__ double trilinear64(const sbrc_volume& v, double px, double py, double pz) {
  if (!(in01(px) && in01(py) && in01(pz))) return 0.0;
  double p[3] = {px, py, pz};
  const int dims[3] = {v.nx, v.ny, v.nz};
  int i0[3], i1[3];
  double f[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double local = dsub(p[c], v.box_lo[c]);
    if (v.box_ext[c] != 1.0) local = ddiv(local, v.box_ext[c]);  // x/1.0 == x exactly
    local = dclip01(local);
    double g = dsub(dmul(local, (double)dims[c]), 0.5);
    double fl = floor(g);
    f[c] = dsub(g, fl);
    int lo = (int)fl;
    i0[c] = min(max(lo, 0), dims[c] - 1);
    i1[c] = min(max(lo + 1, 0), dims[c] - 1);
  }
  const size_t sx = 1, sy = (size_t)v.nx, sz = (size_t)v.nx * (size_t)v.ny;
  const size_t bz0 = (size_t)i0[2] * sz, bz1 = (size_t)i1[2] * sz;
  const size_t by0 = (size_t)i0[1] * sy, by1 = (size_t)i1[1] * sy;
  const size_t x0 = (size_t)i0[0] * sx, x1 = (size_t)i1[0] * sx;
  const double d000 = Voxel<VT>::get(v.data, bz0 + by0 + x0);
  const double d100 = Voxel<VT>::get(v.data, bz0 + by0 + x1);
  const double d010 = Voxel<VT>::get(v.data, bz0 + by1 + x0);
  const double d110 = Voxel<VT>::get(v.data, bz0 + by1 + x1);
  const double d001 = Voxel<VT>::get(v.data, bz1 + by0 + x0);
  const double d101 = Voxel<VT>::get(v.data, bz1 + by0 + x1);
  const double d011 = Voxel<VT>::get(v.data, bz1 + by1 + x0);
  const double d111 = Voxel<VT>::get(v.data, bz1 + by1 + x1);
  const double gx = dsub(1.0, f[0]), gy = dsub(1.0, f[1]), gz = dsub(1.0, f[2]);
  const double c00 = dadd(dmul(d000, gx), dmul(d100, f[0]));
  const double c10 = dadd(dmul(d010, gx), dmul(d110, f[0]));
  const double c01 = dadd(dmul(d001, gx), dmul(d101, f[0]));
  const double c11 = dadd(dmul(d011, gx), dmul(d111, f[0]));
  const double c0 = dadd(dmul(c00, gy), dmul(c10, f[1]));
  const double c1 = dadd(dmul(c01, gy), dmul(c11, f[1]));
  return dadd(dmul(c0, gz), dmul(c1, f[2]));
}

// LUT position: t = clip(s,0,1)*255, i0 = floor(t) (truncation, s >= 0),
// i1 = min(i0+1, 255), f = t - i0 (transfer.py:93-100, lightbuffer.py:188-191).
struct LutPos {
  int i0, i1;
  double f, g;
};
__device__ __forceinline__ LutPos lut_pos(double s) {
  LutPos r;
  const double t = dmul(dclip01(s), 255.0);
  const double fl = floor(t);
  r.i0 = (int)fl;
  r.i1 = min(r.i0 + 1, SBRC_LUT_SIZE - 1);
  r.f = dsub(t, fl);
  r.g = dsub(1.0, r.f);
  return r;
}

// ---------------------------------------------------------------- K1 build
// One thread per light texel; the slice recurrence runs in registers
// (lightbuffer.py:166-198): intensity[k] = T; if the texel-slice point is in
// the cube, alpha = lut(trilinear(p)) and T *= 1 - alpha. Texels are
// independent, so no grid-wide barrier or per-slice launch is needed.
template <int VT>
__global__ void __launch_bounds__(256) build_kernel(const sbrc_build_params P) {
  __shared__ double lut[SBRC_LUT_SIZE];
  for (int i = threadIdx.y * blockDim.x + threadIdx.x; i < SBRC_LUT_SIZE; i += blockDim.x * blockDim.y)
    lut[i] = P.alpha_lut[i];
  __syncthreads();

  const sbrc_light_frame& L = P.light;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = P.row_begin + blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= L.width || y >= P.row_end) return;

  // Texel centre in world (u, v) plane coordinates (_texel_world_grid, :134-141):
  // u0 + (i + 0.5) / W * (u1 - u0).
  const double uc = dadd(L.u_range[0], dmul(ddiv(dadd((double)x, 0.5), (double)L.width),
                                            dsub(L.u_range[1], L.u_range[0])));
  const double vc = dadd(L.v_range[0], dmul(ddiv(dadd((double)y, 0.5), (double)L.height),
                                            dsub(L.v_range[1], L.v_range[0])));
  // base = ug * axis_u + vg * axis_v (:164)
  double base[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) base[c] = dadd(dmul(uc, L.axis_u[c]), dmul(vc, L.axis_v[c]));

  const bool comp = P.compensation_n > 0.0;
  float* out = P.out + (size_t)(y - P.row_begin) * (size_t)P.row_stride + (size_t)x;
  double T = 1.0;
  for (int k = 0; k < L.n_slices; ++k) {
    const double off = __ldg(L.plane_offsets + k);
    // pts = base + offset_k * L (:182); covered = all(0 <= pts <= 1) (:183)
    const double px = dadd(base[0], dmul(off, L.light_dir[0]));
    const double py = dadd(base[1], dmul(off, L.light_dir[1]));
    const double pz = dadd(base[2], dmul(off, L.light_dir[2]));
    float stored = (float)T;  // intensity[k] = trans (:169)
    if (in01(px) && in01(py) && in01(pz)) {
      const double s = trilinear64<VT>(P.volume, px, py, pz);
      const LutPos q = lut_pos(s);
      const double a = dadd(dmul(lut[q.i0], q.g), dmul(lut[q.i1], q.f));
      if (comp) stored = (float)dmul((double)stored, pow(dadd(1.0, a), P.compensation_n));  // :193-196
      T = dmul(T, dsub(1.0, a));  // :197-198
    }
    out[(size_t)k * (size_t)P.layer_stride] = stored;
  }
}

// ---------------------------------------------------------------- K2 march
struct LightTex {
  const float* I;
  size_t ks, ys;  // layer and row strides (elements)
  int W, H, n;
  float fW, fH, fnm1;
};

// Clamp-to-edge bilinear inside one layer (_bilinear_layers, lightbuffer.py:238-253).
__device__ __forceinline__ float bilinear_layer(const float* layer, size_t ys, float fx, float fy,
                                                int x0c, int x1c, int y0c, int y1c) {
  const float* r0 = layer + (size_t)y0c * ys;
  const float* r1 = layer + (size_t)y1c * ys;
  const float c0 = __ldg(r0 + x0c) * (1.0f - fx) + __ldg(r0 + x1c) * fx;
  const float c1 = __ldg(r1 + x0c) * (1.0f - fx) + __ldg(r1 + x1c) * fx;
  return c0 * (1.0f - fy) + c1 * fy;
}

// lookup_light_scalar_many at one light-space position (u, v, idx): outside
// the footprint -> 1 (:268-269); linear: plane k sits at continuous index
// k+0.5, blend the two bracketing layers (:277-285); nearest: one layer (:274-276).
template <int LOOKUP>
__device__ __forceinline__ float light_lookup(const LightTex& t, float u, float v, float idx) {
  if (!(u >= 0.0f && u <= 1.0f && v >= 0.0f && v <= 1.0f)) return 1.0f;
  const float tx = u * t.fW - 0.5f, ty = v * t.fH - 0.5f;
  const float flx = floorf(tx), fly = floorf(ty);
  const float fx = tx - flx, fy = ty - fly;
  const int x0 = (int)flx, y0 = (int)fly;  // >= -1 and <= W-1 inside the footprint
  const int x0c = max(x0, 0), x1c = min(x0 + 1, t.W - 1);
  const int y0c = max(y0, 0), y1c = min(y0 + 1, t.H - 1);
  if (LOOKUP == SBRC_LOOKUP_NEAREST) {
    const int k = min((int)floorf(fminf(fmaxf(idx, 0.0f), t.fnm1)), t.n - 1);
    return bilinear_layer(t.I + (size_t)k * t.ks, t.ys, fx, fy, x0c, x1c, y0c, y1c);
  } else {
    const float li = fminf(fmaxf(idx - 0.5f, 0.0f), t.fnm1);
    const int k0 = min((int)li, t.n - 1);
    const int k1 = min(k0 + 1, t.n - 1);
    const float f = li - (float)k0;
    const float v0 = bilinear_layer(t.I + (size_t)k0 * t.ks, t.ys, fx, fy, x0c, x1c, y0c, y1c);
    const float v1 = bilinear_layer(t.I + (size_t)k1 * t.ks, t.ys, fx, fy, x0c, x1c, y0c, y1c);
    return v0 * (1.0f - f) + v1 * f;
  }
}

struct ShellTap {
  float du, dv, di, w;  // light-space offset of +radius along one world axis
};

template <int SHADING, int LOOKUP, int VT>
__global__ void __launch_bounds__(256) march_kernel(const sbrc_render_params P) {
  __shared__ double2 lut[SBRC_LUT_SIZE * 2];  // 256 x rgba float64
  __shared__ ShellTap shell_taps[SBRC_MAX_SHELLS * 3];
  __shared__ float2 cone_cs[SBRC_MAX_ANGLES];
  for (int i = threadIdx.x; i < SBRC_LUT_SIZE * 2; i += blockDim.x)
    lut[i] = reinterpret_cast<const double2*>(P.lut_rgba)[i];

  const sbrc_light_frame& LF = P.light;
  // Per-frame light-space constants: u = (p.au - u0)/(u1-u0), v likewise,
  // idx = n (p.L - d_min)/(d_max - d_min) (world_to_light_uv_many :202-212,
  // slice_index_many slicing.py:101-105).
  const double su = 1.0 / (LF.u_range[1] - LF.u_range[0]);
  const double sv = 1.0 / (LF.v_range[1] - LF.v_range[0]);
  const double si = (double)LF.n_slices / (LF.d_max - LF.d_min);
  if (SHADING == SBRC_SHADE_SHELL) {
    // p +- r e_a maps to (u,v,idx) +- r (au[a] su, av[a] sv, L[a] si).
    for (int i = threadIdx.x; i < P.shell_count * 3; i += blockDim.x) {
      const int s = i / 3, a = i % 3;
      const double r = P.shell_radius[s];
      shell_taps[i] = ShellTap{(float)(r * LF.axis_u[a] * su), (float)(r * LF.axis_v[a] * sv),
                               (float)(r * LF.light_dir[a] * si), (float)P.shell_weight[s]};
    }
  }
  if (SHADING == SBRC_SHADE_CONE) {
    for (int i = threadIdx.x; i < P.cone_angle_count; i += blockDim.x)
      cone_cs[i] = make_float2((float)P.cone_cos[i], (float)P.cone_sin[i]);
  }
  __syncthreads();

  // Pixel of this lane: a block is 32 x 8 pixels, each warp an 8 x 4 tile.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int px = blockIdx.x * 32 + (warp & 3) * 8 + (lane & 7);
  const int lr = blockIdx.y * 8 + (warp >> 2) * 4 + (lane >> 3);  // rank-local row
  const int band = lr / P.band_rows;
  const int py = (P.rank + band * P.world) * P.band_rows + (lr - band * P.band_rows);
  const bool in_image = px < P.width;  // lr < local rows by construction of the grid
  const bool valid = in_image && py < P.height;

  unsigned int samples = 0;
  if (valid) {
    // ---- Camera.rays (raycaster.py:53-68), numpy op order, float64.
    const double ndc_x = dmul(dmul(dsub(dmul(ddiv(dadd((double)px, 0.5), (double)P.width), 2.0), 1.0),
                                   P.tan_half), P.aspect);
    const double ndc_y = dmul(dsub(1.0, dmul(ddiv(dadd((double)py, 0.5), (double)P.height), 2.0)), P.tan_half);
    double d[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) d[c] = dadd(dadd(P.forward[c], dmul(ndc_x, P.right[c])), dmul(ndc_y, P.up2[c]));
    const double nrm = __dsqrt_rn(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
#pragma unroll
    for (int c = 0; c < 3; ++c) d[c] = ddiv(d[c], nrm);

    // ---- ray_box_intersect (geometry.py:46-67) against the unit cube.
    double t_near = -INFINITY, t_far = INFINITY;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double lo, hi;
      if (d[c] == 0.0) {
        const bool inside = in01(P.eye[c]);
        lo = inside ? -INFINITY : INFINITY;
        hi = inside ? INFINITY : -INFINITY;
      } else {
        const double inv = ddiv(1.0, d[c]);
        lo = dmul(dsub(0.0, P.eye[c]), inv);
        hi = dmul(dsub(1.0, P.eye[c]), inv);
      }
      t_near = fmax(t_near, fmin(lo, hi));
      t_far = fmin(t_far, fmax(lo, hi));
    }
    const double t_enter = fmax(t_near, 0.0);

    if (t_far > t_enter) {
      LightTex tex;
      tex.I = P.intensity;
      tex.ks = (size_t)P.layer_stride;
      tex.ys = (size_t)P.row_stride;
      tex.W = LF.width;
      tex.H = LF.height;
      tex.n = LF.n_slices;
      tex.fW = (float)LF.width;
      tex.fH = (float)LF.height;
      tex.fnm1 = (float)(LF.n_slices - 1);
      // Light-space coordinates are affine in t along the ray.
      double lu0 = 0, lud = 0, lv0 = 0, lvd = 0, li0 = 0, lid = 0;
      float cbu = 1.0f, cbv = 0.0f, dperp = 0.0f;
      if (SHADING != SBRC_SHADE_NONE) {
        double eu = 0, ev = 0, el = 0, du_ = 0, dv_ = 0, dl_ = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          eu += P.eye[c] * LF.axis_u[c];
          ev += P.eye[c] * LF.axis_v[c];
          el += P.eye[c] * LF.light_dir[c];
          du_ += d[c] * LF.axis_u[c];
          dv_ += d[c] * LF.axis_v[c];
          dl_ += d[c] * LF.light_dir[c];
        }
        lu0 = (eu - LF.u_range[0]) * su;
        lud = du_ * su;
        lv0 = (ev - LF.v_range[0]) * sv;
        lvd = dv_ * sv;
        li0 = (el - LF.d_min) * si;
        lid = dl_ * si;
        if (SHADING == SBRC_SHADE_CONE) {
          // Ring basis: normalize(e - (e.L)L) with e = eye - p = -t d, so it is
          // -d_perp/|d_perp| for the whole ray (raycaster.py:276-282); its
          // in-plane coordinates are (-du_, -dv_)/|d_perp|.
          const double pu = -du_, pv = -dv_;
          const double pn = sqrt(pu * pu + pv * pv);
          dperp = (float)pn;
          if (pn > 0.0) {
            cbu = (float)(pu / pn);
            cbv = (float)(pv / pn);
          }
        }
      }
      const double step = P.step, thresh = P.et_alpha;
      double t = dadd(t_enter, 0.5 * step);
      double cr = 0.0, cg = 0.0, cb = 0.0, alpha = 0.0;
      // Front-to-back march (raycaster.py:428-439): the live test precedes
      // each sample, so the sample that crosses the threshold is kept.
      while (t < t_far && alpha < thresh) {
        const double qx = dadd(P.eye[0], dmul(t, d[0]));
        const double qy = dadd(P.eye[1], dmul(t, d[1]));
        const double qz = dadd(P.eye[2], dmul(t, d[2]));
        const double s = trilinear64<VT>(P.volume, qx, qy, qz);
        const LutPos q = lut_pos(s);
        const double2 a_rg = lut[2 * q.i0], a_ba = lut[2 * q.i0 + 1];
        const double2 b_rg = lut[2 * q.i1], b_ba = lut[2 * q.i1 + 1];
        const double sr = dadd(dmul(a_rg.x, q.g), dmul(b_rg.x, q.f));
        const double sg = dadd(dmul(a_rg.y, q.g), dmul(b_rg.y, q.f));
        const double sb = dadd(dmul(a_ba.x, q.g), dmul(b_ba.x, q.f));
        const double sa = dadd(dmul(a_ba.y, q.g), dmul(b_ba.y, q.f));

        float fr = 1.0f, fg = 1.0f, fb = 1.0f;
        if (SHADING != SBRC_SHADE_NONE) {
          const float u = (float)(lu0 + t * lud);
          const float v = (float)(lv0 + t * lvd);
          const float idx = (float)(li0 + t * lid);
          float scalar;
          if (SHADING == SBRC_SHADE_SHADOW) {
            scalar = light_lookup<LOOKUP>(tex, u, v, idx);
          } else if (SHADING == SBRC_SHADE_SHELL) {
            float acc = 0.0f;
            for (int sh = 0; sh < P.shell_count; ++sh) {
              float shell = 0.0f;
#pragma unroll
              for (int a = 0; a < 3; ++a) {
                const ShellTap tp = shell_taps[sh * 3 + a];
                shell += light_lookup<LOOKUP>(tex, u + tp.du, v + tp.dv, idx + tp.di);
                shell += light_lookup<LOOKUP>(tex, u - tp.du, v - tp.dv, idx - tp.di);
              }
              acc += shell_taps[sh * 3].w * shell / 6.0f;
            }
            scalar = acc;
          } else {  // cone
            float bu = cbu, bv = cbv;
            if (!((double)dperp * t > 1e-12)) {  // fallback plane_basis(L)[0] = axis_u
              bu = 1.0f;
              bv = 0.0f;
            }
            float acc = 0.0f;
            for (int i = 1; i <= P.cone_axis_samples; ++i) {
              const float r = (float)(P.cone_ring * (double)i * ((LF.d_max - LF.d_min) / LF.n_slices));
              const float ru = r * (float)su, rv = r * (float)sv;
              const float ki = idx - (float)i;
              for (int j = 0; j < P.cone_angle_count; ++j) {
                const float2 cs = cone_cs[j];
                const float wu = bu * cs.x - bv * cs.y;
                const float wv = bv * cs.x + bu * cs.y;
                acc += light_lookup<LOOKUP>(tex, u + ru * wu, v + rv * wv, ki);
              }
            }
            scalar = acc / (float)(P.cone_axis_samples * P.cone_angle_count);
          }
          // _factor_from_intensity (raycaster.py:197-201)
          const float c0 = P.light_color[0], c1 = P.light_color[1], c2 = P.light_color[2];
          fr = c0 > 0.0f ? fmaxf(scalar * c0, P.ambient_floor) / c0 : 1.0f;
          fg = c1 > 0.0f ? fmaxf(scalar * c1, P.ambient_floor) / c1 : 1.0f;
          fb = c2 > 0.0f ? fmaxf(scalar * c2, P.ambient_floor) / c2 : 1.0f;
        }
        // C += (1-a)*rgb*factor; a += (1-a)*a_src (raycaster.py:436-438)
        const double one_m = dsub(1.0, alpha);
        cr = dadd(cr, dmul(dmul(one_m, sr), (double)fr));
        cg = dadd(cg, dmul(dmul(one_m, sg), (double)fg));
        cb = dadd(cb, dmul(dmul(one_m, sb), (double)fb));
        alpha = dadd(alpha, dmul(one_m, sa));
        t = dadd(t, step);
        ++samples;
      }
      float4* out = reinterpret_cast<float4*>(P.image) + (size_t)lr * P.width + px;
      *out = make_float4((float)cr, (float)cg, (float)cb, (float)alpha);
    } else {
      reinterpret_cast<float4*>(P.image)[(size_t)lr * P.width + px] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else if (in_image) {  // padding row of a partial last band
    reinterpret_cast<float4*>(P.image)[(size_t)lr * P.width + px] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (P.sample_count != nullptr) {
    const unsigned int tot = __reduce_add_sync(0xffffffffu, samples);
    if (lane == 0 && tot) atomicAdd(P.sample_count, (unsigned long long)tot);
  }
}

// ---------------------------------------------------------------- dispatch
bool volume_ok(const sbrc_volume& v) {
  if (v.data == nullptr) return false;
  if (v.nx < 2 || v.ny < 2 || v.nz < 2) return false;  // volume.py:80-81
  if (v.voxel_type < SBRC_VOXEL_F32 || v.voxel_type > SBRC_VOXEL_U16) return false;
  for (int c = 0; c < 3; ++c)
    if (!(v.box_ext[c] > 0.0)) return false;
  return true;
}

bool light_ok(const sbrc_light_frame& L) {
  return L.width >= 1 && L.height >= 1 && L.n_slices >= 1 && L.d_max > L.d_min &&
         L.u_range[1] > L.u_range[0] && L.v_range[1] > L.v_range[0];
}

template <int VT>
void launch_build(const sbrc_build_params& p, cudaStream_t s) {
  dim3 block(32, 8);
  dim3 grid((p.light.width + 31) / 32, (p.row_end - p.row_begin + 7) / 8);
  build_kernel<VT><<<grid, block, 0, s>>>(p);
}

template <int SH, int LK, int VT>
void launch_march3(const sbrc_render_params& p, cudaStream_t s) {
  const int rows = sbrc_local_rows(p.height, p.band_rows, p.rank, p.world);
  dim3 grid((p.width + 31) / 32, (rows + 7) / 8);
  march_kernel<SH, LK, VT><<<grid, 256, 0, s>>>(p);
}
template <int SH, int LK>
void launch_march2(const sbrc_render_params& p, cudaStream_t s) {
  switch (p.volume.voxel_type) {
    case SBRC_VOXEL_F32: launch_march3<SH, LK, SBRC_VOXEL_F32>(p, s); break;
    case SBRC_VOXEL_U8: launch_march3<SH, LK, SBRC_VOXEL_U8>(p, s); break;
    default: launch_march3<SH, LK, SBRC_VOXEL_U16>(p, s); break;
  }
}
template <int SH>
void launch_march1(const sbrc_render_params& p, cudaStream_t s) {
  if (p.lookup == SBRC_LOOKUP_NEAREST) launch_march2<SH, SBRC_LOOKUP_NEAREST>(p, s);
  else launch_march2<SH, SBRC_LOOKUP_LINEAR>(p, s);
}

}  // namespace

extern "C" {

int sbrc_abi_version(void) { return SBRC_ABI_VERSION; }

const char* sbrc_strerror(int status) {
  switch (status) {
    case SBRC_OK: return "ok";
    case SBRC_EINVAL: return "invalid parameter";
    case SBRC_ECONFIG: return "shading mode needs an attenuation buffer";
    case SBRC_ECUDA: return "CUDA error";
    case SBRC_EUNSUPPORTED: return "unsupported shading mode";
    default: return "unknown status";
  }
}

int64_t sbrc_struct_size(int which) {
  switch (which) {
    case 0: return (int64_t)sizeof(sbrc_volume);
    case 1: return (int64_t)sizeof(sbrc_light_frame);
    case 2: return (int64_t)sizeof(sbrc_build_params);
    case 3: return (int64_t)sizeof(sbrc_render_params);
    default: return -1;
  }
}

int sbrc_volume_check(const sbrc_volume* v) { return (v && volume_ok(*v)) ? SBRC_OK : SBRC_EINVAL; }

int sbrc_local_rows(int height, int band_rows, int rank, int world) {
  if (height < 1 || band_rows < 1 || world < 1 || rank < 0 || rank >= world) return 0;
  const int bands = (height + band_rows - 1) / band_rows;
  const int mine = bands > rank ? (bands - rank + world - 1) / world : 0;
  return mine * band_rows;
}

int sbrc_build(const sbrc_build_params* p, void* stream) {
  if (p == nullptr || !volume_ok(p->volume) || !light_ok(p->light)) return SBRC_EINVAL;
  if (p->light.plane_offsets == nullptr || p->alpha_lut == nullptr || p->out == nullptr) return SBRC_EINVAL;
  if (p->row_begin < 0 || p->row_end > p->light.height || p->row_begin >= p->row_end) return SBRC_EINVAL;
  if (p->layer_stride < 1 || p->row_stride < p->light.width) return SBRC_EINVAL;
  if (p->compensation_n < 0.0) return SBRC_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  switch (p->volume.voxel_type) {
    case SBRC_VOXEL_F32: launch_build<SBRC_VOXEL_F32>(*p, s); break;
    case SBRC_VOXEL_U8: launch_build<SBRC_VOXEL_U8>(*p, s); break;
    default: launch_build<SBRC_VOXEL_U16>(*p, s); break;
  }
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_render(const sbrc_render_params* p, void* stream) {
  if (p == nullptr || !volume_ok(p->volume)) return SBRC_EINVAL;
  if (p->width < 1 || p->height < 1 || !(p->step > 0.0)) return SBRC_EINVAL;           // raycaster.py:143-146
  if (!(p->et_alpha > 0.0 && p->et_alpha <= 1.0)) return SBRC_EINVAL;                  // :147-148
  if (p->lut_rgba == nullptr || p->image == nullptr) return SBRC_EINVAL;
  if (p->shading < SBRC_SHADE_NONE || p->shading > SBRC_SHADE_CONE) return SBRC_EUNSUPPORTED;
  if (p->lookup != SBRC_LOOKUP_LINEAR && p->lookup != SBRC_LOOKUP_NEAREST) return SBRC_EINVAL;
  if (p->band_rows < 1 || p->band_rows % 8 != 0 || p->world < 1 || p->rank < 0 || p->rank >= p->world)
    return SBRC_EINVAL;
  if (p->shading != SBRC_SHADE_NONE) {
    if (p->intensity == nullptr) return SBRC_ECONFIG;
    if (!light_ok(p->light)) return SBRC_EINVAL;
    if (p->layer_stride < 1 || p->row_stride < p->light.width) return SBRC_EINVAL;
  }
  if (p->shading == SBRC_SHADE_SHELL && (p->shell_count < 1 || p->shell_count > SBRC_MAX_SHELLS))
    return SBRC_EINVAL;
  if (p->shading == SBRC_SHADE_CONE &&
      (p->cone_axis_samples < 1 || p->cone_angle_count < 1 || p->cone_angle_count > SBRC_MAX_ANGLES ||
       p->cone_ring < 0.0))
    return SBRC_EINVAL;
  if (sbrc_local_rows(p->height, p->band_rows, p->rank, p->world) == 0) return SBRC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  switch (p->shading) {
    case SBRC_SHADE_NONE: launch_march1<SBRC_SHADE_NONE>(*p, s); break;
    case SBRC_SHADE_SHADOW: launch_march1<SBRC_SHADE_SHADOW>(*p, s); break;
    case SBRC_SHADE_SHELL: launch_march1<SBRC_SHADE_SHELL>(*p, s); break;
    default: launch_march1<SBRC_SHADE_CONE>(*p, s); break;
  }
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

}  // extern "C"
