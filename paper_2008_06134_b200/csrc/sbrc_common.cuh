// sbrc_common.cuh — device code shared by the sbrc translation units: the
// float64 reference arithmetic, voxel fetch and trilinear reconstruction,
// light-space lookups, and the K2 march kernel template with its launch
// dispatch. march_inst.cu instantiates one (shading mode, voxel type) per
// compilation, so the kernel variants compile in parallel.
#pragma once

// sbrc.cu — B200 (sm_100a) kernels for slice-based ray casting with volume
// illumination (arXiv 2008.06134), behind the C ABI in include/sbrc.h.
//
//   K1 build_kernel  <- slicecast.lightbuffer.build_attenuation_buffer
//                       (/root/reference/pkg/src/slicecast/lightbuffer.py:144-199)
//   K2 march_kernel  <- slicecast.raycaster.render / _march_rays / _make_shader
//                       (raycaster.py:376-469) with lookup_light_scalar_many
//                       (lightbuffer.py:256-287), _shell_scalar (:239-250),
//                       _cone_scalar (:266-300), _factor_from_intensity (:197-201)
//   pack_quads       <- repacks an externally built (n, H, W) stack
//
// Numerics. Everything that decides WHICH samples exist and
// the alpha that drives early termination — cube coverage of a texel-slice
// point, ray entry/exit, the float64 march counter `t += step`, the
// inside-cube test, trilinear reconstruction, the TF lookup and the alpha
// accumulation — is float64 with numpy's operation order and no FMA
// contraction (explicit __dmul_rn/__dadd_rn/__dsub_rn/__ddiv_rn), so it is
// bit-identical to the reference. The light factor (buffer lookups for
// sbrc/shell/cone) is a continuous function of position and runs in fp32;
// it only scales colour. No hardware texture filtering: its 8-bit weights
// would break 1e-3.
//
// Performance notes (profiles/). The march is issue-bound,
// not HBM-bound (L1 hit rate 94%): the design minimises instructions per
// sample — texel quads turn a two-layer bilinear lookup into two 16-byte
// loads, offsets are 32-bit, edge clamping is folded into saturated
// weights, the trilinear fetch has an unclamped interior fast path, and the
// default cone (2 x 4) and shell (3 shells) kernels are unrolled.
//
// Measured alternatives kept as build switches (default off unless noted;
// numbers: config 3 on one B200, profiles/r2_notes.md):
//   SBRC_PACKED        FFMA2/FADD2 shell taps: ON (shell 4.92 -> 4.73 ms)
//   SBRC_PACKED_CONE   the same for cone taps (2.87 -> 3.17-3.20 ms)
//   SBRC_WARP_VOTE     __any_sync march loop (2.87 -> 3.43 ms)
//   SBRC_PREC          float32 colour / sample paths (2.84 / 2.60 ms, the
//                      latter 1.2e-3 over the contract on 3 pixels)
//   SBRC_PAIRS         layer-pair stack for every mode (cone 3.01, shell
//                      5.63, shadow 1.45 ms) — pairs are chosen at run time
//                      for sbrc_shadow frames instead (quad_layout)
//   SBRC_BRICK         8^3-cell bricks with apron (K2 2.96, K1 0.37 ms)
//   SBRC_BUILD_ASYNC   K1 cp.async gather pipeline (sbrc.cu; 0.36 ms at D=4)
//   SBRC_BUILD_TMA     K1 TMA-staged volume boxes (sbrc.cu; 1.02 ms)

#include "../../include/sbrc.h"

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <type_traits>

// Compile-time variants (A/B'd in profiles/r01_notes.md).
#ifndef SBRC_LATENCY_ALL
#define SBRC_LATENCY_ALL 1  // latency mode also for shell / sbrc_shadow (config 1: 0.576 -> 0.511 ms)
#endif
#ifndef SBRC_LATENCY_MODE_PIXELS
#define SBRC_LATENCY_MODE_PIXELS 196608  // rank-local pixels at or below which K2 runs 1 block/SM
#endif
#ifndef SBRC_WIDE_MAX_PIXELS
#define SBRC_WIDE_MAX_PIXELS 393216  // rank-local pixels at or below which K2 may use 8-warp blocks
#endif
#define SBRC_SM_COUNT 148  // B200
#ifndef SBRC_LAT_GROUP
#define SBRC_LAT_GROUP 4  // lanes per ray for tiny rank-local images (2, 4, 8)
#endif
#ifndef SBRC_GROUP_PIXELS
#define SBRC_GROUP_PIXELS 49152  // rank-local pixels at or below which latency mode uses ray groups
#endif
#ifndef SBRC_NARROW_MINB
#define SBRC_NARROW_MINB 4  // resident 4-warp blocks per SM of the throughput kernel (128 registers)
#endif
#ifndef SBRC_CONE_RING_SERIAL
#define SBRC_CONE_RING_SERIAL 0  // 1: one cone ring's loads in flight at a time (fewer registers)
#endif
#ifndef SBRC_LIGHT_FASTSEG
#define SBRC_LIGHT_FASTSEG 1  // K2: the clamp-free light-lookup samples as one counter interval per ray
#endif
#ifndef SBRC_MARCH_FASTSEG
#define SBRC_MARCH_FASTSEG 1  // K2: samples inside the ray's interior t-range skip the cube/face tests
#endif
#ifndef SBRC_BUILD_FASTSEG
#define SBRC_BUILD_FASTSEG 1  // K1: slices where the whole warp is inside the volume skip the cube/face tests
#endif
#ifndef SBRC_BUILD_UNROLL
#define SBRC_BUILD_UNROLL 1  // slices whose gathers are issued together in K1 (1 + 8 blocks/SM: -3%, r3h)
#endif

// Checked build (SBRC_CHECKED=1, scripts/checked_run.py): every global
// read/write index of the kernels is compared with the extent of its
// buffer and every violation counted by kind in sbrc_violations (the bad
// access itself still happens as in the normal build, so nothing changes
// but the count). compute-sanitizer is closed on this GPU pool; this is the
// bounds evidence instead. Kinds: 0 volume, 1 quad read, 2 quad/plain write,
// 3 image write, 4 peer-image write, 5 tile table, 6 LUT index, 7 plane offset.
#ifndef SBRC_CHECKED
#define SBRC_CHECKED 0
#endif
#if SBRC_CHECKED
// one counter array per translation unit (no relocatable device code):
// sbrc_debug_violations sums the copies of every unit
static __device__ unsigned int sbrc_violations[8];
#define SBRC_CHECK(cond, kind)                                                \
  do {                                                                        \
    if (!(cond)) atomicAdd(&sbrc_violations[kind], 1u);                       \
  } while (0)
#else
#define SBRC_CHECK(cond, kind) \
  do {                         \
  } while (0)
#endif

namespace {


// ---------------------------------------------------------------- float64
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dclip01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }
__device__ __forceinline__ bool in01(double x) { return x >= 0.0 && x <= 1.0; }

// Exact floors without the conversion pipe (F2I/FRND/F2F issue at a quarter
// of the FMA rate and were a third of the march's instructions): adding
// 1.5*2^52 (resp. 1.5*2^23) with round-toward-minus-infinity lands exactly on
// floor(x) + magic for |x| < 2^51 (2^22); the low word is the integer.
struct FloorD {
  double f;
  int i;
};
__device__ __forceinline__ FloorD floor_d(double x) {
  const double m = __dadd_rd(x, 6755399441055744.0);
  return FloorD{__dsub_rn(m, 6755399441055744.0), __double2loint(m)};
}
struct FloorF {
  float f;
  int i;
};
__device__ __forceinline__ FloorF floor_f(float x) {
  const float m = __fadd_rd(x, 12582912.0f);
  return FloorF{__fsub_rn(m, 12582912.0f), __float_as_int(m) - 0x4B400000};
}

// ---------------------------------------------------------------- volume
// Voxel fetch with load_raw's normalisation (volume.py:143-149): u8/u16 are
// kept raw in HBM and normalised at fetch. u8 uses a 256-entry table of
// __fdiv_rn(x, 255.f) (held as double); u16 computes (float)((double)x / 65535) through a
// double product, which rounds to the same float as the IEEE float32
// division because x/65535 is never within 2^-40 of a float midpoint.
// Both are bit-identical to numpy's `astype(float32) / 255.0` etc.
template <int VT> struct Voxel;
template <> struct Voxel<SBRC_VOXEL_F32> {
  using T = float;
  static __device__ __forceinline__ double cvt(float x, const float*) { return (double)x; }
};
template <> struct Voxel<SBRC_VOXEL_U8> {
  using T = unsigned char;
  static __device__ __forceinline__ double cvt(unsigned char x, const float* tab) {
    return reinterpret_cast<const double*>(tab)[x];
  }
};
template <> struct Voxel<SBRC_VOXEL_U16> {
  using T = unsigned short;
  static __device__ __forceinline__ double cvt(unsigned short x, const float*) {
    return (double)__double2float_rn(dmul((double)x, 1.0 / 65535.0));
  }
};
// Cell-centred trilinear reconstruction, clamp-to-edge, 0 outside the unit
// cube: sample_trilinear_many (volume.py:161-194), same op order. Split in
// cell_fetch (indices, fractions, the 8 gathers) and cell_combine (the
// float64 lerps) so callers can issue the gathers of the next slice/sample
// before combining the current one. The voxel index is 32-bit (validated:
// nx*ny*nz < 2^32). UNIT: the volume box is the unit cube (box_lo = 0,
// box_hi = 1: every cubic dataset), where local = (p - 0)/1 = p exactly and
// the clip is a no-op inside the cube.
// Brick layout (SBRC_BRICK = 1, an A/B build): the volume is stored as
// bricks of 8^3 cells, each holding its 9^3 corner voxels (a one-voxel
// apron on the +x/+y/+z sides, edge-replicated at the volume's far faces),
// bricks and voxels x-fastest. A cell's 8 corners then sit in one 2.8 KB
// brick (rows y, y+1 are 36 B apart, slices z, z+1 324 B) instead of four
// rows up to nx*ny*4 bytes apart. 729/512 = 1.42x the voxel bytes.
#ifndef SBRC_BRICK
#define SBRC_BRICK 0
#endif
constexpr int kBrick = 8, kBrickS = 9, kBrickN = 729;
__host__ __device__ __forceinline__ int brick_count(int n) { return n > 1 ? (n - 2) / kBrick + 1 : 1; }
// element offset of voxel (x, y, z) in brick (bx, by, bz): local coordinates in 0..8
__device__ __forceinline__ unsigned brick_voxel(const sbrc_volume& v, int x, int y, int z) {
  const int bx = min(x / kBrick, brick_count(v.nx) - 1), by = min(y / kBrick, brick_count(v.ny) - 1),
            bz = min(z / kBrick, brick_count(v.nz) - 1);
  const unsigned brick = ((unsigned)bz * brick_count(v.ny) + by) * brick_count(v.nx) + bx;
  return brick * kBrickN + ((unsigned)(z - bz * kBrick) * kBrickS + (y - by * kBrick)) * kBrickS + (x - bx * kBrick);
}

template <int VT>
struct Cell {
  typename Voxel<VT>::T r[8];  // d000 d100 d010 d110 d001 d101 d011 d111
  double f[3];
};

template <int VT, bool UNIT>
__device__ __forceinline__ void cell_fetch(const sbrc_volume& v, double px, double py, double pz, Cell<VT>& cl) {
  using T = typename Voxel<VT>::T;
  const double p[3] = {px, py, pz};
  const int dims[3] = {v.nx, v.ny, v.nz};
  int lo[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double local = p[c];
    if (!UNIT) local = dclip01(ddiv(dsub(p[c], v.box_lo[c]), v.box_ext[c]));
    const double g = dsub(dmul(local, (double)dims[c]), 0.5);
    const FloorD fl = floor_d(g);
    cl.f[c] = dsub(g, fl.f);
    lo[c] = fl.i;
  }
  const T* base = reinterpret_cast<const T*>(v.data);
  const unsigned nx = (unsigned)v.nx, nxy = (unsigned)v.nx * (unsigned)v.ny;
  if (SBRC_BRICK) {
    if ((unsigned)lo[0] < (unsigned)(v.nx - 1) && (unsigned)lo[1] < (unsigned)(v.ny - 1) &&
        (unsigned)lo[2] < (unsigned)(v.nz - 1)) {
      // interior: the cell's brick holds all 8 corners (apron)
      const unsigned bx = (unsigned)lo[0] / kBrick, by = (unsigned)lo[1] / kBrick, bz = (unsigned)lo[2] / kBrick;
      const unsigned brick = (bz * (unsigned)brick_count(v.ny) + by) * (unsigned)brick_count(v.nx) + bx;
      const T* c = base + (brick * kBrickN + (((unsigned)lo[2] - bz * kBrick) * kBrickS + ((unsigned)lo[1] - by * kBrick)) *
                                                 kBrickS + ((unsigned)lo[0] - bx * kBrick));
      cl.r[0] = __ldg(c); cl.r[1] = __ldg(c + 1); cl.r[2] = __ldg(c + kBrickS); cl.r[3] = __ldg(c + kBrickS + 1);
      const T* cz = c + kBrickS * kBrickS;
      cl.r[4] = __ldg(cz); cl.r[5] = __ldg(cz + 1); cl.r[6] = __ldg(cz + kBrickS); cl.r[7] = __ldg(cz + kBrickS + 1);
    } else {
      int a[3], b[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        a[c] = min(max(lo[c], 0), dims[c] - 1);
        b[c] = min(max(lo[c] + 1, 0), dims[c] - 1);
      }
      cl.r[0] = __ldg(base + brick_voxel(v, a[0], a[1], a[2])); cl.r[1] = __ldg(base + brick_voxel(v, b[0], a[1], a[2]));
      cl.r[2] = __ldg(base + brick_voxel(v, a[0], b[1], a[2])); cl.r[3] = __ldg(base + brick_voxel(v, b[0], b[1], a[2]));
      cl.r[4] = __ldg(base + brick_voxel(v, a[0], a[1], b[2])); cl.r[5] = __ldg(base + brick_voxel(v, b[0], a[1], b[2]));
      cl.r[6] = __ldg(base + brick_voxel(v, a[0], b[1], b[2])); cl.r[7] = __ldg(base + brick_voxel(v, b[0], b[1], b[2]));
    }
    return;
  }
  if ((unsigned)lo[0] < (unsigned)(v.nx - 1) && (unsigned)lo[1] < (unsigned)(v.ny - 1) &&
      (unsigned)lo[2] < (unsigned)(v.nz - 1)) {
    // interior: the 2x2x2 cell without clamping
    const T* c = base + ((unsigned)lo[0] + nx * (unsigned)lo[1] + nxy * (unsigned)lo[2]);
    SBRC_CHECK((unsigned long long)(c - base) + nxy + nx + 1 < (unsigned long long)nxy * (unsigned)v.nz, 0);
    const T* cy = c + nx;
    const T* cz = c + nxy;
    const T* cyz = cz + nx;
    cl.r[0] = __ldg(c); cl.r[1] = __ldg(c + 1); cl.r[2] = __ldg(cy); cl.r[3] = __ldg(cy + 1);
    cl.r[4] = __ldg(cz); cl.r[5] = __ldg(cz + 1); cl.r[6] = __ldg(cyz); cl.r[7] = __ldg(cyz + 1);
  } else {
    // faces: i0 = clip(lo), i1 = clip(lo + 1) (volume.py:180-182)
    unsigned a[3], b[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      a[c] = (unsigned)min(max(lo[c], 0), dims[c] - 1);
      b[c] = (unsigned)min(max(lo[c] + 1, 0), dims[c] - 1);
    }
    const unsigned z0 = a[2] * nxy, z1 = b[2] * nxy, y0 = a[1] * nx, y1 = b[1] * nx;
    SBRC_CHECK((unsigned long long)z1 + y1 + b[0] < (unsigned long long)nxy * (unsigned)v.nz, 0);
    cl.r[0] = __ldg(base + (z0 + y0 + a[0])); cl.r[1] = __ldg(base + (z0 + y0 + b[0]));
    cl.r[2] = __ldg(base + (z0 + y1 + a[0])); cl.r[3] = __ldg(base + (z0 + y1 + b[0]));
    cl.r[4] = __ldg(base + (z1 + y0 + a[0])); cl.r[5] = __ldg(base + (z1 + y0 + b[0]));
    cl.r[6] = __ldg(base + (z1 + y1 + a[0])); cl.r[7] = __ldg(base + (z1 + y1 + b[0]));
  }
}

// cell_fetch for a point known to be inside the unit-box volume with its
// whole cell (lo in [0, n-2] on every axis): no clamps, no bounds tests.
template <int VT>
__device__ __forceinline__ void cell_fetch_interior(const sbrc_volume& v, double px, double py, double pz,
                                                    Cell<VT>& cl) {
  using T = typename Voxel<VT>::T;
  const double p[3] = {px, py, pz};
  const int dims[3] = {v.nx, v.ny, v.nz};
  int lo[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double g = dsub(dmul(p[c], (double)dims[c]), 0.5);
    const FloorD fl = floor_d(g);
    cl.f[c] = dsub(g, fl.f);
    lo[c] = fl.i;
  }
  const unsigned nx = (unsigned)v.nx, nxy = (unsigned)v.nx * (unsigned)v.ny;
  const T* c = reinterpret_cast<const T*>(v.data) + ((unsigned)lo[0] + nx * (unsigned)lo[1] + nxy * (unsigned)lo[2]);
  SBRC_CHECK(lo[0] >= 0 && lo[1] >= 0 && lo[2] >= 0 && lo[0] < v.nx - 1 && lo[1] < v.ny - 1 && lo[2] < v.nz - 1, 0);
  const T* cy = c + nx;
  const T* cz = c + nxy;
  const T* cyz = cz + nx;
  cl.r[0] = __ldg(c); cl.r[1] = __ldg(c + 1); cl.r[2] = __ldg(cy); cl.r[3] = __ldg(cy + 1);
  cl.r[4] = __ldg(cz); cl.r[5] = __ldg(cz + 1); cl.r[6] = __ldg(cyz); cl.r[7] = __ldg(cyz + 1);
}

template <int VT>
__device__ __forceinline__ double cell_combine(const Cell<VT>& cl, const float* u8tab) {
  using V = Voxel<VT>;
  const double* f = cl.f;
  const double gx = dsub(1.0, f[0]), gy = dsub(1.0, f[1]), gz = dsub(1.0, f[2]);
  const double c00 = dadd(dmul(V::cvt(cl.r[0], u8tab), gx), dmul(V::cvt(cl.r[1], u8tab), f[0]));
  const double c10 = dadd(dmul(V::cvt(cl.r[2], u8tab), gx), dmul(V::cvt(cl.r[3], u8tab), f[0]));
  const double c01 = dadd(dmul(V::cvt(cl.r[4], u8tab), gx), dmul(V::cvt(cl.r[5], u8tab), f[0]));
  const double c11 = dadd(dmul(V::cvt(cl.r[6], u8tab), gx), dmul(V::cvt(cl.r[7], u8tab), f[0]));
  const double c0 = dadd(dmul(c00, gy), dmul(c10, f[1]));
  const double c1 = dadd(dmul(c01, gy), dmul(c11, f[1]));
  return dadd(dmul(c0, gz), dmul(c1, f[2]));
}

__device__ __forceinline__ bool in_cube(double px, double py, double pz) { return in01(px) && in01(py) && in01(pz); }

template <int VT, bool UNIT>
__device__ __forceinline__ double trilinear64(const sbrc_volume& v, const float* u8tab, double px, double py,
                                              double pz) {
  if (!in_cube(px, py, pz)) return 0.0;
  Cell<VT> cl;
  cell_fetch<VT, UNIT>(v, px, py, pz, cl);
  return cell_combine<VT>(cl, u8tab);
}

// u8 normalisation table: tab[x] = (double)((float)x / 255.0f), IEEE division.
__device__ __forceinline__ void fill_u8_table(double* tab) {
  for (int i = threadIdx.y * blockDim.x + threadIdx.x; i < 256; i += blockDim.x * blockDim.y)
    tab[i] = (double)__fdiv_rn((float)i, 255.0f);
}

// LUT position: t = clip(s,0,1)*255, i0 = floor(t) (truncation, s >= 0),
// i1 = min(i0+1, 255), f = t - i0 (transfer.py:93-100, lightbuffer.py:188-191).
struct LutPos {
  int i0, i1;
  double f, g;
  double t;  // LUT coordinate clip(s,0,1)*255
};
__device__ __forceinline__ LutPos lut_pos(double s) {
  LutPos r;
  const double t = dmul(dclip01(s), 255.0);
  const FloorD fl = floor_d(t);
  r.t = t;
  r.i0 = fl.i;
  r.i1 = min(r.i0 + 1, SBRC_LUT_SIZE - 1);
  SBRC_CHECK(r.i0 >= 0 && r.i0 < SBRC_LUT_SIZE, 6);
  r.f = dsub(t, fl.f);
  r.g = dsub(1.0, r.f);
  return r;
}

// ---------------------------------------------------------------- texel quads
// Quad (k, y, x) = (I[k][y][x], I[k+][y][x], I[k][y][x+], I[k+][y][x+]).
// Writing texel x's pair (I[k], I[k+]) fills .xy of quad x and .zw of quad
// x-1 (and .zw of quad x at the right edge, where x+ = x).
__device__ __forceinline__ void emit_pair(float4* row, int x, int w, float a, float b) {
  float2* r2 = reinterpret_cast<float2*>(row);
  r2[2 * x] = make_float2(a, b);
  if (x > 0) r2[2 * x - 1] = make_float2(a, b);
  if (x == w - 1) r2[2 * x + 1] = make_float2(a, b);
}

// ---------------------------------------------------------------- rays
// ray_box_intersect (geometry.py:46-67) for one ray: slab test against the
// unit cube with the reference's parallel-ray handling; t_enter = max(t_near, 0).
__device__ __forceinline__ bool box_hit(const double o[3], const double d[3], double& t_enter, double& t_far) {
  double t_near = -INFINITY;
  t_far = INFINITY;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double lo, hi;
    if (d[c] == 0.0) {
      const bool inside = in01(o[c]);
      lo = inside ? -INFINITY : INFINITY;
      hi = inside ? INFINITY : -INFINITY;
    } else {
      const double inv = ddiv(1.0, d[c]);
      lo = dmul(dsub(0.0, o[c]), inv);
      hi = dmul(dsub(1.0, o[c]), inv);
    }
    t_near = fmax(t_near, fmin(lo, hi));
    t_far = fmin(t_far, fmax(lo, hi));
  }
  t_enter = fmax(t_near, 0.0);
  return t_far > t_enter;
}

// ALPHA_MAX = 1 - 1e-6 (raycaster.py:34)
#define SBRC_ALPHA_MAX (1.0 - 1e-6)

// Straight march from p toward the light (raycaster.py:312-353): EXT returns
// sum(-log1p(-min(a, ALPHA_MAX))) (_extinction_scalar), otherwise
// prod(1 - min(a, ALPHA_MAX)) (_shadow_oracle_scalar). Float64, reference op
// order; only log1p's last ulp can differ from glibc's.
template <int VT, bool UNIT, bool EXT>
__device__ double light_march(const sbrc_volume& v, const double* alut, const float* u8tab, const double p[3],
                              const double tl[3], double step) {
  double t_enter, t_far;
  if (!box_hit(p, tl, t_enter, t_far)) return EXT ? 0.0 : 1.0;
  double acc = EXT ? 0.0 : 1.0;
  for (double t = dadd(t_enter, 0.5 * step); t < t_far; t = dadd(t, step)) {
    const double s = trilinear64<VT, UNIT>(v, u8tab, dadd(p[0], dmul(t, tl[0])), dadd(p[1], dmul(t, tl[1])),
                                           dadd(p[2], dmul(t, tl[2])));
    const LutPos q = lut_pos(s);
    const double a = fmin(dadd(dmul(alut[q.i0], q.g), dmul(alut[q.i1], q.f)), SBRC_ALPHA_MAX);
    if (EXT) acc = dadd(acc, -log1p(-a));
    else acc = dmul(acc, dsub(1.0, a));
  }
  return acc;
}

// _phong_scalar (raycaster.py:204-220) with gradient_many (volume.py:201-220):
// central differences with probes clamped to the cube, divided by the actual
// probe separation; the lit test |g| > 1e-12 sees the same float64 gradient.
template <int VT, bool UNIT>
__device__ double phong_scalar(const sbrc_render_params& P, const float* u8tab, const double p[3]) {
  double g[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double hi[3] = {dclip01(p[0]), dclip01(p[1]), dclip01(p[2])};
    double lo[3] = {hi[0], hi[1], hi[2]};
    hi[a] = dclip01(dadd(p[a], P.voxel_size[a]));
    lo[a] = dclip01(dsub(p[a], P.voxel_size[a]));
    double sep = dsub(hi[a], lo[a]);
    if (sep == 0.0) sep = 1.0;
    g[a] = ddiv(dsub(trilinear64<VT, UNIT>(P.volume, u8tab, hi[0], hi[1], hi[2]),
                     trilinear64<VT, UNIT>(P.volume, u8tab, lo[0], lo[1], lo[2])), sep);
  }
  const double norm = __dsqrt_rn(dadd(dadd(dmul(g[0], g[0]), dmul(g[1], g[1])), dmul(g[2], g[2])));
  const double ambient = P.phong[0];
  if (!(norm > 1e-12)) return ambient;
  double n[3], view[3];
  double vn = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    n[c] = ddiv(-g[c], norm);
    view[c] = dsub(P.eye[c], p[c]);
    vn += view[c] * view[c];
  }
  vn = sqrt(vn);
  double ndl = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) ndl += n[c] * -P.scene_light_dir[c];
  ndl = fmax(0.0, ndl);
  double rdv = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) rdv += (2.0 * ndl * n[c] + P.scene_light_dir[c]) * (view[c] / vn);
  rdv = fmax(0.0, rdv);
  return ambient + (P.phong[1] * ndl + P.phong[2] * pow(rdv, P.phong[3]));
}

// ---------------------------------------------------------------- K2 march
// Light-space lookup state. Texel coordinates tx = u*W - 0.5, ty = v*H - 0.5
// and the layer coordinate li = idx - 0.5 (lightbuffer.py:241-242, :279).
struct QuadTex {
  const float4* q;
  bool pairs;            // sbrc_render_params.quad_layout == 1: float2 layer pairs (sbrc_shadow only)
  unsigned qk, qy;       // layer / row strides in quads
  size_t qy64, qy1_64;   // row step as a 64-bit value; qy1_64: step to row y+1 (0 if H == 1)
  float txmax, tymax;    // footprint: u in [0,1]  <=>  tx in [-0.5, W-0.5]
  float xa_max, ya_max;  // max(W-2, 0), max(H-2, 0)
  float li_max, ka_max;  // n-1, max(n-2, 0)
#if SBRC_CHECKED
  unsigned long long last;  // largest valid quad offset
#endif
};

// The row steps come from the 64-bit parameter, so the compiler cannot fold
// (off + qy) into a 32-bit sum that needs zero-extending before the address
// multiply (3 address instructions per two-row tap instead of 5; config 3
// march 2.92 -> 2.85 ms).
__device__ __forceinline__ QuadTex make_quad_tex(const sbrc_render_params& P) {
  const sbrc_light_frame& LF = P.light;
  QuadTex t;
  t.q = reinterpret_cast<const float4*>(P.quads);
  t.pairs = P.quad_layout == 1;
  t.qk = (unsigned)P.quad_layer_stride;
  t.qy = (unsigned)P.quad_row_stride;
  t.qy64 = (size_t)P.quad_row_stride;
  t.qy1_64 = LF.height > 1 ? t.qy64 : 0;
  t.txmax = (float)LF.width - 0.5f;
  t.tymax = (float)LF.height - 0.5f;
  t.xa_max = (float)max(LF.width - 2, 0);
  t.ya_max = (float)max(LF.height - 2, 0);
  t.li_max = (float)(LF.n_slices - 1);
  t.ka_max = (float)max(LF.n_slices - 2, 0);
#if SBRC_CHECKED
  t.last = (unsigned long long)(LF.n_slices - 1) * t.qk + (unsigned long long)(LF.height - 1) * t.qy + LF.width - 1;
#endif
  return t;
}

__device__ __forceinline__ float lerpf(float a, float b, float t) { return fmaf(t, b, fmaf(-t, a, a)); }

// Layer-pair layout (SBRC_PAIRS = 1, an A/B build): the stack is stored as
// float2 (I[k][y][x], I[k+1][y][x]) per texel, densely at the same (k, y, x)
// offsets the quads use (2x instead of 4x the plain stack); a two-row tap
// then takes four 8-byte loads instead of two 16-byte quads. Valid for W >= 2.
#ifndef SBRC_PAIRS
#define SBRC_PAIRS 0
#endif
// rows y and y+1 of the tap at quad offset `off` as (I[k][x], I[k+1][x], I[k][x+1], I[k+1][x+1])
__device__ __forceinline__ void tap_rows(const float4* q, size_t off, size_t row_step, float4& r0, float4& r1,
                                         bool pairs = false) {
  if (SBRC_PAIRS || pairs) {
    const float2* p = reinterpret_cast<const float2*>(q) + off;
    const float2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + row_step), d = __ldg(p + row_step + 1);
    r0 = make_float4(a.x, a.y, b.x, b.y);
    r1 = make_float4(c.x, c.y, d.x, d.y);
  } else {
    r0 = __ldg(q + off);
    r1 = __ldg(q + off + row_step);
  }
}

#ifndef SBRC_MARCH_PREFETCH
#define SBRC_MARCH_PREFETCH 1  // K2 cell prefetch: 1 in the buffer modes, 0 never, 2 always (A/B)
#endif
#ifndef SBRC_PREC
#define SBRC_PREC 0  // experiment: 0 exact float64 sample path; 1 float32 colour; 2 float32 sample
#endif
template <int VT>
__device__ __forceinline__ float voxel_f(typename Voxel<VT>::T x, const float* u8tab) {
  if constexpr (VT == SBRC_VOXEL_F32) return x;
  else return (float)Voxel<VT>::cvt(x, u8tab);
}
// Trilinear in float32 from the float64-placed cell (fractions rounded to float).
template <int VT>
__device__ __forceinline__ float cell_combine_f(const Cell<VT>& cl, const float* u8tab) {
  const float fx = (float)cl.f[0], fy = (float)cl.f[1], fz = (float)cl.f[2];
  const float c00 = lerpf(voxel_f<VT>(cl.r[0], u8tab), voxel_f<VT>(cl.r[1], u8tab), fx);
  const float c10 = lerpf(voxel_f<VT>(cl.r[2], u8tab), voxel_f<VT>(cl.r[3], u8tab), fx);
  const float c01 = lerpf(voxel_f<VT>(cl.r[4], u8tab), voxel_f<VT>(cl.r[5], u8tab), fx);
  const float c11 = lerpf(voxel_f<VT>(cl.r[6], u8tab), voxel_f<VT>(cl.r[7], u8tab), fx);
  return lerpf(lerpf(c00, c10, fy), lerpf(c01, c11, fy), fz);
}

// lookup_light_scalar_many at one point (lightbuffer.py:256-287): 1 outside
// the footprint (:268-269); linear: bilinear in the two layers bracketing
// plane-centred coordinate li, blended (:277-285); nearest: one layer
// (:274-276). Index clamping (clip(x0,0,W-1), clip(x0+1,0,W-1)) is replaced
// by clamping the cell to [0, W-2] and saturating the weight, which selects
// the same texel values.
// PAIRS_OK: the caller accepts a layer-pair buffer (t.pairs, a uniform
// runtime choice; instantiated only for the one-lookup sbrc_shadow march).
template <int LOOKUP, bool PAIRS_OK = false>
__device__ __forceinline__ float light_lookup(const QuadTex& t, float tx, float ty, float li_raw) {
  // li_raw: idx - 0.5 for linear lookups, idx for nearest
  if (!(tx >= -0.5f && tx <= t.txmax && ty >= -0.5f && ty <= t.tymax)) return 1.0f;
  const float xa = fminf(fmaxf(floor_f(tx).f, 0.0f), t.xa_max);
  const float ya = fminf(fmaxf(floor_f(ty).f, 0.0f), t.ya_max);
  const float fx = __saturatef(tx - xa), fy = __saturatef(ty - ya);
  float ka, f;
  if (LOOKUP == SBRC_LOOKUP_NEAREST) {
    // k = floor(clip(idx, 0, n-1)) (:275); for nearest lookups li_raw is idx
    ka = floor_f(fminf(fmaxf(li_raw, 0.0f), t.li_max)).f;
    f = 0.0f;
  } else {
    const float li = fminf(fmaxf(li_raw, 0.0f), t.li_max);
    ka = fminf(floor_f(li).f, t.ka_max);
    f = li - ka;
  }
  const unsigned off = (unsigned)ka * t.qk + (unsigned)ya * t.qy + (unsigned)xa;
  SBRC_CHECK((unsigned long long)off + t.qy1_64 <= t.last && ka >= 0.f && ya >= 0.f && xa >= 0.f, 1);
  float4 r0, r1;
  tap_rows(t.q, off, t.qy1_64, r0, r1, PAIRS_OK && t.pairs);
  const float a0 = lerpf(r0.x, r0.z, fx), a1 = lerpf(r1.x, r1.z, fx);  // layer ka, rows y, y+1
  const float v0 = lerpf(a0, a1, fy);
  if (LOOKUP == SBRC_LOOKUP_NEAREST) return v0;
  const float b0 = lerpf(r0.y, r0.w, fx), b1 = lerpf(r1.y, r1.w, fx);  // layer ka+1
  return lerpf(v0, lerpf(b0, b1, fy), f);
}

// Interior tap: the caller guarantees 0 <= tx < W-1 and 0 <= ty < H-1, so the
// footprint test passes and no clamp of light_lookup is active; the two
// layers of quad layer offset `kbase` are accumulated separately into v0/v1
// and blended once per layer pair by the caller.
__device__ __forceinline__ void interior_tap(const QuadTex& t, unsigned kbase, float tx, float ty, float& v0,
                                             float& v1) {
  const FloorF xl = floor_f(tx), yl = floor_f(ty);
  const float fx = tx - xl.f, fy = ty - yl.f;
  const unsigned off = kbase + (unsigned)yl.i * t.qy + (unsigned)xl.i;
  SBRC_CHECK((unsigned long long)off + t.qy64 <= t.last, 1);
  float4 r0, r1;
  tap_rows(t.q, off, t.qy64, r0, r1);
  v0 += lerpf(lerpf(r0.x, r0.z, fx), lerpf(r1.x, r1.z, fx), fy);
  v1 += lerpf(lerpf(r0.y, r0.w, fx), lerpf(r1.y, r1.w, fx), fy);
}

#ifndef SBRC_WARP_VOTE
#define SBRC_WARP_VOTE 0  // 1: the march loop runs while __any_sync(live) (A/B)
#endif
#ifndef SBRC_PACKED
#define SBRC_PACKED 3  // shell interior taps in packed float32x2 arithmetic (FFMA2 / FADD2, sm_100)
#endif
#ifndef SBRC_PACKED_CONE
#define SBRC_PACKED_CONE 0  // the same for cone taps: measured slower (config 3 march 2.87 -> 3.17-3.20 ms)
#endif
// Interior tap in packed float32x2 arithmetic: the texel position (tx, ty),
// its floor and fraction, and the two-layer bilinear blend run as FFMA2 /
// FADD2 pairs — layer k and k+1 of a quad row are the (x, y) and (z, w)
// halves of one float4, so each lerp of both layers is one pair of FFMA2
// (per tap ~18 instructions instead of ~28). Same IEEE float32 operations
// per component as interior_tap; returns (layer k, layer k+1) of the tap.
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float t) {
  return __ffma2_rn(make_float2(t, t), b, __ffma2_rn(make_float2(-t, -t), a, a));
}
// SBRC_PACKED bit 0: packed floor / fraction of (tx, ty); bit 1: packed lerps.
__device__ __forceinline__ float2 interior_tap2(const QuadTex& t, unsigned kbase, float2 p) {
  float2 f;
  unsigned xi, yi;
  if (SBRC_PACKED & 1) {
    const float2 m = __fadd2_rd(p, make_float2(12582912.0f, 12582912.0f));
    const float2 fl = __fadd2_rn(m, make_float2(-12582912.0f, -12582912.0f));
    f = __ffma2_rn(fl, make_float2(-1.0f, -1.0f), p);
    xi = (unsigned)(__float_as_int(m.x) - 0x4B400000);
    yi = (unsigned)(__float_as_int(m.y) - 0x4B400000);
  } else {
    const FloorF xl = floor_f(p.x), yl = floor_f(p.y);
    f = make_float2(p.x - xl.f, p.y - yl.f);
    xi = (unsigned)xl.i;
    yi = (unsigned)yl.i;
  }
  const unsigned off = kbase + yi * t.qy + xi;
  SBRC_CHECK((unsigned long long)off + t.qy64 <= t.last, 1);
  float4 r0, r1;
  tap_rows(t.q, off, t.qy64, r0, r1);
  if (SBRC_PACKED & 2) {
    const float2 a = lerp2(make_float2(r0.x, r0.y), make_float2(r0.z, r0.w), f.x);
    const float2 b = lerp2(make_float2(r1.x, r1.y), make_float2(r1.z, r1.w), f.x);
    return lerp2(a, b, f.y);
  } else {
    return make_float2(lerpf(lerpf(r0.x, r0.z, f.x), lerpf(r1.x, r1.z, f.x), f.y),
                       lerpf(lerpf(r0.y, r0.w, f.x), lerpf(r1.y, r1.w, f.x), f.y));
  }
}

struct ShellTap {
  float dtx, dty, dli, w;  // texel-space offset of +radius along one world axis; shell weight
};

#ifndef SBRC_TILE_W
#define SBRC_TILE_W 8  // warp pixel tile width (8 x 4)
#endif
#ifndef SBRC_SKIP_CLEAR
#define SBRC_SKIP_CLEAR 1  // instantiate the zero-emission skip (sbrc_render_params.skip_clear)
#endif
// K2 block shape. NW = 4: 4-warp blocks of 16 x 8 pixels; NW = 8: 8-warp
// blocks of 32 x 8 pixels. The 8-warp shape wins for mid-sized rank-local
// images that still give >= 2 blocks per SM (a rank's share at 4-8 GPUs),
// the 4-warp shape for full frames and tiny images (A/B in
// profiles/r01_notes.md). Host and library use this one rule for the grid.
inline bool march_wide(int width, int local_rows) {
  const long long px = (long long)width * local_rows;
  const long long blocks8 = (long long)((width + 31) / 32) * ((local_rows + 7) / 8);
  return px <= SBRC_WIDE_MAX_PIXELS && blocks8 >= 2 * SBRC_SM_COUNT;
}

// Latency mode (MINB = 1, up to 255 registers; for tiny images also ray
// groups of SBRC_LAT_GROUP lanes) exists for the unrolled default kernels of
// the buffer modes with linear lookups; it is used when the rank-local image
// is small. This must mirror the instantiation choice in
// launch_march_kernel_shape.
inline bool march_latency_kernel(const sbrc_render_params& p) {
  if (p.lookup != SBRC_LOOKUP_LINEAR) return false;
  if (p.shading == SBRC_SHADE_CONE) return p.cone_axis_samples == 2 && p.cone_angle_count == 4;
  if (!SBRC_LATENCY_ALL) return false;
  return (p.shading == SBRC_SHADE_SHELL && p.shell_count == 3) || p.shading == SBRC_SHADE_SHADOW;
}

// The K2 launch shape for these params: the one rule the launch and
// sbrc_render_grid (heavy-first tables on the host) share.
struct MarchShape {
  bool latency;
  int nw, group, bw, bh, tiles_x, tiles_y;
};
inline MarchShape march_shape(const sbrc_render_params& p, int local_rows) {
  MarchShape m{};
  // march_kernel: 0 = by image size (the rule below), 1 = throughput kernel, 2 = latency kernel
  m.latency = march_latency_kernel(p) &&
              (p.march_kernel == 2 ||
               (p.march_kernel == 0 && (long long)p.width * local_rows <= SBRC_LATENCY_MODE_PIXELS));
  m.nw = march_wide(p.width, local_rows) ? 8 : 4;
  m.group = m.latency && (long long)p.width * local_rows <= SBRC_GROUP_PIXELS ? SBRC_LAT_GROUP : 1;
  const int tw = m.group == 1 ? SBRC_TILE_W : 4, th = (32 / m.group) / tw;
  m.bw = (m.nw / 2) * tw;
  m.bh = 2 * th;
  m.tiles_x = (p.width + m.bw - 1) / m.bw;
  m.tiles_y = (local_rows + m.bh - 1) / m.bh;
  return m;
}

// MINB: resident blocks per SM the kernel is compiled for. The throughput
// kernels (MINB = 16 warps per SM / NW: 128 registers) maximise throughput
// when the grid has many blocks per SM; MINB = 1 (up to 255 registers, more
// loads in flight per warp) minimises per-warp latency, which decides the
// kernel time when a rank's share of the image is small (its longest rays run
// nearly alone at the end). SKIP: see sbrc_render_params.skip_clear.
template <int SHADING, int LOOKUP, int VT, bool UNIT, int NSHELL, int CONE_A, int CONE_N, int MINB, bool SKIP,
          int NW, int G>
__global__ void __launch_bounds__(32 * NW, MINB) march_kernel(const sbrc_render_params P) {
  static_assert(G == 1 || SHADING == SBRC_SHADE_SHADOW || SHADING == SBRC_SHADE_SHELL || SHADING == SBRC_SHADE_CONE,
                "ray groups carry float32 light factors (buffer modes)");
  __shared__ double2 lut[SBRC_LUT_SIZE * 2];  // 256 x rgba float64
#if SBRC_PREC
  __shared__ float4 lutf[SBRC_LUT_SIZE];
  for (int i = threadIdx.x; i < SBRC_LUT_SIZE; i += blockDim.x)
    lutf[i] = make_float4((float)P.lut_rgba[4 * i], (float)P.lut_rgba[4 * i + 1], (float)P.lut_rgba[4 * i + 2],
                          (float)P.lut_rgba[4 * i + 3]);
#endif
  __shared__ ShellTap shell_taps[SBRC_MAX_SHELLS * 3];
  __shared__ float2 cone_cs[SBRC_MAX_ANGLES];
  __shared__ double u8tab[256];
  __shared__ double alut[SHADING == SBRC_SHADE_EXTINCTION ? SBRC_LUT_SIZE : 1];
  for (int i = threadIdx.x; i < SBRC_LUT_SIZE * 2; i += blockDim.x)
    lut[i] = reinterpret_cast<const double2*>(P.lut_rgba)[i];
  if (SHADING == SBRC_SHADE_EXTINCTION)
    for (int i = threadIdx.x; i < SBRC_LUT_SIZE; i += blockDim.x) alut[i] = P.lut_rgba[4 * i + 3];
  if (std::is_same<typename Voxel<VT>::T, unsigned char>::value) fill_u8_table(u8tab);

  const sbrc_light_frame& LF = P.light;
  // Light space (world_to_light_uv_many :202-212, slice_index_many slicing.py:101-105):
  // tx = ((p.au - u0)/(u1-u0))*W - 0.5, ty likewise, li = n (p.L - d_min)/(d_max - d_min) - 0.5.
  const double sx = (double)LF.width / (LF.u_range[1] - LF.u_range[0]);
  const double sy = (double)LF.height / (LF.v_range[1] - LF.v_range[0]);
  const double si = (double)LF.n_slices / (LF.d_max - LF.d_min);
  // Interior reach of the scattering kernel in texel / layer units: a sample
  // whose light-space position is at least this far inside the buffer has all
  // its taps inside too, and takes the clamp-free fast path.
  float reach_x = 0.f, reach_y = 0.f, reach_l = 0.f;
  if (SHADING == SBRC_SHADE_SHELL) {
    // p +- r e_a maps to (tx, ty, li) +- r (au[a] sx, av[a] sy, L[a] si).
    for (int i = threadIdx.x; i < P.shell_count * 3; i += blockDim.x) {
      const int s = i / 3, a = i % 3;
      const double r = P.shell_radius[s];
      shell_taps[i] = ShellTap{(float)(r * LF.axis_u[a] * sx), (float)(r * LF.axis_v[a] * sy),
                               (float)(r * LF.light_dir[a] * si), (float)P.shell_weight[s]};
    }
    double rmax = 0.0;
    for (int s = 0; s < P.shell_count; ++s) rmax = fmax(rmax, P.shell_radius[s]);
    double mu = 0.0, mv = 0.0, ml = 0.0;
    for (int a = 0; a < 3; ++a) {
      mu = fmax(mu, fabs(LF.axis_u[a]));
      mv = fmax(mv, fabs(LF.axis_v[a]));
      ml = fmax(ml, fabs(LF.light_dir[a]));
    }
    reach_x = (float)(rmax * mu * sx * 1.001 + 1e-3);
    reach_y = (float)(rmax * mv * sy * 1.001 + 1e-3);
    reach_l = (float)(rmax * ml * si * 1.001 + 1e-3);
  }
  if (SHADING == SBRC_SHADE_CONE) {
    const double rr = P.cone_ring * ((LF.d_max - LF.d_min) / LF.n_slices) * P.cone_axis_samples;
    reach_x = (float)(rr * sx * 1.001 + 1e-3);
    reach_y = (float)(rr * sy * 1.001 + 1e-3);
  }
  const float fast_x_hi = (float)(LF.width - 1), fast_y_hi = (float)(LF.height - 1);
  const float fast_l_hi = (float)(LF.n_slices - 1);
  if (SHADING == SBRC_SHADE_CONE) {
    for (int i = threadIdx.x; i < P.cone_angle_count; i += blockDim.x)
      cone_cs[i] = make_float2((float)P.cone_cos[i], (float)P.cone_sin[i]);
  }
  __shared__ int lut_lit;  // first LUT entry with non-zero emission
  if (threadIdx.x == 0) lut_lit = SBRC_LUT_SIZE;
  __syncthreads();
  if constexpr (SKIP) {
  // Leading run of LUT entries whose (premultiplied) emission is exactly 0:
  // a sample with LUT coordinate t <= lut_lit - 1 interpolates two such
  // entries (or one, with weight 1), so it adds nothing whatever the light
  // factor, and the factor's lookups are skipped (bit-identical).
  for (int i = threadIdx.x; i < SBRC_LUT_SIZE; i += blockDim.x)
    if (lut[2 * i].x != 0.0 || lut[2 * i].y != 0.0 || lut[2 * i + 1].x != 0.0) atomicMin(&lut_lit, i);
  __syncthreads();
  }
  const double clear_t = (double)(lut_lit - 1);

  // Pixel of this lane: each warp owns a TW x TH pixel tile, a block WX x 2
  // warp tiles. Ray groups (G > 1): G adjacent lanes share one ray and take
  // its samples round-robin (lane gl: samples gl, gl+G, ...), so a long ray
  // runs G samples per serial step; warps then own 32/G rays.
  constexpr int TW = G == 1 ? SBRC_TILE_W : 4, TH = (32 / G) / TW;
  constexpr int WX = NW / 2, WY = 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ray = lane / G, gl = lane % G;
  int bx = blockIdx.x, by = blockIdx.y;
  if (P.tile_order != nullptr) {  // heavy-first dispatch: this block renders tile tile_order[b]
    SBRC_CHECK((int)(blockIdx.y * gridDim.x + blockIdx.x) < P.n_tiles, 5);
    const int t = __ldg(P.tile_order + blockIdx.y * gridDim.x + blockIdx.x);
    SBRC_CHECK(t >= 0 && t < (int)(gridDim.x * gridDim.y), 5);
    bx = t % gridDim.x;
    by = t / gridDim.x;
  }
  const int px = bx * (WX * TW) + (warp % WX) * TW + (ray % TW);
  const int lr = by * (WY * TH) + (warp / WX) * TH + (ray / TW);  // rank-local row
  int py;
  if (P.row_count > 0) {  // contiguous partition
    py = P.row_begin + lr;
  } else {
    const int band = lr / P.band_rows;
    py = (P.rank + band * P.world) * P.band_rows + (lr - band * P.band_rows);
  }
  const bool in_image = px < P.width && lr < P.local_rows;
  const bool valid = in_image && py < P.height;

  unsigned int samples = 0;
  float4 result = make_float4(0.f, 0.f, 0.f, 0.f);
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
    // Interior t-range of the ray (unit box): samples whose position lies half
    // a voxel + 1e-9 inside every face are in the cube with their whole cell,
    // so the march skips the float64 cube test and the clamped-cell branch
    // there (the same values; SBRC_MARCH_FASTSEG).
    double t_safe_lo = INFINITY, t_safe_hi = -INFINITY;
    if constexpr (UNIT && SBRC_MARCH_FASTSEG) {
      const int vd[3] = {P.volume.nx, P.volume.ny, P.volume.nz};
      double lo_t = -INFINITY, hi_t = INFINITY;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double m_lo = 0.5 / vd[c] + 1e-9, m_hi = (vd[c] - 0.5) / vd[c] - 1e-9;
        if (fabs(d[c]) < 1e-12) {
          if (!(P.eye[c] > m_lo && P.eye[c] < m_hi)) hi_t = -INFINITY;
        } else {
          const double a = (m_lo - P.eye[c]) / d[c], b = (m_hi - P.eye[c]) / d[c];
          lo_t = fmax(lo_t, fmin(a, b));
          hi_t = fmin(hi_t, fmax(a, b));
        }
      }
      if (lo_t < hi_t) {
        t_safe_lo = lo_t;
        t_safe_hi = hi_t;
      }
    }

    if (t_far > t_enter) {
      QuadTex tex;
      // Light-space coordinates are affine in t along the ray: c(t) = c0 + t*cd.
      double tx0 = 0, txd = 0, ty0 = 0, tyd = 0, li0 = 0, lid = 0;
      float cbu = 1.0f, cbv = 0.0f, dperp = 0.0f;
      float fr_c = 1.f, fg_c = 1.f, fb_c = 1.f, ir = 1.f, ig = 1.f, ib = 1.f;
      constexpr bool BUFFERED = SHADING == SBRC_SHADE_SHADOW || SHADING == SBRC_SHADE_SHELL || SHADING == SBRC_SHADE_CONE;
      if (BUFFERED) {
        tex = make_quad_tex(P);
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
        tx0 = (eu - LF.u_range[0]) * sx - 0.5;
        txd = du_ * sx;
        ty0 = (ev - LF.v_range[0]) * sy - 0.5;
        tyd = dv_ * sy;
        // linear lookups use the plane-centred li = idx - 0.5; nearest uses idx itself
        li0 = (el - LF.d_min) * si - (LOOKUP == SBRC_LOOKUP_NEAREST ? 0.0 : 0.5);
        lid = dl_ * si;
        if (SHADING == SBRC_SHADE_CONE) {
          // Ring basis: normalize(e - (e.L)L) with e = eye - p = -t d, so it is
          // -d_perp/|d_perp| for the whole ray (raycaster.py:276-282); its
          // in-plane coordinates are (-du_, -dv_)/|d_perp|.
          const double pn = sqrt(du_ * du_ + dv_ * dv_);
          dperp = (float)pn;
          if (pn > 0.0) {
            cbu = (float)(-du_ / pn);
            cbv = (float)(-dv_ / pn);
          }
        }
        // _factor_from_intensity (raycaster.py:197-201): max(s*c, floor)/c, 1 where c == 0
        fr_c = P.light_color[0];
        fg_c = P.light_color[1];
        fb_c = P.light_color[2];
        ir = fr_c > 0.f ? 1.0f / fr_c : 0.f;
        ig = fg_c > 0.f ? 1.0f / fg_c : 0.f;
        ib = fb_c > 0.f ? 1.0f / fb_c : 0.f;
      }
      // white light without ambient floor: factor = max(s, 0) on every channel
      const bool white = fr_c == 1.f && fg_c == 1.f && fb_c == 1.f && P.ambient_floor == 0.f;
      // Cone ring geometry per ray (texel units): tap (i, j) sits at
      // (tx + r_i*wx_j, ty + r_i*wy_j, li - i), r_i = ring * i * spacing.
      constexpr int NA = CONE_N > 0 ? CONE_N : 1;
      float wx[NA], wy[NA];
      const float spacing_r = (float)(P.cone_ring * ((LF.d_max - LF.d_min) / LF.n_slices));
      float bu_fb = cbu, bv_fb = cbv;
      if (SHADING == SBRC_SHADE_CONE && CONE_N > 0) {
#pragma unroll
        for (int j = 0; j < NA; ++j) {
          const float c = (float)P.cone_cos[j], s = (float)P.cone_sin[j];
          wx[j] = (float)sx * (cbu * c - cbv * s);
          wy[j] = (float)sy * (cbv * c + cbu * s);
        }
      }
      const double step = P.step, thresh = P.et_alpha;
      double t = dadd(t_enter, 0.5 * step);
      // fp32 light-space centre: c(t) ~= c(t0) + j * step * dc/dt with a float
      // sample counter j (exact below 2^24), so no conversion per sample; the
      // float64 t stays the sample-position authority.
      const float ftx0 = (float)fma(t, txd, tx0), fty0 = (float)fma(t, tyd, ty0), fli0 = (float)fma(t, lid, li0);
      const float ftxs = (float)(txd * step), ftys = (float)(tyd * step), flis = (float)(lid * step);
      // Samples of the clamp-free (fast) light path form one interval of the
      // sample counter: (tx, ty, li) are affine in j, so each bound of the
      // fast test is a half-line in j. Solved once per ray with 0.01 texel /
      // layer of margin (the per-sample fmaf values deviate by < 1e-4), the
      // per-sample test is two compares; samples outside take the general
      // path, which is correct everywhere (SBRC_LIGHT_FASTSEG).
      float jfast_lo = 1.0f, jfast_hi = 0.0f;
      // (cone only: the shell's 18 taps gain nothing from it, 4.70 -> 4.76 ms measured)
      if constexpr (SBRC_LIGHT_FASTSEG && LOOKUP == SBRC_LOOKUP_LINEAR && SHADING == SBRC_SHADE_CONE && CONE_N > 0) {
        double jl = 0.0, jh = 16777216.0;  // float-exact counter range
        auto keep = [&](double v0, double vs, double lo, double hi) {  // lo <= v0 + j vs < hi
          lo += 0.01;
          hi -= 0.01;
          if (!(lo < hi)) {  // no fast sample at all (buffer narrower than the kernel's reach)
            jh = -1.0;
          } else if (vs == 0.0) {
            if (!(v0 >= lo && v0 < hi)) jh = -1.0;
          } else {
            const double a = (lo - v0) / vs, b = (hi - v0) / vs;
            jl = fmax(jl, fmin(a, b));
            jh = fmin(jh, fmax(a, b));
          }
        };
        keep(ftx0, ftxs, reach_x, fast_x_hi - reach_x);
        keep(fty0, ftys, reach_y, fast_y_hi - reach_y);
        keep(fli0, flis, (double)CONE_A, (double)fast_l_hi + 1.0);
        // not degenerate: dperp * t > 1e-12 (with t = t0 + j step, over-estimated for margin)
        if (dperp > 0.f) jl = fmax(jl, (1e-12 / (double)dperp * 1.01 + 1e-12 - t) / step + 1.0);
        else jh = -1.0;
        if (jl <= jh) {
          jfast_lo = (float)ceil(jl);
          jfast_hi = (float)floor(jh);
        }
      }
      float jf = 0.0f;
      if (G > 1) {  // this lane's first sample: gl steps along the exact float64 chain
        for (int i = 0; i < gl; ++i) t = dadd(t, step);
        jf = (float)gl;
      }
      double cr = 0.0, cg = 0.0, cb = 0.0, alpha = 0.0;
      float crf = 0.f, cgf = 0.f, cbf = 0.f, alphaf = 0.f;
      (void)alphaf;
      // Front-to-back march (raycaster.py:428-439): the live test precedes
      // each sample, so the sample that crosses the threshold is kept.
      // the voxel cell of sample j+1 is gathered while sample j is shaded
      // (harmless past the exit: outside the cube nothing is fetched)
      // PF: sample j+1's cell is gathered into registers while sample j is
      // shaded. It pays in the buffer modes, whose light lookups have latency
      // to cover (config 3 cone 2.768 ms vs 3.017 without); `none`, `phong`
      // and `extinction` gather each cell when it is needed (fewer live
      // registers: 1.080 -> 0.936, 7.19 -> 6.43, 195 -> 187 ms;
      // profiles/r2_notes.md). Ray groups always prefetch.
      constexpr bool PF = G > 1 || SBRC_MARCH_PREFETCH == 2 || (SBRC_MARCH_PREFETCH == 1 && BUFFERED);
      Cell<VT> cur;
      bool cur_in = false;
      if (PF) {
        const double qx = dadd(P.eye[0], dmul(t, d[0]));
        const double qy = dadd(P.eye[1], dmul(t, d[1]));
        const double qz = dadd(P.eye[2], dmul(t, d[2]));
        cur_in = in_cube(qx, qy, qz);
        if (cur_in) cell_fetch<VT, UNIT>(P.volume, qx, qy, qz, cur);
      }
      // Light factor of the sample at t (sample counter jf).
      auto light_factor = [&](double& fr, double& fg, double& fb) {
        if (SHADING == SBRC_SHADE_PHONG || SHADING == SBRC_SHADE_EXTINCTION) {
          const double p[3] = {dadd(P.eye[0], dmul(t, d[0])), dadd(P.eye[1], dmul(t, d[1])),
                               dadd(P.eye[2], dmul(t, d[2]))};
          double f;
          if (SHADING == SBRC_SHADE_PHONG) {
            f = phong_scalar<VT, UNIT>(P, reinterpret_cast<const float*>(u8tab), p);  // raycaster.py:385-388
          } else {  // raycaster.py:389-394: max(exp(-tau), floor), alpha LUT at settings.step
            const double tl[3] = {-P.scene_light_dir[0], -P.scene_light_dir[1], -P.scene_light_dir[2]};
            const double tau = light_march<VT, UNIT, true>(P.volume, alut, reinterpret_cast<const float*>(u8tab),
                                                          p, tl, step);
            f = fmax(exp(-tau), (double)P.ambient_floor);
          }
          fr = fg = fb = f;
        } else if (SHADING != SBRC_SHADE_NONE) {
          const float tx = fmaf(jf, ftxs, ftx0);
          const float ty = fmaf(jf, ftys, fty0);
          const float li = fmaf(jf, flis, fli0);
          float scalar;
          if (SHADING == SBRC_SHADE_SHADOW) {
            scalar = light_lookup<LOOKUP, true>(tex, tx, ty, li);
          } else if (SHADING == SBRC_SHADE_SHELL) {
            float acc = 0.0f;
            const int nsh = NSHELL > 0 ? NSHELL : P.shell_count;
            const bool fast = LOOKUP == SBRC_LOOKUP_LINEAR && tx - reach_x >= 0.f && tx + reach_x < fast_x_hi &&
                              ty - reach_y >= 0.f && ty + reach_y < fast_y_hi && li - reach_l >= 0.f &&
                              li + reach_l < fast_l_hi;
            if (fast) {
#pragma unroll
              for (int sh = 0; sh < (NSHELL > 0 ? NSHELL : SBRC_MAX_SHELLS); ++sh) {
                if (NSHELL == 0 && sh >= nsh) break;
                float shell = 0.0f;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                  const ShellTap tp = shell_taps[sh * 3 + a];
#pragma unroll
                  for (int sg = 0; sg < 2; ++sg) {
                    const float sgn = sg ? -1.0f : 1.0f;
                    const float lt = fmaf(sgn, tp.dli, li);
                    const FloorF kl = floor_f(lt);
#if SBRC_PACKED
                    const float2 v = interior_tap2(tex, (unsigned)kl.i * tex.qk,
                                                   __ffma2_rn(make_float2(sgn, sgn), make_float2(tp.dtx, tp.dty),
                                                              make_float2(tx, ty)));
                    shell += lerpf(v.x, v.y, lt - kl.f);
#else
                    float v0 = 0.f, v1 = 0.f;
                    interior_tap(tex, (unsigned)kl.i * tex.qk, fmaf(sgn, tp.dtx, tx), fmaf(sgn, tp.dty, ty), v0, v1);
                    shell += lerpf(v0, v1, lt - kl.f);
#endif
                  }
                }
                acc += shell_taps[sh * 3].w * shell / 6.0f;
              }
            } else {
#pragma unroll
              for (int sh = 0; sh < (NSHELL > 0 ? NSHELL : SBRC_MAX_SHELLS); ++sh) {
                if (NSHELL == 0 && sh >= nsh) break;
                float shell = 0.0f;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                  const ShellTap tp = shell_taps[sh * 3 + a];
                  shell += light_lookup<LOOKUP>(tex, tx + tp.dtx, ty + tp.dty, li + tp.dli);
                  shell += light_lookup<LOOKUP>(tex, tx - tp.dtx, ty - tp.dty, li - tp.dli);
                }
                acc += shell_taps[sh * 3].w * shell / 6.0f;
              }
            }
            scalar = acc;
          } else {  // cone
            const bool degenerate = !((double)dperp * t > 1e-12);  // fallback plane_basis(L)[0] = axis_u
            float acc = 0.0f;
            const bool fast = CONE_N > 0 && LOOKUP == SBRC_LOOKUP_LINEAR &&
                              (SBRC_LIGHT_FASTSEG ? (jf >= jfast_lo && jf <= jfast_hi)
                                                  : (!degenerate && tx - reach_x >= 0.f && tx + reach_x < fast_x_hi &&
                                                     ty - reach_y >= 0.f && ty + reach_y < fast_y_hi &&
                                                     li - (float)CONE_A >= 0.f && li - 1.0f < fast_l_hi));
            if (fast) {
              // every tap inside the buffer: one layer pair per ring, blended once
#if SBRC_CONE_RING_SERIAL
#pragma unroll 1
#else
#pragma unroll
#endif
              for (int i = 1; i <= CONE_A; ++i) {
                const float r = spacing_r * (float)i;
                const float lt = li - (float)i;
                const FloorF kl = floor_f(lt);
                const unsigned kb = (unsigned)kl.i * tex.qk;
#if SBRC_PACKED_CONE
                float2 v = make_float2(0.f, 0.f);
                const float2 c = make_float2(tx, ty);
#pragma unroll
                for (int j = 0; j < NA; ++j)
                  v = __fadd2_rn(v, interior_tap2(tex, kb, __ffma2_rn(make_float2(r, r), make_float2(wx[j], wy[j]), c)));
                acc += lerpf(v.x, v.y, lt - kl.f);
#else
                float v0 = 0.f, v1 = 0.f;
#pragma unroll
                for (int j = 0; j < NA; ++j) interior_tap(tex, kb, fmaf(r, wx[j], tx), fmaf(r, wy[j], ty), v0, v1);
                acc += lerpf(v0, v1, lt - kl.f);
#endif
              }
              scalar = acc * (1.0f / (float)(CONE_A * NA));
            } else if (CONE_N > 0) {
#pragma unroll
              for (int i = 1; i <= CONE_A; ++i) {
                const float r = spacing_r * (float)i;
                const float ki = li - (float)i;
#pragma unroll
                for (int j = 0; j < NA; ++j) {
                  float ox = r * wx[j], oy = r * wy[j];
                  if (degenerate) {
                    const float c = cone_cs[j].x, sn = cone_cs[j].y;
                    ox = r * (float)sx * c;
                    oy = r * (float)sy * sn;
                  }
                  acc += light_lookup<LOOKUP>(tex, tx + ox, ty + oy, ki);
                }
              }
              scalar = acc * (1.0f / (float)(CONE_A * NA));
            } else {
              const float bu = degenerate ? 1.0f : bu_fb, bv = degenerate ? 0.0f : bv_fb;
              for (int i = 1; i <= P.cone_axis_samples; ++i) {
                const float r = spacing_r * (float)i;
                const float ki = li - (float)i;
                for (int j = 0; j < P.cone_angle_count; ++j) {
                  const float2 cs = cone_cs[j];
                  const float ox = r * (float)sx * (bu * cs.x - bv * cs.y);
                  const float oy = r * (float)sy * (bv * cs.x + bu * cs.y);
                  acc += light_lookup<LOOKUP>(tex, tx + ox, ty + oy, ki);
                }
              }
              scalar = acc / (float)(P.cone_axis_samples * P.cone_angle_count);
            }
          }
          if (white) {
            fr = fg = fb = (double)fmaxf(scalar, 0.0f);
          } else {
            fr = fr_c > 0.f ? (double)(fmaxf(scalar * fr_c, P.ambient_floor) * ir) : 1.0;
            fg = fg_c > 0.f ? (double)(fmaxf(scalar * fg_c, P.ambient_floor) * ig) : 1.0;
            fb = fb_c > 0.f ? (double)(fmaxf(scalar * fb_c, P.ambient_floor) * ib) : 1.0;
          }
        }
      };
      if constexpr (G == 1) {
      // One sample: shade the prefetched cell `use` while the next sample's
      // cell is gathered into `fill` (PF), or gather this sample's cell now.
      auto sample = [&](const Cell<VT>& use_pf, const bool use_in_pf, Cell<VT>& fill, bool& fill_in) {
        const double tn = dadd(t, step);
        Cell<VT> use_now;
        bool use_in_now = false;
        {
          const double tc = PF ? tn : t;  // the cell gathered here: the next sample's (PF) or this one's
          Cell<VT>& dst = PF ? fill : use_now;
          bool& dst_in = PF ? fill_in : use_in_now;
          const double qx = dadd(P.eye[0], dmul(tc, d[0]));
          const double qy = dadd(P.eye[1], dmul(tc, d[1]));
          const double qz = dadd(P.eye[2], dmul(tc, d[2]));
          if (UNIT && SBRC_MARCH_FASTSEG && tc >= t_safe_lo && tc <= t_safe_hi) {
            dst_in = true;
            cell_fetch_interior<VT>(P.volume, qx, qy, qz, dst);
          } else {
            dst_in = in_cube(qx, qy, qz);
            if (dst_in) cell_fetch<VT, UNIT>(P.volume, qx, qy, qz, dst);
          }
        }
        if (!PF) fill_in = false;
        const Cell<VT>& use = PF ? use_pf : use_now;
        const bool use_in = PF ? use_in_pf : use_in_now;
#if SBRC_PREC == 0
        const double s = use_in ? cell_combine<VT>(use, reinterpret_cast<const float*>(u8tab)) : 0.0;
        const LutPos q = lut_pos(s);
        const double2 a_rg = lut[2 * q.i0], a_ba = lut[2 * q.i0 + 1];
        const double2 b_rg = lut[2 * q.i1], b_ba = lut[2 * q.i1 + 1];
        const double sr = dadd(dmul(a_rg.x, q.g), dmul(b_rg.x, q.f));
        const double sg = dadd(dmul(a_rg.y, q.g), dmul(b_rg.y, q.f));
        const double sb = dadd(dmul(a_ba.x, q.g), dmul(b_ba.x, q.f));
        const double sa = dadd(dmul(a_ba.y, q.g), dmul(b_ba.y, q.f));

        double fr = 1.0, fg = 1.0, fb = 1.0;
        // premultiplied emission (transfer.py:74) is 0 up to clear_t
        if (!SKIP || !(q.t <= clear_t)) light_factor(fr, fg, fb);
        // C += (1-a)*rgb*factor; a += (1-a)*a_src (raycaster.py:436-438)
        const double one_m = dsub(1.0, alpha);
        cr = dadd(cr, dmul(dmul(one_m, sr), fr));
        cg = dadd(cg, dmul(dmul(one_m, sg), fg));
        cb = dadd(cb, dmul(dmul(one_m, sb), fb));
        alpha = dadd(alpha, dmul(one_m, sa));
#elif SBRC_PREC == 1
        const double s = use_in ? cell_combine<VT>(use, reinterpret_cast<const float*>(u8tab)) : 0.0;
        const LutPos q = lut_pos(s);
        const double sa = dadd(dmul(lut[2 * q.i0 + 1].y, q.g), dmul(lut[2 * q.i1 + 1].y, q.f));
        const float ff = (float)q.f;
        const float4 c0 = lutf[q.i0], c1 = lutf[q.i1];
        double fr = 1.0, fg = 1.0, fb = 1.0;
        if (!SKIP || !(q.t <= clear_t)) light_factor(fr, fg, fb);
        const double one_m = dsub(1.0, alpha);
        const float om = (float)one_m;
        crf = fmaf(om * lerpf(c0.x, c1.x, ff), (float)fr, crf);
        cgf = fmaf(om * lerpf(c0.y, c1.y, ff), (float)fg, cgf);
        cbf = fmaf(om * lerpf(c0.z, c1.z, ff), (float)fb, cbf);
        alpha = dadd(alpha, dmul(one_m, sa));
#else
        const float s = use_in ? cell_combine_f<VT>(use, reinterpret_cast<const float*>(u8tab)) : 0.0f;
        const float lt = __saturatef(s) * 255.0f;
        const FloorF lfl = floor_f(lt);
        const int i0 = lfl.i, i1 = min(lfl.i + 1, SBRC_LUT_SIZE - 1);
        const float ff = lt - lfl.f;
        const float4 c0 = lutf[i0], c1 = lutf[i1];
        double fr = 1.0, fg = 1.0, fb = 1.0;
        if (!SKIP || !(lt <= (float)clear_t)) light_factor(fr, fg, fb);
        const float om = 1.0f - alphaf;
        crf = fmaf(om * lerpf(c0.x, c1.x, ff), (float)fr, crf);
        cgf = fmaf(om * lerpf(c0.y, c1.y, ff), (float)fg, cgf);
        cbf = fmaf(om * lerpf(c0.z, c1.z, ff), (float)fb, cbf);
        alphaf = fmaf(om, lerpf(c0.w, c1.w, ff), alphaf);
        alpha = alphaf;
#endif
        t = tn;
        jf += 1.0f;
        ++samples;
      };
#if SBRC_WARP_VOTE
      // Early ray termination as a warp vote: the warp steps while any lane's
      // ray is live (raycaster.py:429 live test per lane, before each sample).
      // The lanes that reach this loop (valid pixels whose ray hits the cube)
      // vote among themselves.
      const unsigned vmask = __activemask();
      bool live = t < t_far && alpha < thresh;
      while (__any_sync(vmask, live)) {
        if (live) {
          Cell<VT> nxt;
          bool nxt_in;
          sample(cur, cur_in, nxt, nxt_in);
          cur = nxt;
          cur_in = nxt_in;
          live = t < t_far && alpha < thresh;
        }
      }
#else
      while (t < t_far && alpha < thresh) {
        Cell<VT> nxt;
        bool nxt_in;
        sample(cur, cur_in, nxt, nxt_in);
        cur = nxt;
        cur_in = nxt_in;
      }
#endif
      } else {
        // Ray group: each lane shades its own samples; the G samples of a
        // step are then composited in order by every lane of the group with
        // the reference's live test before each (the same float64 operations
        // in the same order as the serial loop). Samples a lane computed past
        // the ray's end are discarded.
        const unsigned gmask = ((1u << G) - 1u) << (lane & ~(G - 1));
        bool done = false;
        while (!done) {
          double tn = t;
#pragma unroll
          for (int i = 0; i < G; ++i) tn = dadd(tn, step);
          Cell<VT> nxt;
          bool nxt_in;
          {
            const double qx = dadd(P.eye[0], dmul(tn, d[0]));
            const double qy = dadd(P.eye[1], dmul(tn, d[1]));
            const double qz = dadd(P.eye[2], dmul(tn, d[2]));
            nxt_in = in_cube(qx, qy, qz);
            if (nxt_in) cell_fetch<VT, UNIT>(P.volume, qx, qy, qz, nxt);
          }
          const bool have = t < t_far;
          double sr = 0.0, sg = 0.0, sb = 0.0, sa = 0.0;
          float fr = 1.0f, fg = 1.0f, fb = 1.0f;
          if (have) {
            const double s = cur_in ? cell_combine<VT>(cur, reinterpret_cast<const float*>(u8tab)) : 0.0;
            const LutPos q = lut_pos(s);
            const double2 a_rg = lut[2 * q.i0], a_ba = lut[2 * q.i0 + 1];
            const double2 b_rg = lut[2 * q.i1], b_ba = lut[2 * q.i1 + 1];
            sr = dadd(dmul(a_rg.x, q.g), dmul(b_rg.x, q.f));
            sg = dadd(dmul(a_rg.y, q.g), dmul(b_rg.y, q.f));
            sb = dadd(dmul(a_ba.x, q.g), dmul(b_ba.x, q.f));
            sa = dadd(dmul(a_ba.y, q.g), dmul(b_ba.y, q.f));
            double dfr = 1.0, dfg = 1.0, dfb = 1.0;
            if (!SKIP || !(q.t <= clear_t)) light_factor(dfr, dfg, dfb);
            fr = (float)dfr;  // buffer-mode factors are float32 values: exact round trip
            fg = (float)dfg;
            fb = (float)dfb;
          }
#pragma unroll
          for (int k = 0; k < G; ++k) {
            const int src = (lane & ~(G - 1)) + k;
            const double ksr = __shfl_sync(gmask, sr, src), ksg = __shfl_sync(gmask, sg, src);
            const double ksb = __shfl_sync(gmask, sb, src), ksa = __shfl_sync(gmask, sa, src);
            const float kfr = __shfl_sync(gmask, fr, src);
            const float kfg = white ? kfr : __shfl_sync(gmask, fg, src);
            const float kfb = white ? kfr : __shfl_sync(gmask, fb, src);
            const bool khave = __shfl_sync(gmask, (int)have, src) != 0;
            if (!done) {
              if (khave && alpha < thresh) {
                const double one_m = dsub(1.0, alpha);
                cr = dadd(cr, dmul(dmul(one_m, ksr), (double)kfr));
                cg = dadd(cg, dmul(dmul(one_m, ksg), (double)kfg));
                cb = dadd(cb, dmul(dmul(one_m, ksb), (double)kfb));
                alpha = dadd(alpha, dmul(one_m, ksa));
                if (gl == 0) ++samples;
              } else {
                done = true;
              }
            }
          }
          t = tn;
          cur = nxt;
          cur_in = nxt_in;
          jf += (float)G;
        }
      }
#if SBRC_PREC
      if constexpr (G == 1) {
        cr = crf;
        cg = cgf;
        cb = cbf;
      }
#endif
      result = make_float4((float)cr, (float)cg, (float)cb, (float)alpha);
    }
  }
  if (in_image && gl == 0) {  // background (and padding rows of a partial last band) is transparent black
    SBRC_CHECK(lr >= 0 && px >= 0 && lr < P.local_rows && px < P.width, 3);
    if (P.image != nullptr) reinterpret_cast<float4*>(P.image)[(size_t)lr * P.width + px] = result;
    // fused assembly: the pixel goes straight into every rank's raster image
    // (peer memory over NVLink); a barrier after the kernel completes the frame
    if (valid)
      for (int i = 0; i < P.n_peers; ++i)
      {
        SBRC_CHECK(py >= 0 && py < P.height && px < P.width, 4);
        reinterpret_cast<float4*>(P.peer_images[i])[(size_t)py * P.width + px] = result;
      }
  }
  if (P.n_peers > 0) __threadfence_system();
  if (P.sample_count != nullptr) {
    const unsigned int tot = __reduce_add_sync(0xffffffffu, samples);
    if (lane == 0 && tot) atomicAdd(P.sample_count, (unsigned long long)tot);
  }
  if (P.tile_steps != nullptr) {  // measured cost of this tile: its longest ray's sample count
    const unsigned int mx = __reduce_max_sync(0xffffffffu, samples);
    SBRC_CHECK(by * (int)gridDim.x + bx < P.n_tiles, 5);
    if (lane == 0 && mx) atomicMax(P.tile_steps + (by * gridDim.x + bx), mx);
  }
}

// ---------------------------------------------------------------- dispatch
inline bool volume_ok(const sbrc_volume& v) {
  if (v.data == nullptr) return false;
  if (v.nx < 2 || v.ny < 2 || v.nz < 2) return false;  // volume.py:80-81
  if ((unsigned long long)v.nx * v.ny * v.nz >= (1ull << 32)) return false;  // 32-bit voxel offsets
  if (v.voxel_type < SBRC_VOXEL_F32 || v.voxel_type > SBRC_VOXEL_U16) return false;
  for (int c = 0; c < 3; ++c)
    if (!(v.box_ext[c] > 0.0)) return false;
  return true;
}

inline bool light_ok(const sbrc_light_frame& L) {
  return L.width >= 1 && L.height >= 1 && L.n_slices >= 1 && L.d_max > L.d_min &&
         L.u_range[1] > L.u_range[0] && L.v_range[1] > L.v_range[0];
}

// Largest quad offset must fit 32 bits (K2 addresses quads with 32-bit offsets).
inline bool quads_ok(const sbrc_light_frame& L, int64_t qk, int64_t qy) {
  if (qk < 1 || qy < L.width) return false;
  const long long last = (long long)(L.n_slices - 1) * qk + (long long)(L.height - 1) * qy + L.width;
  return last < (1ll << 32);
}

// Rank-local image rows of a launch: the contiguous range, or the rank's bands.
inline int rank_rows(const sbrc_render_params& p) {
  return p.row_count > 0 ? p.row_count : sbrc_local_rows(p.height, p.band_rows, p.rank, p.world);
}

inline bool unit_box(const sbrc_volume& v) {
  for (int c = 0; c < 3; ++c)
    if (v.box_lo[c] != 0.0 || v.box_ext[c] != 1.0) return false;
  return true;
}

template <int SH, int LK, int VT, bool UNIT, int NS, int CA, int CN, bool SKIP>
void launch_march_skip(const sbrc_render_params& p, cudaStream_t s) {
  sbrc_render_params q = p;
  q.local_rows = rank_rows(p);
  // latency mode for the default kernels when the rank-local image is small
  // (A/B in profiles/r01_notes.md: 131K px/rank 1.05 -> 0.75 ms; 262K px: 1.16 vs 1.28)
  constexpr bool LAT = LK == SBRC_LOOKUP_LINEAR &&
                       ((SH == SBRC_SHADE_CONE && CN > 0) ||
                        (SBRC_LATENCY_ALL && ((SH == SBRC_SHADE_SHELL && NS > 0) || SH == SBRC_SHADE_SHADOW)));
  const MarchShape m = march_shape(q, q.local_rows);
  const int n_tiles = m.tiles_x * m.tiles_y;
  // A table sized for another grid is stale: dispatch in natural order and
  // record no per-tile costs (tile_steps is indexed by this launch's grid and
  // is only written when the caller sized it for exactly that grid).
  if (q.n_tiles != n_tiles) {
    q.tile_order = nullptr;
    q.tile_steps = nullptr;
  }
  constexpr int LG = SBRC_LAT_GROUP;
  const dim3 grid(m.tiles_x, m.tiles_y);
  if constexpr (LAT) {
    if (m.latency && m.group > 1) {
      if (m.nw == 8) march_kernel<SH, LK, VT, UNIT, NS, CA, CN, 1, SKIP, 8, LG><<<grid, 256, 0, s>>>(q);
      else march_kernel<SH, LK, VT, UNIT, NS, CA, CN, 1, SKIP, 4, LG><<<grid, 128, 0, s>>>(q);
      return;
    }
    if (m.latency) {
      if (m.nw == 8) march_kernel<SH, LK, VT, UNIT, NS, CA, CN, 1, SKIP, 8, 1><<<grid, 256, 0, s>>>(q);
      else march_kernel<SH, LK, VT, UNIT, NS, CA, CN, 1, SKIP, 4, 1><<<grid, 128, 0, s>>>(q);
      return;
    }
  }
  if (m.nw == 8) march_kernel<SH, LK, VT, UNIT, NS, CA, CN, 2, SKIP, 8, 1><<<grid, 256, 0, s>>>(q);
  else march_kernel<SH, LK, VT, UNIT, NS, CA, CN, SBRC_NARROW_MINB, SKIP, 4, 1><<<grid, 128, 0, s>>>(q);
}

// skip_clear (a speed hint; results are identical either way) selects the
// instantiation that skips the light factor of zero-emission samples.
template <int SH, int LK, int VT, bool UNIT, int NS, int CA, int CN>
void launch_march(const sbrc_render_params& p, cudaStream_t s) {
  if constexpr (SBRC_SKIP_CLEAR && SH != SBRC_SHADE_NONE) {
    if (p.skip_clear) {
      launch_march_skip<SH, LK, VT, UNIT, NS, CA, CN, true>(p, s);
      return;
    }
  }
  launch_march_skip<SH, LK, VT, UNIT, NS, CA, CN, false>(p, s);
}

template <int SH, int LK, int VT, bool UNIT>
void launch_march_kernel_shape(const sbrc_render_params& p, cudaStream_t s) {
  if constexpr (SH == SBRC_SHADE_SHELL) {
    if (p.shell_count == 3) launch_march<SH, LK, VT, UNIT, 3, 0, 0>(p, s);
    else launch_march<SH, LK, VT, UNIT, 0, 0, 0>(p, s);
  } else if constexpr (SH == SBRC_SHADE_CONE) {
    if (p.cone_axis_samples == 2 && p.cone_angle_count == 4) launch_march<SH, LK, VT, UNIT, 0, 2, 4>(p, s);
    else launch_march<SH, LK, VT, UNIT, 0, 0, 0>(p, s);
  } else {
    launch_march<SH, LK, VT, UNIT, 0, 0, 0>(p, s);
  }
}
template <int SH, int LK, int VT>
void launch_march_box(const sbrc_render_params& p, cudaStream_t s) {
  if (unit_box(p.volume)) launch_march_kernel_shape<SH, LK, VT, true>(p, s);
  else launch_march_kernel_shape<SH, LK, VT, false>(p, s);
}
template <int SH, int VT>
void launch_march_lookup(const sbrc_render_params& p, cudaStream_t s) {
  if constexpr (SH == SBRC_SHADE_SHADOW || SH == SBRC_SHADE_SHELL || SH == SBRC_SHADE_CONE) {
    if (p.lookup == SBRC_LOOKUP_NEAREST) {
      launch_march_box<SH, SBRC_LOOKUP_NEAREST, VT>(p, s);
      return;
    }
  }
  launch_march_box<SH, SBRC_LOOKUP_LINEAR, VT>(p, s);
}
}  // namespace

// Read (and optionally reset) this translation unit's checked-build counters,
// adding them into acc[8].
inline int tu_violations(unsigned int* acc, int reset) {
#if SBRC_CHECKED
  unsigned int c[8];
  if (cudaMemcpyFromSymbol(c, sbrc_violations, sizeof(c)) != cudaSuccess) return SBRC_ECUDA;
  for (int i = 0; i < 8; ++i) acc[i] += c[i];
  if (reset) {
    const unsigned int zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cudaMemcpyToSymbol(sbrc_violations, zero, sizeof(zero)) != cudaSuccess) return SBRC_ECUDA;
  }
  return SBRC_OK;
#else
  (void)acc;
  (void)reset;
  return SBRC_EUNSUPPORTED;
#endif
}

// K2 dispatch for one (shading mode, voxel type): march_inst.cu compiled
// once per pair (build.py), so the instantiations compile in parallel.
#define SBRC_MARCH_FN_(SH, VT) sbrc_march_##SH##_##VT
#define SBRC_MARCH_FN(SH, VT) SBRC_MARCH_FN_(SH, VT)
#define SBRC_MARCH_VIOL_(SH, VT) sbrc_march_violations_##SH##_##VT
#define SBRC_MARCH_VIOL(SH, VT) SBRC_MARCH_VIOL_(SH, VT)
#define SBRC_MARCH_DECL(SH, VT)                                                   \
  void SBRC_MARCH_FN(SH, VT)(const sbrc_render_params& p, cudaStream_t s);      \
  int SBRC_MARCH_VIOL(SH, VT)(unsigned int* acc, int reset);
#define SBRC_MARCH_DECL_VT(SH) SBRC_MARCH_DECL(SH, 0) SBRC_MARCH_DECL(SH, 1) SBRC_MARCH_DECL(SH, 2)
SBRC_MARCH_DECL_VT(0)
SBRC_MARCH_DECL_VT(1)
SBRC_MARCH_DECL_VT(2)
SBRC_MARCH_DECL_VT(3)
SBRC_MARCH_DECL_VT(4)
SBRC_MARCH_DECL_VT(5)
