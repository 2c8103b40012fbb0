// sbrc.cu — the C ABI of include/sbrc.h: K1 (attenuation build), the
// point-wise light factor, shadow oracle, half-angle baseline, raw-volume
// normalisation, IPC helpers, and K2 dispatch to march_inst.cu instances.
// Kernel documentation and the numerics contract: sbrc_common.cuh.

#include "sbrc_common.cuh"

#include <cudaTypedefs.h>  // CUtensorMap, PFN_cuTensorMapEncodeTiled (driver entry point; no libcuda link)

#include <climits>
#include <cmath>

namespace {

// ---------------------------------------------------------------- K1 build
// One thread per light texel; the slice recurrence runs in registers
// (lightbuffer.py:166-198): intensity[k] = T; if the texel-slice point is in
// the cube, alpha = lut(trilinear(p)) and T *= 1 - alpha. Texels are
// independent, so no grid-wide barrier or per-slice launch is needed. The
// quad of layer k needs layer k+1, so it is emitted one slice late.
// K1 block: 4 warps (light rows) — the finer blocks even out the last wave
// of uneven texel rows (A/B in profiles/r01_notes.md: config 3 build 0.466
// -> 0.417 ms, config 2 0.209 -> 0.179, config 4 3.61 -> 3.47) — compiled
// for 8 blocks/SM (64 registers, 32 warps/SM, one slice's gathers at a time;
// vs 6 blocks/SM with two slices in flight: config 3 0.309 -> 0.299 ms,
// config 2 0.136 -> 0.132, config 4 2.15 -> 2.12, profiles/r2_notes.md).
#ifndef SBRC_BUILD_ROWS
#define SBRC_BUILD_ROWS 4
#endif
#ifndef SBRC_BUILD_MINB
#define SBRC_BUILD_MINB 8
#endif
// Async gather pipeline (float32 volumes): the 8 corner voxels of slice
// k + D - 1 are copied global -> shared with cp.async (LDGSTS, no register
// staging) while slice k is combined, so D - 1 slices of gathers are in
// flight per texel instead of SBRC_BUILD_UNROLL held in registers.
#ifndef SBRC_BUILD_ASYNC
#define SBRC_BUILD_ASYNC 0  // A/B option: slower on config 3 (0.309 -> 0.355 ms at D = 4; profiles/r2_notes.md)
#endif
#ifndef SBRC_BUILD_ASYNC_MINB
#define SBRC_BUILD_ASYNC_MINB 6
#endif

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// TMA-staged volume tiles (D = -1, float32 volumes in the unit box): the
// block's texel-slice points of C consecutive slices lie in a small
// parallelepiped of the volume; its axis-aligned bounding box is loaded into
// shared memory by one cp.async.bulk.tensor.3d (TMA, mbarrier completion),
// double-buffered so the box of the next C slices streams in while this one
// is sampled, and the 8 corner gathers of each point become shared-memory
// loads. Box shape and C come from the light geometry (tma_plan).
#ifndef SBRC_BUILD_TMA
#define SBRC_BUILD_TMA 0  // A/B option: bit-exact but 3.3x slower on config 3 (profiles/r2_notes.md)
#endif
#ifndef SBRC_BUILD_TMA_SMEM
#define SBRC_BUILD_TMA_SMEM (100 * 1024)  // shared-memory budget of the two boxes per block
#endif
#ifndef SBRC_BUILD_TMA_MINB
#define SBRC_BUILD_TMA_MINB 2
#endif

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(m)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            unsigned long long* m) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(m))
      : "memory");
}

template <int VT, bool UNIT, int D>
__global__ void __launch_bounds__(32 * SBRC_BUILD_ROWS,
                                  D > 0 ? SBRC_BUILD_ASYNC_MINB : (D < 0 ? SBRC_BUILD_TMA_MINB : SBRC_BUILD_MINB))
    build_kernel(const sbrc_build_params P, const __grid_constant__ CUtensorMap tmap, const int4 tbox) {
  static_assert(D == 0 || VT == SBRC_VOXEL_F32, "the async gather / TMA pipelines copy 4-byte voxels");
  static_assert(D >= 0 || UNIT, "TMA boxes are placed in unit-box voxel coordinates");
  __shared__ double lut[SBRC_LUT_SIZE];
  __shared__ double u8tab[VT == SBRC_VOXEL_U8 ? 256 : 1];
  for (int i = threadIdx.y * blockDim.x + threadIdx.x; i < SBRC_LUT_SIZE; i += blockDim.x * blockDim.y)
    lut[i] = P.alpha_lut[i];
  if (std::is_same<typename Voxel<VT>::T, unsigned char>::value) fill_u8_table(u8tab);
  __syncthreads();

  const sbrc_light_frame& L = P.light;
  // Warps are 32 consecutive texels of one row overlapping the next warp by
  // one: lane 31 only hands its layer pair to lane 30, so every quad is one
  // 16-byte store (the right neighbour's pair arrives by shuffle).
  const int lane = threadIdx.x;
  const int x = blockIdx.x * 31 + lane;
  const int y = P.row_begin + blockIdx.y * blockDim.y + threadIdx.y;
  const bool row_ok = y < P.row_end;
  if constexpr (D >= 0) {
    if (!row_ok) return;  // whole warp (warps are rows)
  }
  const bool owner = row_ok && lane < 31 && x < L.width;

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
  float4* row = reinterpret_cast<float4*>(P.quads) + (size_t)(y - P.row_begin) * (size_t)P.quad_row_stride;
  float* prow = reinterpret_cast<float*>(P.quads) + (size_t)(y - P.row_begin) * (size_t)P.quad_row_stride;
  const size_t ks = (size_t)P.quad_layer_stride;
  const bool plain = P.output_plain != 0;
  auto put = [&](int kk, const float4& q) {  // texel quad, or its layer-k value in the plain layout
    SBRC_CHECK(kk >= 0 && kk < L.n_slices && x < L.width && y < P.row_end, 2);
    if (plain) prow[(size_t)kk * ks + x] = q.x;
    else if (SBRC_PAIRS || P.quad_layout == 1)  // layer pairs: (I[k], I[k+1]) of this texel at the quad offset
      reinterpret_cast<float2*>(P.quads)[(size_t)(y - P.row_begin) * (size_t)P.quad_row_stride + (size_t)kk * ks + x] =
          make_float2(q.x, q.y);
    else row[(size_t)kk * ks + x] = q;
  };
  const float* tab = reinterpret_cast<const float*>(u8tab);
  double T = 1.0;
  float prev = 0.0f;
  // One slice of the recurrence: stored = T (:169); if covered, alpha from the
  // cell, optional compensation (:193-196), T *= 1 - alpha (:197-198).
  auto step_slice = [&](bool covered, const Cell<VT>& cl) -> float {
    float stored = (float)T;
    if (covered) {
      const LutPos q = lut_pos(cell_combine<VT>(cl, tab));
      const double a = dadd(dmul(lut[q.i0], q.g), dmul(lut[q.i1], q.f));
      if (comp) stored = (float)dmul((double)stored, pow(dadd(1.0, a), P.compensation_n));
      T = dmul(T, dsub(1.0, a));
    }
    return stored;
  };
  // pts = base + offset_k * L (:182); covered = all(0 <= pts <= 1) (:183)
  auto point = [&](int k, double& px, double& py, double& pz) {
    SBRC_CHECK(k >= 0 && k < L.n_slices, 7);
    const double off = __ldg(L.plane_offsets + k);
    px = dadd(base[0], dmul(off, L.light_dir[0]));
    py = dadd(base[1], dmul(off, L.light_dir[1]));
    pz = dadd(base[2], dmul(off, L.light_dir[2]));
  };
  // Slices whose texel-slice point is provably outside the cube need no
  // float64 test: along the texel's line p(o) = base + o*L the cube is the
  // offset interval [o_lo, o_hi] (slab test per axis); slices more than two
  // slice spacings outside it are uncovered with a margin of >= 1.5 spacings
  // times |L_c| >= 1e-6 (far above float64 rounding), so they store T
  // unchanged. The warp runs the exact per-slice test over the union of its
  // lanes' conservative ranges [kA, kB] and only stores before and after it
  // (results bit-identical; near-axis-parallel light falls back to testing
  // every slice).
  const int n = L.n_slices;
  int k_lo = 0, k_hi = n - 1;
  {
    const double spacing = (L.d_max - L.d_min) / n;
    double olo = -INFINITY, ohi = INFINITY;
    bool ranged = true;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double lc = L.light_dir[c];
      if (fabs(lc) < 1e-6) {
        ranged = false;
      } else {
        const double a = (0.0 - base[c]) / lc, b = (1.0 - base[c]) / lc;
        olo = fmax(olo, fmin(a, b));
        ohi = fmin(ohi, fmax(a, b));
      }
    }
    if (ranged) {
      const double kf = fmin(fmax((olo - L.d_min) / spacing - 0.5, -8.0), n + 8.0);
      const double kl = fmin(fmax((ohi - L.d_min) / spacing - 0.5, -8.0), n + 8.0);
      k_lo = max(0, (int)floor(kf) - 2);
      k_hi = min(n - 1, (int)ceil(kl) + 2);
    }
  }
  // Written layers [w_lo, w_hi] of this texel (all of them unless sparse):
  // the slab test of the texel's line against the cube inflated by
  // write_reach, widened by write_below / write_above plus two layers.
  int w_lo = 0, w_hi = n - 1;
  if (P.write_sparse) {
    const double R = P.write_reach, spacing = (L.d_max - L.d_min) / n;
    double olo = -INFINITY, ohi = INFINITY;
    bool empty = false;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double lc = L.light_dir[c];
      if (fabs(lc) < 1e-6) {  // nearly parallel: the coordinate moves < 1e-5 over the stack
        if (base[c] < -R - 1e-5 || base[c] > 1.0 + R + 1e-5) empty = true;
      } else {
        const double a = (-R - base[c]) / lc, b = (1.0 + R - base[c]) / lc;
        olo = fmax(olo, fmin(a, b));
        ohi = fmin(ohi, fmax(a, b));
      }
    }
    // consumer clip half-spaces n.p + c >= 0 along the line: (n.base + c) + o (n.L) >= 0
    for (int i = 0; i < P.n_clip; ++i) {
      const double* h = P.clip[i];
      const double s0 = h[0] * base[0] + h[1] * base[1] + h[2] * base[2] + h[3];
      const double sl = h[0] * L.light_dir[0] + h[1] * L.light_dir[1] + h[2] * L.light_dir[2];
      const double nn = fabs(h[0]) + fabs(h[1]) + fabs(h[2]);
      if (fabs(sl) <= 1e-9 * nn) {  // plane (nearly) parallel to the light: the whole line or nothing
        if (s0 < -1e-9 * nn) empty = true;
      } else if (sl > 0.0) {
        olo = fmax(olo, -s0 / sl);
      } else {
        ohi = fmin(ohi, -s0 / sl);
      }
    }
    if (empty || olo > ohi) {
      w_lo = n;
      w_hi = -1;
    } else {
      const double kf = fmin(fmax((olo - L.d_min) / spacing - 0.5, -8.0 - P.write_below), n + 8.0);
      const double kl = fmin(fmax((ohi - L.d_min) / spacing - 0.5, -8.0), n + 8.0 + P.write_above);
      w_lo = max(0, (int)floor(kf) - 2 - P.write_below);
      w_hi = min(n - 1, (int)ceil(kl) + 2 + P.write_above);
    }
  }
  auto writes = [&](int kk) { return owner && kk >= w_lo && kk <= w_hi; };
  if (!row_ok) {  // (TMA blocks only: rows past the end idle through the block's barriers)
    k_lo = n;
    k_hi = -1;
  }
  const int kA = __reduce_min_sync(0xffffffffu, k_lo <= k_hi ? k_lo : n);
  int kB = __reduce_max_sync(0xffffffffu, k_lo <= k_hi ? k_hi : -1);
  if (P.write_sparse && P.n_clip > 0) {
    // the last quad any texel of the warp writes is w_hi: it needs I[w_hi + 1],
    // the value stored at slice w_hi + 1 (T after slice w_hi) — later slices are not needed
    const int wmax = __reduce_max_sync(0xffffffffu, owner && w_lo <= w_hi ? w_hi : -1);
    kB = min(kB, wmax + 1);
  }
  // before the warp's range: T = 1 on every lane (and its right neighbour)
  const float4 ones = make_float4(1.f, 1.f, 1.f, 1.f);
  const int pre_end = kA > kB ? n : kA - 1;  // quads 0 .. kA-2 hold layers < kA only
  if (owner)
    for (int kk = max(0, w_lo), e = min(pre_end, w_hi + 1); kk < e; ++kk) put(kk, ones);
  if constexpr (D >= 0) {
    if (kA > kB) return;
  }
  auto emit_w = [&](int kk, float a, float b) {  // all lanes shuffle; stores only where written
    float ra = __shfl_down_sync(0xffffffffu, a, 1), rb = __shfl_down_sync(0xffffffffu, b, 1);
    if (x == L.width - 1) {
      ra = a;
      rb = b;
    }
    if (writes(kk)) put(kk, make_float4(a, b, ra, rb));
  };
  prev = 1.0f;
  int k = kA;
  if constexpr (D < 0) {
    extern __shared__ unsigned char tma_smem[];
    __shared__ int kblk[2];
    __shared__ int orig[2][3];
    __shared__ __align__(8) unsigned long long mbar[2];
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int bx = tbox.x, by = tbox.y, bz = tbox.z, C = tbox.w;
    const int bxy = bx * by, box_n = bxy * bz;
    const unsigned box_bytes = (unsigned)box_n * 4u;
    float* bufs[2];
    bufs[0] = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(tma_smem) + 127) & ~(uintptr_t)127);
    bufs[1] = bufs[0] + ((box_n + 31) & ~31);  // 128-byte aligned
    if (tid == 0) {
      kblk[0] = n;
      kblk[1] = -1;
      mbar_init(&mbar[0], 1);
      mbar_init(&mbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (lane == 0 && kA <= kB) {
      atomicMin(&kblk[0], kA);
      atomicMax(&kblk[1], kB);
    }
    __syncthreads();
    const int KA = kblk[0], KB = kblk[1];
    const int nch = KA > KB ? 0 : (KB - KA) / C + 1;
    const int dims[3] = {P.volume.nx, P.volume.ny, P.volume.nz};
    const unsigned nx = (unsigned)dims[0];
    // the block's corner texels (lanes 0..31 of rows row0 .. row0+3, clipped)
    const int xb[2] = {(int)blockIdx.x * 31, min((int)blockIdx.x * 31 + 31, L.width - 1)};
    const int yb0 = P.row_begin + (int)(blockIdx.y * blockDim.y);
    const int yb[2] = {yb0, min(yb0 + (int)blockDim.y - 1, P.row_end - 1)};
    // chunk i: slices [KA + i C, KA + i C + C - 1]; box origin = min over the 8
    // corners of the parallelepiped of floor(g) (the positions are affine in
    // texel and slice index), less one voxel of margin for float64 rounding
    auto issue = [&](int i) {
      const int c0 = KA + i * C, c1 = min(c0 + C - 1, KB);
      int mn[3] = {INT_MAX, INT_MAX, INT_MAX};
#pragma unroll 1
      for (int j = 0; j < 8; ++j) {
        const int xx = xb[j & 1], yy = yb[(j >> 1) & 1], kk = (j & 4) ? c1 : c0;
        const double u = dadd(L.u_range[0], dmul(ddiv(dadd((double)xx, 0.5), (double)L.width),
                                                 dsub(L.u_range[1], L.u_range[0])));
        const double v = dadd(L.v_range[0], dmul(ddiv(dadd((double)yy, 0.5), (double)L.height),
                                                 dsub(L.v_range[1], L.v_range[0])));
        const double off = __ldg(L.plane_offsets + kk);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double pc = dadd(dadd(dmul(u, L.axis_u[c]), dmul(v, L.axis_v[c])), dmul(off, L.light_dir[c]));
          mn[c] = min(mn[c], (int)floor(pc * dims[c] - 0.5));
        }
      }
      const int b = i & 1;
      const int bx0 = (mn[0] - 1) & ~3;  // the box's first x must be 16-byte aligned (TMA faults otherwise)
      orig[b][0] = bx0;
      orig[b][1] = mn[1] - 1;
      orig[b][2] = mn[2] - 1;
      mbar_expect_tx(&mbar[b], box_bytes);
      tma_load_3d(bufs[b], &tmap, bx0, mn[1] - 1, mn[2] - 1, &mbar[b]);
    };
    if (tid == 0 && nch > 0) issue(0);
    for (int i = 0; i < nch; ++i) {
      if (tid == 0 && i + 1 < nch) {
        // buffer (i+1)&1 was last read in chunk i-1, before the barrier that ended it
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(i + 1);
      }
      const int b = i & 1;
      mbar_wait(&mbar[b], (unsigned)((i >> 1) & 1));
      const float* sb = bufs[b];
      const int ox = orig[b][0], oy = orig[b][1], oz = orig[b][2];
      const int c0 = KA + i * C;
      const int k0 = max(c0, kA), k1 = min(c0 + C - 1, kB);  // this warp's slices of the chunk
      for (int kk = k0; kk <= k1; ++kk) {
        double p[3];
        point(kk, p[0], p[1], p[2]);
        const bool cov = in_cube(p[0], p[1], p[2]);
        Cell<VT> cl;
        if (cov) {
          int lo[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {  // cell_fetch's arithmetic (volume.py:175-182), unit box
            const double g = dsub(dmul(p[c], (double)dims[c]), 0.5);
            const FloorD fl = floor_d(g);
            cl.f[c] = dsub(g, fl.f);
            lo[c] = fl.i;
          }
          if ((unsigned)lo[0] < nx - 1 && (unsigned)lo[1] < (unsigned)(dims[1] - 1) &&
              (unsigned)lo[2] < (unsigned)(dims[2] - 1)) {
            const int o = ((lo[2] - oz) * by + (lo[1] - oy)) * bx + (lo[0] - ox);
            SBRC_CHECK(o >= 0 && o + bxy + bx + 1 < box_n, 0);
            cl.r[0] = sb[o]; cl.r[1] = sb[o + 1]; cl.r[2] = sb[o + bx]; cl.r[3] = sb[o + bx + 1];
            cl.r[4] = sb[o + bxy]; cl.r[5] = sb[o + bxy + 1]; cl.r[6] = sb[o + bxy + bx]; cl.r[7] = sb[o + bxy + bx + 1];
          } else {
            int a3[3], b3[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              a3[c] = min(max(lo[c], 0), dims[c] - 1);
              b3[c] = min(max(lo[c] + 1, 0), dims[c] - 1);
            }
            const int z0 = (a3[2] - oz) * bxy, z1 = (b3[2] - oz) * bxy, y0 = (a3[1] - oy) * bx, y1 = (b3[1] - oy) * bx;
            const int x0 = a3[0] - ox, x1 = b3[0] - ox;
            SBRC_CHECK(z0 + y0 + x0 >= 0 && z1 + y1 + x1 < box_n, 0);
            cl.r[0] = sb[z0 + y0 + x0]; cl.r[1] = sb[z0 + y0 + x1]; cl.r[2] = sb[z0 + y1 + x0]; cl.r[3] = sb[z0 + y1 + x1];
            cl.r[4] = sb[z1 + y0 + x0]; cl.r[5] = sb[z1 + y0 + x1]; cl.r[6] = sb[z1 + y1 + x0]; cl.r[7] = sb[z1 + y1 + x1];
          }
        }
        const float st = step_slice(cov, cl);
        if (kk > 0) emit_w(kk - 1, prev, st);
        prev = st;
      }
      __syncthreads();
    }
    if (kA > kB) return;
    k = kB + 1;
  } else if constexpr (D > 0) {
    // Stage st of this thread: corner voxels svox[st][c][tid] (landed by
    // cp.async) and the cell fractions sfr[st][a][tid] (float64, stored at
    // issue; sfr[st][0] = -1 marks an uncovered texel-slice point). Each
    // thread reads only its own slots, so no barrier is needed; a slot is
    // refilled only after the thread consumed it (program order).
    constexpr int NT = 32 * SBRC_BUILD_ROWS;
    __shared__ float svox[D > 0 ? D : 1][8][NT];
    __shared__ double sfr[D > 0 ? D : 1][3][NT];
    const int tid = threadIdx.y * 32 + threadIdx.x;
    const float* vb = reinterpret_cast<const float*>(P.volume.data);
    const int dims[3] = {P.volume.nx, P.volume.ny, P.volume.nz};
    const unsigned nx = (unsigned)P.volume.nx, nxy = (unsigned)P.volume.nx * (unsigned)P.volume.ny;
    auto issue = [&](int kk, int st) {
      double p[3];
      point(kk, p[0], p[1], p[2]);
      if (!in_cube(p[0], p[1], p[2])) {
        sfr[st][0][tid] = -1.0;
        return;
      }
      int lo[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {  // cell_fetch's arithmetic (volume.py:175-182)
        double local = p[c];
        if (!UNIT) local = dclip01(ddiv(dsub(p[c], P.volume.box_lo[c]), P.volume.box_ext[c]));
        const double g = dsub(dmul(local, (double)dims[c]), 0.5);
        const FloorD fl = floor_d(g);
        sfr[st][c][tid] = dsub(g, fl.f);
        lo[c] = fl.i;
      }
      unsigned o[8];
      if ((unsigned)lo[0] < nx - 1 && (unsigned)lo[1] < (unsigned)(dims[1] - 1) &&
          (unsigned)lo[2] < (unsigned)(dims[2] - 1)) {
        const unsigned c0 = (unsigned)lo[0] + nx * (unsigned)lo[1] + nxy * (unsigned)lo[2];
        o[0] = c0; o[1] = c0 + 1; o[2] = c0 + nx; o[3] = c0 + nx + 1;
        o[4] = c0 + nxy; o[5] = c0 + nxy + 1; o[6] = c0 + nxy + nx; o[7] = c0 + nxy + nx + 1;
      } else {
        unsigned a[3], b[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          a[c] = (unsigned)min(max(lo[c], 0), dims[c] - 1);
          b[c] = (unsigned)min(max(lo[c] + 1, 0), dims[c] - 1);
        }
        const unsigned z0 = a[2] * nxy, z1 = b[2] * nxy, y0 = a[1] * nx, y1 = b[1] * nx;
        o[0] = z0 + y0 + a[0]; o[1] = z0 + y0 + b[0]; o[2] = z0 + y1 + a[0]; o[3] = z0 + y1 + b[0];
        o[4] = z1 + y0 + a[0]; o[5] = z1 + y0 + b[0]; o[6] = z1 + y1 + a[0]; o[7] = z1 + y1 + b[0];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        SBRC_CHECK((unsigned long long)o[c] < (unsigned long long)nxy * (unsigned)dims[2], 0);
        cp_async4(&svox[st][c][tid], vb + o[c]);
      }
    };
    int si = 0;
    for (int j = 0; j < D - 1; ++j) {  // prologue: slices kA .. kA+D-2 in flight
      if (kA + j <= kB) issue(kA + j, si);
      cp_async_commit();
      si = si == D - 1 ? 0 : si + 1;
    }
    int sc = 0;
    for (; k <= kB; ++k) {
      if (k + D - 1 <= kB) issue(k + D - 1, si);
      cp_async_commit();
      si = si == D - 1 ? 0 : si + 1;
      cp_async_wait<D - 1>();  // this thread's copies of slice k have landed
      Cell<VT> cl;
      cl.f[0] = sfr[sc][0][tid];
      const bool cov = cl.f[0] >= 0.0;
      if (cov) {
        cl.f[1] = sfr[sc][1][tid];
        cl.f[2] = sfr[sc][2][tid];
#pragma unroll
        for (int c = 0; c < 8; ++c) cl.r[c] = svox[sc][c][tid];
      }
      sc = sc == D - 1 ? 0 : sc + 1;
      const float st = step_slice(cov, cl);
      if (k > 0) emit_w(k - 1, prev, st);
      prev = st;
    }
  } else {
  // Interior segment [kS, kE]: slices at which every lane's point lies inside
  // the volume with its whole trilinear cell (the texel line's interval in the
  // cube shrunk by half a voxel plus 1e-9 per face, one slice of slack each
  // side) — there the float64 cube test and the clamped-cell branch are
  // certainly true / untaken and are skipped (same values, bit-identical).
  int kS = n, kE = -1;
  if constexpr (UNIT && D == 0) {
    if (SBRC_BUILD_FASTSEG) {
      const int dims[3] = {P.volume.nx, P.volume.ny, P.volume.nz};
      const double spacing = (L.d_max - L.d_min) / n;
      double ilo = -INFINITY, ihi = INFINITY;
      bool ok = row_ok;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double lc = L.light_dir[c];
        const double m_lo = 0.5 / dims[c] + 1e-9, m_hi = (dims[c] - 0.5) / dims[c] - 1e-9;
        if (fabs(lc) < 1e-6) {
          ok = false;
        } else {
          const double a = (m_lo - base[c]) / lc, b = (m_hi - base[c]) / lc;
          ilo = fmax(ilo, fmin(a, b));
          ihi = fmin(ihi, fmax(a, b));
        }
      }
      int i_lo = n, i_hi = -1;
      if (ok && ilo < ihi) {
        i_lo = max(0, (int)ceil((ilo - L.d_min) / spacing - 0.5) + 1);
        i_hi = min(n - 1, (int)floor((ihi - L.d_min) / spacing - 0.5) - 1);
      }
      kS = __reduce_max_sync(0xffffffffu, i_lo <= i_hi ? i_lo : n);
      kE = __reduce_min_sync(0xffffffffu, i_lo <= i_hi ? i_hi : -1);
      kS = max(kS, kA);
      kE = min(kE, kB);
    }
  }
  auto fast_slice = [&](int kk) {
    double px, py, pz;
    point(kk, px, py, pz);
    Cell<VT> cl;
    cell_fetch_interior<VT>(P.volume, px, py, pz, cl);
    const float st = step_slice(true, cl);
    if (kk > 0) emit_w(kk - 1, prev, st);
    prev = st;
  };
  // SBRC_BUILD_UNROLL slices at a time: the gathers of all of them are issued
  // before any is combined (the product order of T is unchanged, so the
  // result stays bit-exact).
  constexpr int U = SBRC_BUILD_UNROLL;
  for (; k + U <= kB + 1; k += U) {
    if (k >= kS && k <= kE) {  // warp-uniform: the interior segment, one slice at a time
      for (; k <= kE; ++k) fast_slice(k);
      k -= U;  // (the loop increment)
      continue;
    }
    bool cov[U];
    Cell<VT> cl[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double px, py, pz;
      point(k + u, px, py, pz);
      cov[u] = in_cube(px, py, pz);
      if (cov[u]) cell_fetch<VT, UNIT>(P.volume, px, py, pz, cl[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float st = step_slice(cov[u], cl[u]);
      if (k + u > 0) emit_w(k + u - 1, prev, st);
      prev = st;
    }
  }
  for (; k <= kB; ++k) {
    double ax, ay, az;
    point(k, ax, ay, az);
    const bool ca = in_cube(ax, ay, az);
    Cell<VT> la;
    if (ca) cell_fetch<VT, UNIT>(P.volume, ax, ay, az, la);
    const float sa = step_slice(ca, la);
    if (k > 0) emit_w(k - 1, prev, sa);
    prev = sa;
  }
  }
  if (k == n) {
    emit_w(n - 1, prev, prev);
    return;
  }
  // after the warp's range: every later slice stores the final T
  const float tc = (float)T;
  emit_w(k - 1, prev, tc);
  float tr = __shfl_down_sync(0xffffffffu, tc, 1);
  if (x == L.width - 1) tr = tc;
  const float4 tail = make_float4(tc, tc, tr, tr);
  if (owner)
    for (int e = min(n - 1, w_hi); k <= e; ++k)
      if (k >= w_lo) put(k, tail);
}

// Repack a plain stack into quads (one thread per texel, loop over layers).
__global__ void __launch_bounds__(256) pack_quads_kernel(const float* __restrict__ plain, int64_t pk, int64_t py,
                                                         int n, int h, int w, float* quads, int64_t qk,
                                                         int64_t qy) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  const float* src = plain + (size_t)y * (size_t)py + (size_t)x;
  float4* row = reinterpret_cast<float4*>(quads) + (size_t)y * (size_t)qy;
  float prev = __ldg(src);
  for (int k = 1; k < n; ++k) {
    const float cur = __ldg(src + (size_t)k * (size_t)pk);
    emit_pair(row + (size_t)(k - 1) * (size_t)qk, x, w, prev, cur);
    prev = cur;
  }
  emit_pair(row + (size_t)(n - 1) * (size_t)qk, x, w, prev, prev);
}

// GPU shadow_oracle_many (raycaster.py:356-366): one thread per point.
template <int VT, bool UNIT>
__global__ void __launch_bounds__(256) shadow_oracle_kernel(const sbrc_volume V, const double* __restrict__ alpha_lut,
                                                            const double* __restrict__ pts, int64_t m, double tl0,
                                                            double tl1, double tl2, double step, double* out) {
  __shared__ double alut[SBRC_LUT_SIZE];
  __shared__ double u8tab[256];
  for (int i = threadIdx.x; i < SBRC_LUT_SIZE; i += blockDim.x) alut[i] = alpha_lut[i];
  if (std::is_same<typename Voxel<VT>::T, unsigned char>::value) fill_u8_table(u8tab);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  const double tl[3] = {tl0, tl1, tl2};
  out[i] = light_march<VT, UNIT, false>(V, alut, reinterpret_cast<const float*>(u8tab), p, tl, step);
}

// Light factor at arbitrary world points: lookup_light_scalar_many
// (lightbuffer.py:256-287), _shell_scalar (raycaster.py:239-250) and
// _cone_scalar (:266-300) with the cone basis from `eye - p` per point (or the
// plane_basis fallback when eye is absent), then _factor_from_intensity
// (:197-201). Same device lookup code as K2 (general path); out[i] =
// (scalar, factor_r, factor_g, factor_b).
template <int LOOKUP>
__global__ void __launch_bounds__(256) light_factor_kernel(const sbrc_render_params P, const double* __restrict__ pts,
                                                           int64_t m, int has_eye, double ex, double ey, double ez,
                                                           float4* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const sbrc_light_frame& LF = P.light;
  const double sx = (double)LF.width / (LF.u_range[1] - LF.u_range[0]);
  const double sy = (double)LF.height / (LF.v_range[1] - LF.v_range[0]);
  const double si = (double)LF.n_slices / (LF.d_max - LF.d_min);
  const QuadTex tex = make_quad_tex(P);
  const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  double pu = 0, pv = 0, pl = 0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    pu += p[c] * LF.axis_u[c];
    pv += p[c] * LF.axis_v[c];
    pl += p[c] * LF.light_dir[c];
  }
  const float tx = (float)((pu - LF.u_range[0]) * sx - 0.5);
  const float ty = (float)((pv - LF.v_range[0]) * sy - 0.5);
  const float li = (float)((pl - LF.d_min) * si - (LOOKUP == SBRC_LOOKUP_NEAREST ? 0.0 : 0.5));
  float scalar;
  if (P.shading == SBRC_SHADE_SHADOW) {
    scalar = light_lookup<LOOKUP>(tex, tx, ty, li);
  } else if (P.shading == SBRC_SHADE_SHELL) {
    float acc = 0.0f;
    for (int sh = 0; sh < P.shell_count; ++sh) {
      const double r = P.shell_radius[sh];
      float shell = 0.0f;
      for (int a = 0; a < 3; ++a) {
        const float du = (float)(r * LF.axis_u[a] * sx), dv = (float)(r * LF.axis_v[a] * sy);
        const float dl = (float)(r * LF.light_dir[a] * si);
        shell += light_lookup<LOOKUP>(tex, tx + du, ty + dv, li + dl);
        shell += light_lookup<LOOKUP>(tex, tx - du, ty - dv, li - dl);
      }
      acc += (float)P.shell_weight[sh] * shell / 6.0f;
    }
    scalar = acc;
  } else {  // cone
    float bu = 1.0f, bv = 0.0f;  // plane_basis(L)[0] = axis_u
    if (has_eye) {
      const double e[3] = {ex - p[0], ey - p[1], ez - p[2]};
      const double el = e[0] * LF.light_dir[0] + e[1] * LF.light_dir[1] + e[2] * LF.light_dir[2];
      double b[3], nb = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        b[c] = e[c] - el * LF.light_dir[c];
        nb += b[c] * b[c];
      }
      nb = sqrt(nb);
      if (nb > 1e-12) {
        bu = (float)((b[0] * LF.axis_u[0] + b[1] * LF.axis_u[1] + b[2] * LF.axis_u[2]) / nb);
        bv = (float)((b[0] * LF.axis_v[0] + b[1] * LF.axis_v[1] + b[2] * LF.axis_v[2]) / nb);
      }
    }
    const double spacing = (LF.d_max - LF.d_min) / LF.n_slices;
    float acc = 0.0f;
    for (int a = 1; a <= P.cone_axis_samples; ++a) {
      const double r = P.cone_ring * a * spacing;
      for (int j = 0; j < P.cone_angle_count; ++j) {
        const double c = P.cone_cos[j], sn = P.cone_sin[j];
        const float ox = (float)(r * sx * (bu * c - bv * sn)), oy = (float)(r * sy * (bv * c + bu * sn));
        acc += light_lookup<LOOKUP>(tex, tx + ox, ty + oy, li - (float)a);
      }
    }
    scalar = acc / (float)(P.cone_axis_samples * P.cone_angle_count);
  }
  float f[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float col = P.light_color[c];
    f[c] = col > 0.f ? fmaxf(scalar * col, P.ambient_floor) / col : 1.0f;
  }
  out[i] = make_float4(scalar, f[0], f[1], f[2]);
}

// load_raw's float32 min-max normalisation (volume.py:147-151) in place:
// numpy evaluates (flat - lo) / (hi - lo) in float32 (NEP 50: the Python
// scalars become float32), i.e. fl32(fl32(x - lo) / fl32(hi - lo)).
__global__ void __launch_bounds__(256) normalize_f32_kernel(float* data, long long n, float lo, float range) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    data[i] = __fdiv_rn(__fsub_rn(data[i], lo), range);
}

// K0 widening: a raw u8/u16 volume to float32 with load_raw's IEEE float32
// division (volume.py:143-146: astype(float32) / 255.0 or / 65535.0, the
// Python divisor a float32 under NEP 50) in one pass; the integers convert
// exactly. Vectorised: 4 voxels per thread per step.
template <typename T>
__global__ void __launch_bounds__(256) widen_kernel(const T* __restrict__ src, float* __restrict__ dst, long long n,
                                                   float scale) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long n4 = n / 4;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    T v[4];
    if constexpr (sizeof(T) == 1) {
      const uchar4 q = reinterpret_cast<const uchar4*>(src)[i];
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
      const ushort4 q = reinterpret_cast<const ushort4*>(src)[i];
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    }
    reinterpret_cast<float4*>(dst)[i] = make_float4(__fdiv_rn((float)v[0], scale), __fdiv_rn((float)v[1], scale),
                                                    __fdiv_rn((float)v[2], scale), __fdiv_rn((float)v[3], scale));
  }
  for (long long i = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = __fdiv_rn((float)src[i], scale);
}

// Brick repack (SBRC_BRICK builds): dst element (brick, lz, ly, lx) = src
// voxel (min(8 bx + lx, nx-1), ...) — the apron replicates the far faces.
template <typename T>
__global__ void __launch_bounds__(256) brick_pack_kernel(const T* __restrict__ src, T* __restrict__ dst, int nx,
                                                        int ny, int nz, long long total) {
  const int nbx = brick_count(nx), nby = brick_count(ny);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long brick = i / kBrickN;
    const int e = (int)(i - brick * kBrickN);
    const int lx = e % kBrickS, ly = (e / kBrickS) % kBrickS, lz = e / (kBrickS * kBrickS);
    const int bx = (int)(brick % nbx), by = (int)((brick / nbx) % nby), bz = (int)(brick / ((long long)nbx * nby));
    const int x = min(bx * kBrick + lx, nx - 1), y = min(by * kBrick + ly, ny - 1), z = min(bz * kBrick + lz, nz - 1);
    dst[i] = src[((size_t)z * ny + y) * nx + x];
  }
}

// Heavy-first order from measured tile costs (schedule.TileFeedback): tiles
// by decreasing steps, ties by increasing index — every key
// (~steps << 32 | index) is unique, so its rank among all keys is its slot
// and the order is deterministic. Rank by counting: each thread owns one key
// and compares it with all n keys, staged through shared memory 256 at a
// time (O(n^2) compares; 16K tiles take ~15 us on 148 SMs, no sort library).
__global__ void __launch_bounds__(256) rank_order_kernel(const unsigned* __restrict__ steps, int n,
                                                         int* __restrict__ order) {
  __shared__ unsigned long long tile[256];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned long long mine =
      i < n ? ((unsigned long long)(~__ldg(steps + i)) << 32) | (unsigned)i : ~0ull;
  int rank = 0;
  for (int base = 0; base < n; base += 256) {
    const int j = base + threadIdx.x;
    tile[threadIdx.x] = j < n ? ((unsigned long long)(~__ldg(steps + j)) << 32) | (unsigned)j : ~0ull;
    __syncthreads();
    const int m = min(256, n - base);
#pragma unroll 8
    for (int k = 0; k < m; ++k) rank += tile[k] < mine;
    __syncthreads();
  }
  if (i < n) order[rank] = i;
}

// Image assembly of the NCCL path: raster row y = gathered row perm[y]
// (float4 pixels, one warp-strided row copy per block row).
__global__ void __launch_bounds__(256) permute_rows_kernel(const float4* __restrict__ src,
                                                           const long long* __restrict__ perm, float4* __restrict__ dst,
                                                           int rows, int width) {
  for (int y = blockIdx.x; y < rows; y += gridDim.x) {
    const float4* s = src + (size_t)__ldg(perm + y) * width;
    float4* d = dst + (size_t)y * width;
    for (int x = threadIdx.x; x < width; x += blockDim.x) d[x] = __ldg(s + x);
  }
}

// ---------------------------------------------------------------- half-angle baseline
// halfangle.py:48-142. Float64 throughout, reference op order for the slice
// geometry; alpha correction a = 1 - (1 - alpha)^exponent via pow.
__device__ __forceinline__ double lut_alpha_raw(const double* lut, double s, double* rgb) {
  const LutPos q = lut_pos(s);
#pragma unroll
  for (int c = 0; c < 3; ++c) rgb[c] = dadd(dmul(lut[4 * q.i0 + c], q.g), dmul(lut[4 * q.i1 + c], q.f));
  return dadd(dmul(lut[4 * q.i0 + 3], q.g), dmul(lut[4 * q.i1 + 3], q.f));
}

__global__ void has_init_kernel(double* eye_accum, long long ne, double* light_accum, long long nl) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += (long long)gridDim.x * blockDim.x)
    eye_accum[i] = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += (long long)gridDim.x * blockDim.x)
    light_accum[i] = 1.0;
}

template <int VT, bool UNIT>
__global__ void __launch_bounds__(256) has_eye_kernel(const sbrc_half_angle_params P, int k) {
  __shared__ double lut[SBRC_LUT_SIZE * 4];
  __shared__ double u8tab[256];
  for (int i = threadIdx.x; i < SBRC_LUT_SIZE * 4; i += blockDim.x) lut[i] = P.lut[i];
  if (std::is_same<typename Voxel<VT>::T, unsigned char>::value) fill_u8_table(u8tab);
  __syncthreads();
  const int px = blockIdx.x * 32 + (threadIdx.x & 31);
  const int py = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (px >= P.width || py >= P.height) return;
  // Camera.rays (raycaster.py:53-68)
  const double ndc_x = dmul(dmul(dsub(dmul(ddiv(dadd((double)px, 0.5), (double)P.width), 2.0), 1.0), P.tan_half),
                            P.aspect);
  const double ndc_y = dmul(dsub(1.0, dmul(ddiv(dadd((double)py, 0.5), (double)P.height), 2.0)), P.tan_half);
  double d[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) d[c] = dadd(dadd(P.forward[c], dmul(ndc_x, P.right[c])), dmul(ndc_y, P.up2[c]));
  const double nrm = __dsqrt_rn(dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2])));
#pragma unroll
  for (int c = 0; c < 3; ++c) d[c] = ddiv(d[c], nrm);
  const double hdd = dadd(dadd(dmul(d[0], P.half[0]), dmul(d[1], P.half[1])), dmul(d[2], P.half[2]));
  if (hdd == 0.0) return;
  const double t = ddiv(dsub(P.plane_offsets[k], P.h_dot_e), hdd);  // :107
  if (!(t > 0.0)) return;
  const double q[3] = {dadd(P.eye[0], dmul(t, d[0])), dadd(P.eye[1], dmul(t, d[1])), dadd(P.eye[2], dmul(t, d[2]))};
  if (!in_cube(q[0], q[1], q[2])) return;  // :109
  const double s = trilinear64<VT, UNIT>(P.volume, reinterpret_cast<const float*>(u8tab), q[0], q[1], q[2]);
  double rgb[3];
  const double alpha_raw = lut_alpha_raw(lut, s, rgb);
  const double expo = ddiv(P.delta, dmul(1.0 / 256.0, fabs(hdd)));  // :115
  const double a = dsub(1.0, pow(dsub(1.0, alpha_raw), expo));
  // light transmittance at the sample: _bilinear_scalar of light_accum at uv (:117-118)
  const double u = ((q[0] * P.axis_u[0] + q[1] * P.axis_u[1] + q[2] * P.axis_u[2]) - P.u_range[0]) /
                   (P.u_range[1] - P.u_range[0]);
  const double v = ((q[0] * P.axis_v[0] + q[1] * P.axis_v[1] + q[2] * P.axis_v[2]) - P.v_range[0]) /
                   (P.v_range[1] - P.v_range[0]);
  const int W = P.light_width, H = P.light_height;
  const double tx = u * W - 0.5, ty = v * H - 0.5;
  const double fx0 = floor(tx), fy0 = floor(ty);
  const double fx = tx - fx0, fy = ty - fy0;
  const int x0 = (int)fx0, y0 = (int)fy0;
  const int xa = min(max(x0, 0), W - 1), xb = min(max(x0 + 1, 0), W - 1);
  const int ya = min(max(y0, 0), H - 1), yb = min(max(y0 + 1, 0), H - 1);
  const double* L = P.light_accum;
  const double c0 = L[(size_t)ya * W + xa] * (1 - fx) + L[(size_t)ya * W + xb] * fx;
  const double c1 = L[(size_t)yb * W + xa] * (1 - fx) + L[(size_t)yb * W + xb] * fx;
  const double shade = c0 * (1 - fy) + c1 * fy;
  double* acc = P.eye_accum + 4 * ((size_t)py * P.width + px);
  const double as = dmul(a, shade);
  if (P.front_to_back) {  // :120-123
    const double one_m = dsub(1.0, acc[3]);
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] = dadd(acc[c], dmul(one_m, dmul(rgb[c], as)));
    acc[3] = dadd(acc[3], dmul(one_m, a));
  } else {  // :124-126
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] = dadd(dmul(dsub(1.0, a), acc[c]), dmul(rgb[c], as));
    acc[3] = dadd(a, dmul(dsub(1.0, a), acc[3]));
  }
}

template <int VT, bool UNIT>
__global__ void __launch_bounds__(256) has_light_kernel(const sbrc_half_angle_params P, int k) {
  __shared__ double alut[SBRC_LUT_SIZE];
  __shared__ double u8tab[256];
  for (int i = threadIdx.x; i < SBRC_LUT_SIZE; i += blockDim.x) alut[i] = P.lut[4 * i + 3];
  if (std::is_same<typename Voxel<VT>::T, unsigned char>::value) fill_u8_table(u8tab);
  __syncthreads();
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= P.light_width || y >= P.light_height) return;
  const double ug = dadd(P.u_range[0], dmul(ddiv(dadd((double)x, 0.5), (double)P.light_width),
                                            dsub(P.u_range[1], P.u_range[0])));
  const double vg = dadd(P.v_range[0], dmul(ddiv(dadd((double)y, 0.5), (double)P.light_height),
                                            dsub(P.v_range[1], P.v_range[0])));
  const double tl = ddiv(dsub(dsub(P.plane_offsets[k], dmul(ug, P.h_dot_u)), dmul(vg, P.h_dot_v)), P.hl);  // :130
  double q[3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
    q[c] = dadd(dadd(dmul(ug, P.axis_u[c]), dmul(vg, P.axis_v[c])), dmul(tl, P.light_dir[c]));  // :131
  if (!in_cube(q[0], q[1], q[2])) return;
  const double s = trilinear64<VT, UNIT>(P.volume, reinterpret_cast<const float*>(u8tab), q[0], q[1], q[2]);
  const LutPos lp = lut_pos(s);
  const double alpha_raw = dadd(dmul(alut[lp.i0], lp.g), dmul(alut[lp.i1], lp.f));
  const double a = dsub(1.0, pow(dsub(1.0, alpha_raw), ddiv(P.delta, dmul(1.0 / 256.0, P.hl))));  // :136
  double* T = P.light_accum + (size_t)y * P.light_width + x;
  *T = dmul(*T, dsub(1.0, a));
}

__global__ void has_finish_kernel(const double* eye_accum, float* image, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    image[i] = (float)eye_accum[i];
}

template <int VT, bool UNIT>
void has_passes(const sbrc_half_angle_params& p, int k0, int k1, cudaStream_t s) {
  const dim3 ge((p.width + 31) / 32, (p.height + 7) / 8), gl((p.light_width + 31) / 32, (p.light_height + 7) / 8);
  for (int k = k0; k < k1; ++k) {
    has_eye_kernel<VT, UNIT><<<ge, 256, 0, s>>>(p, k);
    has_light_kernel<VT, UNIT><<<gl, 256, 0, s>>>(p, k);
  }
}

// cuTensorMapEncodeTiled from the driver through the runtime (resolved once;
// the library links only cudart).
static PFN_cuTensorMapEncodeTiled tensor_map_encoder() {
  static const PFN_cuTensorMapEncodeTiled fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (PFN_cuTensorMapEncodeTiled) nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(f);
  }();
  return fn;
}

// TMA plan of a build: the box (voxels) covering one block's texel-slice
// points over C slices plus the cell corners and a rounding margin, the
// largest C whose two boxes fit SBRC_BUILD_TMA_SMEM. False when the volume
// or geometry does not suit TMA (row pitch not a multiple of 16 bytes, box
// dims > 256, unaligned base): the register path is used.
static bool tma_plan(const sbrc_build_params& p, int4* box, size_t* smem) {
  const sbrc_volume& v = p.volume;
  const sbrc_light_frame& L = p.light;
  if ((v.nx % 4) != 0 || (reinterpret_cast<uintptr_t>(v.data) % 16) != 0) return false;
  const double du = (L.u_range[1] - L.u_range[0]) / L.width, dv = (L.v_range[1] - L.v_range[0]) / L.height;
  const double dk = (L.d_max - L.d_min) / L.n_slices;
  const int dims[3] = {v.nx, v.ny, v.nz};
  for (int C = 8; C >= 1; --C) {
    int b[3];
    bool ok = true;
    for (int c = 0; c < 3; ++c) {
      const double ext = (fabs(L.axis_u[c]) * 31.0 * du + fabs(L.axis_v[c]) * (SBRC_BUILD_ROWS - 1) * dv +
                          fabs(L.light_dir[c]) * (C - 1) * dk) * dims[c];
      b[c] = (int)ceil(ext) + 4;
      if (b[c] > 256) ok = false;
    }
    b[0] = (b[0] + 3 + 3) & ~3;  // 16-byte rows; +3: the origin x is rounded down to a multiple of 4
    if (!ok || b[0] > 256) continue;
    const size_t box_n = (size_t)b[0] * b[1] * b[2];
    const size_t bytes = 2 * (((box_n + 31) & ~(size_t)31) * 4) + 128;
    if (bytes > SBRC_BUILD_TMA_SMEM) continue;
    *box = make_int4(b[0], b[1], b[2], C);
    *smem = bytes;
    return true;
  }
  return false;
}

template <int VT>
void launch_build(const sbrc_build_params& p, cudaStream_t s) {
  dim3 block(32, SBRC_BUILD_ROWS);  // warps are rows of 31 owned texels (build_kernel)
  dim3 grid((p.light.width + 30) / 31, (p.row_end - p.row_begin + SBRC_BUILD_ROWS - 1) / SBRC_BUILD_ROWS);
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  const int4 none = make_int4(0, 0, 0, 0);
  if constexpr (VT == SBRC_VOXEL_F32) {
    int4 box;
    size_t smem;
    PFN_cuTensorMapEncodeTiled enc = SBRC_BUILD_TMA && !SBRC_BRICK ? tensor_map_encoder() : nullptr;
    if (enc != nullptr && unit_box(p.volume) && tma_plan(p, &box, &smem)) {
      const cuuint64_t gdim[3] = {(cuuint64_t)p.volume.nx, (cuuint64_t)p.volume.ny, (cuuint64_t)p.volume.nz};
      const cuuint64_t gstride[2] = {(cuuint64_t)p.volume.nx * 4, (cuuint64_t)p.volume.nx * p.volume.ny * 4};
      const cuuint32_t bdim[3] = {(cuuint32_t)box.x, (cuuint32_t)box.y, (cuuint32_t)box.z};
      const cuuint32_t estride[3] = {1, 1, 1};
      if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(p.volume.data), gdim, gstride, bdim,
              estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
        auto kern = build_kernel<VT, true, -1>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, block, smem, s>>>(p, tmap, box);
        return;
      }
    }
  }
  constexpr int D = VT == SBRC_VOXEL_F32 && !SBRC_BRICK ? SBRC_BUILD_ASYNC : 0;
  if (unit_box(p.volume)) build_kernel<VT, true, D><<<grid, block, 0, s>>>(p, tmap, none);
  else build_kernel<VT, false, D><<<grid, block, 0, s>>>(p, tmap, none);
}

}  // namespace

extern "C" {

int sbrc_abi_version(void) { return SBRC_ABI_VERSION; }

int sbrc_debug_violations(unsigned int counts[8], int reset) {
  if (counts == nullptr) return SBRC_EINVAL;
  for (int i = 0; i < 8; ++i) counts[i] = 0;
  int st = tu_violations(counts, reset);
  if (st != SBRC_OK) return st;
  using viol_fn = int (*)(unsigned int*, int);
#define SBRC_VIOL_ROW(SH) SBRC_MARCH_VIOL(SH, 0), SBRC_MARCH_VIOL(SH, 1), SBRC_MARCH_VIOL(SH, 2)
  static const viol_fn kViol[] = {SBRC_VIOL_ROW(0), SBRC_VIOL_ROW(1), SBRC_VIOL_ROW(2),
                                  SBRC_VIOL_ROW(3), SBRC_VIOL_ROW(4), SBRC_VIOL_ROW(5)};
#undef SBRC_VIOL_ROW
  for (viol_fn f : kViol)
    if ((st = f(counts, reset)) != SBRC_OK) return st;
  return SBRC_OK;
}

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
    case 4: return (int64_t)sizeof(sbrc_half_angle_params);
    default: return -1;
  }
}

int sbrc_volume_check(const sbrc_volume* v) { return (v && volume_ok(*v)) ? SBRC_OK : SBRC_EINVAL; }

int sbrc_ipc_alloc(int64_t bytes, void** ptr) {
  if (ptr == nullptr || bytes <= 0) return SBRC_EINVAL;
  return cudaMalloc(ptr, (size_t)bytes) == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_host_device_pointer(const void* host, void** dev) {
  if (host == nullptr || dev == nullptr) return SBRC_EINVAL;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    cudaGetLastError();
    return SBRC_EINVAL;
  }
  if (a.type != cudaMemoryTypeHost || a.devicePointer == nullptr) return SBRC_EINVAL;
  *dev = a.devicePointer;
  return SBRC_OK;
}

int sbrc_ipc_free(void* ptr) { return cudaFree(ptr) == cudaSuccess ? SBRC_OK : SBRC_ECUDA; }

int sbrc_ipc_handle(void* ptr, unsigned char handle[64]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (ptr == nullptr || handle == nullptr) return SBRC_EINVAL;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, ptr) != cudaSuccess) return SBRC_ECUDA;
  memcpy(handle, &h, sizeof(h));
  return SBRC_OK;
}

int sbrc_ipc_open(const unsigned char handle[64], void** ptr) {
  if (ptr == nullptr || handle == nullptr) return SBRC_EINVAL;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_ipc_close(void* ptr) { return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? SBRC_OK : SBRC_ECUDA; }

int sbrc_march_grid(int width, int height, int band_rows, int rank, int world, int* grid) {
  if (grid == nullptr) return SBRC_EINVAL;
  const int rows = sbrc_local_rows(height, band_rows, rank, world);
  const int BW = (march_wide(width, rows) ? 4 : 2) * SBRC_TILE_W, BH = 2 * (32 / SBRC_TILE_W);
  grid[0] = (width + BW - 1) / BW;
  grid[1] = (rows + BH - 1) / BH;
  grid[2] = BW;
  grid[3] = BH;
  return SBRC_OK;
}

// Row partition of a render call: a contiguous range inside the image, or
// bands of a multiple of 8 rows dealt to rank < world.
static bool rows_ok(const sbrc_render_params* p) {
  if (p->row_count > 0) return p->row_begin >= 0 && p->row_begin + p->row_count <= p->height;
  return p->row_count == 0 && p->band_rows >= 1 && p->band_rows % 8 == 0 && p->world >= 1 && p->rank >= 0 &&
         p->rank < p->world;
}

int sbrc_render_grid(const sbrc_render_params* p, int* grid) {
  if (p == nullptr || grid == nullptr || p->width < 1 || p->height < 1 || !rows_ok(p)) return SBRC_EINVAL;
  const MarchShape m = march_shape(*p, rank_rows(*p));
  grid[0] = m.tiles_x;
  grid[1] = m.tiles_y;
  grid[2] = m.bw;
  grid[3] = m.bh;
  return SBRC_OK;
}

int sbrc_local_rows(int height, int band_rows, int rank, int world) {
  if (height < 1 || band_rows < 1 || world < 1 || rank < 0 || rank >= world) return 0;
  const int bands = (height + band_rows - 1) / band_rows;
  const int mine = bands > rank ? (bands - rank + world - 1) / world : 0;
  return mine * band_rows;
}

int sbrc_build(const sbrc_build_params* p, void* stream) {
  if (p == nullptr || !volume_ok(p->volume) || !light_ok(p->light)) return SBRC_EINVAL;
  if (p->light.plane_offsets == nullptr || p->alpha_lut == nullptr || p->quads == nullptr) return SBRC_EINVAL;
  if (p->row_begin < 0 || p->row_end > p->light.height || p->row_begin >= p->row_end) return SBRC_EINVAL;
  if (p->n_clip < 0 || p->n_clip > SBRC_MAX_CLIP || (p->n_clip > 0 && !p->write_sparse)) return SBRC_EINVAL;
  if (p->quad_layout < 0 || p->quad_layout > 1 || (p->quad_layout == 1 && p->output_plain)) return SBRC_EINVAL;
  if (p->quad_layer_stride < 1 || p->quad_row_stride < p->light.width) return SBRC_EINVAL;
  if (p->compensation_n < 0.0) return SBRC_EINVAL;
  if (p->write_sparse && (!(p->write_reach >= 0.0) || p->write_below < 0 || p->write_above < 0)) return SBRC_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  switch (p->volume.voxel_type) {
    case SBRC_VOXEL_F32: launch_build<SBRC_VOXEL_F32>(*p, s); break;
    case SBRC_VOXEL_U8: launch_build<SBRC_VOXEL_U8>(*p, s); break;
    default: launch_build<SBRC_VOXEL_U16>(*p, s); break;
  }
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_pack_quads(const float* plain, int64_t plain_layer_stride, int64_t plain_row_stride, int n, int height,
                    int width, float* quads, int64_t quad_layer_stride, int64_t quad_row_stride, void* stream) {
  if (plain == nullptr || quads == nullptr || n < 1 || height < 1 || width < 1) return SBRC_EINVAL;
  if (plain_layer_stride < 1 || plain_row_stride < width || quad_layer_stride < 1 || quad_row_stride < width)
    return SBRC_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  dim3 block(32, 8);
  dim3 grid((width + 31) / 32, (height + 7) / 8);
  pack_quads_kernel<<<grid, block, 0, s>>>(plain, plain_layer_stride, plain_row_stride, n, height, width, quads,
                                           quad_layer_stride, quad_row_stride);
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_normalize_f32(float* data, int64_t n, float lo, float range, void* stream) {
  if (data == nullptr || n < 0 || !(range > 0.0f)) return SBRC_EINVAL;
  if (n == 0) return SBRC_OK;
  normalize_f32_kernel<<<148 * 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(data, n, lo, range);
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_widen_volume(const void* src, int voxel_type, int64_t n, float* dst, void* stream) {
  if (src == nullptr || dst == nullptr || n < 0) return SBRC_EINVAL;
  if (voxel_type != SBRC_VOXEL_U8 && voxel_type != SBRC_VOXEL_U16) return SBRC_EINVAL;
  if (n == 0) return SBRC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (voxel_type == SBRC_VOXEL_U8)
    widen_kernel<unsigned char><<<148 * 8, 256, 0, s>>>(static_cast<const unsigned char*>(src), dst, n, 255.0f);
  else
    widen_kernel<unsigned short><<<148 * 8, 256, 0, s>>>(static_cast<const unsigned short*>(src), dst, n, 65535.0f);
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_volume_layout(void) { return SBRC_BRICK; }

int64_t sbrc_brick_elems(int nx, int ny, int nz) {
  if (nx < 2 || ny < 2 || nz < 2) return -1;
  return (int64_t)brick_count(nx) * brick_count(ny) * brick_count(nz) * kBrickN;
}

int sbrc_brick_pack(const void* src, int voxel_type, int nx, int ny, int nz, void* dst, void* stream) {
  const int64_t total = sbrc_brick_elems(nx, ny, nz);
  if (src == nullptr || dst == nullptr || total < 0) return SBRC_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int grid = 148 * 8;
  switch (voxel_type) {
    case SBRC_VOXEL_F32:
      brick_pack_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(src), static_cast<float*>(dst), nx, ny,
                                                     nz, total);
      break;
    case SBRC_VOXEL_U8:
      brick_pack_kernel<unsigned char><<<grid, 256, 0, s>>>(static_cast<const unsigned char*>(src),
                                                             static_cast<unsigned char*>(dst), nx, ny, nz, total);
      break;
    case SBRC_VOXEL_U16:
      brick_pack_kernel<unsigned short><<<grid, 256, 0, s>>>(static_cast<const unsigned short*>(src),
                                                              static_cast<unsigned short*>(dst), nx, ny, nz, total);
      break;
    default: return SBRC_EINVAL;
  }
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_tile_order(const unsigned int* steps, int n, int* order, void* stream) {
  if (steps == nullptr || order == nullptr || n < 0) return SBRC_EINVAL;
  if (n == 0) return SBRC_OK;
  rank_order_kernel<<<(n + 255) / 256, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(steps, n, order);
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_permute_rows(const float* src, const int64_t* perm, float* dst, int rows, int width, void* stream) {
  if (src == nullptr || perm == nullptr || dst == nullptr || rows < 0 || width < 1) return SBRC_EINVAL;
  if (rows == 0) return SBRC_OK;
  permute_rows_kernel<<<min(rows, 148 * 8), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4*>(src), reinterpret_cast<const long long*>(perm), reinterpret_cast<float4*>(dst),
      rows, width);
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_light_factor(const sbrc_render_params* p, const double* pts, int64_t m, const double* eye, float* out,
                      void* stream) {
  if (p == nullptr || out == nullptr || m < 0 || (m > 0 && pts == nullptr)) return SBRC_EINVAL;
  if (p->shading < SBRC_SHADE_SHADOW || p->shading > SBRC_SHADE_CONE) return SBRC_EINVAL;
  if (p->lookup != SBRC_LOOKUP_LINEAR && p->lookup != SBRC_LOOKUP_NEAREST) return SBRC_EINVAL;
  if (p->quads == nullptr) return SBRC_ECONFIG;
  if (!light_ok(p->light) || !quads_ok(p->light, p->quad_layer_stride, p->quad_row_stride)) return SBRC_EINVAL;
  if (p->quad_layout != 0) return SBRC_EINVAL;  // the point API reads texel quads
  if (p->shading == SBRC_SHADE_SHELL && (p->shell_count < 1 || p->shell_count > SBRC_MAX_SHELLS)) return SBRC_EINVAL;
  if (p->shading == SBRC_SHADE_CONE && (p->cone_axis_samples < 1 || p->cone_angle_count < 1 ||
                                        p->cone_angle_count > SBRC_MAX_ANGLES))
    return SBRC_EINVAL;
  if (m == 0) return SBRC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const unsigned blocks = (unsigned)((m + 255) / 256);
  const int he = eye != nullptr;
  const double ex = he ? eye[0] : 0.0, ey = he ? eye[1] : 0.0, ez = he ? eye[2] : 0.0;
  if (p->lookup == SBRC_LOOKUP_NEAREST)
    light_factor_kernel<SBRC_LOOKUP_NEAREST><<<blocks, 256, 0, s>>>(*p, pts, m, he, ex, ey, ez, reinterpret_cast<float4*>(out));
  else
    light_factor_kernel<SBRC_LOOKUP_LINEAR><<<blocks, 256, 0, s>>>(*p, pts, m, he, ex, ey, ez, reinterpret_cast<float4*>(out));
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_half_angle(const sbrc_half_angle_params* p, int first_slice, int last_slice, int init, int finish,
                    int* pass_count, void* stream) {
  if (p == nullptr || !volume_ok(p->volume) || p->lut == nullptr || p->plane_offsets == nullptr) return SBRC_EINVAL;
  if (p->width < 1 || p->height < 1 || p->light_width < 1 || p->light_height < 1 || p->n_slices < 1)
    return SBRC_EINVAL;
  if (p->eye_accum == nullptr || p->light_accum == nullptr || p->image == nullptr || !(p->hl > 0.0))
    return SBRC_EINVAL;
  if (first_slice < 0 || last_slice > p->n_slices || first_slice > last_slice) return SBRC_EINVAL;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const long long ne = 4ll * p->width * p->height, nl = (long long)p->light_width * p->light_height;
  if (init) has_init_kernel<<<148 * 4, 256, 0, s>>>(p->eye_accum, ne, p->light_accum, nl);
  const bool unit = unit_box(p->volume);
  switch (p->volume.voxel_type) {
#define SBRC_HAS(VT) (unit ? has_passes<VT, true>(*p, first_slice, last_slice, s) \
                           : has_passes<VT, false>(*p, first_slice, last_slice, s))
    case SBRC_VOXEL_F32: SBRC_HAS(SBRC_VOXEL_F32); break;
    case SBRC_VOXEL_U8: SBRC_HAS(SBRC_VOXEL_U8); break;
    default: SBRC_HAS(SBRC_VOXEL_U16); break;
#undef SBRC_HAS
  }
  if (finish) has_finish_kernel<<<148 * 4, 256, 0, s>>>(p->eye_accum, p->image, ne);
  if (pass_count) *pass_count = 2 * (last_slice - first_slice);
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_shadow_oracle(const sbrc_volume* v, const double* alpha_lut, const double* pts, int64_t m,
                       const double* to_light, double step, double* out, void* stream) {
  if (v == nullptr || !volume_ok(*v) || alpha_lut == nullptr || to_light == nullptr || out == nullptr)
    return SBRC_EINVAL;
  if (!(step > 0.0) || m < 0 || (m > 0 && pts == nullptr)) return SBRC_EINVAL;  // raycaster.py:361-362
  if (m == 0) return SBRC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const unsigned blocks = (unsigned)((m + 255) / 256);
  const bool unit = unit_box(*v);
#define SBRC_ORACLE(VT)                                                                                        \
  (unit ? shadow_oracle_kernel<VT, true><<<blocks, 256, 0, s>>>(*v, alpha_lut, pts, m, to_light[0], to_light[1], \
                                                                to_light[2], step, out)                        \
        : shadow_oracle_kernel<VT, false><<<blocks, 256, 0, s>>>(*v, alpha_lut, pts, m, to_light[0], to_light[1], \
                                                                 to_light[2], step, out))
  switch (v->voxel_type) {
    case SBRC_VOXEL_F32: SBRC_ORACLE(SBRC_VOXEL_F32); break;
    case SBRC_VOXEL_U8: SBRC_ORACLE(SBRC_VOXEL_U8); break;
    default: SBRC_ORACLE(SBRC_VOXEL_U16); break;
  }
#undef SBRC_ORACLE
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

int sbrc_render(const sbrc_render_params* p, void* stream) {
  if (p == nullptr || !volume_ok(p->volume)) return SBRC_EINVAL;
  if (p->width < 1 || p->height < 1 || !(p->step > 0.0)) return SBRC_EINVAL;           // raycaster.py:143-146
  if (!(p->et_alpha > 0.0 && p->et_alpha <= 1.0)) return SBRC_EINVAL;                  // :147-148
  if (p->lut_rgba == nullptr || p->n_peers < 0 || p->n_peers > SBRC_MAX_PEERS) return SBRC_EINVAL;
  if (p->image == nullptr && p->n_peers == 0) return SBRC_EINVAL;
  for (int i = 0; i < p->n_peers; ++i)
    if (p->peer_images[i] == nullptr) return SBRC_EINVAL;
  if (p->shading < SBRC_SHADE_NONE || p->shading > SBRC_SHADE_EXTINCTION) return SBRC_EUNSUPPORTED;
  if (p->lookup != SBRC_LOOKUP_LINEAR && p->lookup != SBRC_LOOKUP_NEAREST) return SBRC_EINVAL;
  if (!rows_ok(p)) return SBRC_EINVAL;
  if (p->march_kernel < 0 || p->march_kernel > 2) return SBRC_EINVAL;
  if (p->quad_layout < 0 || p->quad_layout > 1 ||
      (p->quad_layout == 1 && (p->shading != SBRC_SHADE_SHADOW || p->light.width < 2)))
    return SBRC_EINVAL;
  if (p->shading >= SBRC_SHADE_SHADOW && p->shading <= SBRC_SHADE_CONE) {
    if (p->quads == nullptr) return SBRC_ECONFIG;
    if (!light_ok(p->light)) return SBRC_EINVAL;
    if (!quads_ok(p->light, p->quad_layer_stride, p->quad_row_stride)) return SBRC_EINVAL;
  }
  if (p->shading == SBRC_SHADE_SHELL && (p->shell_count < 1 || p->shell_count > SBRC_MAX_SHELLS))
    return SBRC_EINVAL;
  if (p->shading == SBRC_SHADE_CONE &&
      (p->cone_axis_samples < 1 || p->cone_angle_count < 1 || p->cone_angle_count > SBRC_MAX_ANGLES ||
       p->cone_ring < 0.0))
    return SBRC_EINVAL;
  if (rank_rows(*p) == 0) return SBRC_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  using march_fn = void (*)(const sbrc_render_params&, cudaStream_t);
#define SBRC_MARCH_ROW(SH) {SBRC_MARCH_FN(SH, 0), SBRC_MARCH_FN(SH, 1), SBRC_MARCH_FN(SH, 2)}
  static const march_fn kMarch[6][3] = {SBRC_MARCH_ROW(0), SBRC_MARCH_ROW(1), SBRC_MARCH_ROW(2),
                                        SBRC_MARCH_ROW(3), SBRC_MARCH_ROW(4), SBRC_MARCH_ROW(5)};
#undef SBRC_MARCH_ROW
  kMarch[p->shading][p->volume.voxel_type](*p, s);
  return cudaGetLastError() == cudaSuccess ? SBRC_OK : SBRC_ECUDA;
}

}  // extern "C"
