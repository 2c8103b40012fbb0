// Microbenchmark: cone-tap loads from the attenuation stack three ways on B200.
//   0: texel quads (float4 layer pairs, 4x the plain stack) - two LDG.128 per tap (K2 today)
//   1: plain stack in a 2D layered CUDA array - two TLD4 (gather) per tap, HW addressing
//   2: plain stack in linear memory - eight LDG.32 per tap
// Rays mimic K2 at config 3: warps of 8x4 lanes 0.25 texel apart, stepping
// (0.45, 0.3, 0.29) texels/layers per sample, 8 taps (2 rings x 4) per sample.
// Prints ms per launch and a checksum (modes must agree).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ float val(int k, int y, int x) {
  unsigned h = (unsigned)(k * 73856093) ^ (unsigned)(y * 19349663) ^ (unsigned)(x * 83492791);
  h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
  return (h & 0xFFFF) * (1.0f / 65536.0f);
}
__global__ void fill_plain(float* p, int n, int H, int W) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, tot = (size_t)n * H * W;
  for (; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    int x = i % W, y = (i / W) % H, k = i / ((size_t)W * H);
    p[i] = val(k, y, x);
  }
}
__global__ void fill_quads(float4* q, int n, int H, int W) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, tot = (size_t)n * H * W;
  for (; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    int x = i % W, y = (i / W) % H, k = i / ((size_t)W * H);
    int k1 = min(k + 1, n - 1), x1 = min(x + 1, W - 1);
    q[i] = make_float4(val(k, y, x), val(k1, y, x), val(k, y, x1), val(k1, y, x1));
  }
}
__global__ void fill_surface(cudaSurfaceObject_t s, int n, int H, int W) {
  int x = blockIdx.x * 32 + threadIdx.x, y = blockIdx.y * 8 + threadIdx.y;
  if (x >= W || y >= H) return;
  for (int k = 0; k < n; ++k) surf2DLayeredwrite(val(k, y, x), s, x * 4, y, k);
}

__device__ __forceinline__ float lerpf(float a, float b, float t) { return fmaf(t, b, fmaf(-t, a, a)); }
struct FloorF { float f; int i; };
__device__ __forceinline__ FloorF floor_f(float x) {
  const float m = __fadd_rd(x, 12582912.0f);
  return FloorF{__fsub_rn(m, 12582912.0f), __float_as_int(m) - 0x4B400000};
}
__device__ __forceinline__ float4 tld4_a2d(cudaTextureObject_t t, int layer, float x, float y) {
  float4 r;
  asm volatile("tld4.r.a2d.v4.f32.f32 {%0, %1, %2, %3}, [%4, {%5, %6, %7, %8}];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(t), "r"(layer), "f"(x), "f"(y), "f"(x));
  return r;
}

struct Args {
  const float4* quads; const float* plain; cudaTextureObject_t tex;
  int n, H, W; int samples; float* out;
};

template <int MODE>
__global__ void __launch_bounds__(128, 4) taps(const Args a) {
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * 4) + (threadIdx.x >> 5);
  unsigned h = warp * 2654435761u; h ^= h >> 16; h *= 0x45d9f3bu; h ^= h >> 16;
  float tx = 8.f + (h % (a.W - 300)) + 0.25f * (lane & 7);
  float ty = 8.f + ((h >> 10) % (a.H - 200)) + 0.25f * (lane >> 3);
  float li = 4.f + ((h >> 20) % (a.n / 4));
  const float dx = 0.45f, dy = 0.3f, dl = 0.29f;
  const float wx[4] = {1.1f, 0.f, -1.1f, 0.f}, wy[4] = {0.f, 1.1f, 0.f, -1.1f};
  const unsigned qk = a.W * a.H, qy = a.W;
  float acc = 0.f;
  for (int s = 0; s < a.samples; ++s) {
#pragma unroll
    for (int i = 1; i <= 2; ++i) {
      const float r = (float)i;
      const float lt = li - (float)i;
      const FloorF kl = floor_f(lt);
      float v0 = 0.f, v1 = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float x = fmaf(r, wx[j], tx), y = fmaf(r, wy[j], ty);
        const FloorF xl = floor_f(x), yl = floor_f(y);
        const float fx = x - xl.f, fy = y - yl.f;
        if (MODE == 0) {
          const float4* p = a.quads + ((unsigned)kl.i * qk + (unsigned)yl.i * qy + (unsigned)xl.i);
          const float4 r0 = __ldg(p), r1 = __ldg(p + qy);
          v0 += lerpf(lerpf(r0.x, r0.z, fx), lerpf(r1.x, r1.z, fx), fy);
          v1 += lerpf(lerpf(r0.y, r0.w, fx), lerpf(r1.y, r1.w, fx), fy);
        } else if (MODE == 1) {
          // corner between texels (xl, yl) and (xl+1, yl+1): unnormalised coordinate xl + 1
          const float cx = xl.f + 1.0f, cy = yl.f + 1.0f;
          const float4 g0 = tld4_a2d(a.tex, kl.i, cx, cy), g1 = tld4_a2d(a.tex, kl.i + 1, cx, cy);
          // gather order: x = (x0, y1), y = (x1, y1), z = (x1, y0), w = (x0, y0)
          v0 += lerpf(lerpf(g0.w, g0.z, fx), lerpf(g0.x, g0.y, fx), fy);
          v1 += lerpf(lerpf(g1.w, g1.z, fx), lerpf(g1.x, g1.y, fx), fy);
        } else {
          const float* p = a.plain + ((unsigned)kl.i * qk + (unsigned)yl.i * qy + (unsigned)xl.i);
          const float* q = p + qk;
          v0 += lerpf(lerpf(__ldg(p), __ldg(p + 1), fx), lerpf(__ldg(p + qy), __ldg(p + qy + 1), fx), fy);
          v1 += lerpf(lerpf(__ldg(q), __ldg(q + 1), fx), lerpf(__ldg(q + qy), __ldg(q + qy + 1), fx), fy);
        }
      }
      acc += lerpf(v0, v1, lt - kl.f);
    }
    tx += dx; ty += dy; li += dl;
    if (li > a.n - 4) li -= a.n / 2;
    if (tx > a.W - 8) tx -= a.W / 2;
    if (ty > a.H - 8) ty -= a.H / 2;
  }
  a.out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 256, H = argc > 2 ? atoi(argv[2]) : 512, W = H;
  int samples = 128, blocks = 148 * 64;
  size_t cnt = (size_t)n * H * W;
  float *plain, *out; float4* quads;
  CK(cudaMalloc(&plain, cnt * 4)); CK(cudaMalloc(&quads, cnt * 16)); CK(cudaMalloc(&out, blocks * 128 * 4));
  fill_plain<<<148 * 8, 256>>>(plain, n, H, W);
  fill_quads<<<148 * 8, 256>>>(quads, n, H, W);
  cudaChannelFormatDesc fd = cudaCreateChannelDesc<float>();
  cudaArray_t arr;
  CK(cudaMalloc3DArray(&arr, &fd, make_cudaExtent(W, H, n), cudaArrayLayered | cudaArraySurfaceLoadStore));
  cudaResourceDesc rd = {}; rd.resType = cudaResourceTypeArray; rd.res.array.array = arr;
  cudaSurfaceObject_t surf; CK(cudaCreateSurfaceObject(&surf, &rd));
  cudaTextureDesc td = {}; td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModePoint; td.readMode = cudaReadModeElementType; td.normalizedCoords = 0;
  cudaTextureObject_t tex; CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // surface fill timing (the K1 store path into the layered array) vs linear fill
  dim3 sb(32, 8), sg((W + 31) / 32, (H + 7) / 8);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); fill_surface<<<sg, sb>>>(surf, n, H, W); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  }
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("surface fill (%d x %d x %d floats): %.3f ms = %.1f GB/s\n", n, H, W, ms, cnt * 4 / ms / 1e6);
  Args a{quads, plain, tex, n, H, W, samples, out};
  double sums[3];
  for (int mode = 0; mode < 3; ++mode) {
    auto launch = [&]() {
      if (mode == 0) taps<0><<<blocks, 128>>>(a);
      else if (mode == 1) taps<1><<<blocks, 128>>>(a);
      else taps<2><<<blocks, 128>>>(a);
    };
    for (int w = 0; w < 3; ++w) launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    float* h = (float*)malloc(blocks * 128 * 4);
    CK(cudaMemcpy(h, out, blocks * 128 * 4, cudaMemcpyDeviceToHost));
    double sum = 0; for (int i = 0; i < blocks * 128; ++i) sum += h[i];
    sums[mode] = sum; free(h);
    double taps_total = (double)blocks * 128 * samples * 8;
    printf("mode %d (%s): %.3f ms/launch  %.2f Gtaps/s  checksum %.6f\n", mode,
           mode == 0 ? "quads LDG.128" : mode == 1 ? "layered TLD4" : "plain LDG.32", ms / 10,
           taps_total / (ms / 10 * 1e-3) / 1e9, sum);
  }
  printf("checksum rel diff tld4 vs quads %.3e, plain vs quads %.3e\n", (sums[1] - sums[0]) / sums[0],
         (sums[2] - sums[0]) / sums[0]);
  return 0;
}
