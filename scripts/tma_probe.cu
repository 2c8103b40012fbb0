// TMA probe: 3D tiled box load (cp.async.bulk.tensor.3d + mbarrier) of a
// float volume into shared memory, copied back out and checked on the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/tma_probe scripts/tma_probe.cu && /tmp/tma_probe
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap tmap, int ox, int oy, int oz, int n, float* out) {
  extern __shared__ unsigned char sm[];
  __shared__ __align__(8) unsigned long long mbar;
  float* buf = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sm) + 127) & ~(uintptr_t)127);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&mbar)), "r"(1) : "memory");
    if (MODE == 1) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    else asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&mbar)), "r"(n * 4)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(smem_u32(buf)), "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(ox), "r"(oy), "r"(oz),
        "r"(smem_u32(&mbar))
        : "memory");
  }
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(&mbar)),
      "r"(0)
      : "memory");
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int N = 64;
  std::vector<float> h(N * N * N);
  for (int i = 0; i < N * N * N; ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(f);
  int fails = 0;
  const int boxes[][3] = {{8, 4, 2}, {48, 10, 25}, {48, 13, 28}};
  const int origins[][3] = {{0, 7, 9}, {4, 0, 0}, {-4, -2, -1}, {40, 61, 50}, {-8, 3, 62}, {60, 60, 60}};
  for (auto& b : boxes)
    for (auto& og : origins)
      for (int mode = 0; mode < 2; ++mode) {
        CUtensorMap tm;
        memset(&tm, 0, sizeof(tm));
        const cuuint64_t gd[3] = {N, N, N}, gs[2] = {N * 4, N * N * 4};
        const cuuint32_t bd[3] = {(cuuint32_t)b[0], (cuuint32_t)b[1], (cuuint32_t)b[2]}, es[3] = {1, 1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, gd, gs, bd, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int n = b[0] * b[1] * b[2];
        cudaMalloc(&o, n * 4);
        const size_t smem = n * 4 + 128;
        auto k = mode ? probe<1> : probe<0>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<1, 128, smem>>>(tm, og[0], og[1], og[2], n, o);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> got(n);
        cudaMemcpy(got.data(), o, n * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int z = 0; z < b[2]; ++z)
          for (int y = 0; y < b[1]; ++y)
            for (int x = 0; x < b[0]; ++x) {
              const int gx = og[0] + x, gy = og[1] + y, gz = og[2] + z;
              const bool in = gx >= 0 && gy >= 0 && gz >= 0 && gx < N && gy < N && gz < N;
              const float want = in ? (float)(gx + N * (gy + N * gz)) : 0.0f;
              if (got[(z * b[1] + y) * b[0] + x] != want) ++bad;
            }
        printf("box %d %d %d origin %d %d %d mode %d: encode %d launch %s bad %d\n", b[0], b[1], b[2], og[0], og[1],
               og[2], mode, (int)r, cudaGetErrorString(e), bad);
        fails += bad != 0 || e != cudaSuccess;
        cudaFree(o);
        if (e != cudaSuccess) { cudaDeviceReset(); cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice); }
      }
  printf("fails %d\n", fails);
  return fails != 0;
}
