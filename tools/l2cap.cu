// Effective L2 capacity for random atomics: G ops/s of returning f32 atomicAdd
// over arrays of increasing size, with and without an evict_last policy and
// the persisting-L2 carve-out.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template <int POL>
__global__ void k(float* a, uint32_t n, uint64_t opt, float* sink) {
  uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t pol;
  if (POL) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  float acc = 0;
  for (uint64_t i = 0; i < opt; i += 4) {
    float o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t idx = hash32(tid * 0x9E3779B9u + (uint32_t)(i + j) * 0x85EBCA6Bu) % n;
      if (POL) asm volatile("atom.relaxed.gpu.global.add.L2::cache_hint.f32 %0, [%1], %2, %3;" : "=f"(o[j]) : "l"(a + idx), "f"(1e-7f), "l"(pol));
      else o[j] = atomicAdd(a + idx, 1e-7f);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) acc += o[j];
  }
  if (acc == 12345.f) *sink = acc;
}
int main() {
  int dev = 0, maxp = 0, l2 = 0, sms = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  printf("L2 %d MB, max persisting %d MB\n", l2 >> 20, maxp >> 20);
  float *a, *s; cudaMalloc(&a, 512u << 20); cudaMalloc(&s, 4); cudaMemset(a, 0, 512u << 20);
  for (int carve = 0; carve < 2; ++carve) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve ? maxp : 0);
    for (int mb : {8, 16, 32, 48, 64, 80, 96, 128, 256}) {
      uint32_t n = (uint32_t)((size_t)mb << 20) / 4;
      for (int pol = 0; pol < 2; ++pol) {
        int blocks = sms * 8, threads = 256; uint64_t opt = 512;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(e0);
          if (pol) k<1><<<blocks, threads>>>(a, n, opt, s); else k<0><<<blocks, threads>>>(a, n, opt, s);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("carve=%d array=%4d MB evict_last=%d : %7.1f G atomics/s\n", carve, mb, pol, (double)blocks * threads * opt / ms / 1e6);
      }
    }
  }
  return 0;
}
