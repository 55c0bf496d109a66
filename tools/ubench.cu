// Microbenchmarks for the secondary (L2-atomic) ceiling of the Atos hot path:
// random-address atomics / loads over an n-element array (n = 2^24 = RMAT-24's
// vertex count, 64 MB), all SMs.  Prints G ops/s.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template <int MODE>
__global__ void k(float* a, uint32_t* u, uint32_t mask, uint64_t ops_per_thread, float* sink, uint32_t skew) {
  uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0;
  for (uint64_t i = 0; i < ops_per_thread; i += 4) {
    uint32_t idx[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t h = hash32(tid * 0x9E3779B9u + (uint32_t)(i + j) * 0x85EBCA6Bu);
      idx[j] = skew ? ((h & mask) >> (h % skew)) : (h & mask);  // skew: RMAT-like hot low ids
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (MODE == 0) acc += atomicAdd(a + idx[j], 1e-7f);
      if (MODE == 1) atomicAdd(a + idx[j], 1e-7f);
      if (MODE == 2) acc += (float)atomicMin(u + idx[j], 5u);
      if (MODE == 3) acc += __ldcg(a + idx[j]);
      if (MODE == 4) { float v; asm volatile("ld.relaxed.cta.global.f32 %0, [%1];" : "=f"(v) : "l"(a + idx[j])); acc += v; }
    }
  }
  if (acc == 12345.f) *sink = acc;
}
__global__ void krand_big(const float* a, uint64_t mask, uint64_t ops_per_thread, float* sink) {
  uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0;
  for (uint64_t i = 0; i < ops_per_thread; i += 8) {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint64_t h = hash32(tid * 0x9E3779B9u + (uint32_t)(i + j) * 0x85EBCA6Bu);
      h = (h << 32) | hash32((uint32_t)h ^ 0x1234567u);
      v[j] = __ldcg(a + ((h & mask) << 3));  // one float per 32-byte sector
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j];
  }
  if (acc == 12345.f) *sink = acc;
}

int main() {
  {
    // random 32-byte sectors over 4 GB (L2 misses): DRAM random-access rate
    const uint64_t bytes = 4ull << 30;
    float* big; float* s0;
    cudaMalloc(&big, bytes); cudaMalloc(&s0, 4); cudaMemset(big, 0, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t sectors = bytes / 32;
    int blocks = sms * 8, threads = 256; uint64_t opt = 512;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      krand_big<<<blocks, threads>>>(big, sectors - 1, opt, s0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * opt;
    printf("%-34s           %8.1f G sectors/s = %7.1f GB/s of 32-B sectors (%.2f ms)\n", "random sector loads over 4 GB", ops / ms / 1e6, ops * 32 / ms / 1e6, ms);
    cudaFree(big);
  }
  const uint32_t n = 1u << 24;
  float* a; uint32_t* u; float* s;
  cudaMalloc(&a, n * 4); cudaMalloc(&u, n * 4); cudaMalloc(&s, 4);
  cudaMemset(a, 0, n * 4); cudaMemset(u, 0xff, n * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"atomicAdd f32 (ATOM, returning)", "atomicAdd f32 (RED)", "atomicMin u32 (ATOM)", "ld.cg f32 (L2)", "ld.relaxed.cta f32 (L1)"};
  for (int skew : {0, 12}) {
    for (int mode = 0; mode < 5; ++mode) {
      int blocks = sms * 8, threads = 256;
      uint64_t opt = 1024;
      double ops = (double)blocks * threads * opt;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        switch (mode) {
          case 0: k<0><<<blocks, threads>>>(a, u, n - 1, opt, s, skew); break;
          case 1: k<1><<<blocks, threads>>>(a, u, n - 1, opt, s, skew); break;
          case 2: k<2><<<blocks, threads>>>(a, u, n - 1, opt, s, skew); break;
          case 3: k<3><<<blocks, threads>>>(a, u, n - 1, opt, s, skew); break;
          case 4: k<4><<<blocks, threads>>>(a, u, n - 1, opt, s, skew); break;
        }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("%-34s skew=%2d  %8.1f G ops/s  (%.2f ms)\n", names[mode], skew, ops / ms / 1e6, ms);
    }
  }
  return 0;
}
