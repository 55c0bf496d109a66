// racecheck probe: does compute-sanitizer racecheck accept an mbarrier producer/consumer handoff?
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ void mb_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory"); }
__device__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ bool mb_try(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
  return ok;
}
__global__ void k(int* out, int iters) {
  __shared__ int buf[2][256];
  __shared__ uint64_t full[2], empty[2];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x / 32 - 1;
  if (threadIdx.x < 2) { mb_init(&full[threadIdx.x], 1); mb_init(&empty[threadIdx.x], nw); }
  __syncthreads();
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    const int b = i & 1, pass = i >> 1;
    if (wid == 0) {
      if (pass > 0) while (!mb_try(&empty[b], (pass - 1) & 1)) {}
      for (int j = lane; j < 256; j += 32) buf[b][j] = i * 1000 + j;
      __syncwarp();
      if (lane == 0) mb_arrive(&full[b]);
    } else {
      while (!mb_try(&full[b], pass & 1)) {}
      for (int j = lane; j < 256; j += 32) acc += buf[b][j];
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[b]);
    }
  }
  atomicAdd(out, acc);
}
int main() { int* o; cudaMalloc(&o, 4); cudaMemset(o, 0, 4); k<<<4, 128>>>(o, 64); int h = 0; cudaMemcpy(&h, o, 4, cudaMemcpyDeviceToHost); printf("probe %d %s\n", h, cudaGetErrorString(cudaGetLastError())); }
