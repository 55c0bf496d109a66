// Microbenchmarks for the secondary (L2-atomic) ceiling of the Atos hot path
// ("measure it with a microbenchmark"; sweep
// in-flight depth, occupancy and address locality).  Random-address atomics /
// loads over an n-element array (n = 2^24 = RMAT-24's vertex count), all SMs.
// Prints G ops/s.  Not part of the product.
//
// usage: ubench            full sweep (op x skew x in-flight x warps/SM)
//        ubench quick      the round-1 table (4 in flight, 64 warps/SM)
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
enum { ATOM_F32, RED_F32, ATOM_F64, RED_F64, ATOM_MIN_U32, LD_CG_F32, LD_CTA_F32, NMODES };
static const char* NAMES[] = {"atom.add.f32 (returning)", "red.add.f32", "atom.add.f64 (returning)", "red.add.f64",
                              "atom.min.u32 (returning)", "ld.cg.f32 (L2)", "ld.relaxed.cta.f32 (L1)"};

// DEPTH ops in flight per thread: all DEPTH addresses are computed, then all
// DEPTH ops issued, then (returning ops) all results consumed.
template <int MODE, int DEPTH>
__global__ void k(float* a, double* d, uint32_t* u, uint32_t mask, uint32_t iters, float* sink, uint32_t skew) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0;
  double accd = 0;
  for (uint32_t i = 0; i < iters; ++i) {
    uint32_t idx[DEPTH];
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) {
      const uint32_t h = hash32(tid * 0x9E3779B9u + (i * DEPTH + j) * 0x85EBCA6Bu);
      idx[j] = skew ? ((h & mask) >> (h % skew)) : (h & mask);  // skew: RMAT-like hot low ids
    }
    float r[DEPTH];
    double rd[DEPTH];
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) {
      r[j] = 0.f;
      rd[j] = 0.0;
      if (MODE == ATOM_F32) r[j] = atomicAdd(a + idx[j], 1e-7f);
      if (MODE == RED_F32) asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(a + idx[j]), "f"(1e-7f));
      if (MODE == ATOM_F64) rd[j] = atomicAdd(d + idx[j], 1e-7);
      if (MODE == RED_F64) asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(d + idx[j]), "d"(1e-7));
      if (MODE == ATOM_MIN_U32) r[j] = (float)atomicMin(u + idx[j], 5u);
      if (MODE == LD_CG_F32) r[j] = __ldcg(a + idx[j]);
      if (MODE == LD_CTA_F32) asm volatile("ld.relaxed.cta.global.f32 %0, [%1];" : "=f"(r[j]) : "l"(a + idx[j]));
    }
#pragma unroll
    for (int j = 0; j < DEPTH; ++j) {
      acc += r[j];
      accd += rd[j];
    }
  }
  if (acc == 12345.f || accd == 12345.0) *sink = acc;
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

template <int MODE, int DEPTH>
static float run1(int blocks, int threads, float* a, double* d, uint32_t* u, uint32_t n, uint32_t iters, float* s,
                  uint32_t skew) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<MODE, DEPTH><<<blocks, threads>>>(a, d, u, n - 1, iters, s, skew);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms;
}

template <int MODE>
static float run_depth(int depth, int blocks, int threads, float* a, double* d, uint32_t* u, uint32_t n, uint32_t ops,
                       float* s, uint32_t skew) {
  switch (depth) {
    case 1: return run1<MODE, 1>(blocks, threads, a, d, u, n, ops / 1, s, skew);
    case 4: return run1<MODE, 4>(blocks, threads, a, d, u, n, ops / 4, s, skew);
    case 8: return run1<MODE, 8>(blocks, threads, a, d, u, n, ops / 8, s, skew);
    default: return run1<MODE, 16>(blocks, threads, a, d, u, n, ops / 16, s, skew);
  }
}

static float run_mode(int mode, int depth, int blocks, int threads, float* a, double* d, uint32_t* u, uint32_t n,
                      uint32_t ops, float* s, uint32_t skew) {
  switch (mode) {
    case ATOM_F32: return run_depth<ATOM_F32>(depth, blocks, threads, a, d, u, n, ops, s, skew);
    case RED_F32: return run_depth<RED_F32>(depth, blocks, threads, a, d, u, n, ops, s, skew);
    case ATOM_F64: return run_depth<ATOM_F64>(depth, blocks, threads, a, d, u, n, ops, s, skew);
    case RED_F64: return run_depth<RED_F64>(depth, blocks, threads, a, d, u, n, ops, s, skew);
    case ATOM_MIN_U32: return run_depth<ATOM_MIN_U32>(depth, blocks, threads, a, d, u, n, ops, s, skew);
    case LD_CG_F32: return run_depth<LD_CG_F32>(depth, blocks, threads, a, d, u, n, ops, s, skew);
    default: return run_depth<LD_CTA_F32>(depth, blocks, threads, a, d, u, n, ops, s, skew);
  }
}

int main(int argc, char** argv) {
  const bool quick = argc > 1 && !strcmp(argv[1], "quick");
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  {
    // random 32-byte sectors over 4 GB (L2 misses): DRAM random-access rate
    const uint64_t bytes = 4ull << 30;
    float* big;
    float* s0;
    cudaMalloc(&big, bytes);
    cudaMalloc(&s0, 4);
    cudaMemset(big, 0, bytes);
    const uint64_t sectors = bytes / 32;
    int blocks = sms * 8, threads = 256;
    uint64_t opt = 512;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      krand_big<<<blocks, threads>>>(big, sectors - 1, opt, s0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * opt;
    printf("random 32-B sector loads over 4 GB: %.1f G sectors/s = %.1f GB/s (%.2f ms)\n", ops / ms / 1e6,
           ops * 32 / ms / 1e6, ms);
    cudaFree(big);
  }
  const uint32_t n = 1u << 24;
  float* a;
  double* d;
  uint32_t* u;
  float* s;
  cudaMalloc(&a, n * 4);
  cudaMalloc(&d, n * 8ull);
  cudaMalloc(&u, n * 4);
  cudaMalloc(&s, 4);
  cudaMemset(a, 0, n * 4);
  cudaMemset(d, 0, n * 8ull);
  cudaMemset(u, 0xff, n * 4);
  const uint32_t ops = 1024;  // per thread
  printf("| op | skew | in flight / thread | warps / SM | G ops/s |\n|---|---|---|---|---|\n");
  const int depths[] = {4, 1, 8, 16}, wpsm[] = {64, 16, 32};
  const int nd = quick ? 1 : 4, nwp = quick ? 1 : 3;
  for (int mode = 0; mode < NMODES; ++mode)
    for (int skew : {0, 12})
      for (int di = 0; di < nd; ++di)
        for (int wi = 0; wi < nwp; ++wi) {
          const int depth = depths[di], w = wpsm[wi];
          const int threads = 256, blocks = sms * (w * 32 / threads);
          const float ms = run_mode(mode, depth, blocks, threads, a, d, u, n, ops, s, (uint32_t)skew);
          const double total = (double)blocks * threads * (double)(ops / depth * depth);
          printf("| %s | %d | %d | %d | %.1f |\n", NAMES[mode], skew, depth, w, total / ms / 1e6);
        }
  return 0;
}
