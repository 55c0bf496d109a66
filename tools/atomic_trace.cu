// atomic_trace.cu — the L2 atomic ceiling for a GRAPH's own target
// distribution ("tighten the ceiling").  tools/ubench.cu
// measures random and mildly skewed addresses; PageRank's pushes land on
// RMAT in-degree hubs far more often.  This program replays a graph's column
// array — every edge's target, in CSR order, i.e. the multiset of addresses one
// full sweep of edge pushes hits — through the same operations the PageRank
// kernel issues, at full occupancy with 8 operations in flight per thread:
//   atom   returning f32 atomicAdd on every target (the threshold-crossing push)
//   red    red.add.f32 on every target
//   mixed  red.add.f64 for targets whose column carries HUB_TAG (bit 31; in-degree
//          >= the threshold tools/atomic_trace.py tags with, 2048 in the product,
//          R34/R35) and returning f32 atomicAdd for the others
//   mixed, R replicas  the same with each hub's fp64 residue spread over R
//          arrays n elements apart (replica = lane bits); R = 4 is the product's
//          push (R38)
//   mode 6  4 hub replicas and the non-hub returning atomics over 2 fp32
//          arrays (measured worse: the non-hub lines are not contended)
// Input: a raw int32 file of column entries (tools/atomic_trace.py writes it).
// Prints G ops/s per mode.  Not part of the product.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

template <int MODE>
__global__ void k(const uint32_t* __restrict__ col, int64_t m, float* res, double* res64, float* sink, int64_t nrep) {
  constexpr int U = 8;
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * U; base < m; base += stride) {
    uint32_t w[U];
#pragma unroll
    for (int j = 0; j < U; ++j) w[j] = base + j < m ? __ldg(col + base + j) : 0xFFFFFFFFu;
    float r[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      r[j] = 0.f;
      if (w[j] == 0xFFFFFFFFu) continue;
      const uint32_t v = w[j] & 0x3FFFFFFFu;
      if (MODE == 0) r[j] = atomicAdd(res + v, 1e-7f);
      if (MODE == 1) asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(res + v), "f"(1e-7f));
      if (MODE == 2) {
        if (w[j] & 0x80000000u) asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(res64 + v), "d"(1e-7));
        else r[j] = atomicAdd(res + v, 1e-7f);
      }
      if (MODE == 6) {  // hubs over 4 replicas AND non-hub returning atomics over 2 fp32 replica arrays
        const int64_t rep = (int64_t)(threadIdx.x & 3) * (int64_t)nrep;
        if (w[j] & 0x80000000u) asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(res64 + rep + v), "d"(1e-7));
        else r[j] = atomicAdd(res + (int64_t)(threadIdx.x & 1) * nrep + v, 1e-7f);
      }
      if (MODE >= 3 && MODE <= 5) {  // hub residues spread over R = 2^(MODE-2) replica arrays (replica = lane bits)
        constexpr int R = 1 << (MODE >= 3 && MODE <= 5 ? MODE - 2 : 0);
        const int64_t rep = (int64_t)(threadIdx.x & (R - 1)) * (int64_t)nrep;
        if (w[j] & 0x80000000u) asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(res64 + rep + v), "d"(1e-7));
        else r[j] = atomicAdd(res + v, 1e-7f);
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) acc += r[j];
  }
  if (acc == 12345.f) *sink = acc;
}

int main(int argc, char** argv) {
  if (argc != 3) {
    fprintf(stderr, "usage: atomic_trace COLS.bin n\n");
    return 64;
  }
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 2;
  fseek(f, 0, SEEK_END);
  const int64_t m = ftell(f) / 4;
  fseek(f, 0, SEEK_SET);
  std::vector<uint32_t> h(m);
  if (fread(h.data(), 4, m, f) != (size_t)m) return 3;
  fclose(f);
  const int64_t n = atoll(argv[2]);
  uint32_t* col;
  float *res, *s;
  double* res64;
  cudaMalloc(&col, m * 4);
  cudaMalloc(&res, n * 4 * 2);  // 2 fp32 replicas (mode 6)
  cudaMalloc(&res64, n * 8 * 8);  // up to 8 replica arrays (modes 3-5)
  cudaMalloc(&s, 4);
  cudaMemcpy(col, h.data(), m * 4, cudaMemcpyHostToDevice);
  cudaMemset(res, 0, n * 4 * 2);
  cudaMemset(res64, 0, n * 8 * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"atom.add.f32 (returning) on every target", "red.add.f32 on every target",
                         "mixed: red.add.f64 at hub targets, returning atom.add.f32 elsewhere (R35)",
                         "mixed, hub residues over 2 replica arrays", "mixed, hub residues over 4 replica arrays",
                         "mixed, hub residues over 8 replica arrays",
                         "mixed, hubs over 4 replicas and the non-hub returning atomics over 2"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("| op | targets (edges) | ms | G ops/s |\n|---|---|---|---|\n");
  for (int mode = 0; mode < 7; ++mode) {
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<sms * 8, 256>>>(col, m, res, res64, s, n);
      if (mode == 1) k<1><<<sms * 8, 256>>>(col, m, res, res64, s, n);
      if (mode == 2) k<2><<<sms * 8, 256>>>(col, m, res, res64, s, n);
      if (mode == 3) k<3><<<sms * 8, 256>>>(col, m, res, res64, s, n);
      if (mode == 4) k<4><<<sms * 8, 256>>>(col, m, res, res64, s, n);
      if (mode == 5) k<5><<<sms * 8, 256>>>(col, m, res, res64, s, n);
      if (mode == 6) k<6><<<sms * 8, 256>>>(col, m, res, res64, s, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("| %s | %lld | %.2f | %.1f |\n", names[mode], (long long)m, ms, m / (ms * 1e6));
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
