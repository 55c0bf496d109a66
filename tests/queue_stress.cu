// queue_stress.cu — TEST PROGRAM (tests/test_queue_stress.py): the product's
// shared task queue (paper_2112_00132_b200/csrc/device.cuh: warp-aggregated
// push, count-reservation pop, q_read_batch, termination detector) under a
// unique-tag workload, without any graph app on top (PAPER.md P:240-242,
// "atomic operations to ensure exclusive pops"; SURVEY §8c queue pins).
//
// K chains of unique tags: task t (t < N) spawns task t + K.  So exactly N
// tasks exist, each must be processed exactly once, and at most K are live —
// with a ring of `cap` >= K slots the ring wraps ~N/cap times.  With K = 0 the
// tags form a binary tree from root 0 (t spawns 2t+1, 2t+2 < N): the live set
// grows to ~N/2, which must overflow a small ring — detected, not hung.  Workers (one
// warp each) pop FETCH-sized batches, read them with q_read_batch, sleep a
// pseudo-random time (race widening) before pushing the children and before
// marking the batch processed, then poll for termination exactly like the
// persistent kernels.  The host checks: every tag seen exactly once (multiset
// equality), processed == pushed == N, no abort, and that no worker exited
// while tasks remained (early-exit detector: a worker records the processed
// count it saw when it quit; it must equal N).
//
// Message-passing litmus (SURVEY hard part 5, DESIGN §5 "memory ordering"):
// before pushing child c the producer writes payload[c] = sig(c) with an
// atomicExch whose RETURNED value feeds the push predicate — the pattern the
// apps rely on (BFS atomicMin, PageRank atomicAdd decide the push) — and the
// slot is then published with a relaxed store.  A consumer that read c from
// its slot loads payload[c] with ld.relaxed.gpu and counts a violation if it
// does not see sig(c).  The test requires zero violations.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2112_00132_b200/csrc/device.cuh"

using namespace atos;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t sig(uint32_t t) { return mix(t ^ 0x5bd1e995u) | 1u; }

__global__ void k_stress(Queue q0, uint32_t N, uint32_t K, uint32_t fetch, uint32_t sleep_mask, unsigned int* seen,
                         unsigned long long* quit_seen, unsigned long long* early, uint32_t* payload,
                         unsigned long long* mp_viol) {
  extern __shared__ uint32_t stage_all[];
  Queue q = q0;
  q_arm(q);
  uint32_t* stage = stage_all + (threadIdx.x >> 5) * fetch;
  const uint32_t lane = lane_id();
  uint32_t rng = mix(blockIdx.x * 977u + threadIdx.x);
  for (;;) {
    uint64_t first = 0, hw = 0;
    uint32_t n = 0;
    if (lane == 0) n = q_pop_or_quit(q, fetch, first, hw);
    n = __shfl_sync(FULL_MASK, n, 0);
    first = __shfl_sync(FULL_MASK, first, 0);
    if (n == 0) break;
    q_read_batch(q, first, n, stage, lane, 32);
    __syncwarp();
    for (uint32_t b = 0; b < n; b += 32) {
      const uint32_t i = b + lane;
      bool child = false;
      uint32_t t = 0;
      bool child2 = false;
      if (i < n) {
        t = stage[i];
        if (t != EMPTY_ITEM) {
          atomicAdd(seen + t, 1u);
          if (ld_relaxed_u32(payload + t) != sig(t)) atomicAdd(mp_viol, 1ull);  // the producer's atomic visible?
          child = K ? t + K < N : 2 * t + 1 < N;
          child2 = !K && 2 * t + 2 < N;
        }
      }
      rng = mix(rng + t);
      if (sleep_mask) __nanosleep(rng & sleep_mask);  // widen push races
      // write each child's payload with an atomic whose returned value decides the push
      if (child) {
        const uint32_t c = K ? t + K : 2 * t + 1;
        child = atomicExch(payload + c, sig(c)) != sig(c);
      }
      if (child2) child2 = atomicExch(payload + 2 * t + 2, sig(2 * t + 2)) != sig(2 * t + 2);
      q_warp_push(q, child, K ? t + K : 2 * t + 1);
      q_warp_push(q, child2, 2 * t + 2);
    }
    __syncwarp();
    rng = mix(rng);
    if (sleep_mask) __nanosleep(rng & sleep_mask);  // widen the processed-after-push window
    if (lane == 0) q_done(q, n);
  }
  if (lane == 0) {
    const unsigned long long p = ld_acquire_u64(&q.ctl->processed.v);
    atomicMax(quit_seen, p);
    if (p != N && !q_aborted(q)) atomicAdd(early, 1ull);  // quit while work remained
  }
}

int main(int argc, char** argv) {
  if (argc != 7) {
    fprintf(stderr, "usage: queue_stress N K cap fetch blocks sleep_mask\n");
    return 64;
  }
  const uint32_t N = (uint32_t)atol(argv[1]), K = (uint32_t)atol(argv[2]), cap = (uint32_t)atol(argv[3]);
  const uint32_t fetch = (uint32_t)atol(argv[4]), blocks = (uint32_t)atol(argv[5]), sleep_mask = (uint32_t)strtoul(argv[6], 0, 0);
  uint64_t* ring;
  QueueCtl* ctl;
  unsigned int* seen;
  unsigned long long *quit_seen, *early, *mp_viol;
  uint32_t* payload;
  cudaMalloc(&ring, cap * 8ull);
  cudaMalloc(&ctl, sizeof(QueueCtl));
  cudaMalloc(&seen, N * 4ull);
  cudaMalloc(&quit_seen, 8);
  cudaMalloc(&early, 8);
  cudaMalloc(&mp_viol, 8);
  cudaMalloc(&payload, N * 4ull);
  cudaMemset(mp_viol, 0, 8);
  cudaMemset(payload, 0, N * 4ull);
  cudaMemset(ring, 0, cap * 8ull);
  cudaMemset(ctl, 0, sizeof(QueueCtl));
  cudaMemset(seen, 0, N * 4ull);
  cudaMemset(quit_seen, 0, 8);
  cudaMemset(early, 0, 8);
  // roots: tags 0..R-1 published at positions 0..R-1 (lap 0, full)
  const uint32_t R = K ? K : 1;
  if (R > cap) return 64;
  std::vector<uint64_t> init(R);
  for (uint32_t i = 0; i < R; ++i) init[i] = (1ull << 32) | i;
  cudaMemcpy(ring, init.data(), R * 8ull, cudaMemcpyHostToDevice);
  {  // the roots' payloads (sig(t), computed on the host with the same mix)
    auto hmix = [](uint32_t x) {
      x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
    };
    std::vector<uint32_t> pl(R);
    for (uint32_t i = 0; i < R; ++i) pl[i] = hmix(i ^ 0x5bd1e995u) | 1u;
    cudaMemcpy(payload, pl.data(), R * 4ull, cudaMemcpyHostToDevice);
  }
  QueueCtl h{};
  h.tail.v = R;
  h.count.v = R;
  cudaMemcpy(ctl, &h, sizeof h, cudaMemcpyHostToDevice);
  Queue q{};
  q.ring = ring;
  q.mask = cap - 1;
  q.log2cap = 0;
  while ((1u << q.log2cap) < cap) q.log2cap++;
  q.ctl = ctl;
  q.timeout_ns = 60ull * 1000000000ull;
  q.backoff_ns = 256;
  const int threads = 256;
  k_stress<<<blocks, threads, (threads / 32) * fetch * 4>>>(q, N, K, fetch, sleep_mask, seen, quit_seen, early,
                                                           payload, mp_viol);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "cuda: %s\n", cudaGetErrorString(e));
    return 2;
  }
  cudaMemcpy(&h, ctl, sizeof h, cudaMemcpyDeviceToHost);
  std::vector<unsigned int> s(N);
  cudaMemcpy(s.data(), seen, N * 4ull, cudaMemcpyDeviceToHost);
  unsigned long long qs = 0, ea = 0;
  cudaMemcpy(&qs, quit_seen, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&ea, early, 8, cudaMemcpyDeviceToHost);
  unsigned long long mv = 0;
  cudaMemcpy(&mv, mp_viol, 8, cudaMemcpyDeviceToHost);
  uint64_t zero = 0, dup = 0;
  for (uint32_t t = 0; t < N; ++t) {
    zero += s[t] == 0;
    dup += s[t] > 1;
  }
  printf("{\"N\": %u, \"K\": %u, \"cap\": %u, \"fetch\": %u, \"blocks\": %u, \"missing\": %llu, \"duplicated\": %llu, "
         "\"processed\": %llu, \"tail\": %llu, \"abort\": %llu, \"early_exits\": %llu, \"laps\": %llu, \"mp_violations\": %llu}\n",
         N, K, cap, fetch, blocks, (unsigned long long)zero, (unsigned long long)dup,
         (unsigned long long)h.processed.v, (unsigned long long)h.tail.v, (unsigned long long)h.abort.v, ea,
         (unsigned long long)(h.tail.v / cap), mv);
  return (zero || dup || h.processed.v != N || h.tail.v != N || h.abort.v || ea || mv) ? 1 : 0;
}
