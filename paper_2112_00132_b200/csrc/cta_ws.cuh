// cta_ws.cuh — warp-specialised persistent CTA worker for the edge-map apps
// (BFS, PageRank): SURVEY §8a rows a4 + a5 on sm_100a.
//
// Warp 0 is the CTA's queue agent: it pops the next FETCH-sized batch, reads
// the claimed slots, runs begin()/chunk/split for every item and scans the
// degrees into one of two shared-memory batch buffers, while warps 1..W-1
// expand the other buffer with the load-balancing search.  Pop latency (two
// L2 atomics), slot reads and the per-vertex begin() loads (dist/off/atomics)
// thereby overlap the previous batch's edge expansion instead of stalling the
// whole CTA at a barrier (measured: 24.5% of BFS stall samples sat at the
// post-pop barrier, profiles/r01_bfs_rmat24_v3).
//
// Sync: named barriers.  READY[b] (ids 1,2): agent bar.arrive, workers
// bar.sync.  FREE[b] (ids 3,4): workers bar.arrive, agent bar.sync.  DONE (id
// 5): workers only, before the batch's `processed` increment.  The agent reads
// every claimed slot before it pushes anything (split chunks), so it never
// waits on a wrapped slot it holds itself.
#pragma once
#include "engine.cuh"

namespace atos {

__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive_n(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <class Payload>
__host__ __device__ constexpr size_t ws_buf_bytes(int F) {
  return (size_t)F * 8 + ((size_t)F + 1) * 8 + (((size_t)F * sizeof(Payload) + 15) & ~(size_t)15);
}
template <class Payload>
__host__ __device__ constexpr size_t ws_smem_bytes(int F) {
  return 2 * ws_buf_bytes<Payload>(F) + 64;
}

// Warp-cooperative exclusive scan of a[0..n) into a[0..n], a[n] = total.
__device__ __forceinline__ void warp_exclusive_scan(int64_t* a, int n) {
  const int lane = lane_id();
  const int per = (n + 31) / 32;
  const int b = min(n, lane * per), e = min(n, b + per);
  int64_t s = 0;
  for (int i = b; i < e; ++i) s += a[i];
  int64_t x = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int64_t y = __shfl_up_sync(FULL_MASK, x, d);
    if (lane >= d) x += y;
  }
  int64_t run = x - s;
  for (int i = b; i < e; ++i) {
    int64_t d = a[i];
    a[i] = run;
    run += d;
  }
  if (lane == 31) a[n] = x;
  __syncwarp();
}

template <class App>
__device__ void cta_ws_persistent(const App& app, const GraphView& g, const Queue& q, int F, unsigned char* smem,
                                  LocalStats& st) {
  using Payload = typename App::Payload;
  const int T = blockDim.x, tid = threadIdx.x, wid = tid >> 5, lane = lane_id();
  const size_t bb = ws_buf_bytes<Payload>(F);
  uint32_t* hdr = reinterpret_cast<uint32_t*>(smem + 2 * bb);  // n of buffer 0 / 1
  auto buf_e0 = [&](int b) { return reinterpret_cast<int64_t*>(smem + b * bb); };
  auto buf_pre = [&](int b) { return reinterpret_cast<int64_t*>(smem + b * bb) + F; };
  auto buf_pay = [&](int b) { return reinterpret_cast<Payload*>(reinterpret_cast<int64_t*>(smem + b * bb) + 2 * F + 1); };
  const Queue* cq = q.chunks ? &q : nullptr;

  if (wid == 0) {
    // ------------------------------------------------ queue agent (warp 0)
    int b = 0;
    for (int round = 0;; ++round) {
      if (round >= 2) bar_sync_n(3 + b, T);  // workers released buffer b
      uint64_t first = 0;
      uint32_t n = 0;
      if (lane == 0) n = q_pop_or_quit(q, (uint32_t)F, first, st.hw);
      n = __shfl_sync(FULL_MASK, n, 0);
      first = __shfl_sync(FULL_MASK, first, 0);
      int64_t* e0 = buf_e0(b);
      int64_t* pre = buf_pre(b);
      Payload* pay = buf_pay(b);
      if (n) {
        for (uint32_t i = lane; i < n; i += 32) {  // read every claimed slot first
          uint32_t it = 0xFFFFFFFFu;
          if (!q_load_slot(q, first + i, it)) it = 0xFFFFFFFFu;
          pre[i] = it;
        }
        __syncwarp();
        for (uint32_t i = lane; i < n; i += 32) {
          const uint32_t it = (uint32_t)pre[i];
          int64_t a = 0, z = 0;
          Payload p{};
          const bool ok = it != 0xFFFFFFFFu && prepare_item(app, g, cq, it, a, z, p);
          e0[i] = a;
          pre[i] = ok ? z - a : 0;
          pay[i] = p;
        }
        __syncwarp();
        warp_exclusive_scan(pre, (int)n);
      }
      if (lane == 0) hdr[b] = n;
      bar_arrive_n(1 + b, T);  // buffer b ready (n == 0: quit)
      if (n == 0) {
        if (round >= 1) bar_sync_n(3 + (b ^ 1), T);  // consume the workers' last release
        break;
      }
      b ^= 1;
    }
  } else {
    // ------------------------------------------------ edge workers (warps 1..W-1)
    RingSink sink{q};
    const int nw = (T >> 5) - 1;
    int b = 0;
    uint32_t pushed = 0;
    uint64_t edges = 0;
    for (;;) {
      bar_sync_n(1 + b, T);
      const uint32_t n = hdr[b];
      if (n == 0) break;
      const int64_t* pre = buf_pre(b);
      const int64_t total = pre[n];
      pushed += lbs_expand(app, g, sink, pre, buf_e0(b), buf_pay(b), (int)n, total, wid - 1, nw);
      edges += total;
      bar_sync_n(5, T - 32);  // every worker's pushes for this batch are reserved
      if (tid == 32) {
        st.popped += n;
        q_done(q, n);
        q_trace(q, n, (uint64_t)total);
      }
      bar_arrive_n(3 + b, T);  // release buffer b
      b ^= 1;
    }
    if (lane == 0) st.pushed += pushed;
    if (tid == 32) st.edges += edges;
  }
}

}  // namespace atos
