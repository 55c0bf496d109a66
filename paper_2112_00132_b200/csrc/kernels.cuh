// kernels.cuh — the three kernel strategies (PAPER.md
// P:264) over any worker policy:
//   k_persistent  one launch; workers loop pop -> process -> push until the
//                 termination detector fires (Listing 2).
//   k_discrete    one launch per round over the queue snapshot [h, t) with
//                 static slot assignment (no pop atomics); pushes land beyond t.
//   k_bsp         one launch per BSP step over an explicit frontier array
//                 (Alg. 1/3/5), appending to an out-frontier.
#pragma once
#include "cta_ws2.cuh"
#include "gc.cuh"

namespace atos {

enum WorkerKind : int { W_THREAD = 0, W_WARP = 1, W_CTA = 2 };

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------- policies
template <class App>
struct EdgeMapPolicy {
  static constexpr bool kSplit = true;  // CTA workers split hubs into chunk tasks
  static constexpr bool kWarpSpecialised = true;
  using Payload = typename App::Payload;
  static __host__ __device__ size_t smem_bytes(int F) { return cta_smem_bytes<Payload>(F); }
  static __host__ __device__ size_t ws_smem(int F, int S) { return ws2_smem_bytes<Payload>(F, S); }
  static __device__ __forceinline__ void cta_persistent(const App& app, const GraphView& g, const Queue& q, int F,
                                                        unsigned char* smem, LocalStats& st) {
    cta_ws2_persistent(app, g, q, F, smem, st);
  }
  template <class Src, class Sink>
  static __device__ __forceinline__ void cta(const App& app, const GraphView& g, const Src& src, const Sink& sink,
                                             uint32_t n, unsigned char* smem, int F, LocalStats& st) {
    CtaSmem<Payload> sm = cta_smem_carve<Payload>(smem, F);
    cta_batch(app, g, src, sink, n, sm, st);
  }
  template <class Src, class Sink>
  static __device__ __forceinline__ void warp(const App& app, const GraphView& g, const Src& src, const Sink& sink,
                                              uint32_t n, LocalStats& st) {
    warp_batch(app, g, src, sink, n, st);
  }
  template <class Src, class Sink>
  static __device__ __forceinline__ void thread(const App& app, const GraphView& g, const Src& src,
                                                const Sink& sink, uint32_t n, LocalStats& st) {
    thread_batch(app, g, src, sink, n, st);
  }
};

template <int MODE>
struct GcPolicy {
  static constexpr bool kSplit = false;
  static constexpr bool kWarpSpecialised = false;
  static __host__ __device__ size_t ws_smem(int, int) { return 0; }
  static __device__ __forceinline__ void cta_persistent(const GcApp&, const GraphView&, const Queue&, int,
                                                        unsigned char*, LocalStats&) {}
  static __host__ __device__ size_t smem_bytes(int F) { return gc_cta_smem_bytes(F); }
  template <class Src, class Sink>
  static __device__ __forceinline__ void cta(const GcApp& app, const GraphView& g, const Src& src, const Sink& sink,
                                             uint32_t n, unsigned char* smem, int F, LocalStats& st) {
    GcCtaSmem sm = gc_smem_carve(smem, F);
    gc_cta_batch<MODE>(app, g, src, sink, n, sm, st);
  }
  template <class Src, class Sink>
  static __device__ __forceinline__ void warp(const GcApp& app, const GraphView& g, const Src& src, const Sink& sink,
                                              uint32_t n, LocalStats& st) {
    uint64_t edges = 0;
    uint32_t pushed = 0;
    for (uint32_t j = 0; j < n; ++j) {
      uint32_t t = 0;
      bool ok = true;
      if (lane_id() == 0) ok = src.get(j, t);
      ok = __shfl_sync(FULL_MASK, ok, 0);
      t = __shfl_sync(FULL_MASK, t, 0);
      if (!ok) continue;
      if (MODE == GC_BSP_DETECT) t |= GC_CHECK_BIT;
      pushed += gc_warp_task<MODE>(app, g, sink, t, edges);
    }
    if (lane_id() == 0) {
      st.pushed += pushed;
      st.edges += edges;
    }
  }
  template <class Src, class Sink>
  static __device__ __forceinline__ void thread(const GcApp& app, const GraphView& g, const Src& src,
                                                const Sink& sink, uint32_t n, LocalStats& st) {
    uint64_t edges = 0;
    uint32_t pushed = 0;
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t j = base + lane_id();
      uint32_t t = 0;
      bool ok = j < n && src.get(j, t);
      if (MODE == GC_BSP_DETECT) t |= GC_CHECK_BIT;
      pushed += gc_thread_task<MODE>(app, g, sink, ok, t, edges);
    }
    st.edges += edges;
    if (lane_id() == 0) st.pushed += pushed;
  }
};

// Stage claimed ring positions [first, first+n) into shared memory (warp-collective).
__device__ __forceinline__ void stage_items(const Queue& q, uint64_t first, uint32_t n, uint32_t* stage) {
  q_read_batch(q, first, n, stage, lane_id(), 32);
  __syncwarp();
}
struct StageSrc {
  const uint32_t* a;
  __device__ __forceinline__ bool get(uint32_t i, uint32_t& item) const {
    item = a[i];
    return item != EMPTY_ITEM;
  }
};

// dynamic shared memory per block for a worker kind
template <class P>
__host__ __device__ inline size_t worker_smem_bytes(int W, int F, int T, bool persistent = false, int S = 0) {
  if (W == W_CTA) {
    if (persistent && P::kWarpSpecialised) return P::ws_smem(F, S);
    return persistent ? align16(P::smem_bytes(F)) + (size_t)F * 4 : P::smem_bytes(F);  // + the staged items
  }
  if (W == W_WARP) return (size_t)(T / 32) * (size_t)F * 4;
  return (size_t)T * (size_t)F * 4;
}

// ------------------------------------------------------------ persistent
template <class P, class App, int W>
__global__ void __launch_bounds__((W == W_CTA && P::kWarpSpecialised) ? CTA_MAX_THREADS : 1024,
                                  (W == W_CTA && P::kWarpSpecialised) ? CTA_MIN_BLOCKS : 1)
    k_persistent(App app, GraphView g, Queue q0, int F) {
  extern __shared__ __align__(16) unsigned char smem[];
  Queue q = q0;
  q_arm(q);
  LocalStats st;
  RingSink sink{q};
  if (W == W_CTA && P::kWarpSpecialised) {
    P::cta_persistent(app, g, q, F, smem, st);
  } else if (W == W_CTA) {
    __shared__ uint64_t s_first;
    __shared__ uint32_t s_n;
    for (;;) {
      if (threadIdx.x == 0) {
        uint64_t first = 0;
        uint32_t n = q_pop_or_quit(q, (uint32_t)F, first, st.hw);
        s_first = first;
        s_n = n;
      }
      __syncthreads();
      const uint32_t n = s_n;
      const uint64_t first = s_first;
      if (n == 0) break;
      // every claimed slot is read and released before the batch pushes anything (q_read_batch)
      uint32_t* stage = reinterpret_cast<uint32_t*>(smem + align16(P::smem_bytes(F)));
      q_read_batch(q, first, n, stage, threadIdx.x, blockDim.x);
      __syncthreads();
      StageSrc src{stage};
      const uint64_t e_before = st.edges;
      P::cta(app, g, src, sink, n, smem, F, st);  // ends with __syncthreads
      if (threadIdx.x == 0) {
        st.popped += n;
        q_done(q, n);
        q_trace(q, n, st.edges - e_before);
      }
    }
  } else {
    // Warp / thread workers stage their claimed items in shared memory right
    // after the pop (eager read): a worker never holds a claimed-but-unread
    // slot while it pushes, so a producer waiting on a wrapped slot (lap > 0)
    // can never wait on itself.
    const uint32_t want = (W == W_WARP) ? (uint32_t)F : 32u * (uint32_t)F;
    uint32_t* stage = reinterpret_cast<uint32_t*>(smem) + (size_t)(threadIdx.x >> 5) * want;
    for (;;) {
      uint64_t first = 0;
      uint32_t n = 0;
      if (lane_id() == 0) n = q_pop_or_quit(q, want, first, st.hw);
      n = __shfl_sync(FULL_MASK, n, 0);
      first = __shfl_sync(FULL_MASK, first, 0);
      if (n == 0) break;
      stage_items(q, first, n, stage);
      StageSrc src{stage};
      const uint64_t e_before = st.edges;
      if (W == W_WARP) P::warp(app, g, src, sink, n, st);
      else P::thread(app, g, src, sink, n, st);
      __syncwarp();
      uint64_t de = st.edges - e_before;
      if (W == W_THREAD) de = __reduce_add_sync(FULL_MASK, (unsigned)min(de, (uint64_t)0xFFFFFFFFu));
      if (lane_id() == 0) {
        st.popped += n;
        q_done(q, n);
        q_trace(q, n, de);
      }
    }
  }
  st.flush(q);
}

// ------------------------------------------------------------ discrete
// Round over queue positions [h, t); worker k owns [h + k*chunk, ...).
template <class P, class App, int W>
__device__ __forceinline__ void discrete_round(const App& app, const GraphView& g, Queue& q, uint64_t h, uint64_t t,
                                               int F, unsigned char* smem, unsigned long long* claim = nullptr) {
  q_arm(q);
  q.head_floor = t;
  LocalStats st;
  RingSink sink{q};
  const uint64_t S = t - h;
  if (W == W_CTA) {
    __shared__ unsigned long long s_k;
    // static striding for a grid sized to the round (host loop); dynamic
    // claiming for the fixed persistent-sized grid of the device loop
    for (uint64_t k = blockIdx.x;; k += gridDim.x) {
      if (claim) {
        __syncthreads();
        if (threadIdx.x == 0) s_k = atomicAdd(claim, 1ull);
        __syncthreads();
        k = s_k;
      }
      if (k * (uint64_t)F >= S) break;
      const uint64_t first = h + k * (uint64_t)F;
      const uint32_t n = (uint32_t)umin64((uint64_t)F, t - first);
      RingSrc src{q, first};
      P::cta(app, g, src, sink, n, smem, F, st);
      if (threadIdx.x == 0) st.popped += n;
    }
  } else {
    const uint64_t chunk = (W == W_WARP) ? (uint64_t)F : 32ull * (uint64_t)F;
    const uint64_t wpb = blockDim.x >> 5;
    const uint64_t nw = (uint64_t)gridDim.x * wpb;
    uint32_t* stage = reinterpret_cast<uint32_t*>(smem) + (size_t)(threadIdx.x >> 5) * chunk;
    for (uint64_t k = blockIdx.x * wpb + (threadIdx.x >> 5);; k += nw) {
      if (claim) {
        unsigned long long kk = 0;
        if (lane_id() == 0) kk = atomicAdd(claim, 1ull);
        k = __shfl_sync(FULL_MASK, kk, 0);
      }
      if (k * chunk >= S) break;
      const uint64_t first = h + k * chunk;
      const uint32_t n = (uint32_t)umin64(chunk, t - first);
      stage_items(q, first, n, stage);
      StageSrc src{stage};
      if (W == W_WARP) P::warp(app, g, src, sink, n, st);
      else P::thread(app, g, src, sink, n, st);
      __syncwarp();
      if (lane_id() == 0) st.popped += n;
    }
  }
  st.flush(q);
}

template <class P, class App, int W>
__global__ void __launch_bounds__(1024, 1) k_discrete(App app, GraphView g, Queue q0, uint64_t h, uint64_t t, int F) {
  extern __shared__ __align__(16) unsigned char smem[];
  Queue q = q0;
  discrete_round<P, App, W>(app, g, q, h, t, F, smem);
}

// Device-driven discrete strategy: the round snapshot [h, t) lives in device
// memory and a CUDA-graph WHILE node repeats {k_discrete_dev, k_round_end}
// until a round produces nothing — one launch of the graph instead of one
// host round trip per round (the launch overhead the paper measures).
struct DevRound {
  uint64_t h, t, rounds;
  unsigned long long next;  // dynamic chunk claims of the current round
};

template <class P, class App, int W>
__global__ void __launch_bounds__(1024, 1) k_discrete_dev(App app, GraphView g, Queue q0, int F, DevRound* r) {
  extern __shared__ __align__(16) unsigned char smem[];
  Queue q = q0;
  discrete_round<P, App, W>(app, g, q, r->h, r->t, F, smem, &r->next);
}

__global__ void k_round_end(DevRound* r, const QueueCtl* ctl, cudaGraphConditionalHandle hnd) {
  r->h = r->t;
  r->t = *(volatile const uint64_t*)&ctl->tail.v;
  r->rounds++;
  r->next = 0;
  const bool more = r->t > r->h && *(volatile const uint64_t*)&ctl->abort.v == 0;
  cudaGraphSetConditional(hnd, more ? 1u : 0u);
}

// ------------------------------------------------------------ BSP
struct OffsetSrc {
  const uint32_t* a;
  __device__ __forceinline__ bool get(uint32_t i, uint32_t& item) const {
    item = a[i];
    return true;
  }
};
struct IotaSrc {
  uint32_t base;
  __device__ __forceinline__ bool get(uint32_t i, uint32_t& item) const {
    item = base + i;
    return true;
  }
};
struct NullSink {
  template <int U>
  __device__ __forceinline__ uint32_t warp_push_multi(const bool (&)[U], const uint32_t (&)[U]) const { return 0; }
  __device__ __forceinline__ uint32_t warp_push(bool, uint32_t) const { return 0; }
  __device__ __forceinline__ uint32_t active_push(bool, uint32_t) const { return 0; }
};

// in == nullptr: the frontier is all vertices [0, count).
template <class P, class App, int W>
__global__ void __launch_bounds__(1024, 1) k_bsp(App app, GraphView g, const uint32_t* in, uint64_t count,
                                              uint32_t* out, unsigned long long* out_count, QueueCtl* ctl, int F) {
  extern __shared__ __align__(16) unsigned char smem[];
  LocalStats st;
  ArraySink sink{out, out_count};
  const uint64_t chunk = (W == W_CTA) ? (uint64_t)F : (W == W_WARP ? (uint64_t)F : 32ull * (uint64_t)F);
  uint64_t k, step;
  if (W == W_CTA) { k = blockIdx.x; step = gridDim.x; }
  else { k = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); step = (uint64_t)gridDim.x * (blockDim.x >> 5); }
  for (; k * chunk < count; k += step) {
    const uint64_t first = k * chunk;
    const uint32_t n = (uint32_t)umin64(chunk, count - first);
    if (in) {
      OffsetSrc src{in + first};
      if (W == W_CTA) P::cta(app, g, src, sink, n, smem, F, st);
      else if (W == W_WARP) P::warp(app, g, src, sink, n, st);
      else P::thread(app, g, src, sink, n, st);
    } else {
      IotaSrc src{(uint32_t)first};
      if (W == W_CTA) P::cta(app, g, src, sink, n, smem, F, st);
      else if (W == W_WARP) P::warp(app, g, src, sink, n, st);
      else P::thread(app, g, src, sink, n, st);
    }
    if ((W == W_CTA && threadIdx.x == 0) || (W != W_CTA && lane_id() == 0)) st.popped += n;
  }
  if (ctl) {
    Queue q{};
    q.ctl = ctl;
    st.hw = 0;
    st.flush(q);
  }
}

// ------------------------------------------------------------ small kernels
template <class T>
__global__ void k_fill(T* a, int64_t n, T v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) a[i] = v;
}

// ring[p] = full(lap 0) | item(p) for p < n; item = p (| tag)
__global__ void k_ring_prefill(uint64_t* ring, int64_t n, uint32_t tag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    ring[i] = (1ull << 32) | (uint64_t)((uint32_t)i | tag);
}

// Initialise the control block: head = 0, tail = processed-base, etc.
__global__ void k_ctl_init(QueueCtl* ctl, uint64_t tail, uint64_t* ring, int64_t src_item) {
  ctl->head.v = 0;
  ctl->tail.v = tail;
  ctl->count.v = tail;
  ctl->processed.v = 0;
  ctl->abort.v = 0;
  ctl->high_water.v = tail;
  ctl->chunk_tail.v = 0;
  ctl->chunk_done.v = 0;
  ctl->trace_count.v = 0;
  for (int i = 0; i < 4; ++i) { ctl->stats[i].v = 0; ctl->aux[i].v = 0; }
  if (src_item >= 0) ring[0] = (1ull << 32) | (uint64_t)(uint32_t)src_item;
}

// BFS init: dist[:] = MAX, dist[src] = 0 (R1); done[:] = MAX; near mirrors dist
__global__ void k_bfs_init(uint32_t* dist, uint32_t* done, uint16_t* near, int64_t n, int64_t src) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    dist[i] = (i == src) ? 0u : 0xFFFFFFFFu;
    if (done) done[i] = 0xFFFFFFFFu;
    if (near) near[i] = (i == src) ? (uint16_t)0 : (uint16_t)0xFFFFu;
  }
}

// PR residue seeding (reading R4 of Alg. 3 lines 5-7): every edge v->w adds
// c = (1-a) a / deg(v) to r(w), no activation.  With R34's storage the add to a
// hub target (column HUB_TAG) accumulates in fp64 (red.add.f64 into the hub's
// replica lane & 3, R38 — hundreds of thousands of equal adds, R30), every
// other target in its fp32 residue directly (< 2048 adds, R34's argument); with
// all-fp64 residues (!SPLIT) every add is fp64.
//
// One flat pass over the edge array rather than an edge map over the
// all-vertex frontier: the (vertex, edge) sequence — vertex i's end offset
// off[i+1] merged with the edge indices 0..m-1 — is cut into tiles of SEED_D
// items along the merge path, so every tile holds at most SEED_D vertices +
// edges whatever the degree mix (runs of empty vertices, out-degree hubs).
// Each CTA walks a contiguous run of tiles, locating only its first tile in
// HBM and every later one inside the offsets it has staged in shared memory.
// Edges of a tile go to threads round-robin (coalesced column reads); an
// edge's source is the last staged vertex whose offset is <= the edge index.
// Every edge issues one non-returning atomic, so the pass runs at the L2
// atomic rate of the graph's own targets (profiles/r02_seed.md).
constexpr int SEED_T = 256, SEED_D = 2048;
__device__ __forceinline__ int64_t seed_path(const int64_t* off, int64_t n, int64_t m, int64_t diag) {
  // vertices fully consumed at merge-path diagonal `diag` (Merrill & Garland's CSR merge path)
  int64_t lo = diag > m ? diag - m : 0, hi = diag < n ? diag : n;
  while (lo < hi) {
    const int64_t p = (lo + hi) >> 1;
    if (off[p + 1] <= diag - p - 1) lo = p + 1;
    else hi = p;
  }
  return lo;
}
template <bool SPLIT>
__global__ void __launch_bounds__(SEED_T) k_pr_seed(const int64_t* __restrict__ off, const uint32_t* __restrict__ col,
                                                    int64_t n, int64_t m, float* res, double* res64, int64_t r2,
                                                    double c0) {
  __shared__ int64_t s_off[SEED_D + 2];
  __shared__ int64_t s_end[2];
  const int64_t tiles = (n + m + SEED_D - 1) / SEED_D;
  const int64_t t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
  if (t0 >= t1) return;
  int64_t i0 = seed_path(off, n, m, t0 * SEED_D);  // first vertex of the CTA's run
  int64_t j0 = t0 * SEED_D - i0;                   // first edge
  const uint32_t rep = lane_id() & (ATOS_HUB_REPLICAS - 1u);
  for (int64_t t = t0; t < t1; ++t) {
    const int64_t nv = n - i0 < SEED_D + 1 ? n - i0 + 1 : SEED_D + 2;  // staged entries off[i0 ..]
    for (int k = threadIdx.x; k < nv; k += SEED_T) s_off[k] = __ldg(off + i0 + k);
    __syncthreads();
    if (threadIdx.x == 0) {  // the tile's end point, by the same merge-path search over the staged offsets
      const int64_t d = (t + 1) * SEED_D < n + m ? SEED_D : n + m - t * SEED_D;
      int64_t lo = d > m - j0 ? d - (m - j0) : 0, hi = d < n - i0 ? d : n - i0;
      while (lo < hi) {
        const int64_t p = (lo + hi) >> 1;
        if (s_off[p + 1] <= j0 + (d - p - 1)) lo = p + 1;
        else hi = p;
      }
      s_end[0] = i0 + lo;
      s_end[1] = j0 + d - lo;
    }
    __syncthreads();
    const int64_t i1 = s_end[0], j1 = s_end[1];
    const int last = (int)(i1 - i0 < nv - 2 ? i1 - i0 : nv - 2);  // last staged vertex that can own an edge
    for (int64_t e = j0 + threadIdx.x; e < j1; e += SEED_T) {
      int lo = 0, hi = last;  // largest k with s_off[k] <= e
      while (lo < hi) {
        const int p = (lo + hi + 1) >> 1;
        if (s_off[p] <= e) lo = p;
        else hi = p - 1;
      }
      const double c = c0 / (double)(s_off[lo + 1] - s_off[lo]);
      const uint32_t raw = __ldg(col + e), w = raw & VID_MASK;
      if (SPLIT) {
        if ((raw >> TAG_SHIFT) & TAG_HUB) red_add_hot(res64 + rep * r2 + w, c);
        else red_add_hot(res + w, (float)c);
      } else {
        red_add_hot(res64 + w, c);
      }
    }
    __syncthreads();  // s_off / s_end are restaged
    i0 = i1;
    j0 = j1;
  }
}

// zero the fp64 residue of every hub (bit set in the hub bitmap)
__global__ void k_zero_hubs(const uint32_t* bits, int64_t n, double* res64, int64_t r2) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < (n + 31) / 32; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t m = bits[w];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      for (int k = 0; k < (int)ATOS_HUB_REPLICAS; ++k) res64[k * r2 + w * 32 + b] = 0.0;  // R38 replicas
    }
  }
}

__device__ __forceinline__ bool bit_of(const uint32_t* bits, int64_t v) {
  return bits && ((bits[v >> 5] >> (v & 31)) & 1u);
}

// Round the fp64 seeding sums (R30) to the residue storage (R34): a hub keeps
// its sum in fp64 (res64 is the sums array itself) and its fp32 word is 0;
// every other vertex takes the sum rounded once to R.
template <class R>
__global__ void k_f64_to_res(const double* a, R* b, const uint32_t* hub, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = bit_of(hub, i) ? R(0) : (R)a[i];
}

__global__ void k_f64_to_f32(const double* a, float* b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}

// Sink bitmap for PageRank sink deferral (R29): bit v of word v/32 = (deg(v) == 0).
__global__ void k_sink_bitmap(const int64_t* off, int64_t n, uint32_t* bits) {
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; b < n; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = b + lane_id();
    const uint32_t m = __ballot_sync(FULL_MASK, v < n && off[v + 1] == off[v]);
    if (lane_id() == 0) bits[b >> 5] = m;
  }
}

// Column tagging (R34, R37), at graph create: in-degree histogram, then bit
// 31 of every column entry whose target has in-degree >= thr, bit 30 if the
// target is dangling (the sink bitmap), and the hub bitmap.
// Tags (HUB_TAG: in-degree >= HUB_IN_DEG, SINK_TAG: out-degree 0) from one
// interleaved 4-MB map — word i holds the hub bits of vertices 16i..16i+15 in
// its low half and their sink bits in the high half — so each column costs one
// random gather that stays in L2 (the gathers' L1 wavefronts bound this
// kernel: with the two 2-MB bitmaps read separately it took 2.05 ms on RMAT-24).
__global__ void k_tag_map(const uint32_t* hub, const uint32_t* sink, int64_t n, uint32_t* map) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n + 15) / 16; i += (int64_t)gridDim.x * blockDim.x) {
    const int sh = (int)(i & 1) * 16;
    const uint32_t h = (hub[i >> 1] >> sh) & 0xFFFFu, k = (sink[i >> 1] >> sh) & 0xFFFFu;
    map[i] = h | (k << 16);
  }
}
__device__ __forceinline__ uint32_t tag_of(uint32_t raw, int64_t n, const uint32_t* map) {
  const uint32_t w = ATOS_CHK(raw & VID_MASK, (uint32_t)n);
  const uint32_t t = __ldg(map + (w >> 4)) >> (w & 15);
  return w | ((t & 1u) ? HUB_TAG : 0u) | ((t & 0x10000u) ? SINK_TAG : 0u);
}
// four columns per thread (one 16-B load; col is 16-B aligned and padded, capi.cu)
__global__ void k_tag_hubs(int32_t* col, int64_t m, int64_t n, const uint32_t* map) {
  const int64_t q = m >> 2;
  uint4* c4 = reinterpret_cast<uint4*>(col);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < q; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = c4[i];
    v.x = tag_of(v.x, n, map);
    v.y = tag_of(v.y, n, map);
    v.z = tag_of(v.z, n, map);
    v.w = tag_of(v.w, n, map);
    c4[i] = v;
  }
  const int64_t e = 4 * q + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < m) col[e] = (int32_t)tag_of((uint32_t)col[e], n, map);
}
__global__ void k_hub_bitmap(const uint32_t* indeg, int64_t n, uint32_t thr, uint32_t* bits,
                             unsigned long long* count) {
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; b < n; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = b + lane_id();
    const uint32_t m = __ballot_sync(FULL_MASK, v < n && indeg[v] >= thr);
    if (lane_id() == 0) {
      bits[b >> 5] = m;
      if (m) atomicAdd(count, (unsigned long long)__popc(m));
    }
  }
}

// R35: list of hub vertices with out-degree > 0, in id order within each warp's 32 ids.
__global__ void k_hub_list(const uint32_t* bits, const int64_t* off, int64_t n, uint32_t* list,
                           unsigned long long* count) {
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; b < n; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = b + lane_id();
    const bool h = v < n && ((bits[v >> 5] >> (v & 31)) & 1u) && off[v + 1] > off[v];
    const uint32_t m = __ballot_sync(FULL_MASK, h);
    if (!m) continue;
    unsigned long long base = 0;
    if (lane_id() == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
    base = __shfl_sync(FULL_MASK, base, 0);
    if (h) list[base + __popc(m & lanemask_lt())] = (uint32_t)v;
  }
}
// R35: every listed hub starts queued (the initial queue holds all vertices)
__global__ void k_hub_mark(const uint32_t* list, int64_t k, uint32_t* hq) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    hq[list[i]] = 1u;
}

// Sink absorption (R29): after quiescence every dangling vertex performs its
// deferred task body `rank[v] += exch(res[v], 0)` (Alg. 4 line 8 with deg 0, R5).
template <class R>
__global__ void k_pr_absorb_sinks(const uint32_t* __restrict__ bits, Residues<R> rs, double* rank, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    if ((bits[v >> 5] >> (v & 31)) & 1u) {
      const bool h = rs.res64 && bit_of(rs.hub, v);
      const double r = h ? rs.hub_read((uint32_t)v) : (double)rs.res[v];
      if (r != 0.0) {
        rank[v] += r;
        if (h) for (int k = 0; k < (int)ATOS_HUB_REPLICAS; ++k) rs.res64[k * rs.r2 + v] = 0.0;
        else rs.res[v] = R(0);
      }
    }
  }
}

// BSP PageRank filter kernel (Alg. 3 lines 18-22): residue > eps -> frontier
template <class R>
__global__ void k_pr_filter(Residues<R> rs, int64_t n, R eps, uint32_t* out, unsigned long long* count) {
  ArraySink sink{out, count};
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; b < n; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = b + lane_id();
    bool a = false;
    if (v < n) a = (rs.res64 && bit_of(rs.hub, v)) ? rs.hub_read((uint32_t)v) > (double)eps : rs.res[v] > eps;
    sink.warp_push(a, (uint32_t)v);
  }
}

// max over v of the residue (stats.max_residue), as float bits
template <class R>
__global__ void k_max_res(Residues<R> rs, int64_t n, unsigned int* out_bits) {
  float m = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, (rs.res64 && bit_of(rs.hub, i)) ? (float)rs.hub_read((uint32_t)i) : (float)rs.res[i]);
  for (int d = 16; d; d >>= 1) m = fmaxf(m, __shfl_xor_sync(FULL_MASK, m, d));
  if (lane_id() == 0) atomicMax(out_bits, __float_as_uint(m));  // m >= 0 so bit order == value order
}

// max reduction helpers for stats
__global__ void k_max_s32(const int32_t* a, int64_t n, int* out) {
  int m = -1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) m = max(m, a[i]);
  for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(FULL_MASK, m, d));
  if (lane_id() == 0) atomicMax(out, m);
}

}  // namespace atos
