// cta_ws2.cuh — decoupled warp-specialised persistent CTA worker for the
// edge-map apps (BFS, PageRank; SURVEY §8a rows a4 + a5).
//
// Warp 0 (the queue agent) pops FETCH-sized batches, reads their slots, runs
// begin()/chunk/split and scans degrees into a ring of NBUF shared-memory batch
// buffers, up to NBUF-1 batches ahead.  Worker warps 1..W-1 consume the ring
// in order, claiming 32*UNROLL-edge steps of the current batch with a
// shared-memory atomic; a warp that finds the batch exhausted moves on to the
// next batch at once — no CTA barrier per batch.  The last warp to leave a
// batch increments `processed` (a7; every warp's pushes for the batch are
// reserved before it leaves) and frees the buffer.  (The double-buffered
// version with bar.sync hand-offs spent 20-27% of its stall samples in
// barriers, profiles/r01_*_ncu.md.)
#pragma once
#include "cta_ws.cuh"

namespace atos {

constexpr int NBUF = 4;
// CTA-local continuation (small-frontier regime): while the global queue is
// short, a worker warp keeps the vertices it activates in its own SPSC ring in
// shared memory and the CTA's agent takes them next, skipping the global
// push -> poll -> pop round trip on the critical path of high-diameter
// graphs (9.5 us per hop on the 4899^2 grid without it).  Kept items are
// counted in ctl->kept (they take no ring position), and quiescence (a7) is
// processed == tail + kept.
constexpr int LCAP = 128;  // per worker warp
constexpr int STEP_CAP = 2048;  // per-buffer step-owner table (steps beyond it search)
// Register budget vs occupancy of the persistent CTA kernel (build-time knobs).
// Measured on RMAT-24 (PR kernel ms / BFS ms): 1024x1 bound (64 regs, some
// spills) + unroll 8: 209 / 4.1 — best; 512x1 (128 regs) + unroll 16:
// 259 / 6.9; 256x3 (85 regs) + unroll 8: 257 / 4.0; 512x1 + unroll 8: 228 / 6.1.
// Occupancy beats per-warp memory-level parallelism here.
#ifndef ATOS_CTA_MAX_THREADS
#define ATOS_CTA_MAX_THREADS 1024
#endif
#ifndef ATOS_CTA_MIN_BLOCKS
#define ATOS_CTA_MIN_BLOCKS 1
#endif
#ifndef ATOS_WS_UNROLL
#define ATOS_WS_UNROLL 8
#endif
constexpr int CTA_MAX_THREADS = ATOS_CTA_MAX_THREADS;
constexpr int CTA_MIN_BLOCKS = ATOS_CTA_MIN_BLOCKS;
constexpr int WS_UNROLL = ATOS_WS_UNROLL;
constexpr int64_t STEP_EDGES = 32 * WS_UNROLL;
enum : int { BUF_FREE = 0, BUF_READY = 1, BUF_QUIT = 2 };

struct BufHdr {
  int state;     // BUF_*
  int seq;       // ring pass this batch belongs to (a fast warp must not re-enter an older batch)
  int n;         // items
  int next;      // next step index to claim
  int left;      // warps that have left this batch
  long long total;
};

template <class Payload>
__host__ __device__ constexpr size_t ws2_buf_bytes(int F) {
  return ws_buf_bytes<Payload>(F) + (size_t)STEP_CAP * 4;
}
template <class Payload>
__host__ __device__ constexpr size_t ws2_smem_bytes(int F) {
  // + local rings (31 worker warps max) + their head/tail + the agent's gather scratch
  return (size_t)NBUF * ws2_buf_bytes<Payload>(F) + NBUF * sizeof(BufHdr) + 64 + 31 * LCAP * 4 + 64 * 4 +
         ((size_t)F * 4 + 16);
}

// Worker-side sink: keep activated items in the warp's local ring when the
// agent says the global queue is short and the ring has room; else push globally.
struct KeepSink {
  Queue q;
  uint32_t* ring;          // this warp's LCAP slots
  int* tail;               // producer index (this warp)
  const int* head;         // consumer index (agent)
  const int* keep;         // agent's "queue is short" flag
  template <int U>
  __device__ __forceinline__ uint32_t warp_push_multi(const bool (&pred)[U], const uint32_t (&item)[U]) const {
    unsigned m[U];
    uint32_t total = 0;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      m[k] = __ballot_sync(FULL_MASK, pred[k]);
      total += __popc(m[k]);
    }
    if (total == 0) return 0;
    const int t = *(volatile const int*)tail;
    const bool local = *(volatile const int*)keep && (int)total <= LCAP - (t - *(volatile const int*)head);
    if (!local) return q_warp_push_multi<U>(q, pred, item);
    if (lane_id() == 0)  // count the kept items as enqueued (termination); wait for it to be performed
      (void)atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->kept.v), (unsigned long long)total);
    const unsigned lt = lanemask_lt();
    int base = t;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (pred[k]) ring[(base + __popc(m[k] & lt)) % LCAP] = item[k];
      base += __popc(m[k]);
    }
    __syncwarp();
    if (lane_id() == 0) {
      __threadfence_block();
      *(volatile int*)tail = t + (int)total;
    }
    __syncwarp();
    return total;
  }
};

__device__ __forceinline__ int vload(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ void vstore(int* p, int v) { *(volatile int*)p = v; }

// Agent pop: CTA-local continuation items first, then the global queue; the
// idle path polls both and runs the termination check (a7).  Also maintains
// the `keep` flag (global queue short => workers keep their activations).
__device__ __forceinline__ uint32_t agent_pop(const Queue& q, uint32_t want, uint64_t& first, uint64_t& hw, int nw,
                                              const uint32_t* lrings, int* lhead, const int* ltail, int* keep,
                                              uint32_t* gather, bool& from_local, bool allow_keep,
                                              long long& last_count) {
  const int lane = lane_id();
  unsigned ns = 0;
  for (;;) {
    // 1. local rings (lane w drains worker warp w's ring)
    uint32_t got = 0;
    if (*(volatile int*)keep || true) {
      int avail = 0, h = 0;
      if (lane < nw) {
        h = lhead[lane];
        avail = *(volatile const int*)(ltail + lane) - h;
      }
      // exclusive scan of avail over lanes, capped at want
      int x = avail;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(FULL_MASK, x, d);
        if (lane >= d) x += y;
      }
      const int before = x - avail;
      const int take = max(0, min(avail, (int)want - before));
      __threadfence_block();
      for (int i = 0; i < take; ++i) gather[before + i] = lrings[lane * LCAP + (h + i) % LCAP];
      got = (uint32_t)min(__shfl_sync(FULL_MASK, x, 31), (int)want);
      __syncwarp();
      if (take) *(volatile int*)(lhead + lane) = h + take;
      __syncwarp();
    }
    if (got) {
      from_local = true;
      return got;
    }
    from_local = false;
    // 2. global queue (abort / watchdog are checked on the idle path only)
    uint32_t n = 0;
    uint64_t qlen = 0;
    bool quit = false;
    if (lane == 0) {
      n = q_try_pop(q, want, first, qlen, last_count);
      last_count = (long long)qlen - (long long)n;
      if (allow_keep) *(volatile int*)keep = last_count < (long long)q.workers * 2 ? 1 : 0;
      if (n) {
        if (qlen > hw) hw = qlen;
      } else if (q_aborted(q) || q_timed_out(q)) {
        quit = true;
      } else {
        const uint64_t p = ld_acquire_u64(&q.ctl->processed.v);
        const uint64_t t = q_enqueued(q);
        quit = p == t;
      }
    }
    n = __shfl_sync(FULL_MASK, n, 0);
    first = __shfl_sync(FULL_MASK, first, 0);
    if (n) return n;
    if (__shfl_sync(FULL_MASK, quit, 0)) return 0;
    if (ns) __nanosleep(ns);
    ns = ns == 0 ? 32 : (ns < q.backoff_ns ? ns * 2 : ns);
  }
}

template <class App>
__device__ void cta_ws2_persistent(const App& app, const GraphView& g, const Queue& q, int F, unsigned char* smem,
                                   LocalStats& st) {
  using Payload = typename App::Payload;
  const int T = blockDim.x, tid = threadIdx.x, wid = tid >> 5, lane = lane_id();
  const size_t bb = ws2_buf_bytes<Payload>(F);
  BufHdr* hdr = reinterpret_cast<BufHdr*>(smem + NBUF * bb);
  auto buf_own = [&](int b) { return reinterpret_cast<int*>(smem + b * bb + ws_buf_bytes<Payload>(F)); };
  auto buf_e0 = [&](int b) { return reinterpret_cast<int64_t*>(smem + b * bb); };
  auto buf_pre = [&](int b) { return reinterpret_cast<int64_t*>(smem + b * bb) + F; };
  auto buf_pay = [&](int b) { return reinterpret_cast<Payload*>(reinterpret_cast<int64_t*>(smem + b * bb) + 2 * F + 1); };
  const Queue* cq = q.chunks ? &q : nullptr;
  const int nw = (T >> 5) - 1;
  uint32_t* lrings = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(hdr + NBUF) + 64);
  int* lhead = reinterpret_cast<int*>(lrings + 31 * LCAP);  // [32]
  int* ltail = lhead + 32;                                  // [32]
  int* keep = ltail + 31;                                   // shares the last tail slot (31 warps max)
  uint32_t* gather = reinterpret_cast<uint32_t*>(ltail + 32);
  if (tid < 64) lhead[tid] = 0;
  if (tid == 0) *keep = 0;
  if (tid < NBUF) hdr[tid] = BufHdr{BUF_FREE, -1, 0, 0, 0, 0};
  __syncthreads();

  if (wid == 0) {
    // ------------------------------------------------ queue agent
    long long last_count = 0;  // lane 0: queue length seen at the last pop
    for (int i = 0;; ++i) {
      const int b = i % NBUF;
      // wait until the workers have released buffer b
      bool dead = false;
      for (unsigned ns = 8; vload(&hdr[b].state) != BUF_FREE; ns = ns < 256 ? ns * 2 : ns) {
        __nanosleep(ns);
        if (q_aborted(q) || q_timed_out(q)) { dead = true; break; }
      }
      if (dead) {  // workers are stuck on an unreleased batch only if they died; publish QUIT anyway
        if (lane == 0) { hdr[b].seq = i / NBUF; __threadfence_block(); vstore(&hdr[b].state, BUF_QUIT); }
        __syncwarp();
        break;
      }
      uint64_t first = 0;
      uint32_t n = 0;
      bool from_local = false;
      if constexpr (App::kWindow) {
        n = window_pop(app, q, (uint32_t)F, first, st.hw);
      } else {
        n = agent_pop(q, (uint32_t)F, first, st.hw, nw, lrings, lhead, ltail, keep, gather, from_local, App::kKeep,
                      last_count);
      }
      if (n) {
        agent_prepare(app, g, q, cq, first, n, buf_e0(b), buf_pre(b), buf_pay(b), from_local ? gather : nullptr);
        int64_t* pre = buf_pre(b);
        warp_exclusive_scan(pre, (int)n);
        // step-owner table: own[c] = item holding flattened edge c*STEP_EDGES
        int* own = buf_own(b);
        for (uint32_t it = lane; it < n; it += 32) {
          const int64_t c0 = (pre[it] + STEP_EDGES - 1) / STEP_EDGES;
          const int64_t c1 = min((pre[it + 1] + STEP_EDGES - 1) / STEP_EDGES, (int64_t)STEP_CAP);
          for (int64_t c = c0; c < c1; ++c) own[c] = (int)it;
        }
        __syncwarp();
      }
      if (lane == 0) {
        hdr[b].n = (int)n;
        hdr[b].total = n ? buf_pre(b)[n] : 0;
        hdr[b].next = 0;
        hdr[b].left = 0;
        hdr[b].seq = i / NBUF;
        __threadfence_block();
        vstore(&hdr[b].state, n ? BUF_READY : BUF_QUIT);
      }
      __syncwarp();
      if (n == 0) break;
    }
  } else {
    // ------------------------------------------------ edge workers
    const int wi = wid - 1;
    KeepSink sink{q, lrings + wi * LCAP, ltail + wi, lhead + wi, keep};
    uint32_t pushed = 0;
    uint64_t edges = 0;
    for (int i = 0;; ++i) {
      const int b = i % NBUF, pass = i / NBUF;
      int s = BUF_FREE;
      for (unsigned ns = 8;; ns = ns < 128 ? ns * 2 : ns) {
        s = vload(&hdr[b].state);
        if (s != BUF_FREE && vload(&hdr[b].seq) == pass) break;
        __nanosleep(ns);
        if (ns >= 128 && (q_aborted(q) || q_timed_out(q))) { s = BUF_QUIT; break; }
      }
      if (s == BUF_QUIT) break;
      __threadfence_block();
      const int n = hdr[b].n;
      const int64_t total = hdr[b].total;
      const int64_t* pre = buf_pre(b);
      const int64_t* e0 = buf_e0(b);
      const Payload* pay = buf_pay(b);
      const int* own = buf_own(b);
      const int64_t steps = (total + STEP_EDGES - 1) / STEP_EDGES;
      for (;;) {
        int c = 0;
        if (lane == 0) c = atomicAdd(&hdr[b].next, 1);
        c = __shfl_sync(FULL_MASK, c, 0);
        if ((int64_t)c >= steps) break;
        int hlo = -1, hhi = -1;
        if (c < STEP_CAP) {
          hlo = own[c];
          hhi = (c + 1 < steps && c + 1 < STEP_CAP) ? own[c + 1] : n - 1;
        }
        const uint32_t p = lbs_step<App, KeepSink, WS_UNROLL>(app, g, sink, pre, e0, pay, n, total,
                                                               (int64_t)c * STEP_EDGES, hlo, hhi);
        if (lane == 0) pushed += p;
        if (lane == 0) edges += (uint64_t)min(STEP_EDGES, total - (int64_t)c * STEP_EDGES);
      }
      if constexpr (App::kWindow) {
        // Alg. 4 lines 11-14: each popped vertex checks a Check_Size window
        pushed += window_sweep(app, q, ((uint32_t)n * (uint32_t)app.check_size + nw - 1) / nw);
      }
      __syncwarp();
      int last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&hdr[b].left, 1) == nw - 1;
      }
      last = __shfl_sync(FULL_MASK, last, 0);
      if (last && lane == 0) {
        st.popped += (uint64_t)n;
        if constexpr (App::kWindow) {
          __threadfence();
          atomicMax(reinterpret_cast<unsigned long long*>(&q.ctl->aux[2].v),
                    (unsigned long long)ld_relaxed_u64(&q.ctl->aux[0].v));
        }
        q_done(q, (uint32_t)n);
        q_trace(q, (uint32_t)n, (uint64_t)total);
        vstore(&hdr[b].state, BUF_FREE);
      }
    }
    if (lane == 0) {
      st.pushed += pushed;
      st.edges += edges;
    }
  }
}

}  // namespace atos
