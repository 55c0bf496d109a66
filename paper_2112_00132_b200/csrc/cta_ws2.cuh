// cta_ws2.cuh — decoupled warp-specialised persistent CTA worker for the
// edge-map apps (BFS, PageRank; SURVEY §8a rows a4 + a5).
//
// Warp 0 (the queue agent) pops FETCH-sized batches, reads their slots, runs
// begin()/chunk/split and scans degrees into a ring of NBUF shared-memory batch
// buffers, up to NBUF-1 batches ahead.  It also stages the batch's column lists
// into the buffer with TMA 1-D bulk copies (cp.async.bulk, completion on a
// per-buffer mbarrier), so worker warps read neighbour ids from shared memory
// instead of waiting on DRAM ("lists ... staged into smem
// by cp.async.bulk (TMA 1-D bulk copy), double-buffered" — here NBUF-buffered).
// Worker warps 1..W-1 consume the ring in order, claiming 32*UNROLL-edge steps
// of the current batch with a shared-memory atomic; a warp that finds the
// batch exhausted moves on to the next batch at once — no CTA barrier per
// batch.  The last warp to leave a batch increments `processed` (a7; every
// warp's pushes for the batch are reserved before it leaves) and frees the
// buffer.  (The double-buffered version with bar.sync hand-offs spent 20-27%
// of its stall samples in barriers, profiles/r01_*_ncu.md.)
#pragma once
#include "cta_ws.cuh"

namespace atos {

#ifndef ATOS_NBUF
#define ATOS_NBUF 4
#endif
constexpr int NBUF = ATOS_NBUF;
// Queue-agent warps per CTA, per app (App::kAgents, default 1): agent a
// prepares ring batches i = a, a + A, ... (buffer i % NBUF); workers consume
// every batch in order and skip the batches of an agent that has published
// QUIT.  PageRank runs two agents per 1,024-thread CTA: with one, the agent
// was busy the whole run and the 31 worker warps waited for it 30% of their
// cycles (profiles/r02_wait_prof.md); two measured -3.7% on RMAT-24
// (profiles/r02_agents.md).  BFS keeps one (two: +20% at 256 threads).
template <class A, class = void>
struct AgentsTrait : std::integral_constant<int, 1> {};
template <class A>
struct AgentsTrait<A, std::void_t<decltype(A::kAgents)>> : std::integral_constant<int, A::kAgents> {};
constexpr int STEP_CAP = 512;
// A prepared batch with at most this many edges is expanded by the queue agent
// itself (0 = off; must be <= STEP_EDGES: one LBS step).
#ifndef ATOS_AGENT_FAST
#define ATOS_AGENT_FAST 0
#endif  // per-buffer step-owner table (u16; steps beyond it binary-search)
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
constexpr int64_t AGENT_FAST_EDGES = ATOS_AGENT_FAST;
static_assert(AGENT_FAST_EDGES <= STEP_EDGES, "ATOS_AGENT_FAST must fit one LBS step");
// Column staging: item i of a batch is staged at element offset
// roundup4(pre[i] + STAGE_PAD * i) of the buffer's stage area, covering its
// 16-B aligned superset [e0 & ~3, roundup4(e1)) (at most 6 extra elements), so
// slots never overlap and need no second scan; an item is staged iff its slot
// ends within the stage capacity (so the staged items are a prefix).
constexpr int STAGE_PAD = 10;
enum : int { BUF_FREE = 0, BUF_READY = 1, BUF_QUIT = 2 };

// ATOS_WAIT_PROF builds (tuning experiments only) accumulate clock64 cycles per
// phase into ctl->prof: 0 agent waits for a free buffer, 1 agent pop, 2 agent
// prepare + scan + staging issue, 3 workers wait for a ready buffer (and its
// staged columns), 4 workers in steps, 5 worker batch exits.
#ifdef ATOS_WAIT_PROF
#define WPROF_DECL long long wp_t = clock64(); unsigned long long wp_acc[6] = {0, 0, 0, 0, 0, 0};
#define WPROF_MARK(i) do { const long long wp_n = clock64(); wp_acc[i] += (unsigned long long)(wp_n - wp_t); wp_t = wp_n; } while (0)
#define WPROF_FLUSH(q) do { if (lane_id() == 0) for (int wp_i = 0; wp_i < 6; ++wp_i) if (wp_acc[wp_i]) atomicAdd(reinterpret_cast<unsigned long long*>(&(q).ctl->prof[wp_i].v), wp_acc[wp_i]); } while (0)
#else
#define WPROF_DECL
#define WPROF_MARK(i) do {} while (0)
#define WPROF_FLUSH(q) do {} while (0)
#endif

struct BufHdr {
  int state;     // BUF_*
  int seq;       // ring pass this batch belongs to (a fast warp must not re-enter an older batch)
  int n;         // items
  int next;      // next step index to claim
  int left;      // warps that have left this batch
  int pad;
  long long total;
};

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
// Per-buffer layout: e0 (F x i64) | pre ((F+1) x i64) | payload (F) |
// own (STEP_CAP x u16) | sofs (F x i32) | stage (S x i32, 16-B aligned).
template <class Payload>
__host__ __device__ constexpr size_t ws2_sofs_offset(int F) {
  return align16(ws_buf_bytes<Payload>(F) + (size_t)STEP_CAP * 2);
}
template <class Payload>
__host__ __device__ constexpr size_t ws2_stage_offset(int F) {
  return ws2_sofs_offset<Payload>(F) + align16((size_t)F * 4);
}
template <class Payload>
__host__ __device__ constexpr size_t ws2_buf_bytes(int F, int S) {
  return ws2_stage_offset<Payload>(F) + (size_t)S * 4;
}
template <class Payload>
__host__ __device__ constexpr size_t ws2_smem_bytes(int F, int S) {
  // buffers + headers + one mbarrier per buffer
  return (size_t)NBUF * ws2_buf_bytes<Payload>(F, S) + NBUF * sizeof(BufHdr) + NBUF * 8;
}

__device__ __forceinline__ int vload(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ void vstore(int* p, int v) { *(volatile int*)p = v; }

// Agent pop from the global queue; the idle path runs the termination check
// (a7) — for apps with sweep-activated hubs (R35) quiescence must also pass a
// clean hub sweep.
constexpr uint32_t AGENT_SKIP = 0xFFFFFFFFu;
// With several agents per CTA the workers consume batches in ring order, so an
// agent that finds the queue empty (but the run not quiescent) must not wait
// for work: its ring slot may be the one the workers wait on while another
// agent's claimed batch (whose pushes would feed it) sits behind it.  It
// publishes an empty batch instead (AGENT_SKIP) and moves on.
template <class App, bool kSkip = true>
__device__ __forceinline__ uint32_t agent_pop(const App& app, const Queue& q, uint32_t want, uint64_t& first,
                                              uint64_t& hw, long long& last_count) {
  const int lane = lane_id();
  unsigned ns = 0;
  for (;;) {
    // abort / watchdog are checked on the idle path only
    uint32_t n = 0;
    uint64_t qlen = 0, t = 0;
    bool quit = false, quiescent = false;
    if (lane == 0) {
      n = q_try_pop(q, want, first, qlen, last_count);
      last_count = (long long)qlen - (long long)n;
      if (n) {
        if (qlen > hw) hw = qlen;
      } else if (q_aborted(q) || q_timed_out(q)) {
        quit = true;
      } else {
        const uint64_t p = ld_acquire_u64(&q.ctl->processed.v);
        t = q_enqueued(q);
        quiescent = p == t;
      }
    }
    n = __shfl_sync(FULL_MASK, n, 0);
    first = __shfl_sync(FULL_MASK, first, 0);
    if (n) return n;
    if (__shfl_sync(FULL_MASK, quit, 0)) return 0;
    if (__shfl_sync(FULL_MASK, quiescent, 0)) {
      if constexpr (HubSweepTrait<App>::value) {
        const int r = hub_final_sweep(app, q, __shfl_sync(FULL_MASK, t, 0));
        if (r == 2) return 0;
        if (r == 1) { ns = 0; continue; }
      } else {
        return 0;
      }
    } else if (kSkip && AgentsTrait<App>::value > 1) {
      return AGENT_SKIP;
    }
    if (ns) __nanosleep(ns);
    ns = ns == 0 ? 32 : (ns < q.backoff_ns ? ns * 2 : ns);
  }
}

// Agent: stage the column lists of the batch's leading items into `stage`
// (capacity S elements) with one TMA bulk copy per item, all completing on
// `bar`; sofs[i] = stage offset of item i's first edge, or -1 (the workers
// read it from global memory).  Exactly one arrival per batch, so the
// barrier's k-th phase completes with the k-th use of the buffer.
__device__ __forceinline__ void agent_stage(const GraphView& g, uint32_t n, const int64_t* e0s, const int64_t* pre,
                                            int* sofs, int32_t* stage, uint32_t S, uint64_t* bar) {
  const uint32_t lane = lane_id();
  uint32_t bytes = 0;
  for (uint32_t it = lane; it < n; it += 32) {
    const int64_t deg = pre[it + 1] - pre[it];
    const int64_t a = e0s[it];
    const int64_t as = a & ~(int64_t)3, ae = (a + deg + 3) & ~(int64_t)3;
    const bool st = deg > 0 && pre[it + 1] + (int64_t)STAGE_PAD * (it + 1) <= (int64_t)S && ae <= g.col_cap;
    const int64_t slot = (pre[it] + (int64_t)STAGE_PAD * it + 3) & ~(int64_t)3;
    sofs[it] = st ? (int)(slot + (a - as)) : -1;
    if (st) bytes += (uint32_t)(ae - as) * 4u;
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) bytes += __shfl_xor_sync(FULL_MASK, bytes, d);
  if (lane == 0) {
    fence_proxy_async_smem();  // order the workers' reads of the buffer's last batch before the async writes
    mbar_arrive_expect_tx(bar, bytes);
  }
  __syncwarp();
  if (bytes == 0) return;
  for (uint32_t it = lane; it < n; it += 32) {
    const int o = sofs[it];
    if (o < 0) continue;
    const int64_t a = e0s[it], deg = pre[it + 1] - pre[it];
    const int64_t as = a & ~(int64_t)3, ae = (a + deg + 3) & ~(int64_t)3;
    tma_load_1d(stage + (o - (int)(a - as)), g.col + as, (uint32_t)(ae - as) * 4u, bar);
  }
}

template <class App>
__device__ void cta_ws2_persistent(const App& app, const GraphView& g, const Queue& q, int F, unsigned char* smem,
                                   LocalStats& st) {
  using Payload = typename App::Payload;
  constexpr int AGENTS = AgentsTrait<App>::value;
  static_assert(NBUF % AGENTS == 0, "NBUF must be a multiple of the agents per CTA");
  const int T = blockDim.x, tid = threadIdx.x, wid = tid >> 5, lane = lane_id();
  const uint32_t S = q.stage_cap;
  const size_t bb = ws2_buf_bytes<Payload>(F, (int)S);
  BufHdr* hdr = reinterpret_cast<BufHdr*>(smem + NBUF * bb);
  uint64_t* bars = reinterpret_cast<uint64_t*>(hdr + NBUF);
  auto buf_own = [&](int b) { return reinterpret_cast<uint16_t*>(smem + b * bb + ws_buf_bytes<Payload>(F)); };
  auto buf_e0 = [&](int b) { return reinterpret_cast<int64_t*>(smem + b * bb); };
  auto buf_pre = [&](int b) { return reinterpret_cast<int64_t*>(smem + b * bb) + F; };
  auto buf_pay = [&](int b) { return reinterpret_cast<Payload*>(reinterpret_cast<int64_t*>(smem + b * bb) + 2 * F + 1); };
  auto buf_sofs = [&](int b) { return reinterpret_cast<int*>(smem + b * bb + ws2_sofs_offset<Payload>(F)); };
  auto buf_stage = [&](int b) { return reinterpret_cast<int32_t*>(smem + b * bb + ws2_stage_offset<Payload>(F)); };
  const Queue* cq = q.chunks ? &q : nullptr;
  const int nw = (T >> 5) - AGENTS;
  if (tid < NBUF) {
    hdr[tid] = BufHdr{BUF_FREE, -1, 0, 0, 0, 0, 0};
    if (S) mbar_init(&bars[tid], 1);
  }
  if (S && tid == 0) fence_mbar_init();
  __syncthreads();

  if (wid < AGENTS) {
    // ------------------------------------------------ queue agent(s)
    long long last_count = 0;  // lane 0: queue length seen at the last pop
    WPROF_DECL
    for (int i = wid;;) {
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
      WPROF_MARK(0);
      uint64_t first = 0;
      uint32_t n = 0;
      if constexpr (App::kWindow) {
        n = window_pop(app, q, (uint32_t)F, first, st.hw);
      } else {
        n = agent_pop(app, q, (uint32_t)F, first, st.hw, last_count);
      }
      const bool skip = n == AGENT_SKIP;
      if (skip) {
        n = 0;
        // an empty batch still completes its buffer's staging phase (workers wait on it)
        if (S) agent_stage(g, 0u, buf_e0(b), buf_pre(b), buf_sofs(b), buf_stage(b), S, &bars[b]);
      }
      WPROF_MARK(1);
      if (n) {
        const uint32_t dfr = agent_prepare(app, g, q, cq, first, n, buf_e0(b), buf_pre(b), buf_pay(b));
        if (lane == 0) st.pushed += dfr;
        int64_t* pre = buf_pre(b);
        warp_exclusive_scan(pre, (int)n);
        if constexpr (AGENT_FAST_EDGES > 0 && !App::kWindow) {
          // Small batch (high-diameter frontiers): the agent expands it itself —
          // one LBS step, no hand-off to the workers — and keeps ring index i
          // (buffer b was never published, so it is still free).
          const int64_t total = pre[n];
          if (S == 0 && total <= (int64_t)AGENT_FAST_EDGES) {
            RingSink sink{q};
            uint32_t p = total ? lbs_step<App, RingSink, WS_UNROLL>(app, g, sink, pre, buf_e0(b), buf_pay(b),
                                                                    (int)n, total, 0) : 0u;
            if constexpr (HubSweepTrait<App>::value) p += hub_sweep(app, q);  // R35, before q_done
            if (lane == 0) {
              st.pushed += p;
              st.edges += (uint64_t)total;
              st.popped += n;
              q_done(q, n);
              q_trace(q, n, (uint64_t)total);
            }
            __syncwarp();
            continue;
          }
        }
        if (S) agent_stage(g, n, buf_e0(b), pre, buf_sofs(b), buf_stage(b), S, &bars[b]);
        // step-owner table: own[c] = item holding flattened edge c*STEP_EDGES
        uint16_t* own = buf_own(b);
        for (uint32_t it = lane; it < n; it += 32) {
          const int64_t c0 = (pre[it] + STEP_EDGES - 1) / STEP_EDGES;
          const int64_t c1 = min((pre[it + 1] + STEP_EDGES - 1) / STEP_EDGES, (int64_t)STEP_CAP);
          for (int64_t c = c0; c < c1; ++c) own[c] = (uint16_t)it;
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
        vstore(&hdr[b].state, n || skip ? BUF_READY : BUF_QUIT);
      }
      __syncwarp();
      WPROF_MARK(2);
      if (n == 0 && !skip) break;
      if (skip) __nanosleep(256);
      i += AGENTS;
    }
    WPROF_FLUSH(q);
  } else {
    // ------------------------------------------------ edge workers
    RingSink sink{q};
    uint32_t pushed = 0;
    uint64_t edges = 0;
    unsigned quit_mask = 0;  // agents that have published QUIT
    WPROF_DECL
    for (int i = 0;; ++i) {
      const int b = i % NBUF, pass = i / NBUF;
      if ((quit_mask >> (i % AGENTS)) & 1u) continue;
      int s = BUF_FREE;
      for (unsigned ns = 8;; ns = ns < 128 ? ns * 2 : ns) {
        s = vload(&hdr[b].state);
        if (s != BUF_FREE && vload(&hdr[b].seq) == pass) break;
        __nanosleep(ns);
        if (ns >= 128 && (q_aborted(q) || q_timed_out(q))) { s = BUF_QUIT; quit_mask = (1u << AGENTS) - 1; break; }
      }
      if (s == BUF_QUIT) {
        quit_mask |= 1u << (i % AGENTS);
        if (quit_mask == (1u << AGENTS) - 1) break;
        continue;
      }
      __threadfence_block();
      // this batch's staged columns complete the buffer's pass-th mbarrier phase
      if (S) {
        bool dead = false;
        for (unsigned ns = 8; !mbar_try_wait(&bars[b], (uint32_t)pass & 1u); ns = ns < 128 ? ns * 2 : ns) {
          __nanosleep(ns);
          if (ns >= 128 && (q_aborted(q) || q_timed_out(q))) { dead = true; break; }
        }
        if (dead) break;
      }
      WPROF_MARK(3);
      const int n = hdr[b].n;
      const int64_t total = hdr[b].total;
      const int64_t* pre = buf_pre(b);
      const int64_t* e0 = buf_e0(b);
      const Payload* pay = buf_pay(b);
      const uint16_t* own = buf_own(b);
      const int* sofs = S ? buf_sofs(b) : nullptr;
      const int32_t* stage = buf_stage(b);
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
        const uint32_t p = lbs_step<App, RingSink, WS_UNROLL>(app, g, sink, pre, e0, pay, n, total,
                                                               (int64_t)c * STEP_EDGES, hlo, hhi, sofs, stage);
        if (lane == 0) pushed += p;
        if (lane == 0) edges += (uint64_t)min(STEP_EDGES, total - (int64_t)c * STEP_EDGES);
      }
      if constexpr (App::kWindow) {
        // Alg. 4 lines 11-14: each popped vertex checks a Check_Size window
        pushed += window_sweep(app, q, ((uint32_t)n * (uint32_t)app.check_size + nw - 1) / nw);
      }
      __syncwarp();
      WPROF_MARK(4);
      int last = 0;
      if (lane == 0) {
        __threadfence_block();
        last = atomicAdd(&hdr[b].left, 1) == nw - 1;
      }
      last = __shfl_sync(FULL_MASK, last, 0);
      if constexpr (HubSweepTrait<App>::value) {
        if (last) pushed += hub_sweep(app, q);  // R35, before this batch's q_done
      }
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
      WPROF_MARK(5);
    }
    WPROF_FLUSH(q);
    if (lane == 0) {
      st.pushed += pushed;
      st.edges += edges;
    }
  }
}

}  // namespace atos
