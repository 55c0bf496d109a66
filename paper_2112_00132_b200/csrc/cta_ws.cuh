// cta_ws.cuh — queue-agent helpers of the persistent CTA worker (SURVEY §8a
// rows a4 + a5): batch preparation (slot reads, begin loads/atomics, hub
// splitting) phased for memory-level parallelism, the warp scan, and the
// Check_Size window activation of Alg. 4 (row f1).  The worker itself is in
// cta_ws2.cuh.
#pragma once
#include <type_traits>

#include "engine.cuh"

namespace atos {


template <class Payload>
__host__ __device__ constexpr size_t ws_buf_bytes(int F) {
  return (size_t)F * 8 + ((size_t)F + 1) * 8 + (((size_t)F * sizeof(Payload) + 15) & ~(size_t)15);
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

// Queue agent: turn the claimed positions [first, first+n) into a prepared
// batch (e0 / degree / payload per item).  Items are handled AGENT_G per lane
// at a time in phases — slot loads, then every item's begin loads, then every
// item's begin atomics — so ~3 L2 round trips cover 32*AGENT_G items instead
// of ~3 per item (the agent warp was the bottleneck on low-degree frontiers).
// AGENT_G sweep on RMAT-24 (tools/gpu_jobs/agentg.sh, 3 alternating reps):
// PageRank 166.6 / 164.4 / 166.6 / 175.0 ms and BFS 3.51 / 3.46 / 3.48 / 3.63 ms
// at AGENT_G 4 / 2 / 1 / 8 — two items per lane per phase is the best balance
// of in-flight L2 requests and agent registers.
#ifndef ATOS_AGENT_G
#define ATOS_AGENT_G 2
#endif
constexpr int AGENT_G = ATOS_AGENT_G;
// Phase 0 (slot reads) holds one u64 per item, so it takes more items per L2
// round trip than the later phases.
#ifndef ATOS_AGENT_SLOT_G
#define ATOS_AGENT_SLOT_G 2
#endif
constexpr int AGENT_SLOT_G = ATOS_AGENT_SLOT_G;

// Apps that may defer a popped task (PageRank hub deferral, R31) declare kDefer.
template <class A, class = void>
struct DeferTrait : std::false_type {};
template <class A>
struct DeferTrait<A, std::void_t<decltype(A::kDefer)>> : std::integral_constant<bool, A::kDefer> {};

// Apps with sweep-activated hubs (PageRank R35) declare kHubSweep.
template <class A, class = void>
struct HubSweepTrait : std::false_type {};
template <class A>
struct HubSweepTrait<A, std::void_t<decltype(A::kHubSweep)>> : std::integral_constant<bool, A::kHubSweep> {};

// R35 sweep step (warp-collective; the warp that closes a batch, before its
// q_done, so the pushes are reserved while the batch still counts as
// unprocessed — a7): check app.hub_check hubs from the round-robin cursor
// ctl->aux[0] and push those whose fp64 residue exceeds eps and that are not
// queued (hq 0 -> 1).  Returns the pushes (warp-uniform).
template <class App>
__device__ __forceinline__ uint32_t hub_sweep(const App& app, const Queue& q) {
  uint64_t s = 0;
  if (lane_id() == 0)
    s = atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->aux[0].v), (unsigned long long)app.hub_check);
  s = __shfl_sync(FULL_MASK, s, 0);
  uint32_t pushed = 0;
  for (uint32_t i = 0; i < app.hub_check; i += 32 * AGENT_G) {
    uint32_t v[AGENT_G];
    double r[AGENT_G];
#pragma unroll
    for (int k = 0; k < AGENT_G; ++k) {
      const uint32_t j = i + lane_id() + 32 * k;
      v[k] = j < app.hub_check ? __ldg(app.hubs + (uint32_t)((s + j) % app.num_hubs)) : 0xFFFFFFFFu;
      r[k] = v[k] != 0xFFFFFFFFu ? app.rs.hub_read(v[k]) : 0.0;
    }
    bool act[AGENT_G];
#pragma unroll
    for (int k = 0; k < AGENT_G; ++k)
      act[k] = r[k] > (double)app.eps && ld_relaxed_u32(app.hq + v[k]) == 0u && atomicExch(app.hq + v[k], 1u) == 0u;
    pushed += q_warp_push_multi<AGENT_G>(q, act, v);
  }
  return pushed;
}

// R35 termination (R9's clean-sweep protocol over the hubs): called by an
// idle agent warp that saw the queue quiescent (processed == tail == t0).
// One warp at a time (lock ctl->aux[3]: 0 free, 1 sweeping, 2 done) checks
// EVERY hub and pushes each with residue > eps (flags are ignored: with the
// queue quiescent no copy is queued).  Returns 2 = the run is over (a clean
// sweep with the queue unchanged), 1 = it pushed or the queue moved (keep
// popping), 0 = another warp holds the lock (poll again).
template <class App>
__device__ __forceinline__ int hub_final_sweep(const App& app, const Queue& q, uint64_t t0) {
  int state = 0;
  if (lane_id() == 0) {
    const uint64_t flag = ld_relaxed_u64(&q.ctl->aux[3].v);
    if (flag == 2) state = 2;
    else if (atomicCAS(reinterpret_cast<unsigned long long*>(&q.ctl->aux[3].v), 0ull, 1ull) == 0ull) state = 1;
  }
  state = __shfl_sync(FULL_MASK, state, 0);
  if (state != 1) return state;
  uint32_t found = 0;
  for (uint32_t b = 0; b < app.num_hubs; b += 32 * AGENT_G) {
    uint32_t v[AGENT_G];
    double r[AGENT_G];
#pragma unroll
    for (int k = 0; k < AGENT_G; ++k) {
      const uint32_t j = b + lane_id() + 32 * k;
      v[k] = j < app.num_hubs ? __ldg(app.hubs + j) : 0xFFFFFFFFu;
      r[k] = v[k] != 0xFFFFFFFFu ? app.rs.hub_read(v[k]) : 0.0;
    }
    bool act[AGENT_G];
#pragma unroll
    for (int k = 0; k < AGENT_G; ++k) {
      act[k] = r[k] > (double)app.eps;
      if (act[k]) atomicExch(app.hq + v[k], 1u);
    }
    found += q_warp_push_multi<AGENT_G>(q, act, v);
  }
  bool done = false;
  if (lane_id() == 0) {
    __threadfence();
    const uint64_t p = ld_acquire_u64(&q.ctl->processed.v);
    const uint64_t t = q_enqueued(q);
    done = found == 0 && p == t && t == t0;
    st_relaxed_u64(&q.ctl->aux[3].v, done ? 2ull : 0ull);
  }
  return __shfl_sync(FULL_MASK, done, 0) ? 2 : 1;
}

// Per-item state of a batch between the agent's phases, kept in pre[i]:
// a vertex item (>= 0, may carry DEFER_BIT), a resolved chunk task
// (-2 - edges), an item lost to an abort (-1), or not yet read (PENDING).
constexpr int64_t STASH_PENDING = -0x7fffffffffffffffLL - 1;
constexpr int64_t STASH_INVALID = -1;

// Take the item of claimed position pos from its slot word `raw` if it is
// full.  A chunk task is resolved on the spot — its table entry is read while
// the slot is still held, then the slot is released with st.release (device.cuh,
// Chunk) — a vertex item is stashed and its slot released.  Returns false if
// the slot is not published yet.
template <class App>
__device__ __forceinline__ bool agent_take(const App& app, const Queue& q, uint64_t pos, uint64_t raw, uint32_t i,
                                           int64_t* e0s, int64_t* pre, typename App::Payload* pay) {
  const uint32_t want = 2u * (uint32_t)(pos >> q.log2cap) + 1u;
  if ((uint32_t)(raw >> 32) != want) return false;
  const uint32_t it = (uint32_t)raw;
  if (q.chunks && (it & CHUNK_BIT)) {
    int64_t a = 0, z = 0;
    typename App::Payload p{};
    const bool cur = read_chunk(app, q, pos, a, z, p);
    e0s[i] = a;
    pay[i] = p;
    pre[i] = -2 - (cur ? z - a : 0);
    q_release_slot_ordered(q, pos);
  } else {
    pre[i] = (int64_t)it;
    q_release_slot(q, pos);
  }
  return true;
}

// Returns the tasks the agent re-pushed (deferred, R31; warp-uniform).
template <class App>
__device__ __forceinline__ uint32_t agent_prepare(const App& app, const GraphView& g, const Queue& q, const Queue* cq,
                                                  uint64_t first, uint32_t n, int64_t* e0s, int64_t* pre,
                                                  typename App::Payload* pay) {
  using Payload = typename App::Payload;
  using Pre = typename App::Pre;
  constexpr bool kDefer = DeferTrait<App>::value;
  const uint32_t lane = lane_id();
  uint32_t deferred = 0;
  // phase 0: read and release EVERY claimed slot before this agent pushes
  // anything (hub chunk tasks, deferrals), and never hold a published slot
  // while spinning on an unpublished one (the batch is re-scanned with backoff
  // until every item is in).  So a producer waiting for one of these slots to
  // be released for its next lap (ring wrap-around) never waits on this agent
  // (the agent used to push between sub-rounds of unread claims).
  bool pending = false;
  for (uint32_t base = 0; base < n; base += 32 * AGENT_SLOT_G) {
    uint64_t raw[AGENT_SLOT_G];
#pragma unroll
    for (int k = 0; k < AGENT_SLOT_G; ++k) {
      const uint32_t i = base + lane + 32 * k;
      raw[k] = i < n ? ld_relaxed_u64(q.ring + ((first + i) & q.mask)) : 0;
    }
#pragma unroll
    for (int k = 0; k < AGENT_SLOT_G; ++k) {
      const uint32_t i = base + lane + 32 * k;
      if (i < n && !agent_take(app, q, first + i, raw[k], i, e0s, pre, pay)) {
        pre[i] = STASH_PENDING;
        pending = true;
      }
    }
  }
  for (unsigned ns = 16; __any_sync(FULL_MASK, pending); ns = ns < 256 ? ns * 2 : ns) {
    const bool dead = q_aborted(q) || q_timed_out(q);
    pending = false;
    if (!dead) __nanosleep(ns);
    for (uint32_t i = lane; i < n; i += 32) {
      if (pre[i] != STASH_PENDING) continue;
      if (dead) { pre[i] = STASH_INVALID; continue; }
      if (!agent_take(app, q, first + i, ld_relaxed_u64(q.ring + ((first + i) & q.mask)), i, e0s, pre, pay))
        pending = true;
    }
  }
  __syncwarp();
  for (uint32_t base = 0; base < n; base += 32 * AGENT_G) {
    int64_t sv[AGENT_G];
    uint32_t it[AGENT_G];
#pragma unroll
    for (int k = 0; k < AGENT_G; ++k) {
      const uint32_t i = base + lane + 32 * k;
      sv[k] = i < n ? pre[i] : STASH_INVALID;
      it[k] = sv[k] >= 0 ? (uint32_t)sv[k] : 0xFFFFFFFFu;
    }
    // phase B: begin loads (per-vertex state)
    Pre x[AGENT_G];
    bool was_deferred[AGENT_G];
#pragma unroll
    for (int k = 0; k < AGENT_G; ++k) {
      was_deferred[k] = false;
      if constexpr (kDefer) {
        if (app.defer_deg && it[k] != 0xFFFFFFFFu && (it[k] & DEFER_BIT)) {
          was_deferred[k] = true;
          it[k] &= ~DEFER_BIT;
        }
      }
      if (it[k] != 0xFFFFFFFFu) x[k] = app.begin_load(it[k], g);
    }
    bool dpush[AGENT_G];
    uint32_t ditem[AGENT_G];
#pragma unroll
    for (int k = 0; k < AGENT_G; ++k) {
      dpush[k] = false;
      ditem[k] = 0;
    }
    // phase C: commits and splitting; write the batch
#pragma unroll
    for (int k = 0; k < AGENT_G; ++k) {
      const uint32_t i = base + lane + 32 * k;
      if (i >= n) continue;
      if (sv[k] < STASH_INVALID) {  // chunk task, resolved in phase 0
        pre[i] = -2 - sv[k];
        continue;
      }
      int64_t a = 0, z = 0;
      Payload p{};
      bool ok = false;
      if (it[k] != 0xFFFFFFFFu) {
        a = x[k].e0;
        z = x[k].e1;
        bool held = false;
        if constexpr (kDefer) {
          if (!was_deferred[k] && app.should_defer(x[k])) {
            held = true;  // residue put back; re-pushed with DEFER_BIT unless another copy exists
            dpush[k] = app.put_back(it[k], x[k]);
            ditem[k] = it[k] | DEFER_BIT;
          }
        }
        if (!held) {
          ok = app.begin_commit(it[k], x[k], p);
          if (ok && cq && z - a > SPLIT_DEG) z = split_hub(cq, it[k], a, z, p);
        }
      }
      e0s[i] = a;
      pre[i] = ok ? z - a : 0;
      pay[i] = p;
    }
    if constexpr (kDefer) {
      if (app.defer_deg) deferred += q_warp_push_multi<AGENT_G>(q, dpush, ditem);
    }
  }
  __syncwarp();
  return deferred;
}

// Check_Size window sweep (f1): the warp reserves `span` ids from the global
// cursor and pushes every id with residue > eps that is not already queued.
// Returns the number pushed (warp-uniform).  ctl->aux[0] = cursor,
// aux[1] = cursor position of the last push, aux[2] = cursor at the last
// completed task.
template <class App>
__device__ __forceinline__ uint32_t window_sweep(const App& app, const Queue& q, uint32_t span);

// Warp-collective pop for window activation: try the queue; on a failed pop
// sweep one window (the paper's f2 hook continues the check sweep); quit on a
// clean full sweep with an empty queue (R9).  Per successful pop the warp also
// sweeps n * Check_Size ids (Alg. 4: every popped vertex checks a window).
template <class App>
__device__ __forceinline__ uint32_t window_pop(const App& app, const Queue& q, uint32_t want, uint64_t& first,
                                               uint64_t& hw) {
  unsigned ns = 0;
  for (;;) {
    uint32_t n = 0;
    uint64_t qlen = 0;
    if (lane_id() == 0) {
      n = q_aborted(q) || q_timed_out(q) ? 0xFFFFFFFFu : q_try_pop(q, want, first, qlen);
      if (n && n != 0xFFFFFFFFu && qlen > hw) hw = qlen;
    }
    n = __shfl_sync(FULL_MASK, n, 0);
    first = __shfl_sync(FULL_MASK, first, 0);
    if (n == 0xFFFFFFFFu) return 0;
    if (n) return n;
    if (window_sweep(app, q, 32u * (uint32_t)app.check_size)) {
      ns = 0;
      continue;
    }
    // Termination (R9): with the queue empty, one warp (lock aux[3]: 0 -> 1)
    // sweeps ALL n residues itself; if it finds none > eps and the queue stayed
    // empty and unchanged (no task could run, so residues were stable) the run
    // is over (aux[3] = 2).
    int state = 0;  // 0 = keep going, 1 = sweeper, 2 = quit
    uint64_t t0 = 0;
    if (lane_id() == 0) {
      const uint64_t flag = ld_relaxed_u64(&q.ctl->aux[3].v);
      if (flag == 2) {
        state = 2;
      } else {
        const uint64_t p = ld_acquire_u64(&q.ctl->processed.v);
        t0 = q_enqueued(q);
        if (p == t0 && atomicCAS(reinterpret_cast<unsigned long long*>(&q.ctl->aux[3].v), 0ull, 1ull) == 0ull) state = 1;
      }
    }
    state = __shfl_sync(FULL_MASK, state, 0);
    if (state == 2) return 0;
    if (state == 1) {
      uint32_t found = 0;
      for (int64_t b = 0; b < app.n; b += 32) {
        const int64_t v = b + lane_id();
        bool act = false;
        if (v < app.n) act = app.rs.peek((uint32_t)v) > (double)app.eps && atomicExch(app.queued + v, 1u) == 0u;
        found += q_warp_push(q, act, (uint32_t)v);
      }
      bool done = false;
      if (lane_id() == 0) {
        __threadfence();
        const uint64_t p = ld_acquire_u64(&q.ctl->processed.v);
        const uint64_t t = q_enqueued(q);
        done = found == 0 && p == t && t == t0;
        st_relaxed_u64(&q.ctl->aux[3].v, done ? 2ull : 0ull);
      }
      if (__shfl_sync(FULL_MASK, done, 0)) return 0;
      ns = 0;
      continue;
    }
    if (ns) __nanosleep(ns);
    ns = ns == 0 ? 32 : (ns < 256 ? ns * 2 : ns);
  }
}

template <class App>
__device__ __forceinline__ uint32_t window_sweep(const App& app, const Queue& q, uint32_t span) {
  uint64_t s = 0;
  if (lane_id() == 0) s = atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->aux[0].v), (unsigned long long)span);
  s = __shfl_sync(FULL_MASK, s, 0);
  uint32_t pushed = 0;
  constexpr int G = 8;
  for (uint32_t i = 0; i < span; i += 32 * G) {
    double r[G];
    uint32_t v[G];
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const uint32_t j = i + lane_id() + 32 * k;
      v[k] = (uint32_t)((s + j) % (uint64_t)app.n);
      r[k] = j < span ? app.rs.peek(v[k]) : 0.0;
    }
    bool act[G];
#pragma unroll
    for (int k = 0; k < G; ++k) act[k] = r[k] > (double)app.eps && atomicExch(app.queued + v[k], 1u) == 0u;
    pushed += q_warp_push_multi<G>(q, act, v);
  }
  if (pushed && lane_id() == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(&q.ctl->aux[1].v), (unsigned long long)(s + span));
  return pushed;
}

}  // namespace atos
