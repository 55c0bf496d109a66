// engine.cuh — worker expansion and the edge-map
// applications BFS (a6-BFS) and push PageRank (a6-PR) for sm_100a.
//
// A worker takes a batch of popped vertices and, for each, visits its CSR
// out-edges, applies the app's relaxed update to the neighbour and pushes the
// neighbour if it was activated (Listing 2).  Worker
// sizes:
//   THREAD  one lane per vertex, serial neighbour walk (SIMT cursor loop);
//   WARP    the paper's persist-32: the warp walks one vertex's list
//           at a time, lanes striding with 16-byte int4 loads of col[];
//   CTA     the paper's persist-CTA: block exclusive scan of the
//           batch's degrees, then load-balancing search over the
//           flattened edge range — thread e finds its vertex by binary search
//           of the shared-memory prefix.  Each thread carries UNROLL edges per
//           step so UNROLL col loads and UNROLL atomics are in flight.
// Item sources and push sinks are templates so the same expansion serves the
// persistent and discrete schedulers (ring queue) and the BSP variant
// (frontier arrays).
#pragma once
#include <type_traits>

#include "device.cuh"

namespace atos {

struct GraphView {
  const int64_t* off;
  const int32_t* col;
  int64_t n;
  int64_t col_cap;  // readable elements of col (>= m; TMA staging may read up to 3 past a list's end)
};

// ------------------------------------------------------------------ apps ---

// Speculative BFS relax (Alg. 2): d = current dist[v] (R3);
// per edge: optional read filter, atomicMin(&dist[w], d+1), push iff d+1 < old
// (strict, R2).
#ifndef ATOS_BFS_AGENTS
#define ATOS_BFS_AGENTS 1
#endif
struct BfsApp {
  static constexpr bool kWindow = false;
  static constexpr int kAgents = ATOS_BFS_AGENTS;  // queue agents per persistent CTA (cta_ws2.cuh)
  __device__ __forceinline__ uint32_t item_of(uint32_t w) const { return w; }
  uint32_t* dist;
  // near[v] = min(dist[v], 0xFFFF) as of some moment (stale values are larger,
  // never smaller): a 2-byte mirror of dist that the per-edge filter probes.
  // At 32 MB (RMAT-24) it stays L2-resident where the 64 MB dist array
  // missed 38% of probes into random DRAM sectors (profiles/r01_bfs_*).
  uint16_t* near;
  int filter;
  // R29: bit w set = deg(w) == 0.  A dangling vertex's task expands no edge,
  // so an improvement of dist[w] is final without pushing w.  nullptr = off.
  const uint32_t* sink;
  uint32_t sink_tagged;  // R37: read the column's SINK_TAG instead of the bitmap
  using Payload = uint32_t;
  using Probe = uint32_t;
  // Chunk task of v created with payload nd: still current iff dist[v]+1 == nd.
  // If v improved since, a newer task of v exists and covers every edge.
  __device__ __forceinline__ bool chunk_current(uint32_t v, Payload nd) const { return ld_relaxed_u32(dist + v) + 1u >= nd; }
  // Two-phase edge: all probes of a thread's UNROLL edges are issued before
  // any atomic (memory-level parallelism).  The probe may hit a stale L1 copy
  // (>= the current value): it only lets through atomics that turn out not to
  // improve, never suppresses one that would.
  // Probe = the filter's bound (low 31 bits; 0x7FFFFFFF = none) | the
  // column's SINK tag in bit 31 (R37).
  __device__ __forceinline__ Probe probe(uint32_t w, uint32_t tag) const {
    uint32_t v = 0x7FFFFFFFu;
    if (filter) {
      v = ld_probe_u16(near + w);
      if (v == 0xFFFFu) v = 0x7FFFFFFFu;
    }
    return v | ((tag & TAG_SINK) << 31);
  }
  __device__ __forceinline__ bool commit(Payload nd, uint32_t w, Probe pr) const {
    return decide(nd, w, pr, issue(nd, w, pr));
  }
  // commit split into issue (the atomic) and decide (uses its result), so a
  // thread's UNROLL atomics are all in flight before any result is consumed.
  using Raw = uint32_t;
  __device__ __forceinline__ Raw issue(Payload nd, uint32_t w, Probe pr) const {
    return nd < (pr & 0x7FFFFFFFu) ? atom_min_hot(dist + w, nd) : 0u;
  }
  __device__ __forceinline__ bool decide(Payload nd, uint32_t w, Probe pr, Raw old) const {
    const bool improved = nd < (pr & 0x7FFFFFFFu) && nd < old;
    if (!improved) return false;
    st_u16_hot(near + w, nd < 0xFFFFu ? (uint16_t)nd : (uint16_t)0xFFFFu);
    if (sink == nullptr) return true;
    return sink_tagged ? !(pr >> 31) : !((ld_nc_u32(sink + (w >> 5)) >> (w & 31)) & 1u);
  }
  __device__ __forceinline__ bool begin(uint32_t v, const GraphView& g, int64_t& e0, int64_t& e1,
                                        Payload& p) const {
    Pre x = begin_load(v, g);
    e0 = x.e0;
    e1 = x.e1;
    return begin_commit(v, x, p);
  }
  // begin() in two phases so a queue agent can overlap many items' loads.
  struct Pre {
    int64_t e0, e1;
    uint32_t d;
  };
  __device__ __forceinline__ Pre begin_load(uint32_t v, const GraphView& g) const {
    v = ATOS_CHK(v, (uint32_t)g.n);  // a popped task word
    Pre x;
    x.e0 = ld_nc_s64(g.off + v);
    x.e1 = ld_nc_s64(g.off + v + 1);
    x.d = ld_relaxed_hot(dist + v);
    return x;
  }
  // Expand v at its CURRENT depth d (R3).  No "expanded once per depth"
  // dedupe (R25): its atomicMin on a per-vertex word sat on the queue agent's
  // critical path (one more dependent L2 round trip per batch) and cost more
  // than the duplicate expansions it saved (RMAT-24: 3.5 -> 2.75 ms for +2.5%
  // edge visits, profiles/r02_bfs_variants.md).
  __device__ __forceinline__ bool begin_commit(uint32_t, const Pre& x, Payload& p) const {
    p = x.d + 1u;
    return x.e1 != x.e0;
  }
  __device__ __forceinline__ bool edge(Payload nd, uint32_t w, uint32_t tag) const {
    const Probe pr = probe(w, tag);
    return decide(nd, w, pr, issue(nd, w, pr));
  }
};

#ifndef ATOS_HUB_REPLICAS
#define ATOS_HUB_REPLICAS 4u  // R38: hub-residue replicas (a power of two)
#endif
// PageRank residue storage (R34).  Residues are fp32 (4 B per edge push)
// except at HUB vertices — in-degree >= HUB_IN_DEG, tagged in the CSR at
// graph create (device.cuh HUB_TAG) — whose residues are fp64 in res64.  A
// residue that keeps growing while its vertex waits in the queue rounds away
// the small pushes it receives: each of k adds onto an fp32 sum rounds by at
// most half an ulp, 2^-25 of the sum, and identical pushes (a fan-in hub fed
// by equal-degree chains) round the same way every time — measured 2.3e-4 of
// max x* on a 40,000-way fan-in (above the 1e-4 gate).  A vertex receives at
// most about in-degree adds per queue cycle, so below HUB_IN_DEG = 2048 the
// loss is < 2048 2^-25 = 6.1e-5 of its rank even if every rounding had the
// same sign; at hubs fp64 makes it negligible.  RMAT-24: 12,951 hubs take
// 27% of the edge pushes.  (A TwoSum-compensated fp32 add, tried first,
// cost +40% on RMAT-24; fp64 residues everywhere +10%.)  With R = double
// (atos_config.pr_residue_fp64, untagged graphs) every residue is fp64.
__device__ __forceinline__ float atomic_take(float* p) { return atomicExch(p, 0.0f); }
__device__ __forceinline__ double atomic_take(double* p) {
  return __longlong_as_double((long long)atomicExch(reinterpret_cast<unsigned long long*>(p), 0ull));
}
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ void red_add_hot(float* p, float v) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol_evict_last()));
}
__device__ __forceinline__ void red_add_hot(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol_evict_last()));
}
__device__ __forceinline__ bool test_bit(const uint32_t* bits, uint32_t v) {
  return bits && ((ld_nc_u32(bits + (v >> 5)) >> (v & 31)) & 1u);
}

template <class R>
struct Residues {
  R* res;                // fp32 (or fp64 with R = double) residue per vertex
  double* res64;         // hub residues (R == float on a tagged graph), indexed by vertex id; else nullptr
  const uint32_t* hub;   // bit v = v is a hub (pops); nullptr when res64 is
  // R38: a hub's fp64 residue is the sum of ATOS_HUB_REPLICAS = 4 replicas,
  // res64[k r2 + v] (r2 = n): R35's fire-and-forget hub pushes spread over
  // them by lane, dividing the contention on a hub's L2 line (RMAT-24 target
  // replay at the 2048 threshold: 92.7 -> 118.6 G ops/s,
  // profiles/r02_atomic_trace.md).  Every reader sums them; paths that test a
  // crossing write replica 0 only (the R4 seeding scatter spreads too).
  int64_t r2;
  __device__ __forceinline__ double hub_read(uint32_t v) const {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < (int)ATOS_HUB_REPLICAS; ++k) s += __ldcg(res64 + k * r2 + v);
    return s;
  }
  __device__ __forceinline__ double hub_take(uint32_t v) const {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < (int)ATOS_HUB_REPLICAS; ++k) s += atomic_take(res64 + k * r2 + v);
    return s;
  }
  __device__ __forceinline__ bool is_hub(uint32_t v) const { return res64 && test_bit(hub, v); }
  // Alg. 4 line 7, r = atomicExch(residue[v], 0), in two phases so the hub
  // test never delays the common case: take_issue starts the fp32 exchange
  // and the hub-bitmap load together (a hub's fp32 word is always 0);
  // take_finish adds the fp64 exchange for hubs only.
  struct Take {
    R r;
    uint32_t word;  // hub bitmap word of v (0 without hubs)
  };
  __device__ __forceinline__ Take take_issue(uint32_t v) const {
    Take t;
    t.word = res64 && hub ? ld_nc_u32(hub + (v >> 5)) : 0u;
    t.r = atomic_take(res + v);
    return t;
  }
  __device__ __forceinline__ double take_finish(uint32_t v, const Take& t) const {
    return ((t.word >> (v & 31)) & 1u) ? hub_take(v) + (double)t.r : (double)t.r;
  }
  __device__ __forceinline__ double take(uint32_t v) const { return take_finish(v, take_issue(v)); }
  // residue[w] += c at the storage the column's hub tag names; returns the old value
  __device__ __forceinline__ double add(uint32_t w, uint32_t tag, R c) const {
    if ((tag & TAG_HUB) && res64) return atom_add_hot(res64 + w, (double)c);
    return (double)atom_add_hot(res + w, c);
  }
  __device__ __forceinline__ void add_noret(uint32_t w, uint32_t tag, R c) const {
    if ((tag & TAG_HUB) && res64) red_add_hot(res64 + w, (double)c);
    else red_add_hot(res + w, c);
  }
  // did the add of c that returned `old` cross eps (old <= eps < old + c, in the add's own precision)?
  __device__ __forceinline__ bool crossed(uint32_t tag, double old, R c, R eps) const {
    if ((tag & TAG_HUB) && res64) return old <= (double)eps && old + (double)c > (double)eps;
    return (R)old <= eps && add_rn((R)old, c) > eps;
  }
  __device__ __forceinline__ double peek(uint32_t v) const {  // L2 read (sweeps)
    return is_hub(v) ? hub_read(v) : (double)__ldcg(res + v);
  }
  // put a taken residue back (deferral); returns the old value
  __device__ __forceinline__ double put(uint32_t v, double r) const {
    return is_hub(v) ? atom_add_hot(res64 + v, r) : (double)atom_add_hot(res + v, (R)r);
  }
};

// Push PageRank (Alg. 4 body; dangling R5; activation R6):
// r = atomicExch(res[v], 0); rank[v] += r; c = alpha r / deg(v);
// per edge: old = atomicAdd(res[w], c); push w iff old <= eps < old + c.
// rank accumulates in fp64 (a per-pop cost): a hub receives 10^4+ pops.
#ifndef ATOS_PR_AGENTS
#define ATOS_PR_AGENTS 2
#endif
template <class R, bool HS = false>
struct PrAppT {
  static constexpr bool kWindow = false;
  __device__ __forceinline__ uint32_t item_of(uint32_t w) const { return w; }
  double* rank;
  Residues<R> rs;
  R alpha, eps;
  // Sink deferral (R29): bit w set = deg(w) == 0.  A dangling vertex's task is
  // `rank += exch(res)` with no effect on any other vertex, so its activation
  // push is skipped and k_pr_absorb_sinks applies it once after quiescence.
  // nullptr = off (every crossing is pushed, Alg. 4 literally).
  const uint32_t* sink;
  // R37: the columns carry SINK_TAG (library-owned CSR), so the test reads
  // the tag instead of the bitmap; 0 with sink == nullptr or an untagged CSR.
  uint32_t sink_tagged;
  // Hub deferral (R31, persistent CTA workers): a popped vertex with at least
  // defer_deg out-edges whose residue is below defer_res (a few eps) is not
  // expanded yet — its residue goes back and it is re-queued once (DEFER_BIT),
  // so it comes back with the residue accumulated over a second queue cycle
  // instead of scattering an eps-sized residue over thousands of edges.
  static constexpr bool kDefer = true;
  static constexpr bool kHubSweep = HS;
  static constexpr int kAgents = ATOS_PR_AGENTS;  // queue agents per persistent CTA (cta_ws2.cuh)
  uint32_t defer_deg;  // 0 = off
  R defer_res;
  // Sweep activation of hubs (R35, persistent CTA workers; HS = true):
  // an edge push to a hub target (column HUB_TAG) is a fire-and-forget fp64
  // `red` with no threshold test, and hubs are activated instead by sweeps —
  // the worker warp that closes a batch checks hub_check hubs of `hubs` (a
  // round-robin cursor) and pushes those with residue > eps not already
  // queued (hq[v] = 1 while a copy is queued; cleared at pop).  With the queue
  // quiescent one warp sweeps every hub (hub_final_sweep) and the run ends
  // only after a clean sweep (R9's protocol over the hubs alone).
  const uint32_t* hubs;
  uint32_t num_hubs;
  uint32_t hub_check;
  uint32_t* hq;
  using Payload = R;
  using Probe = uint32_t;  // the column's hub tag
  using Raw = double;
  struct Pre {
    int64_t e0, e1;
    typename Residues<R>::Take t;
  };
  __device__ __forceinline__ bool begin(uint32_t v, const GraphView& g, int64_t& e0, int64_t& e1,
                                        Payload& p) const {
    Pre x = begin_load(v, g);
    e0 = x.e0;
    e1 = x.e1;
    return begin_commit(v, x, p);
  }
  // (deferral only inspects the fp32 part: a hub is never deferred)
  __device__ __forceinline__ bool should_defer(const Pre& x) const {
    return defer_deg && x.e1 - x.e0 >= (int64_t)defer_deg && x.t.word == 0u && x.t.r < defer_res && x.t.r > R(0);
  }
  // Put the taken residue back.  If it was <= eps just before (nobody re-pushed
  // v since our take), the caller re-queues v; otherwise a copy is queued already.
  __device__ __forceinline__ bool put_back(uint32_t v, const Pre& x) const { return rs.put(v, (double)x.t.r) <= (double)eps; }
  // the residue exchange is issued in the load phase (its result is only used in commit)
  __device__ __forceinline__ Pre begin_load(uint32_t v, const GraphView& g) const {
    v = ATOS_CHK(v, (uint32_t)g.n);  // a popped task word
    Pre x;
    x.e0 = ld_nc_s64(g.off + v);
    x.e1 = ld_nc_s64(g.off + v + 1);
    x.t = rs.take_issue(v);
    return x;
  }
  __device__ __forceinline__ bool begin_commit(uint32_t v, const Pre& x, Payload& p) const {
    // R35: a popped hub is no longer queued; a sweep may re-queue it as soon as
    // its residue exceeds eps again (an extra copy only pops a small residue)
    if constexpr (HS) {
      if ((x.t.word >> (v & 31)) & 1u) atomicExch(hq + v, 0u);
    }
    const double r = rs.take_finish(v, x.t);
    if (r == 0.0) return false;
    red_add_cold(rank + v, r);
    if (x.e1 == x.e0) return false;
    p = std::is_same<R, float>::value && x.t.word == 0u ? alpha * x.t.r / (R)(x.e1 - x.e0)
                                                         : (R)((double)alpha * r / (double)(x.e1 - x.e0));
    return true;
  }
  __device__ __forceinline__ Probe probe(uint32_t, uint32_t tag) const { return tag; }
  __device__ __forceinline__ Raw issue(Payload c, uint32_t w, Probe tag) const {
    if constexpr (HS) {
      if (tag & TAG_HUB) {  // R35: hub target, activated by sweeps
        red_add_hot(rs.res64 + (lane_id() & (ATOS_HUB_REPLICAS - 1u)) * rs.r2 + w, (double)c);  // R38 replica by lane
        return 0.0;
      }
    }
    return rs.add(w, tag, c);
  }
  __device__ __forceinline__ bool decide(Payload c, uint32_t w, Probe tag, Raw old) const {
    if constexpr (HS) {
      if (tag & TAG_HUB) return false;
    }
    if (!rs.crossed(tag, old, c, eps)) return false;
    if (sink == nullptr) return true;  // sink deferral off: push every crossing
    return sink_tagged ? !(tag & TAG_SINK) : !test_bit(sink, w);
  }
  __device__ __forceinline__ bool commit(Payload c, uint32_t w, Probe tag) const { return decide(c, w, tag, issue(c, w, tag)); }
  __device__ __forceinline__ bool edge(Payload c, uint32_t w, uint32_t tag) const { return commit(c, w, tag); }
  __device__ __forceinline__ bool chunk_current(uint32_t, Payload) const { return true; }
};

// Asynchronous PageRank with the paper's own activation rule (Alg. 4 lines
// 11-14): residue adds are fire-and-forget
// (`red`, no threshold test per edge) and vertices are (re)activated by a
// sweeping window — each worker reserves Check_Size ids from a global cursor
// (atomicAdd(check, Check_Size)) and pushes those with residue > eps (R6/R7,
// check_id mod n).  queued[v] keeps a vertex in the queue at most once (set on
// push, cleared at pop before the residue exchange).  Termination (R9): the
// queue is empty AND the cursor has swept n ids since the last push and the
// last completed task — a clean full sweep over unchanging residues.
template <class R>
struct PrWindowAppT {
  static constexpr bool kWindow = true;
  double* rank;
  Residues<R> rs;
  uint32_t* queued;
  R alpha, eps;
  int64_t n;
  int check_size;
  using Payload = R;
  using Probe = uint32_t;
  using Raw = int;
  __device__ __forceinline__ uint32_t item_of(uint32_t w) const { return w; }
  __device__ __forceinline__ bool chunk_current(uint32_t, Payload) const { return true; }
  struct Pre {
    int64_t e0, e1;
    typename Residues<R>::Take t;
  };
  __device__ __forceinline__ Pre begin_load(uint32_t v, const GraphView& g) const {
    v = ATOS_CHK(v, (uint32_t)g.n);  // a popped task word
    Pre x;
    x.e0 = ld_nc_s64(g.off + v);
    x.e1 = ld_nc_s64(g.off + v + 1);
    atomicExch(queued + v, 0u);  // a later sweep may re-queue v
    x.t = rs.take_issue(v);
    return x;
  }
  __device__ __forceinline__ bool begin_commit(uint32_t v, const Pre& x, Payload& p) const {
    const double r = rs.take_finish(v, x.t);
    if (r == 0.0) return false;
    red_add_cold(rank + v, r);
    if (x.e1 == x.e0) return false;
    p = (R)((double)alpha * r / (double)(x.e1 - x.e0));
    return true;
  }
  __device__ __forceinline__ bool begin(uint32_t v, const GraphView& g, int64_t& e0, int64_t& e1, Payload& p) const {
    Pre x = begin_load(v, g);
    e0 = x.e0;
    e1 = x.e1;
    return begin_commit(v, x, p);
  }
  __device__ __forceinline__ Probe probe(uint32_t, uint32_t tag) const { return tag; }
  __device__ __forceinline__ Raw issue(Payload c, uint32_t w, Probe tag) const {
    rs.add_noret(w, tag, c);
    return 0;
  }
  __device__ __forceinline__ bool decide(Payload, uint32_t, Probe, Raw) const { return false; }
  __device__ __forceinline__ bool commit(Payload c, uint32_t w, Probe p) const { return decide(c, w, p, issue(c, w, p)); }
  __device__ __forceinline__ bool edge(Payload c, uint32_t w, uint32_t tag) const { return commit(c, w, tag); }
};

// BSP PageRank push kernel body (Alg. 3 lines 11-16): same push
// but the frontier is rebuilt by the filter kernel, so nothing is appended
// and the adds need no returned value.
template <class R>
struct PrBspAppT {
  static constexpr bool kWindow = false;
  __device__ __forceinline__ uint32_t item_of(uint32_t w) const { return w; }
  PrAppT<R> base;
  using Payload = R;
  __device__ __forceinline__ bool begin(uint32_t v, const GraphView& g, int64_t& e0, int64_t& e1,
                                        Payload& p) const {
    return base.begin(v, g, e0, e1, p);
  }
  using Probe = uint32_t;
  using Raw = int;
  __device__ __forceinline__ Probe probe(uint32_t, uint32_t tag) const { return tag; }
  __device__ __forceinline__ Raw issue(Payload c, uint32_t w, Probe tag) const {
    base.rs.add_noret(w, tag, c);
    return 0;
  }
  __device__ __forceinline__ bool decide(Payload, uint32_t, Probe, Raw) const { return false; }
  __device__ __forceinline__ bool commit(Payload c, uint32_t w, Probe tag) const { return decide(c, w, tag, issue(c, w, tag)); }
  __device__ __forceinline__ bool edge(Payload c, uint32_t w, uint32_t tag) const { return commit(c, w, tag); }
  __device__ __forceinline__ bool chunk_current(uint32_t, Payload) const { return true; }
};

// ------------------------------------------------------- sources / sinks ---

struct RingSrc {
  Queue q;
  uint64_t first;
  __device__ __forceinline__ bool get(uint32_t i, uint32_t& item) const { return q_load_slot(q, first + i, item); }
};
struct ArraySrc {
  const uint32_t* a;
  __device__ __forceinline__ bool get(uint32_t i, uint32_t& item) const {
    item = a[i];
    return true;
  }
};

struct RingSink {
  Queue q;
  template <int U>
  __device__ __forceinline__ uint32_t warp_push_multi(const bool (&pred)[U], const uint32_t (&item)[U]) const {
    return q_warp_push_multi<U>(q, pred, item);
  }
  __device__ __forceinline__ uint32_t warp_push(bool pred, uint32_t item) const { return q_warp_push(q, pred, item); }
  __device__ __forceinline__ uint32_t active_push(bool pred, uint32_t item) const { return q_active_push(q, pred, item); }
};
// BSP out-frontier: warp-aggregated append to out[count++].
struct ArraySink {
  uint32_t* out;
  unsigned long long* count;
  template <int U>
  __device__ __forceinline__ uint32_t warp_push_multi(const bool (&pred)[U], const uint32_t (&item)[U]) const {
    uint32_t t = 0;
#pragma unroll
    for (int k = 0; k < U; ++k) t += warp_push(pred[k], item[k]);
    return t;
  }
  __device__ __forceinline__ uint32_t warp_push(bool pred, uint32_t item) const {
    const unsigned mask = __ballot_sync(FULL_MASK, pred);
    if (!mask) return 0;
    const int leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(count, (unsigned long long)__popc(mask));
    base = __shfl_sync(FULL_MASK, base, leader);
    if (pred) out[base + __popc(mask & lanemask_lt())] = item;
    return __popc(mask);
  }
  __device__ __forceinline__ uint32_t active_push(bool pred, uint32_t item) const {
    const unsigned act = __activemask();
    const unsigned mask = __ballot_sync(act, pred);
    if (!mask) return 0;
    const int leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if ((int)lane_id() == leader) base = atomicAdd(count, (unsigned long long)__popc(mask));
    base = __shfl_sync(act, base, leader);
    if (pred) out[base + __popc(mask & lanemask_lt())] = item;
    return __popc(mask);
  }
};

// ------------------------------------------------------ CTA worker (LBS) ---

template <class Payload>
struct CtaSmem {
  int64_t* e0;    // [F]   first edge of batch item i
  int64_t* pre;   // [F+1] exclusive prefix of degrees (LBS offsets)
  Payload* pay;   // [F]
  int64_t* wsum;  // [32]  scan scratch
};

template <class Payload>
__host__ __device__ constexpr size_t cta_smem_bytes(int F) {
  return (size_t)F * 8 + ((size_t)F + 1) * 8 + (size_t)F * sizeof(Payload) + 32 * 8 + 64;
}

template <class Payload>
__device__ __forceinline__ CtaSmem<Payload> cta_smem_carve(unsigned char* base, int F) {
  CtaSmem<Payload> s;
  s.e0 = reinterpret_cast<int64_t*>(base);
  s.pre = s.e0 + F;
  s.wsum = s.pre + F + 1;
  s.pay = reinterpret_cast<Payload*>(s.wsum + 32);
  return s;
}

// In-place exclusive scan of a[0..n) (n <= F) into a[0..n], a[n] = total.
// Each thread scans a contiguous segment; warp shuffles; one smem pass.
__device__ __forceinline__ void block_exclusive_scan(int64_t* a, int n, int64_t* wsum) {
  const int T = blockDim.x, tid = threadIdx.x;
  const int per = (n + T - 1) / T;
  const int b = min(n, tid * per), e = min(n, b + per);
  int64_t s = 0;
  for (int i = b; i < e; ++i) s += a[i];
  // inclusive warp scan of s
  int64_t x = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    int64_t y = __shfl_up_sync(FULL_MASK, x, d);
    if ((int)lane_id() >= d) x += y;
  }
  const int wid = tid >> 5, nw = (T + 31) >> 5;
  if ((int)lane_id() == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int64_t v = (int)lane_id() < nw ? wsum[lane_id()] : 0;
    int64_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      int64_t y = __shfl_up_sync(FULL_MASK, inc, d);
      if ((int)lane_id() >= d) inc += y;
    }
    if ((int)lane_id() < nw) wsum[lane_id()] = inc - v;  // exclusive warp offsets
  }
  __syncthreads();
  int64_t run = wsum[wid] + x - s;  // exclusive prefix of this thread's segment
  for (int i = b; i < e; ++i) {
    int64_t d = a[i];
    a[i] = run;
    run += d;
  }
  if (tid == T - 1) a[n] = run;  // last thread's segment ends at n
  __syncthreads();
}

// largest i in [0, n) with pre[i] <= e  (pre is non-decreasing, pre[0] = 0)
__device__ __forceinline__ int lbs_find(const int64_t* pre, int n, int64_t e) {
  int lo = 0, hi = n;  // invariant: pre[lo] <= e < pre[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (pre[mid] <= e) lo = mid; else hi = mid;
  }
  return lo;
}

// largest i in [lo, hi) with pre[i] <= e, given pre[lo] <= e < pre[hi]
__device__ __forceinline__ int lbs_find_range(const int64_t* pre, int lo, int hi, int64_t e) {
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (pre[mid] <= e) lo = mid; else hi = mid;
  }
  return lo;
}

constexpr int LBS_UNROLL = 8;

// Hub splitting (persistent CTA workers): a popped vertex with more than
// SPLIT_DEG edges keeps its first CHUNK_EDGES edges and publishes the rest as
// CHUNK_EDGES-sized chunk tasks on the same queue, so all SMs expand a hub in
// parallel instead of one CTA walking it serially while the rest of the GPU
// speculates on depths the hub has not yet fixed (the measured source of
// RMAT-24 BFS overwork).
#ifndef ATOS_CHUNK_EDGES
#define ATOS_CHUNK_EDGES 1024
#endif
#ifndef ATOS_SPLIT_DEG
#define ATOS_SPLIT_DEG (2 * ATOS_CHUNK_EDGES)
#endif
constexpr int64_t CHUNK_EDGES = ATOS_CHUNK_EDGES;
constexpr int64_t SPLIT_DEG = ATOS_SPLIT_DEG;

template <class P>
__device__ __forceinline__ uint64_t pack_payload(P p) {
  uint64_t u = 0;
  memcpy(&u, &p, sizeof(P));
  return u;
}
template <class P>
__device__ __forceinline__ P unpack_payload(uint64_t u) {
  P p;
  memcpy(&p, &u, sizeof(P));
  return p;
}

// Load-balancing search expansion of a prepared batch: pre[0..n] is the
// exclusive prefix of the items' degrees, e0/pay their first edge and payload.
// Warp `wi` of `nw` takes 32*UNROLL consecutive flattened edges per step; each
// lane locates its edges' items by binary search bounded by the owners of the
// warp's first and last edge, loads UNROLL columns, issues UNROLL probes, then
// UNROLL commits, then ONE aggregated push.  Returns the pushes (per lane 0).


// One LBS step: the warp expands flattened edges [eb, eb + 32*UNROLL) of a
// prepared batch (see lbs_expand).  Returns the pushes (warp-uniform).
// hint_lo/hint_hi (>= 0): owners of the step's first edge and of the first
// edge of the next step, precomputed by the queue agent (no per-step search).
template <class App, class Sink, int U = LBS_UNROLL>
__device__ __forceinline__ uint32_t lbs_step(const App& app, const GraphView& g, const Sink& sink, const int64_t* pre,
                                             const int64_t* e0s, const typename App::Payload* pay, int n,
                                             int64_t total, int64_t eb, int hint_lo = -1, int hint_hi = -1,
                                             const int* sofs = nullptr, const int32_t* stage = nullptr) {
  const int lane = lane_id();
  int lo, hi;
  if (hint_lo >= 0) {
    lo = hint_lo;
    hi = hint_hi + 1;
  } else {
    const int64_t elast = min(total, eb + 32 * U) - 1;
    int bound = 0;
    if (lane == 0) bound = lbs_find(pre, n, eb);
    if (lane == 31) bound = lbs_find(pre, n, elast);
    lo = __shfl_sync(FULL_MASK, bound, 0);
    hi = __shfl_sync(FULL_MASK, bound, 31) + 1;
  }
  uint32_t w[U];
  int idx[U];
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int64_t e = eb + lane + 32 * k;
    idx[k] = -1;
    w[k] = 0;
    if (e < total) {
      lo = ATOS_CHK(lbs_find_range(pre, lo, hi, e), n);
      idx[k] = lo;
      const int so = sofs ? sofs[lo] : -1;  // staged in shared memory by the agent's TMA copy?
      w[k] = so >= 0 ? (uint32_t)stage[so + (int)(e - pre[lo])]
                     : ld_col_tagged(g.col + ATOS_CHK(e0s[lo] + (e - pre[lo]), g.col_cap));
    }
  }
  // (value-initialised: an uninitialised raw[k] on lanes without an edge made
  // the compiler carry it across steps through local memory — an LDL/STL
  // pair around every atomic)
  typename App::Probe pr[U];
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const uint32_t tag = w[k] >> TAG_SHIFT;  // TAG_HUB | TAG_SINK (device.cuh)
    w[k] = ATOS_CHK(w[k] & VID_MASK, g.n);
    pr[k] = typename App::Probe{};
    if (idx[k] >= 0) pr[k] = app.probe(w[k], tag);
  }
  typename App::Raw raw[U];
  typename App::Payload pk[U];
#pragma unroll
  for (int k = 0; k < U; ++k) {
    raw[k] = typename App::Raw{};
    pk[k] = idx[k] >= 0 ? pay[idx[k]] : typename App::Payload{};
    if (idx[k] >= 0) raw[k] = app.issue(pk[k], w[k], pr[k]);
  }
  bool act[U];
#pragma unroll
  for (int k = 0; k < U; ++k) act[k] = idx[k] >= 0 && app.decide(pk[k], w[k], pr[k], raw[k]);
  uint32_t item[U];
#pragma unroll
  for (int k = 0; k < U; ++k) item[k] = app.item_of(w[k]);
  return sink.template warp_push_multi<U>(act, item);
}

template <class App, class Sink>
__device__ __forceinline__ uint32_t lbs_expand(const App& app, const GraphView& g, const Sink& sink, const int64_t* pre,
                                               const int64_t* e0s, const typename App::Payload* pay, int n,
                                               int64_t total, int wi, int nw) {
  const int lane = lane_id();
  const int64_t stride = (int64_t)nw * 32 * LBS_UNROLL;
  uint32_t pushed = 0;
  // Locate the items of the edges of step `eb` and issue their column loads.
  auto fetch = [&](int64_t eb, uint32_t (&w)[LBS_UNROLL], int (&idx)[LBS_UNROLL]) {
    const int64_t elast = min(total, eb + 32 * LBS_UNROLL) - 1;
    int bound = 0;
    if (lane == 0) bound = lbs_find(pre, n, eb);
    if (lane == 31) bound = lbs_find(pre, n, elast);
    int lo = __shfl_sync(FULL_MASK, bound, 0);
    const int hi = __shfl_sync(FULL_MASK, bound, 31) + 1;
#pragma unroll
    for (int k = 0; k < LBS_UNROLL; ++k) {
      const int64_t e = eb + lane + 32 * k;
      idx[k] = -1;
      w[k] = 0;
      if (e < total) {
        lo = ATOS_CHK(lbs_find_range(pre, lo, hi, e), n);
        idx[k] = lo;
        w[k] = ld_col_tagged(g.col + ATOS_CHK(e0s[lo] + (e - pre[lo]), g.col_cap));
      }
    }
  };
  // Software pipeline: the next step's column loads are in flight while this
  // step's probes / atomics / push wait on L2 (two dependent memory latencies
  // per step otherwise — col load then probe).
  uint32_t wn[LBS_UNROLL];
  int idxn[LBS_UNROLL];
  int64_t eb = (int64_t)wi * 32 * LBS_UNROLL;
  if (eb < total) fetch(eb, wn, idxn);
  for (; eb < total; eb += stride) {
    uint32_t w[LBS_UNROLL];
    int idx[LBS_UNROLL];
#pragma unroll
    for (int k = 0; k < LBS_UNROLL; ++k) {
      w[k] = wn[k];
      idx[k] = idxn[k];
    }
    if (eb + stride < total) fetch(eb + stride, wn, idxn);
    typename App::Probe pr[LBS_UNROLL];
#pragma unroll
    for (int k = 0; k < LBS_UNROLL; ++k) {
      const uint32_t tag = w[k] >> TAG_SHIFT;  // TAG_HUB | TAG_SINK
      w[k] = ATOS_CHK(w[k] & VID_MASK, g.n);
      pr[k] = typename App::Probe{};
      if (idx[k] >= 0) pr[k] = app.probe(w[k], tag);
    }
    typename App::Raw raw[LBS_UNROLL];
    typename App::Payload pk[LBS_UNROLL];
#pragma unroll
    for (int k = 0; k < LBS_UNROLL; ++k) {
      pk[k] = idx[k] >= 0 ? pay[idx[k]] : typename App::Payload{};
      if (idx[k] >= 0) raw[k] = app.issue(pk[k], w[k], pr[k]);
    }
    bool act[LBS_UNROLL];
#pragma unroll
    for (int k = 0; k < LBS_UNROLL; ++k) act[k] = idx[k] >= 0 && app.decide(pk[k], w[k], pr[k], raw[k]);
    uint32_t item[LBS_UNROLL];
#pragma unroll
    for (int k = 0; k < LBS_UNROLL; ++k) item[k] = app.item_of(w[k]);
    pushed += sink.template warp_push_multi<LBS_UNROLL>(act, item);
  }
  return pushed;
}

// Publish edges [e0 + CHUNK_EDGES, e1) of hub `v` as chunk tasks; returns the
// new end of the range the caller keeps (its first chunk).  The entry of the
// task at ring position p is written to chunks[p & mask] once that slot is
// free for its lap, then all entries are fenced before the slots are
// published (device.cuh, Chunk).
template <class Payload>
__device__ __noinline__ int64_t split_hub(const Queue* cq, uint32_t v, int64_t e0, int64_t e1, Payload p) {
  const Queue& q = *cq;
  const uint32_t k = (uint32_t)((e1 - e0 - 1) / CHUNK_EDGES);  // chunks beyond the first
  const unsigned long long base = atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->tail.v), (unsigned long long)k);
  red_add_relaxed_s64(&q.ctl->count.v, (int64_t)k);
  red_add_relaxed_s64(&q.ctl->chunk_tail.v, (int64_t)k);
  uint64_t pv = pack_payload(p);
  if (sizeof(Payload) == 4) pv |= (uint64_t)v << 32;
  for (uint32_t j = 0; j < k; ++j) {
    const uint64_t pos = base + j;
    if (!q_wait_free(q, pos)) return e1;  // aborted: the run is over
    const int64_t c0 = e0 + CHUNK_EDGES * (int64_t)(j + 1);
    const int64_t c1 = min(e1, c0 + CHUNK_EDGES);
    Chunk* c = q.chunks + (pos & q.mask);
    c->range = (uint64_t)c0 | ((uint64_t)(c1 - c0) << 48);
    c->pv = pv;
  }
  __threadfence();  // chunk entries visible before their tasks
  for (uint32_t j = 0; j < k; ++j) q_publish(q, base + j, CHUNK_BIT | (uint32_t)((base + j) & q.mask));
  return e0 + CHUNK_EDGES;
}

// Read the chunk task at ring position `pos` (its slot read, NOT yet
// released): edge range + payload, and whether it is still current (BFS: the
// hub has not improved since).  The caller releases the slot afterwards with
// q_release_slot_ordered.
template <class App>
__device__ __forceinline__ bool read_chunk(const App& app, const Queue& q, uint64_t pos, int64_t& e0, int64_t& e1,
                                           typename App::Payload& p) {
  using Payload = typename App::Payload;
  const Chunk* c = q.chunks + (pos & q.mask);
  const uint64_t range = ld_cg_u64(&c->range);  // L2: entries are rewritten on wrap
  const uint64_t pv = ld_cg_u64(&c->pv);
  e0 = (int64_t)(range & ((1ull << 48) - 1));
  e1 = e0 + (int64_t)(range >> 48);
  p = unpack_payload<Payload>(sizeof(Payload) == 4 ? (pv & 0xFFFFFFFFull) : pv);
  atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->chunk_done.v), 1ull);
  return app.chunk_current((uint32_t)(pv >> 32), p);
}

// Process batch items [0, n) with the whole CTA.  Every thread must call.
template <class App, class Src, class Sink>
__device__ __forceinline__ void cta_batch(const App& app, const GraphView& g, const Src& src, const Sink& sink,
                                          uint32_t n, CtaSmem<typename App::Payload>& sm, LocalStats& st) {
  using Payload = typename App::Payload;
  const int T = blockDim.x, tid = threadIdx.x;
  for (int i = tid; i < (int)n; i += T) {
    uint32_t item = 0;
    int64_t e0 = 0, e1 = 0;
    Payload p{};
    bool ok = src.get(i, item) && app.begin(item, g, e0, e1, p);
    sm.e0[i] = e0;
    sm.pre[i] = ok ? e1 - e0 : 0;
    sm.pay[i] = p;
  }
  __syncthreads();
  block_exclusive_scan(sm.pre, (int)n, sm.wsum);
  const int64_t total = sm.pre[n];
  const int lane = lane_id();
  const uint32_t pushed = lbs_expand(app, g, sink, sm.pre, sm.e0, sm.pay, (int)n, total, tid >> 5, T >> 5);
  if (lane == 0) st.pushed += pushed;
  if (tid == 0) st.edges += total;
  __syncthreads();
}

// ---------------------------------------------------------- warp worker ---

// Visit edges [e0, e1) of one vertex with the whole warp: scalar head up to a
// 16-byte boundary, int4 body (4 edges per lane per step), scalar tail.
template <class App, class Sink>
__device__ __forceinline__ uint32_t warp_walk(const App& app, const GraphView& g, const Sink& sink, int64_t e0,
                                              int64_t e1, typename App::Payload p) {
  const int lane = lane_id();
  uint32_t pushed = 0;
  int64_t a0 = (e0 + 3) & ~int64_t(3);
  if (a0 > e1) a0 = e1;
  // head (< 4 edges) + tail share one scalar step each
  {
    const int64_t e = e0 + lane;
    const bool v = e < a0;
    const uint32_t raw = v ? ld_col_tagged(g.col + ATOS_CHK(e, g.col_cap)) : 0u;
    const uint32_t w = ATOS_CHK(raw & VID_MASK, g.n);
    bool act = v && app.edge(p, w, raw >> TAG_SHIFT);
    pushed += sink.warp_push(act, app.item_of(w));
  }
  const int64_t a1 = a0 + ((e1 - a0) & ~int64_t(3));
  const int4* body = reinterpret_cast<const int4*>(g.col + a0);
  const int64_t nv = (a1 - a0) >> 2;
  for (int64_t vb = 0; vb < nv; vb += 32) {
    const int64_t vi = vb + lane;
    const bool v = vi < nv;
    int4 w4 = v ? ld_stream_v4(body + ATOS_CHK(vi, (g.col_cap - a0) >> 2)) : make_int4(0, 0, 0, 0);
    const uint32_t raw[4] = {(uint32_t)w4.x, (uint32_t)w4.y, (uint32_t)w4.z, (uint32_t)w4.w};
    const uint32_t w[4] = {ATOS_CHK(raw[0] & VID_MASK, g.n), ATOS_CHK(raw[1] & VID_MASK, g.n),
                           ATOS_CHK(raw[2] & VID_MASK, g.n), ATOS_CHK(raw[3] & VID_MASK, g.n)};
    typename App::Probe pr[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (v) pr[k] = app.probe(w[k], raw[k] >> TAG_SHIFT);
    typename App::Raw old[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (v) old[k] = app.issue(p, w[k], pr[k]);
    bool act[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) act[k] = v && app.decide(p, w[k], pr[k], old[k]);
    uint32_t item[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) item[k] = app.item_of(w[k]);
    pushed += sink.template warp_push_multi<4>(act, item);
  }
  {
    const int64_t e = a1 + lane;
    const bool v = e < e1;
    const uint32_t raw = v ? ld_col_tagged(g.col + ATOS_CHK(e, g.col_cap)) : 0u;
    const uint32_t w = ATOS_CHK(raw & VID_MASK, g.n);
    bool act = v && app.edge(p, w, raw >> TAG_SHIFT);
    pushed += sink.warp_push(act, app.item_of(w));
  }
  return pushed;
}

// Process batch items [0, n) with one warp (persist-32: no in-worker LB).
template <class App, class Src, class Sink>
__device__ __forceinline__ void warp_batch(const App& app, const GraphView& g, const Src& src, const Sink& sink,
                                           uint32_t n, LocalStats& st) {
  using Payload = typename App::Payload;
  const int lane = lane_id();
  uint32_t pushed = 0;
  uint64_t edges = 0;
  for (uint32_t c = 0; c < n; c += 32) {
    const uint32_t k = min(32u, n - c);
    int64_t e0 = 0, e1 = 0;
    Payload p{};
    bool ok = false;
    if ((uint32_t)lane < k) {
      uint32_t item;
      ok = src.get(c + lane, item) && app.begin(item, g, e0, e1, p);
    }
    unsigned todo = __ballot_sync(FULL_MASK, ok);
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const int64_t je0 = __shfl_sync(FULL_MASK, e0, j);
      const int64_t je1 = __shfl_sync(FULL_MASK, e1, j);
      const Payload jp = __shfl_sync(FULL_MASK, p, j);
      pushed += warp_walk(app, g, sink, je0, je1, jp);
      edges += je1 - je0;
    }
  }
  if (lane == 0) {
    st.pushed += pushed;
    st.edges += edges;
  }
}

// -------------------------------------------------------- thread worker ---

// Each lane owns items lane, lane+32, ... of the warp's batch [0, n) and walks
// their edges serially; pushes aggregate over the lanes active in a step.
template <class App, class Src, class Sink>
__device__ __forceinline__ void thread_batch(const App& app, const GraphView& g, const Src& src, const Sink& sink,
                                             uint32_t n, LocalStats& st) {
  using Payload = typename App::Payload;
  const uint32_t lane = lane_id();
  uint32_t next = lane;
  int64_t e = 0, e1 = 0;
  Payload p{};
  uint32_t pushed = 0;
  uint64_t edges = 0;
  auto refill = [&]() {
    while (e >= e1 && next < n) {
      uint32_t item;
      int64_t b = 0, c = 0;
      bool ok = src.get(next, item) && app.begin(item, g, b, c, p);
      next += 32;
      if (ok) { e = b; e1 = c; edges += c - b; }
    }
  };
  refill();
  while (__any_sync(FULL_MASK, e < e1)) {
    bool act = false;
    uint32_t w = 0;
    if (e < e1) {
      const uint32_t raw = ld_col_tagged(g.col + ATOS_CHK(e, g.col_cap));
      w = ATOS_CHK(raw & VID_MASK, g.n);
      ++e;
      act = app.edge(p, w, raw >> TAG_SHIFT);
    }
    pushed += sink.warp_push(act, app.item_of(w));
    refill();
  }
  st.edges += edges;
  if (lane == 0) st.pushed += pushed;
}

}  // namespace atos
