// device.cuh — memory-model helpers, the shared task queue and the termination
// detector of the Atos hot path, sm_100a.
//
// The queue is ONE ring shared by every worker of the GPU (PAPER.md P:97,
// "a single queue balances load more quickly"; Listing 2).
//
//  * ring: uint64 slots, capacity a power of two.  A slot word is
//    (tag << 32) | item.  For queue position p (lap L = p >> log2cap) the slot
//    is "empty for lap L" when tag == 2L and "full for lap L" when
//    tag == 2L+1.  All tags start at 0 (empty for lap 0).  A consumer that has
//    read position p writes tag 2L+2 (empty for lap L+1).  This bounded-MPMC
//    discipline makes wrap-around safe without assuming anything about how
//    fast other workers are.
//  * head (next position to pop), tail (next position to push) and processed
//    (items fully processed, including their pushes) are 64-bit counters, each
//    on its own 128-byte line.
//  * push (a3): warp-aggregated — __ballot_sync/__popc, ONE atomicAdd(tail)
//    per warp (plus one red.add(count) that publishes the batch), then each
//    lane writes its slot (see q_store_slot for the ordering argument).
//  * pop (a4): the worker leader reserves n = min(FETCH, count) items from a
//    signed `count` of published items (fetch-and-add, excess returned), then
//    claims positions with atomicAdd(head, n).  Reservations never exceed
//    published items, so head never passes tail: no overshoot, and a claimed
//    slot is at worst an in-flight store.  (A CAS on head serialises badly
//    with thousands of poppers: measured 0.5 M pops/s at FETCH 1.)
//  * termination (a7): a worker adds its batch size to `processed` (release)
//    only after all pushes of that batch are reserved.  An idle worker reads
//    processed (acquire) THEN tail; processed == tail means every pushed item
//    has been fully processed and nobody holds work: quiescence, exit.
//  * overflow: a producer whose slot still holds an unconsumed item of the
//    previous lap while head <= p - cap (more than cap live items) raises
//    ATOS_ERR_QUEUE_OVERFLOW and aborts the run.
//  * watchdog: idle/spin loops compare %globaltimer with a deadline and abort
//    with ATOS_ERR_TIMEOUT.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace atos {

constexpr unsigned FULL_MASK = 0xffffffffu;
constexpr uint32_t GC_CHECK_BIT = 0x80000000u;  // colouring CHECK(v) tag (R10)

enum : uint32_t { ABORT_NONE = 0, ABORT_OVERFLOW = 1, ABORT_TIMEOUT = 2 };

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int32_t ld_relaxed_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float ld_relaxed_f32(const float* p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// relaxed at CTA scope: may hit in L1 and return a stale (older) value; used
// only where a stale value is safe (BFS probe: dist only decreases).
__device__ __forceinline__ uint32_t ld_relaxed_cta_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.cta.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32_nc(const uint32_t* p) {  // no compiler memory clobber
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_cg_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int64_t ld_cg_s64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.global.cg.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_s32(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_relaxed_s64(uint64_t* p, int64_t v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void atom_add_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// L2 cache policies.  The CSR column array streams through L2 once per
// expansion (1 GB at RMAT-24, re-read ~67x by PageRank) and would evict the
// per-vertex state that every edge hits at random (dist: 64 MB, residue:
// 64 MB) — measured L2 hit rate 54% and 160 GB of DRAM reads per PR launch.
// Columns are therefore loaded evict_first and the hot state is accessed
// evict_last.  (createpolicy is pure, so the compiler hoists it.)
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Column entries carry two TAG bits (vertex ids are < 2^30 - 1, R10/R37),
// set at graph create on library-owned CSRs: bit 31 (HUB_TAG) when the
// target's in-degree is >= HUB_IN_DEG, so the PageRank edge push knows without
// any extra load that the target keeps its residue in fp64 (R34/R35); bit 30
// (SINK_TAG) when the target has out-degree 0, so an activation test needs no
// load of the dangling bitmap (R29/R37).  Every reader masks them off with
// VID_MASK; the hot loops pass `raw >> TAG_SHIFT` (TAG_HUB | TAG_SINK bits)
// to the apps.
constexpr uint32_t HUB_TAG = 0x80000000u;
constexpr uint32_t SINK_TAG = 0x40000000u;
constexpr uint32_t VID_MASK = 0x3FFFFFFFu;
constexpr int TAG_SHIFT = 30;
constexpr uint32_t TAG_HUB = HUB_TAG >> TAG_SHIFT;    // 2
constexpr uint32_t TAG_SINK = SINK_TAG >> TAG_SHIFT;  // 1
#ifndef ATOS_HUB_IN_DEG
#define ATOS_HUB_IN_DEG 2048  // R34 (512 until the R38 replicas; 2048: -8% PageRank, profiles/r02_hub_threshold.md)
#endif
constexpr uint32_t HUB_IN_DEG = ATOS_HUB_IN_DEG;
// streaming read-only loads of immutable CSR arrays (no L1 allocation, L2 evict-first)
__device__ __forceinline__ uint32_t ld_col_tagged(const int32_t* p) {  // raw entry: vertex id | HUB_TAG
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol_evict_first()));
  return v;
}
__device__ __forceinline__ int32_t ld_stream_s32(const int32_t* p) { return (int32_t)(ld_col_tagged(p) & VID_MASK); }
__device__ __forceinline__ int4 ld_stream_v4(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol_evict_first()));
  return v;
}
// ---- TMA 1-D bulk copies + mbarriers (column staging for CTA workers, a5)
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// one arrival that also adds `bytes` to the phase's expected transaction count
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// global -> shared bulk copy (cp.async.bulk, the TMA unit's 1-D mode): 16-B
// aligned addresses, size a multiple of 16; completion is signalled on `bar`.
// Columns stream once per expansion, so the copy reads them L2 evict_first.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol_evict_first())
      : "memory");
}

// hot per-vertex state: relaxed gpu-scope atomics / loads with L2 evict_last
__device__ __forceinline__ uint32_t atom_min_hot(uint32_t* p, uint32_t v) {
  uint32_t o;
  asm volatile("atom.relaxed.gpu.global.min.L2::cache_hint.u32 %0, [%1], %2, %3;" : "=r"(o) : "l"(p), "r"(v), "l"(pol_evict_last()));
  return o;
}
__device__ __forceinline__ float atom_add_hot(float* p, float v) {
  float o;
  asm volatile("atom.relaxed.gpu.global.add.L2::cache_hint.f32 %0, [%1], %2, %3;" : "=f"(o) : "l"(p), "f"(v), "l"(pol_evict_last()));
  return o;
}
__device__ __forceinline__ double atom_add_hot(double* p, double v) {
  double o;
  asm volatile("atom.relaxed.gpu.global.add.L2::cache_hint.f64 %0, [%1], %2, %3;" : "=d"(o) : "l"(p), "d"(v), "l"(pol_evict_last()));
  return o;
}
__device__ __forceinline__ uint32_t ld_probe_hot(const uint32_t* p) {  // cta scope: may hit a stale L1 copy
  uint32_t v;
  asm volatile("ld.relaxed.cta.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol_evict_last()));
  return v;
}
__device__ __forceinline__ uint32_t ld_probe_u16(const uint16_t* p) {  // cta scope, L1-cacheable, evict_last
  uint16_t v;
  asm volatile("ld.relaxed.cta.global.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol_evict_last()));
  return v;
}
__device__ __forceinline__ void st_u16_hot(uint16_t* p, uint16_t v) {
  asm volatile("st.relaxed.gpu.global.L2::cache_hint.u16 [%0], %1, %2;" ::"l"(p), "h"(v), "l"(pol_evict_last()));
}
__device__ __forceinline__ uint32_t ld_relaxed_hot(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol_evict_last()));
  return v;
}
__device__ __forceinline__ int64_t ld_nc_s64(const int64_t* p) {  // CSR offsets: read-only, evict_first
  int64_t v;
  asm volatile("ld.global.nc.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol_evict_first()));
  return v;
}
__device__ __forceinline__ uint32_t ld_nc_u32(const uint32_t* p) {  // immutable per-vertex bitmaps: keep in L2
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol_evict_last()));
  return v;
}
__device__ __forceinline__ void st_stream_u64(uint64_t* p, uint64_t v) {  // queue slot writes
  asm volatile("st.relaxed.gpu.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol_evict_first()) : "memory");
}
// per-pop accumulation into a large array (PR rank): keep it from evicting the residues
__device__ __forceinline__ void red_add_cold(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol_evict_first()));
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// ---- bounds-checked builds (-DATOS_CHECKED; tests/test_queue_stress.py).  Every
// index the hot path derives from device data (a popped task word, a CSR offset,
// a column entry, a shared-memory batch offset) passes through chk(): in a
// checked build an out-of-range index records (file hash, line, value) in
// g_atos_check — the first failure wins — and is clamped to 0 so the access
// stays in bounds; the call then returns ATOS_ERR_CUDA naming the check.  In
// product builds chk() is the identity.  (compute-sanitizer is not available
// on this pool, so this is the out-of-bounds detector.)
__host__ __device__ constexpr uint32_t chk_fnv(const char* s, uint32_t h = 2166136261u) {
  return *s ? chk_fnv(s + 1, (h ^ (uint32_t)(unsigned char)*s) * 16777619u) : h;
}
__host__ __device__ constexpr const char* chk_base(const char* s, const char* b = nullptr) {
  return *s ? chk_base(s + 1, *s == '/' ? s + 1 : (b ? b : s)) : (b ? b : s);
}
__host__ __device__ constexpr uint32_t chk_fhash(const char* path) { return chk_fnv(chk_base(path)); }
struct CheckRec {
  unsigned long long hit;  // 0 = clean
  uint32_t file, line;
  long long value, bound;
};
#ifdef ATOS_CHECKED
__device__ CheckRec g_atos_check;
__device__ __noinline__ void chk_fail(uint32_t file, uint32_t line, long long v, long long bound) {
  if (atomicCAS(&g_atos_check.hit, 0ull, 1ull) == 0ull) {
    g_atos_check.file = file;
    g_atos_check.line = line;
    g_atos_check.value = v;
    g_atos_check.bound = bound;
    __threadfence();
  }
}
#define ATOS_CHK(i, bound) \
  (((unsigned long long)(long long)(i) < (unsigned long long)(long long)(bound)) ? (i) \
   : (::atos::chk_fail(::atos::chk_fhash(__FILE__), __LINE__, (long long)(i), (long long)(bound)), decltype(i)(0)))
#else
#define ATOS_CHK(i, bound) (i)
#endif

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- queue state
struct alignas(128) Line64 {
  uint64_t v;
  uint64_t pad[15];
};

// Device-resident control block (one per run).
struct QueueCtl {
  Line64 head;
  Line64 tail;
  Line64 count;  // published, unclaimed items (signed; see q_try_pop)
  Line64 processed;
  Line64 abort;         // ABORT_* code (u32 in .v)
  Line64 high_water;    // max observed tail - head
  Line64 chunk_tail;    // hub chunk tasks pushed
  Line64 chunk_done;    // hub chunk tasks consumed
  Line64 trace_count;   // timeline records produced
  Line64 stats[4];      // popped, pushed, edges, spare
  Line64 aux[4];        // app-specific counters (e.g. PR check cursor, colours)
  Line64 prof[12];       // clock64 cycle counters of ATOS_WAIT_PROF builds (tuning experiments only)
};

// Kernel-side view of the queue (passed by value).
struct Queue {
  uint64_t* ring;
  uint64_t mask;      // cap - 1
  uint32_t log2cap;
  QueueCtl* ctl;
  uint64_t deadline;    // %globaltimer deadline (ns); 0 = none (armed by q_arm)
  uint64_t timeout_ns;  // 0 = no watchdog
  uint64_t head_floor;  // discrete rounds: every position < head_floor is claimed
  struct Chunk* chunks; // hub chunk table, ring-capacity entries (persistent CTA edge-map workers); nullptr = no splitting
  struct TraceRec* trace;  // optional timeline (atos_trace_rec); nullptr = off
  uint64_t trace_cap;
  uint32_t trace_kind;
  uint32_t workers;  // adaptive fetch: number of concurrent poppers (0 = off)
  uint32_t backoff_ns;  // idle-poll backoff cap
  uint32_t stage_cap;   // persistent CTA workers: staged column elements per batch buffer (0 = off)
};

// Timeline record (layout == atos_trace_rec in include/atos.h).
struct TraceRec {
  uint64_t t_ns;
  uint32_t items, edges, sm, kind;
};
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
// One record per processed batch (single thread).
__device__ __forceinline__ void q_trace(const Queue& q, uint32_t items, uint64_t edges) {
  if (!q.trace) return;
  const unsigned long long i = atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->trace_count.v), 1ull);
  if (i < q.trace_cap) {
    TraceRec r;
    r.t_ns = globaltimer_ns();
    r.items = items;
    r.edges = (uint32_t)(edges > 0xFFFFFFFFull ? 0xFFFFFFFFull : edges);
    r.sm = smid();
    r.kind = q.trace_kind;
    q.trace[i] = r;
  }
}

// A slice [e0, e1) of a hub's adjacency list, queued as its own task (R24;
// item = CHUNK_BIT | (p & mask), p = the task's ring position).  The entry of
// the chunk task at ring position p is chunks[p & mask]: the table has the
// ring's capacity, a producer writes the entry only after the slot is free for
// its lap (q_wait_free), and the consumer reads the entry before it releases
// the slot (st.release) — so an entry is live exactly while its slot is, and
// the table can neither overflow nor be overwritten under a straggler.
constexpr uint32_t CHUNK_BIT = 0x80000000u;
constexpr uint32_t DEFER_BIT = 0x40000000u;  // PageRank: a task deferred once (R31); needs n <= 2^30
struct Chunk {
  uint64_t range;  // e0 | (e1 - e0) << 48   (m < 2^48, e1 - e0 <= CHUNK_EDGES)
  uint64_t pv;     // payload bits; 4-byte payloads carry the hub vertex in bits 32..63
};

__device__ __forceinline__ bool q_aborted(const Queue& q) {
  return ld_relaxed_u64(&q.ctl->abort.v) != 0;
}
__device__ __forceinline__ void q_raise(const Queue& q, uint32_t code) {
  atomicCAS(reinterpret_cast<unsigned long long*>(&q.ctl->abort.v), 0ull, (unsigned long long)code);
}
__device__ __forceinline__ bool q_timed_out(const Queue& q) {
  if (q.deadline == 0) return false;
  if (globaltimer_ns() > q.deadline) { q_raise(q, ABORT_TIMEOUT); return true; }
  return false;
}
// Arm the watchdog at kernel entry (deadline = now + timeout).
__device__ __forceinline__ void q_arm(Queue& q) {
  q.deadline = q.timeout_ns ? globaltimer_ns() + q.timeout_ns : 0;
}

// Wait until ring position p may be written: in the wrap-around case (lap >
// 0) the previous lap's item must have been consumed.  Detects overflow (more
// than cap live, unclaimed items).  Returns false on abort.
__device__ __forceinline__ bool q_wait_free(const Queue& q, uint64_t p) {
  const uint32_t lap = (uint32_t)(p >> q.log2cap);
  if (lap == 0) return true;
  const uint64_t* slot = q.ring + (p & q.mask);
  unsigned ns = 32;
  for (;;) {
    uint32_t tag = (uint32_t)(ld_relaxed_u64(slot) >> 32);
    if (tag == 2u * lap) return true;
    uint64_t h = ld_relaxed_u64(&q.ctl->head.v);
    if (h < q.head_floor) h = q.head_floor;
    if (h + q.mask + 1 <= p) {  // more than cap live (unclaimed) items
      q_raise(q, ABORT_OVERFLOW);
      return false;
    }
    if (q_aborted(q) || q_timed_out(q)) return false;
    __nanosleep(ns);
    ns = ns < 1024 ? ns * 2 : ns;
  }
}

// Store `item` as the full slot word of position p (slot known to be free).
__device__ __forceinline__ void q_publish(const Queue& q, uint64_t p, uint32_t item) {
  // Relaxed (strong, L2) store: every push predicate is computed from the
  // RETURNED value of the atomic that produced the state its consumer reads
  // (BFS atomicMin, PR atomicAdd, GC atomicExch after __threadfence), so that
  // atomic is performed at L2 — the point of coherence — before this store
  // issues.  A st.release here cost a MEMBAR+ERRBAR per push (19% of BFS
  // stall samples, profiles/r01_bfs_rmat24_v1).  (Hub chunk entries are plain
  // stores and are ordered before their slots by a __threadfence in split_hub.)
  const uint32_t lap = (uint32_t)(p >> q.log2cap);
  asm volatile("st.relaxed.gpu.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(q.ring + (p & q.mask)),
               "l"(((uint64_t)(2u * lap + 1u) << 32) | item), "l"(pol_evict_first())
               : "memory");
}

// Publish `item` at queue position p (a3).  Waits only in the wrap-around case
// for the previous lap's consumer; detects overflow.  Returns false on abort.
__device__ __forceinline__ bool q_store_slot(const Queue& q, uint64_t p, uint32_t item) {
  if (!q_wait_free(q, p)) return false;
  q_publish(q, p, item);
  return true;
}

// Read the item at position p (claimed by this worker) without releasing the
// slot.  Returns false only on abort/timeout.
__device__ __forceinline__ bool q_read_slot(const Queue& q, uint64_t p, uint32_t& item) {
  const uint64_t* slot = q.ring + (p & q.mask);
  const uint32_t want = 2u * (uint32_t)(p >> q.log2cap) + 1u;
  // Relaxed (strong, L2) load: everything the consumer then reads about the
  // item is addressed THROUGH the item (dist[v], res[v], off[v], chunk entry)
  // and read from L2, so it cannot be issued before this load returns.  An
  // ld.acquire here adds CCTL.IVALL (L1 invalidate) per item, which would also
  // defeat the L1-cached BFS filter probes.
  uint64_t w = ld_relaxed_u64(slot);
  if ((uint32_t)(w >> 32) != want) {
    unsigned ns = 16;
    for (;;) {
      __nanosleep(ns);
      w = ld_relaxed_u64(slot);
      if ((uint32_t)(w >> 32) == want) break;
      if (q_aborted(q) || q_timed_out(q)) return false;
      ns = ns < 256 ? ns * 2 : ns;
    }
  }
  item = (uint32_t)w;
  return true;
}

// Mark position p's slot empty for the next lap (after its item was read).
__device__ __forceinline__ void q_release_slot(const Queue& q, uint64_t p) {
  asm volatile("st.relaxed.gpu.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(q.ring + (p & q.mask)),
               "l"((uint64_t)(2u * (uint32_t)(p >> q.log2cap) + 2u) << 32), "l"(pol_evict_first())
               : "memory");
}
// Release with st.release: every load this thread issued before (the hub
// chunk entry of the slot) is performed before a producer can see the slot
// free and rewrite the entry.
__device__ __forceinline__ void q_release_slot_ordered(const Queue& q, uint64_t p) {
  st_release_u64(q.ring + (p & q.mask), (uint64_t)(2u * (uint32_t)(p >> q.log2cap) + 2u) << 32);
}

// Read the item at position p (claimed by this worker) and mark the slot
// empty for the next lap.  Returns false only on abort/timeout.
__device__ __forceinline__ bool q_load_slot(const Queue& q, uint64_t p, uint32_t& item) {
  if (!q_read_slot(q, p, item)) return false;
  q_release_slot(q, p);
  return true;
}

constexpr uint32_t EMPTY_ITEM = 0xFFFFFFFFu;  // never a task word (n < 2^31 - 1, R10)

// Read the claimed positions [first, first + n) into stage[] — participant
// `me` of `parts` takes items me, me + parts, ... — releasing every slot as
// soon as its item is read.  An unpublished slot never holds up the others:
// the participant re-scans its items with backoff until all are in, so a
// producer waiting for one of these slots to be released for its next lap
// (ring wrap-around) is never waiting on a consumer that waits on it.
// Returns false on abort (unread entries stay EMPTY_ITEM).
__device__ __forceinline__ bool q_read_batch(const Queue& q, uint64_t first, uint32_t n, uint32_t* stage, uint32_t me,
                                             uint32_t parts) {
  bool pending = false;
  for (uint32_t i = me; i < n; i += parts) {
    const uint64_t p = first + i;
    const uint64_t w = ld_relaxed_u64(q.ring + (p & q.mask));
    if ((uint32_t)(w >> 32) == 2u * (uint32_t)(p >> q.log2cap) + 1u) {
      stage[i] = (uint32_t)w;
      q_release_slot(q, p);
    } else {
      stage[i] = EMPTY_ITEM;
      pending = true;
    }
  }
  for (unsigned ns = 16; pending; ns = ns < 256 ? ns * 2 : ns) {
    if (q_aborted(q) || q_timed_out(q)) return false;
    __nanosleep(ns);
    pending = false;
    for (uint32_t i = me; i < n; i += parts) {
      if (stage[i] != EMPTY_ITEM) continue;
      const uint64_t p = first + i;
      const uint64_t w = ld_relaxed_u64(q.ring + (p & q.mask));
      if ((uint32_t)(w >> 32) == 2u * (uint32_t)(p >> q.log2cap) + 1u) {
        stage[i] = (uint32_t)w;
        q_release_slot(q, p);
      } else {
        pending = true;
      }
    }
  }
  return true;
}

// Warp-collective push (every lane of the warp must call; `pred` per lane).
// One atomicAdd on tail per warp.  Returns the number of items pushed.
__device__ __forceinline__ uint32_t q_warp_push(const Queue& q, bool pred, uint32_t item) {
  const unsigned mask = __ballot_sync(FULL_MASK, pred);
  if (mask == 0) return 0;
  const unsigned lane = lane_id();
  const int leader = __ffs(mask) - 1;
  const uint32_t cnt = __popc(mask);
  unsigned long long base = 0;
  if ((int)lane == leader) {
    base = atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->tail.v), (unsigned long long)cnt);
    red_add_relaxed_s64(&q.ctl->count.v, (int64_t)cnt);  // publish (consumers spin on slot tags)
  }
  base = __shfl_sync(FULL_MASK, base, leader);
  if (pred) q_store_slot(q, base + __popc(mask & lanemask_lt()), item);
  return cnt;
}

// Push from a subset of converged lanes (thread workers with divergent loops):
// aggregates over __activemask().
__device__ __forceinline__ uint32_t q_active_push(const Queue& q, bool pred, uint32_t item) {
  const unsigned act = __activemask();
  const unsigned mask = __ballot_sync(act, pred);
  if (mask == 0) return 0;
  const unsigned lane = lane_id();
  const int leader = __ffs(mask) - 1;
  const uint32_t cnt = __popc(mask);
  unsigned long long base = 0;
  if ((int)lane == leader) {
    base = atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->tail.v), (unsigned long long)cnt);
    red_add_relaxed_s64(&q.ctl->count.v, (int64_t)cnt);
  }
  base = __shfl_sync(act, base, leader);
  if (pred) q_store_slot(q, base + __popc(mask & lanemask_lt()), item);
  return cnt;
}

// Warp-collective push of up to U items per lane with ONE atomicAdd on tail.
template <int U>
__device__ __forceinline__ uint32_t q_warp_push_multi(const Queue& q, const bool (&pred)[U], const uint32_t (&item)[U]) {
  unsigned m[U];
  uint32_t total = 0;
#pragma unroll
  for (int k = 0; k < U; ++k) {
    m[k] = __ballot_sync(FULL_MASK, pred[k]);
    total += __popc(m[k]);
  }
  if (total == 0) return 0;
  unsigned long long base = 0;
  if (lane_id() == 0) {
    base = atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->tail.v), (unsigned long long)total);
    red_add_relaxed_s64(&q.ctl->count.v, (int64_t)total);
  }
  base = __shfl_sync(FULL_MASK, base, 0);
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int k = 0; k < U; ++k) {
    if (pred[k]) q_store_slot(q, base + __popc(m[k] & lt), item[k]);
    base += __popc(m[k]);
  }
  return total;
}

// Single-thread push of k items item_of(j), j < k (hub chunk tasks).
template <class F>
__device__ __forceinline__ void q_thread_push(const Queue& q, uint32_t k, F item_of) {
  const unsigned long long base = atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->tail.v), (unsigned long long)k);
  red_add_relaxed_s64(&q.ctl->count.v, (int64_t)k);
  for (uint32_t j = 0; j < k; ++j) q_store_slot(q, base + j, item_of(j));
}

// Single-thread pop (a4): claim up to `want` published items with two
// fetch-and-adds and no retry loop.  `count` = items published by producers
// minus items reserved by consumers; a consumer reserves n = min(want, count)
// from it (returning any excess), then takes positions [head, head+n) with
// atomicAdd(head, n).  Because reservations never exceed published items,
// head never passes tail (no overshoot).  Producers publish after reserving
// tail and storing, so a claimed slot is at worst an in-flight store.
// Returns the count claimed (0 if nothing is published right now).
#ifndef ATOS_POP_HINT_MIN
#define ATOS_POP_HINT_MIN 8ll  // skip the pre-read when the caller last saw > this many batches queued
#endif
__device__ __forceinline__ uint32_t q_try_pop(const Queue& q, uint32_t want, uint64_t& first, uint64_t& qlen,
                                              long long hint = 0) {
  long long* cnt = reinterpret_cast<long long*>(&q.ctl->count.v);
  // Skip the pre-read when the caller's last observation says the queue is
  // long (saves one L2 round trip per pop on the critical path).
  const long long seen = hint > ATOS_POP_HINT_MIN * (long long)want ? hint : (long long)ld_relaxed_u64(&q.ctl->count.v);
  if (seen <= 0) return 0;
  // Adaptive fetch: while the queue is short, take only a fair share
  // ceil(count / workers) (>= 1) so a small frontier — e.g. the ~200 chunk
  // tasks of the source hub — spreads over all workers instead of landing in
  // one FETCH-sized batch (measured: 28 batches on 24 SMs in the first 0.7 ms
  // of RMAT-24 BFS).  FETCH_SIZE stays the upper bound.
  if (q.workers) {
    const long long share = (seen + q.workers - 1) / q.workers;
    if (share < (long long)want) want = (uint32_t)share;
  }
  const long long old = atomicAdd(reinterpret_cast<unsigned long long*>(cnt), (unsigned long long)(-(long long)want));
  uint32_t n;
  if (old >= (long long)want) {
    n = want;
  } else if (old > 0) {
    n = (uint32_t)old;
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt), (unsigned long long)(long long)(want - n));
  } else {
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt), (unsigned long long)(long long)want);
    qlen = 0;
    return 0;
  }
  first = atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->head.v), (unsigned long long)n);
  qlen = old > 0 ? (uint64_t)old : 0;
  return n;
}

// Tasks ever enqueued = ring positions handed out.  Read AFTER `processed`:
// processed <= enqueued always, so equality at the reads implies equality
// (quiescence) at the processed read.
__device__ __forceinline__ uint64_t q_enqueued(const Queue& q) {
  return ld_relaxed_u64(&q.ctl->tail.v);
}

// Leader-side pop with the idle path (the paper's f2 hook): backoff,
// termination poll (a7) and watchdog.  Returns n > 0 with `first`, or 0 when
// the run is over (quiescent or aborted).
__device__ __forceinline__ uint32_t q_pop_or_quit(const Queue& q, uint32_t want, uint64_t& first, uint64_t& hw) {
  unsigned ns = 0;
  if (q_aborted(q) || q_timed_out(q)) return 0;
  for (;;) {
    uint64_t qlen = 0;
    uint32_t n = q_try_pop(q, want, first, qlen);
    if (n) {
      if (qlen > hw) hw = qlen;
      return n;
    }
    // f2: failed pop.  Quiescence: processed (acquire) read BEFORE tail.
    const uint64_t p = ld_acquire_u64(&q.ctl->processed.v);
    const uint64_t t = q_enqueued(q);
    if (p == t) return 0;
    if (q_aborted(q) || q_timed_out(q)) return 0;
    if (ns) __nanosleep(ns);
    ns = ns == 0 ? 32 : (ns < q.backoff_ns ? ns * 2 : ns);
  }
}

// Mark `n` claimed items as fully processed (after all their pushes).
__device__ __forceinline__ void q_done(const Queue& q, uint32_t n) {
  atom_add_release_u64(&q.ctl->processed.v, (uint64_t)n);
}

// Per-worker statistics accumulated in registers and flushed once at exit.
struct LocalStats {
  uint64_t popped = 0, pushed = 0, edges = 0, hw = 0;
  __device__ __forceinline__ void flush(const Queue& q) {
    if (popped) atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->stats[0].v), (unsigned long long)popped);
    if (pushed) atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->stats[1].v), (unsigned long long)pushed);
    if (edges) atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->stats[2].v), (unsigned long long)edges);
    if (hw) atomicMax(reinterpret_cast<unsigned long long*>(&q.ctl->high_water.v), (unsigned long long)hw);
  }
};

}  // namespace atos
