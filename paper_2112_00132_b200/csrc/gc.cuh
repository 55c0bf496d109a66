// gc.cuh — speculative greedy colouring workers.
//
// Asynchronous uberkernel (Alg. 6): a task word is
// ASSIGN(v) = v or CHECK(v) = v | bit31 (R10: the paper's sign trick cannot
// tag vertex 0).
//   ASSIGN(v): pend[v] <- 0 (atomicExch) ; fence ; first-fit: smallest colour
//              not held by any neighbour (window bitmap, R11) ; store
//              color[v] ; __threadfence() (fence.sc: forbids the
//              store-buffering race between two adjacent ASSIGNs) ; push CHECK(v).
//   CHECK(v):  for every neighbour u != v with color[u] == color[v]: let
//              w = max(u, v) (R13 tie-break — the paper-literal "both
//              endpoints recolour" livelocks under lockstep) ; fence ; push
//              ASSIGN(w) only if atomicExch(&pend[w], 1) == 0 (dedupe: at most
//              one pending ASSIGN per vertex, R12).
// BSP variant (Alg. 5): an assign kernel over the frontier (no
// pend, no CHECK push) and a detect kernel that appends v iff some neighbour
// u < v has its colour (R13 applied to Alg. 5).
//
// The forbidden set is a WIN-bit window of colours [base, base+WIN); when a
// vertex sees its whole window used, it rescans with base += WIN.
#pragma once
#include "engine.cuh"

namespace atos {

// Queue items and pend[] are LOCAL vertex ids; colours are indexed by GLOBAL
// id (v + vb).  On one GPU vb = 0 and the range is everything.  On a 1-D
// partition `color` is this rank's replica of all N
// colours (owned entries authoritative, ghosts as last received), a conflict
// whose larger endpoint is remote is left to its owner, and every ASSIGN
// marks chg[v] so the round's end sends the new colour to the neighbours'
// owners (dist_impl.cuh).
struct GcApp {
  int32_t* color;
  uint32_t* pend;
  uint32_t vb = 0, ve = 0xFFFFFFFFu;  // owned global ids [vb, ve)
  uint8_t* chg = nullptr;             // partitioned runs: colour changed this round (local ids)
  __device__ __forceinline__ bool owned(uint32_t u) const { return u >= vb && u < ve; }
  __device__ __forceinline__ void assigned(uint32_t v) const {
    if (chg) chg[v] = 1;
  }
};

enum GcMode : int { GC_UBER = 0, GC_BSP_ASSIGN = 1, GC_BSP_DETECT = 2 };

constexpr int GC_WIN_WORDS = 8;  // 256-colour window per pass (CTA and warp workers)
#ifndef ATOS_GC_WIN_MAX
#define ATOS_GC_WIN_MAX 1024  // largest per-item window of a short CTA batch, in words
#endif

// ------------------------------------------------------------ CTA worker ---
struct GcCtaSmem {
  int64_t* e0;     // [F]
  int64_t* pre;    // [F+1]
  uint32_t* task;  // [F] task word; 0xFFFFFFFF = done/empty
  int32_t* col_v;  // [F] CHECK: colour of v ; ASSIGN: window base
  uint32_t* bits;  // [F * GC_WIN_WORDS] ASSIGN forbidden windows, ww words per item of a batch
  int win_total;   // F * GC_WIN_WORDS
  int32_t* flag;   // [F] CHECK: self-conflict flag ; ASSIGN: needs another pass
  int64_t* wsum;   // [32]
  int32_t* cnt;    // [2]
};

__host__ __device__ constexpr size_t gc_cta_smem_bytes(int F) {
  return (size_t)F * 8 + ((size_t)F + 1) * 8 + (size_t)F * 4 * 3 + (size_t)F * GC_WIN_WORDS * 4 + 32 * 8 + 64;
}

__device__ __forceinline__ GcCtaSmem gc_smem_carve(unsigned char* base, int F) {
  GcCtaSmem s;
  s.e0 = reinterpret_cast<int64_t*>(base);
  s.pre = s.e0 + F;
  s.wsum = s.pre + F + 1;
  s.task = reinterpret_cast<uint32_t*>(s.wsum + 32);
  s.col_v = reinterpret_cast<int32_t*>(s.task + F);
  s.flag = s.col_v + F;
  s.bits = reinterpret_cast<uint32_t*>(s.flag + F);
  s.cnt = reinterpret_cast<int32_t*>(s.bits + (size_t)F * GC_WIN_WORDS);
  s.win_total = F * GC_WIN_WORDS;
  return s;
}

__device__ __forceinline__ int gc_first_free(const uint32_t* w, int words = GC_WIN_WORDS) {
  for (int k = 0; k < words; ++k)
    if (w[k] != 0xFFFFFFFFu) return k * 32 + __ffs(~w[k]) - 1;
  return -1;
}
// Colour-window words per item of a CTA batch of n tasks: the batch's whole
// bitmap area is shared out, so a short batch — typically one hub task in a
// run's tail — scans its neighbours' colours in one pass instead of one pass
// per 256 colours (a hub of RMAT-24 sees ~870 colours).
__device__ __forceinline__ int gc_window_words(int win_total, uint32_t n) {
  const int w = n ? win_total / (int)n : win_total;
  return max(GC_WIN_WORDS, min(ATOS_GC_WIN_MAX, w));
}

template <int MODE, class Src, class Sink>
__device__ void gc_cta_batch(const GcApp& app, const GraphView& g, const Src& src, const Sink& sink, uint32_t n,
                             GcCtaSmem& sm, LocalStats& st) {
  const int T = blockDim.x, tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
  const int ww = gc_window_words(sm.win_total, n);
  // phase 1: read tasks
  bool fenced = false;
  for (int i = tid; i < (int)n; i += T) {
    uint32_t t = 0xFFFFFFFFu;
    if (!src.get(i, t)) t = 0xFFFFFFFFu;
    if (MODE == GC_BSP_DETECT) t |= (t == 0xFFFFFFFFu ? 0u : GC_CHECK_BIT);
    sm.task[i] = t;
    sm.flag[i] = 0;
    if (t != 0xFFFFFFFFu) {
      const uint32_t v = t & ~GC_CHECK_BIT;
      sm.e0[i] = ld_nc_s64(g.off + ATOS_CHK(v, g.n));
      sm.pre[i] = ld_nc_s64(g.off + v + 1) - sm.e0[i];
      if (t & GC_CHECK_BIT) {
        sm.col_v[i] = ld_relaxed_s32(app.color + app.vb + v);
      } else {
        if (MODE == GC_UBER) { atomicExch(app.pend + v, 0u); fenced = true; }
        sm.col_v[i] = 0;  // window base
#pragma unroll
        for (int k = 0; k < ww; ++k) sm.bits[i * ww + k] = 0;
      }
    } else {
      sm.e0[i] = 0;
      sm.pre[i] = 0;
    }
  }
  if (fenced) __threadfence();
  __syncthreads();
  block_exclusive_scan(sm.pre, (int)n, sm.wsum);
  uint64_t edges = 0;
  uint32_t pushed = 0;
  // ASSIGN items may need several window passes; CHECK items take one.
  for (int pass = 0;; ++pass) {
    const int64_t total = sm.pre[n];
    edges += (tid == 0) ? (uint64_t)total : 0;
    for (int64_t eb = (int64_t)wid * 32; eb < total; eb += T) {
      const int64_t e = eb + lane;
      bool act = false;
      uint32_t push_item = 0;
      if (e < total) {
        const int i = lbs_find(sm.pre, (int)n, e);
        const uint32_t t = sm.task[i];
        const uint32_t v = (t & ~GC_CHECK_BIT) + app.vb;  // global id
        const uint32_t u = (uint32_t)ld_stream_s32(g.col + ATOS_CHK(sm.e0[i] + (e - sm.pre[i]), g.col_cap));
        if (u != v) {
          const int32_t cu = ld_relaxed_s32(app.color + u);
          if (t & GC_CHECK_BIT) {
            if (cu == sm.col_v[i]) {
              if (MODE == GC_BSP_DETECT) {
                if (u < v) sm.flag[i] = 1;
              } else if (u < v) {
                sm.flag[i] = 1;  // v itself must recolour (one push per task, R12)
              } else if (app.owned(u)) {  // a remote larger endpoint is its owner's to recolour
                __threadfence();
                if (atomicExch(app.pend + (u - app.vb), 1u) == 0u) { act = true; push_item = u - app.vb; }
              }
            }
          } else {
            const int32_t r = cu - sm.col_v[i];
            if (r >= 0 && r < 32 * ww) atomicOr(sm.bits + i * ww + (r >> 5), 1u << (r & 31));
          }
        }
      }
      if (MODE == GC_UBER) pushed += sink.warp_push(act, push_item);
    }
    __syncthreads();
    // resolve: ASSIGN items pick a colour or need another pass
    if (tid == 0) sm.cnt[0] = 0;
    __syncthreads();
    int again = 0;
    bool stored = false;
    for (int i = tid; i < (int)n; i += T) {
      const uint32_t t = sm.task[i];
      int64_t deg = 0;
      if (t != 0xFFFFFFFFu && !(t & GC_CHECK_BIT)) {
        const int f = gc_first_free(sm.bits + i * ww, ww);
        const uint32_t v = t;
        if (f >= 0) {
          st_relaxed_s32(app.color + app.vb + v, sm.col_v[i] + f);
          app.assigned(v);
          stored = true;
          sm.flag[i] = 2;  // assigned in this batch
        } else {
          sm.col_v[i] += 32 * ww;
          for (int k = 0; k < ww; ++k) sm.bits[i * ww + k] = 0;
          deg = ld_nc_s64(g.off + v + 1) - sm.e0[i];
          again = 1;
        }
      }
      if (pass == 0 || true) sm.pre[i] = deg;  // next pass visits only unresolved ASSIGNs
    }
    if (stored) __threadfence();  // colour stores before CHECK pushes (fence.sc)
    if (again) atomicOr(sm.cnt, 1);
    __syncthreads();
    const bool more = sm.cnt[0] != 0;
    if (!more) break;
    block_exclusive_scan(sm.pre, (int)n, sm.wsum);
  }
  // final pushes: CHECK(v) for assigned, ASSIGN(v) for self-conflicted CHECKs
  for (int ib = wid * 32; ib < (int)n; ib += T) {
    const int i = ib + lane;
    bool act = false;
    uint32_t item = 0;
    if (i < (int)n) {
      const uint32_t t = sm.task[i];
      if (t != 0xFFFFFFFFu) {
        const uint32_t v = t & ~GC_CHECK_BIT;
        if (MODE == GC_UBER) {
          if (!(t & GC_CHECK_BIT)) {
            act = true;
            item = v | GC_CHECK_BIT;
          } else if (sm.flag[i] == 1) {
            __threadfence();
            if (atomicExch(app.pend + v, 1u) == 0u) { act = true; item = v; }
          }
        } else if (MODE == GC_BSP_DETECT) {
          act = sm.flag[i] == 1;
          item = v;
        }
      }
    }
    if (MODE != GC_BSP_ASSIGN) pushed += sink.warp_push(act, item);
  }
  if (lane == 0) st.pushed += pushed;
  if (tid == 0) st.edges += edges;
  __syncthreads();
}

// ----------------------------------------------------------- warp worker ---
// One task at a time per warp; lanes stride the neighbour list; the 256-colour
// window is OR-reduced across the warp.
template <int MODE, class Sink>
__device__ __forceinline__ uint32_t gc_warp_task(const GcApp& app, const GraphView& g, const Sink& sink, uint32_t t,
                                                 uint64_t& edges) {
  const int lane = lane_id();
  const uint32_t v = t & ~GC_CHECK_BIT;  // local id
  const uint32_t vg = v + app.vb;        // global id
  const int64_t e0 = ld_nc_s64(g.off + ATOS_CHK(v, g.n)), e1 = ld_nc_s64(g.off + v + 1);
  uint32_t pushed = 0;
  if (t & GC_CHECK_BIT) {
    const int32_t c = ld_relaxed_s32(app.color + vg);
    bool self = false;
    edges += e1 - e0;
    for (int64_t eb = e0; eb < e1; eb += 32) {
      const int64_t e = eb + lane;
      bool act = false;
      uint32_t u = 0;
      if (e < e1) {
        u = (uint32_t)ld_stream_s32(g.col + ATOS_CHK(e, g.col_cap));
        if (u != vg && ld_relaxed_s32(app.color + u) == c) {
          if (u < vg) self = true;
          else if (MODE == GC_UBER && app.owned(u)) {
            __threadfence();
            act = atomicExch(app.pend + (u - app.vb), 1u) == 0u;
          }
        }
      }
      if (MODE == GC_UBER) pushed += sink.warp_push(act, u - app.vb);
    }
    self = __any_sync(FULL_MASK, self);
    bool act = false;
    if (self && lane == 0) {
      if (MODE == GC_UBER) {
        __threadfence();
        act = atomicExch(app.pend + v, 1u) == 0u;
      } else {
        act = true;
      }
    }
    pushed += sink.warp_push(act, v);
    return pushed;
  }
  // ASSIGN(v)
  if (MODE == GC_UBER && lane == 0) {
    atomicExch(app.pend + v, 0u);
    __threadfence();
  }
  __syncwarp();
  int32_t base = 0;
  int32_t chosen = -1;
  while (chosen < 0) {
    uint32_t m[GC_WIN_WORDS];
#pragma unroll
    for (int k = 0; k < GC_WIN_WORDS; ++k) m[k] = 0;
    edges += e1 - e0;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const uint32_t u = (uint32_t)ld_stream_s32(g.col + ATOS_CHK(e, g.col_cap));
      if (u == vg) continue;
      const int32_t r = ld_relaxed_s32(app.color + u) - base;
      if (r >= 0 && r < 32 * GC_WIN_WORDS) {
#pragma unroll
        for (int k = 0; k < GC_WIN_WORDS; ++k) m[k] |= ((r >> 5) == k) ? (1u << (r & 31)) : 0u;
      }
    }
#pragma unroll
    for (int k = 0; k < GC_WIN_WORDS; ++k) m[k] = __reduce_or_sync(FULL_MASK, m[k]);
    const int f = gc_first_free(m);
    if (f >= 0) chosen = base + f;
    else base += 32 * GC_WIN_WORDS;
  }
  bool act = false;
  if (lane == 0) {
    st_relaxed_s32(app.color + vg, chosen);
    app.assigned(v);
    __threadfence();
    act = (MODE == GC_UBER);
  }
  pushed += (MODE == GC_UBER) ? sink.warp_push(act, v | GC_CHECK_BIT) : 0u;
  return pushed;
}

// ---------------------------------------------------------- thread worker ---
// One task per lane, serial neighbour walks, 64-colour register window.
template <int MODE, class Sink>
__device__ __forceinline__ uint32_t gc_thread_task(const GcApp& app, const GraphView& g, const Sink& sink,
                                                   bool valid, uint32_t t, uint64_t& edges) {
  uint32_t pushed = 0;
  const uint32_t v = t & ~GC_CHECK_BIT;  // local id
  const uint32_t vg = v + app.vb;        // global id
  int64_t e0 = 0, e1 = 0;
  if (valid) { e0 = ld_nc_s64(g.off + ATOS_CHK(v, g.n)); e1 = ld_nc_s64(g.off + v + 1); }
  const bool is_check = valid && (t & GC_CHECK_BIT);
  const bool is_assign = valid && !(t & GC_CHECK_BIT);
  // CHECK
  {
    const int32_t c = is_check ? ld_relaxed_s32(app.color + vg) : 0;
    bool self = false;
    int64_t e = is_check ? e0 : 0, ee = is_check ? e1 : 0;
    if (is_check) edges += ee - e;
    while (__any_sync(FULL_MASK, e < ee)) {
      bool act = false;
      uint32_t u = 0;
      if (e < ee) {
        u = (uint32_t)ld_stream_s32(g.col + ATOS_CHK(e, g.col_cap));
        ++e;
        if (u != vg && ld_relaxed_s32(app.color + u) == c) {
          if (u < vg) self = true;
          else if (MODE == GC_UBER && app.owned(u)) {
            __threadfence();
            act = atomicExch(app.pend + (u - app.vb), 1u) == 0u;
          }
        }
      }
      if (MODE == GC_UBER) pushed += sink.warp_push(act, u - app.vb);
    }
    bool act = false;
    if (self) {
      if (MODE == GC_UBER) {
        __threadfence();
        act = atomicExch(app.pend + v, 1u) == 0u;
      } else {
        act = true;
      }
    }
    if (MODE != GC_BSP_ASSIGN) pushed += sink.warp_push(act, v);
  }
  // ASSIGN
  {
    if (is_assign && MODE == GC_UBER) {
      atomicExch(app.pend + v, 0u);
      __threadfence();
    }
    int32_t base = 0, chosen = is_assign ? -1 : 0;
    while (__any_sync(FULL_MASK, chosen < 0)) {
      uint64_t m = 0;
      int64_t e = chosen < 0 ? e0 : 0, ee = chosen < 0 ? e1 : 0;
      edges += ee - e;
      for (; e < ee; ++e) {
        const uint32_t u = (uint32_t)ld_stream_s32(g.col + ATOS_CHK(e, g.col_cap));
        if (u == vg) continue;
        const int32_t r = ld_relaxed_s32(app.color + u) - base;
        if (r >= 0 && r < 64) m |= 1ull << r;
      }
      if (chosen < 0) {
        if (~m) chosen = base + __ffsll((long long)~m) - 1;
        else base += 64;
      }
    }
    bool act = false;
    if (is_assign) {
      st_relaxed_s32(app.color + vg, chosen);
      app.assigned(v);
      __threadfence();
      act = (MODE == GC_UBER);
    }
    if (MODE == GC_UBER) pushed += sink.warp_push(act, v | GC_CHECK_BIT);
  }
  return pushed;
}

}  // namespace atos
