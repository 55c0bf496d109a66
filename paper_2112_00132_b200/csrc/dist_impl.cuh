// dist_impl.cuh — multi-GPU BFS / PageRank over a 1-D vertex partition
// (SURVEY §8e), included at the end of capi.cu.
//
// Every rank runs the single-GPU persistent queue kernel (same queue, same
// workers) over its own vertices; the apps below route each relaxed update to
// the local state or, for a vertex owned by another rank, to a per-round
// outbox.  The caller exchanges outboxes with an all-to-all (torch.distributed
// over NCCL/NVLink) and applies what arrives (atos_part_apply); a round with no
// message anywhere ends the run.  Queue items are LOCAL vertex ids; columns are
// global ids.

namespace atos {

// Owner of global vertex w among `world` contiguous blocks (bounds[world+1]).
__device__ __forceinline__ int owner_of(const int64_t* bounds, int world, uint32_t w) {
  int lo = 0, hi = world;  // bounds[lo] <= w < bounds[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if ((int64_t)w >= bounds[mid]) lo = mid; else hi = mid;
  }
  return lo;
}

struct Outbox {
  uint64_t* buf;                // per-destination segments
  const int64_t* seg;           // segment start per destination (world + 1)
  unsigned long long* cnt;      // messages per destination this round
  unsigned int* overflow;
  __device__ __forceinline__ void put(int r, uint64_t msg) const {
    const unsigned long long i = atomicAdd(cnt + r, 1ull);
    if ((int64_t)i < seg[r + 1] - seg[r]) buf[seg[r] + (int64_t)i] = msg;
    else atomicOr(overflow, 1u);
  }
};

// BFS on a partition: dist/done are local; sent_min (global n) filters remote
// sends so a remote vertex is sent once per improvement of its tentative depth.
struct BfsPartApp {
  static constexpr bool kWindow = false;
  uint32_t* dist;
  uint32_t* done;
  uint32_t* sent_min;
  int filter;
  uint32_t vb, ve;
  const int64_t* bounds;
  int world;
  Outbox out;
  using Payload = uint32_t;
  using Probe = uint32_t;
  using Raw = uint32_t;
  __device__ __forceinline__ bool local(uint32_t w) const { return w >= vb && w < ve; }
  __device__ __forceinline__ uint32_t item_of(uint32_t w) const { return w - vb; }
  __device__ __forceinline__ bool chunk_current(uint32_t v, Payload nd) const { return ld_relaxed_u32(dist + v) + 1u >= nd; }
  struct Pre {
    int64_t e0, e1;
    uint32_t d;
  };
  __device__ __forceinline__ Pre begin_load(uint32_t v, const GraphView& g) const {
    Pre x;
    x.e0 = ld_nc_s64(g.off + v);
    x.e1 = ld_nc_s64(g.off + v + 1);
    x.d = ld_relaxed_hot(dist + v);
    return x;
  }
  __device__ __forceinline__ bool begin_commit(uint32_t v, const Pre& x, Payload& p) const {
    p = x.d + 1u;
    if (x.e1 == x.e0) return false;
    return atomicMin(done + v, x.d) > x.d;
  }
  __device__ __forceinline__ bool begin(uint32_t v, const GraphView& g, int64_t& e0, int64_t& e1, Payload& p) const {
    Pre x = begin_load(v, g);
    e0 = x.e0;
    e1 = x.e1;
    return begin_commit(v, x, p);
  }
  __device__ __forceinline__ Probe probe(uint32_t w) const {
    if (!filter) return 0xFFFFFFFFu;
    return local(w) ? ld_probe_hot(dist + (w - vb)) : ld_probe_hot(sent_min + w);
  }
  __device__ __forceinline__ Raw issue(Payload nd, uint32_t w, Probe pr) const {
    if (nd >= pr) return 0u;
    return local(w) ? atom_min_hot(dist + (w - vb), nd) : atom_min_hot(sent_min + w, nd);
  }
  __device__ __forceinline__ bool decide(Payload nd, uint32_t w, Probe pr, Raw old) const {
    if (nd >= pr || nd >= old) return false;
    if (local(w)) return true;
    const int r = owner_of(bounds, world, w);
    out.put(r, ((uint64_t)(w - (uint32_t)bounds[r]) << 32) | nd);
    return false;
  }
  __device__ __forceinline__ bool commit(Payload nd, uint32_t w, Probe pr) const { return decide(nd, w, pr, issue(nd, w, pr)); }
  __device__ __forceinline__ bool edge(Payload nd, uint32_t w) const { return commit(nd, w, probe(w)); }
};

// PageRank on a partition: residues of remote vertices accumulate in racc
// (global n, fp32) and are flushed as messages at the end of every round.
template <class R>
struct PrPartAppT {
  static constexpr bool kWindow = false;
  double* rank;
  R* res;
  R alpha, eps;
  uint32_t vb, ve;
  float* racc;
  using Payload = R;
  using Probe = int;
  using Raw = R;
  __device__ __forceinline__ bool local(uint32_t w) const { return w >= vb && w < ve; }
  __device__ __forceinline__ uint32_t item_of(uint32_t w) const { return w - vb; }
  __device__ __forceinline__ bool chunk_current(uint32_t, Payload) const { return true; }
  struct Pre {
    int64_t e0, e1;
    R r;
  };
  __device__ __forceinline__ Pre begin_load(uint32_t v, const GraphView& g) const {
    Pre x;
    x.e0 = ld_nc_s64(g.off + v);
    x.e1 = ld_nc_s64(g.off + v + 1);
    x.r = atomic_take(res + v);
    return x;
  }
  __device__ __forceinline__ bool begin_commit(uint32_t v, const Pre& x, Payload& p) const {
    if (x.r == R(0)) return false;
    red_add_cold(rank + v, (double)x.r);
    if (x.e1 == x.e0) return false;
    p = alpha * x.r / (R)(x.e1 - x.e0);
    return true;
  }
  __device__ __forceinline__ bool begin(uint32_t v, const GraphView& g, int64_t& e0, int64_t& e1, Payload& p) const {
    Pre x = begin_load(v, g);
    e0 = x.e0;
    e1 = x.e1;
    return begin_commit(v, x, p);
  }
  __device__ __forceinline__ Probe probe(uint32_t) const { return 0; }
  __device__ __forceinline__ Raw issue(Payload c, uint32_t w, Probe) const {
    if (local(w)) return atom_add_hot(res + (w - vb), c);
    atomicAdd(racc + w, (float)c);
    return R(1e30);  // never a crossing
  }
  __device__ __forceinline__ bool decide(Payload c, uint32_t w, Probe, Raw old) const {
    return local(w) && old <= eps && add_rn(old, c) > eps;
  }
  __device__ __forceinline__ bool commit(Payload c, uint32_t w, Probe p) const { return decide(c, w, p, issue(c, w, p)); }
  __device__ __forceinline__ bool edge(Payload c, uint32_t w) const { return commit(c, w, 0); }
};

// PR residue seeding on a partition (R4): local targets add to res, remote to racc.
template <class R>
struct PrPartInitAppT {
  static constexpr bool kWindow = false;
  R* res;
  R* racc;
  R c0;
  uint32_t vb, ve;
  using Payload = R;
  using Probe = int;
  using Raw = int;
  __device__ __forceinline__ uint32_t item_of(uint32_t w) const { return w; }
  __device__ __forceinline__ bool chunk_current(uint32_t, Payload) const { return true; }
  __device__ __forceinline__ bool begin(uint32_t v, const GraphView& g, int64_t& e0, int64_t& e1, Payload& p) const {
    e0 = ld_nc_s64(g.off + v);
    e1 = ld_nc_s64(g.off + v + 1);
    if (e1 == e0) return false;
    p = c0 / (R)(e1 - e0);
    return true;
  }
  __device__ __forceinline__ Probe probe(uint32_t) const { return 0; }
  __device__ __forceinline__ Raw issue(Payload c, uint32_t w, Probe) const {
    if (w >= vb && w < ve) atomicAdd(res + (w - vb), c);
    else atomicAdd(racc + w, c);
    return 0;
  }
  __device__ __forceinline__ bool decide(Payload, uint32_t, Probe, Raw) const { return false; }
  __device__ __forceinline__ bool commit(Payload c, uint32_t w, Probe p) const { return decide(c, w, p, issue(c, w, p)); }
  __device__ __forceinline__ bool edge(Payload c, uint32_t w) const { return commit(c, w, 0); }
};

// Flush remote PR accumulations of destination r's range into messages: only
// those above `thr` (= eps) in a regular round — a smaller amount cannot
// re-activate its target on its own and keeps accumulating at the sender — and
// everything (thr = 0) in a closing round, so no mass is stranded.
__global__ void k_pr_flush(float* racc, int64_t b0, int64_t b1, int r, Outbox out, float thr) {
  for (int64_t w = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < b1; w += (int64_t)gridDim.x * blockDim.x) {
    const float v = racc[w];
    if (v != 0.0f && v > thr) {
      racc[w] = 0.0f;
      out.put(r, ((uint64_t)(uint32_t)(w - b0) << 32) | (uint64_t)__float_as_uint(v));
    }
  }
}

// Pack the per-destination segments contiguously (rank order).
__global__ void k_part_pack(const uint64_t* buf, const int64_t* seg, const unsigned long long* cnt, int world,
                            uint64_t* dst) {
  int64_t base = 0;
  for (int r = 0; r < world; ++r) {
    const int64_t c = (int64_t)cnt[r];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c; i += (int64_t)gridDim.x * blockDim.x)
      dst[base + i] = buf[seg[r] + i];
    base += c;
  }
}

// Apply received messages: BFS atomicMin + push; PR atomicAdd + push on a crossing.
template <int APP, class R>
__global__ void k_part_apply(const uint64_t* msgs, int64_t count, uint32_t* dist, R* res, R eps, Queue q) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; b < count; b += stride) {
    const int64_t i = b + lane_id();
    bool act = false;
    uint32_t l = 0;
    if (i < count) {
      const uint64_t m = msgs[i];
      l = (uint32_t)(m >> 32);
      const uint32_t pay = (uint32_t)m;
      if (APP == 0) {
        act = pay < atomicMin(dist + l, pay);
      } else {
        const R c = (R)__uint_as_float(pay);
        const R old = atomicAdd(res + l, c);
        act = old <= eps && add_rn(old, c) > eps;
      }
    }
    q_warp_push(q, act, l);
  }
}

// ------------------------------------------------ partitioned colouring (f4)
// Round structure: every rank runs the uberkernel (Alg. 6)
// on its own vertices to local quiescence, reading neighbours' colours from a
// replica of all N colours (ghost entries as last received).  At the round's
// end each vertex whose colour changed sends (global id, colour) once to every
// other rank owning one of its neighbours; the receiver updates its replica
// and re-checks its vertices against the changed ghosts: a local v whose
// colour equals a changed neighbour u's and v > u is re-ASSIGNed (R13 across
// ranks: the larger endpoint recolours, so the smallest id in a conflict
// never moves and the rounds terminate).  A cut edge left monochromatic would
// need its larger endpoint's owner to have missed the other endpoint's last
// change, which every change is sent to — so the final colouring is proper.

// One warp per changed local vertex: the set of remote owners of its
// neighbours (columns are sorted global ids; owners are a 64-bit mask, world
// <= 64) gets one message (vg << 32 | colour) each.
__global__ void k_gc_pack(const GraphView g, const int32_t* color, uint8_t* chg, uint32_t vb, const int64_t* bounds,
                          int world, int rank, Outbox out) {
  const int lane = lane_id();
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t base = warp * 32; base < g.n; base += nwarps * 32) {
    const int64_t my = base + lane;
    const bool c = my < g.n && chg[my];
    unsigned todo = __ballot_sync(FULL_MASK, c);
    if (c) chg[my] = 0;
    while (todo) {
      const int j = __ffs(todo) - 1;
      todo &= todo - 1;
      const uint32_t v = (uint32_t)(base + j);
      const int64_t e0 = ld_nc_s64(g.off + v), e1 = ld_nc_s64(g.off + v + 1);
      unsigned long long mask = 0;
      for (int64_t e = e0 + lane; e < e1; e += 32) {
        const int r = owner_of(bounds, world, (uint32_t)g.col[e]);
        if (r != rank) mask |= 1ull << r;
      }
#pragma unroll
      for (int d = 16; d; d >>= 1) mask |= __shfl_xor_sync(FULL_MASK, mask, d);
      const uint32_t c_v = (uint32_t)ld_relaxed_s32(color + vb + v);
      const unsigned long long msg = ((unsigned long long)(vb + v) << 32) | c_v;
      for (int r = lane; r < world; r += 32)
        if ((mask >> r) & 1ull) out.put(r, msg);
    }
  }
}

// Received ghost colours: replica update + changed-ghost mark.
__global__ void k_gc_apply(const uint64_t* msgs, int64_t count, int32_t* color, uint8_t* gchg, uint8_t val) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t m = msgs[i];
    const uint32_t u = (uint32_t)(m >> 32);
    if (val) color[u] = (int32_t)(uint32_t)m;
    gchg[u] = val;
  }
}

// Re-check every local vertex against the ghosts that changed this round
// (warp per vertex): a conflict with a smaller changed ghost re-ASSIGNs v
// (pend dedupe, as a local CHECK would).
__global__ void k_gc_ghost_scan(const GraphView g, const int32_t* color, const uint8_t* gchg, uint32_t* pend,
                                uint32_t vb, Queue q) {
  const int lane = lane_id();
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < g.n; v += nwarps) {
    const uint32_t vg = vb + (uint32_t)v;
    const int64_t e0 = ld_nc_s64(g.off + v), e1 = ld_nc_s64(g.off + v + 1);
    const int32_t cv = ld_relaxed_s32(color + vg);
    bool hit = false;
    for (int64_t e = e0 + lane; e < e1 && !hit; e += 32) {
      const uint32_t u = (uint32_t)g.col[e];
      hit = u < vg && gchg[u] && color[u] == cv;
    }
    hit = __any_sync(FULL_MASK, hit);
    bool act = false;
    if (hit && lane == 0) {
      __threadfence();
      act = atomicExch(pend + v, 1u) == 0u;
    }
    q_warp_push(q, act, (uint32_t)v);
  }
}

}  // namespace atos

struct DistState {
  int world = 1, rank = 0;
  std::vector<int64_t> bounds;
  int64_t* d_bounds = nullptr;
  int64_t* d_seg = nullptr;
  std::vector<int64_t> seg;
  uint64_t* outbox = nullptr;
  unsigned long long* d_cnt = nullptr;  // [world] + overflow flag
  unsigned long long* h_cnt = nullptr;  // pinned
  uint32_t* sent_min = nullptr;
  float* racc = nullptr;
  double* racc64 = nullptr;     // seeding sums of remote targets (R30), rounded into racc
  int32_t* gc_color = nullptr;  // colouring: replica of all N colours
  uint8_t* gc_chg = nullptr;    // colouring: local vertex changed colour this round
  uint8_t* gc_gchg = nullptr;   // colouring: ghost changed this round (global ids)
  int app = -1;
  float alpha = 0.85f, eps = 1e-6f;
  atos_config cfg{};
  int64_t rounds = 0, bytes_sent = 0, launches = 0;
  double ms = 0, kernel_ms = 0;
  bool r64 = false;
  uint64_t next_h = 0;  // discrete rounds: first unprocessed queue position
};

void dist_free(atos_graph g) {
  if (!g || !g->dist) return;
  DistState* d = g->dist;
  cudaFree(d->d_bounds);
  cudaFree(d->d_seg);
  cudaFree(d->outbox);
  cudaFree(d->d_cnt);
  if (d->h_cnt) cudaFreeHost(d->h_cnt);
  cudaFree(d->sent_min);
  cudaFree(d->racc);
  cudaFree(d->racc64);
  cudaFree(d->gc_color);
  cudaFree(d->gc_chg);
  cudaFree(d->gc_gchg);
  delete d;
  g->dist = nullptr;
}

extern "C" atos_status atos_graph_create_partitioned(int64_t global_n, int32_t world, int32_t rank,
                                                     const int64_t* bounds, const int64_t* off, const int32_t* col,
                                                     int64_t m, uint32_t flags, atos_graph* out) {
  if (!out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "out == NULL");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world || !bounds || global_n < 0 || m < 0 || !off || (m > 0 && !col))
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bad partition arguments");
  if (global_n >= 0x7FFFFFFFLL) return atos_set_error(ATOS_ERR_UNSUPPORTED, "global_n >= 2^31-1");
  if (bounds[0] != 0 || bounds[world] != global_n)
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bounds[0] != 0 or bounds[world] != global_n");
  for (int r = 0; r < world; ++r)
    if (bounds[r + 1] < bounds[r]) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bounds not monotone");
  const int64_t vb = bounds[rank], ve = bounds[rank + 1], n = ve - vb;
  atos_graph g = new (std::nothrow) atos_graph_s();
  if (!g) return atos_set_error(ATOS_ERR_OUT_OF_MEMORY, "host allocation");
  atos_status s = graph_init_common(g, off, col, n, m, flags & ~(uint32_t)ATOS_GRAPH_BORROW, global_n);
  if (s != ATOS_OK) {
    graph_free(g);
    return s;
  }
  g->global_n = global_n;
  g->v_begin = vb;
  g->v_end = ve;
  DistState* d = new (std::nothrow) DistState();
  if (!d) {
    graph_free(g);
    return atos_set_error(ATOS_ERR_OUT_OF_MEMORY, "host allocation");
  }
  g->dist = d;
  d->world = world;
  d->rank = rank;
  d->bounds.assign(bounds, bounds + world + 1);
  // outbox segment r: room for 2x destination r's vertex count (BFS sends each
  // remote vertex once per improvement; PR flushes each at most once per round)
  d->seg.assign(world + 1, 0);
  for (int r = 0; r < world; ++r) d->seg[r + 1] = d->seg[r] + (r == rank ? 0 : 2 * (bounds[r + 1] - bounds[r]) + 1024);
  auto fail = [&](atos_status st) {
    graph_free(g);
    return st;
  };
  if (cudaMalloc(&d->d_bounds, (world + 1) * sizeof(int64_t)) != cudaSuccess ||
      cudaMalloc(&d->d_seg, (world + 1) * sizeof(int64_t)) != cudaSuccess ||
      cudaMalloc(&d->outbox, std::max<int64_t>(d->seg[world], 1) * sizeof(uint64_t)) != cudaSuccess ||
      cudaMalloc(&d->d_cnt, (world + 1) * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMallocHost(&d->h_cnt, (world + 1) * sizeof(unsigned long long)) != cudaSuccess)
    return fail(atos_set_error(ATOS_ERR_OUT_OF_MEMORY, "partition buffers"));
  cudaMemcpy(d->d_bounds, bounds, (world + 1) * sizeof(int64_t), cudaMemcpyHostToDevice);
  cudaMemcpy(d->d_seg, d->seg.data(), (world + 1) * sizeof(int64_t), cudaMemcpyHostToDevice);
  if (cudaGetLastError() != cudaSuccess) return fail(atos_set_error(ATOS_ERR_CUDA, "partition setup copy"));
  *out = g;
  return ATOS_OK;
}

static atos_status part_ctx(atos_graph g, LaunchCtx& c) {
  if (!g || !g->dist) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "not a partitioned graph");
  if (g->dist->app < 0) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "atos_part_begin not called");
  c.g = g;
  c.cfg = g->dist->cfg;
  c.s = reinterpret_cast<cudaStream_t>(c.cfg.stream);
  c.gv = GraphView{g->d_off, g->d_col, g->n, g->col_cap};
  c.t0 = std::chrono::steady_clock::now();
  return ATOS_OK;
}

extern "C" atos_status atos_part_begin(atos_graph g, int32_t app, int64_t src, float alpha, float eps,
                                       const atos_config* cfg) {
  LaunchCtx c;
  CKS(begin_call(g, cfg, c, nullptr));
  if (!g->dist) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "not a partitioned graph");
  DistState* d = g->dist;
  if (app < 0 || app > 2)
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "app must be 0 (BFS), 1 (PageRank) or 2 (colouring)");
  if (app == 2 && !g->symmetric)
    return atos_set_error(ATOS_ERR_INVALID_GRAPH, "partitioned colouring needs ATOS_GRAPH_SYMMETRIC");
  if (app == 2 && d->world > 64) return atos_set_error(ATOS_ERR_UNSUPPORTED, "partitioned colouring: world > 64");
  if (app == 2 && c.cfg.worker != ATOS_WORKER_CTA && c.cfg.worker != ATOS_WORKER_WARP && c.cfg.worker != ATOS_WORKER_THREAD)
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bad worker");
  if (app == 0 && (src < 0 || src >= g->global_n)) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "src out of range");
  if (app == 1 && (!(alpha > 0.f && alpha < 1.f) || !(eps > 0.f)))
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "alpha/eps");
  if (c.cfg.kernel == ATOS_KERNEL_BSP)
    return atos_set_error(ATOS_ERR_UNSUPPORTED, "partitioned runs use the persistent or discrete kernel");
  d->next_h = 0;
  d->app = app;
  d->alpha = alpha;
  d->eps = eps;
  d->cfg = c.cfg;
  d->rounds = d->bytes_sent = d->launches = 0;
  d->ms = d->kernel_ms = 0;
  d->r64 = c.cfg.pr_residue_fp64 != 0;
  const int64_t n = g->n, N = g->global_n;
  Workspace& w = g->ws;
  CKS(ws_prepare(g, c.cfg, n, (app == 2 ? 4 : 2) * (uint64_t)std::max<int64_t>(n, 1), true, c.s));
  if (app >= 1 && (uint64_t)n > w.cap) return atos_set_error(ATOS_ERR_QUEUE_OVERFLOW, "queue_capacity < n");
  CK(cudaMemsetAsync(d->d_cnt, 0, (d->world + 1) * sizeof(unsigned long long), c.s));
  CK(cudaEventRecord(w.ev[0], c.s));
  if (app == 0) {
    CKS(ensure(w.u32a, w.u32a_n, (size_t)std::max<int64_t>(n, 1)));
    CKS(ensure(w.u32b, w.u32b_n, (size_t)std::max<int64_t>(n, 1)));
    if (!d->sent_min) CK(cudaMalloc(&d->sent_min, (size_t)N * sizeof(uint32_t)));
    const bool mine = src >= g->v_begin && src < g->v_end;
    k_bfs_init<<<fill_blocks(std::max<int64_t>(n, 1), g->sms), 256, 0, c.s>>>(w.u32a, w.u32b, nullptr, n,
                                                                               mine ? src - g->v_begin : -1);
    k_fill<uint32_t><<<fill_blocks(N, g->sms), 256, 0, c.s>>>(d->sent_min, N, 0xFFFFFFFFu);
    k_ctl_init<<<1, 1, 0, c.s>>>(w.ctl, mine ? 1 : 0, w.ring, mine ? src - g->v_begin : -1);
    d->launches += 3;
  } else if (app == 2) {
    // colouring: replica colours -1, pend = 1 (every vertex has its initial ASSIGN queued), ASSIGN(v) in id order
    CKS(ensure(w.u32a, w.u32a_n, (size_t)std::max<int64_t>(n, 1)));
    if (!d->gc_color) CK(cudaMalloc(&d->gc_color, (size_t)std::max<int64_t>(N, 1) * sizeof(int32_t)));
    if (!d->gc_gchg) {
      CK(cudaMalloc(&d->gc_gchg, (size_t)std::max<int64_t>(N, 1)));
      CK(cudaMemsetAsync(d->gc_gchg, 0, (size_t)std::max<int64_t>(N, 1), c.s));
    }
    if (!d->gc_chg) CK(cudaMalloc(&d->gc_chg, (size_t)std::max<int64_t>(n, 1)));
    CK(cudaMemsetAsync(d->gc_chg, 0, (size_t)std::max<int64_t>(n, 1), c.s));
    k_fill<int32_t><<<fill_blocks(std::max<int64_t>(N, 1), g->sms), 256, 0, c.s>>>(d->gc_color, N, -1);
    k_fill<uint32_t><<<fill_blocks(std::max<int64_t>(n, 1), g->sms), 256, 0, c.s>>>(w.u32a, n, 1u);
    k_ctl_init<<<1, 1, 0, c.s>>>(w.ctl, (uint64_t)n, w.ring, -1);
    if (n) k_ring_prefill<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.ring, n, 0u);
    d->launches += 4;
  } else {
    CKS(ensure(w.f32a, w.f32a_n, (size_t)std::max<int64_t>(n, 1)));
    CKS(ensure(w.f64a, w.f64a_n, (size_t)std::max<int64_t>(n, 1)));
    CKS(ensure(w.f64b, w.f64b_n, (size_t)std::max<int64_t>(n, 1)));  // residues or the fp64 seeding sums (R30)
    if (!d->r64) CKS(ensure(w.f32b, w.f32b_n, (size_t)std::max<int64_t>(n, 1)));
    if (!d->racc) CK(cudaMalloc(&d->racc, (size_t)N * sizeof(float)));
    CK(cudaMemsetAsync(d->racc, 0, (size_t)N * sizeof(float), c.s));
    k_fill<double><<<fill_blocks(std::max<int64_t>(n, 1), g->sms), 256, 0, c.s>>>(w.f64a, n, 1.0 - (double)alpha);
    k_ctl_init<<<1, 1, 0, c.s>>>(w.ctl, (uint64_t)n, w.ring, -1);
    if (n) k_ring_prefill<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.ring, n, 0u);
    // R30: local seeding sums accumulate in fp64 and are rounded once (remote ones go to racc)
    if (n) {
      k_fill<double><<<fill_blocks(std::max<int64_t>(n, 1), g->sms), 256, 0, c.s>>>(w.f64b, n, 0.0);
      if (!d->racc64) CK(cudaMalloc(&d->racc64, (size_t)N * sizeof(double)));
      k_fill<double><<<fill_blocks(N, g->sms), 256, 0, c.s>>>(d->racc64, N, 0.0);
      PrPartInitAppT<double> ia{w.f64b, d->racc64, (1.0 - (double)alpha) * (double)alpha, (uint32_t)g->v_begin,
                                (uint32_t)g->v_end};
      LaunchCtx ci = c;
      ci.cfg.worker = ATOS_WORKER_CTA;
      CKS((bsp_step_w<EdgeMapPolicy<PrPartInitAppT<double>>, PrPartInitAppT<double>, W_CTA>(
          ci, ia, nullptr, (uint64_t)n, nullptr, nullptr, 256, nullptr)));
      if (!d->r64) k_f64_to_res<float><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.f64b, w.f32b, n);
      k_f64_to_res<float><<<fill_blocks(N, g->sms), 256, 0, c.s>>>(d->racc64, d->racc, N);
    }
    d->launches += n ? (d->r64 ? 7 : 8) : 2;
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(w.ev[1], c.s));
  CK(cudaStreamSynchronize(c.s));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, w.ev[0], w.ev[1]));
  d->ms += ms;
  return ATOS_OK;
}

extern "C" atos_status atos_part_run(atos_graph g, int32_t flush_all, int64_t* send_counts) {
  LaunchCtx c;
  CKS(part_ctx(g, c));
  DistState* d = g->dist;
  if (!send_counts) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "send_counts == NULL");
  Workspace& w = g->ws;
  Outbox ob{d->outbox, d->d_seg, d->d_cnt, reinterpret_cast<unsigned int*>(d->d_cnt + d->world)};
  CK(cudaMemsetAsync(d->d_cnt, 0, (d->world + 1) * sizeof(unsigned long long), c.s));
  CK(cudaEventRecord(w.ev[0], c.s));
  Queue q = make_queue(g, c.cfg, (uint32_t)d->app);
  const uint32_t vb = (uint32_t)g->v_begin, ve = (uint32_t)g->v_end;
  // persistent: drain the local queue to quiescence; discrete: process the
  // current snapshot [next_h, tail) once (one superstep per exchange round)
  const bool disc = c.cfg.kernel == ATOS_KERNEL_DISCRETE;
  uint64_t tail_now = 0;
  if (disc) {
    CK(cudaMemcpyAsync(&w.h_ctl->tail.v, &w.ctl->tail.v, sizeof(uint64_t), cudaMemcpyDeviceToHost, c.s));
    CK(cudaStreamSynchronize(c.s));
    tail_now = w.h_ctl->tail.v;
  }
  auto go = [&](const auto& app) -> atos_status {
    using A = std::decay_t<decltype(app)>;
    if (disc) return run_discrete<EdgeMapPolicy<A>>(c, app, q, tail_now, d->next_h, 1, &d->next_h);
    return run_persistent<EdgeMapPolicy<A>>(c, app, q);
  };
  if (d->app == 2) {
    GcApp app{d->gc_color, w.u32a, vb, ve, d->gc_chg};
    if (disc) CKS(run_discrete<GcPolicy<GC_UBER>>(c, app, q, tail_now, d->next_h, 1, &d->next_h));
    else CKS(run_persistent<GcPolicy<GC_UBER>>(c, app, q));
    if (g->n) {
      k_gc_pack<<<fill_blocks(g->n, g->sms), 256, 0, c.s>>>(c.gv, d->gc_color, d->gc_chg, vb, d->d_bounds, d->world,
                                                             d->rank, ob);
      c.launches++;
    }
  } else if (d->app == 0) {
    CKS(go(BfsPartApp{w.u32a, w.u32b, d->sent_min, c.cfg.bfs_filter, vb, ve, d->d_bounds, d->world, ob}));
  } else if (d->r64) {
    CKS(go(PrPartAppT<double>{w.f64a, w.f64b, (double)d->alpha, (double)d->eps, vb, ve, d->racc}));
  } else {
    CKS(go(PrPartAppT<float>{w.f64a, w.f32b, d->alpha, d->eps, vb, ve, d->racc}));
  }
  if (d->app == 1) {
    for (int r = 0; r < d->world; ++r) {
      if (r == d->rank || d->bounds[r + 1] == d->bounds[r]) continue;
      k_pr_flush<<<fill_blocks(d->bounds[r + 1] - d->bounds[r], g->sms), 256, 0, c.s>>>(
          d->racc, d->bounds[r], d->bounds[r + 1], r, ob, flush_all ? 0.0f : d->eps);
      c.launches++;
    }
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(w.ev[2], c.s));
  CK(cudaMemcpyAsync(d->h_cnt, d->d_cnt, (d->world + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c.s));
  CKS(read_ctl(g, c.s));  // synchronises; checks overflow / timeout
  if (d->h_cnt[d->world])
    return atos_set_error(ATOS_ERR_QUEUE_OVERFLOW, "partition outbox overflow");
  float ms = 0, kms = 0;
  CK(cudaEventElapsedTime(&ms, w.ev[0], w.ev[2]));
  CK(cudaEventElapsedTime(&kms, w.ev[0], w.ev[2]));
  d->ms += ms;
  d->kernel_ms += kms;
  d->launches += c.launches;
  d->rounds++;
  for (int r = 0; r < d->world; ++r) {
    send_counts[r] = (int64_t)d->h_cnt[r];
    d->bytes_sent += (int64_t)d->h_cnt[r] * 8;
  }
  // local work still queued (discrete rounds leave the next superstep queued)
  send_counts[d->world] = disc ? (int64_t)(w.h_ctl->tail.v - d->next_h) : 0;
  return ATOS_OK;
}

extern "C" atos_status atos_part_pack(atos_graph g, uint64_t* dst, int64_t cap) {
  LaunchCtx c;
  CKS(part_ctx(g, c));
  DistState* d = g->dist;
  int64_t total = 0;
  for (int r = 0; r < d->world; ++r) total += (int64_t)d->h_cnt[r];
  if (cap < total) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "pack capacity %lld < %lld", (long long)cap, (long long)total);
  if (!total) return ATOS_OK;
  if (!dst) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "dst == NULL");
  cudaPointerAttributes pa{};
  const bool dev = cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
  (void)cudaGetLastError();
  if (dev) {
    k_part_pack<<<fill_blocks(total, g->sms), 256, 0, c.s>>>(d->outbox, d->d_seg, d->d_cnt, d->world, dst);
    CK(cudaGetLastError());
  } else {
    int64_t base = 0;
    for (int r = 0; r < d->world; ++r) {
      const int64_t cnt = (int64_t)d->h_cnt[r];
      if (cnt) CK(cudaMemcpyAsync(dst + base, d->outbox + d->seg[r], cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost, c.s));
      base += cnt;
    }
  }
  CK(cudaStreamSynchronize(c.s));
  return ATOS_OK;
}

extern "C" atos_status atos_part_apply(atos_graph g, const uint64_t* msgs, int64_t count) {
  LaunchCtx c;
  CKS(part_ctx(g, c));
  DistState* d = g->dist;
  if (count < 0 || (count > 0 && !msgs)) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bad message buffer");
  if (!count) return ATOS_OK;
  Workspace& w = g->ws;
  const uint64_t* dm = msgs;
  uint64_t* tmp = nullptr;
  cudaPointerAttributes pa{};
  const bool dev = cudaPointerGetAttributes(&pa, msgs) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
  (void)cudaGetLastError();
  if (!dev) {
    CK(cudaMallocAsync(&tmp, count * sizeof(uint64_t), c.s));
    CK(cudaMemcpyAsync(tmp, msgs, count * sizeof(uint64_t), cudaMemcpyHostToDevice, c.s));
    dm = tmp;
  }
  Queue q = make_queue(g, c.cfg, (uint32_t)d->app);
  q.deadline = 0;
  const int blocks = fill_blocks(count, g->sms);
  if (d->app == 2) {
    k_gc_apply<<<blocks, 256, 0, c.s>>>(dm, count, d->gc_color, d->gc_gchg, 1);
    if (g->n)
      k_gc_ghost_scan<<<fill_blocks(g->n * 32, g->sms), 256, 0, c.s>>>(c.gv, d->gc_color, d->gc_gchg, w.u32a,
                                                                        (uint32_t)g->v_begin, q);
    k_gc_apply<<<blocks, 256, 0, c.s>>>(dm, count, nullptr, d->gc_gchg, 0);
    d->launches += g->n ? 3 : 2;
  } else if (d->app == 0) k_part_apply<0, float><<<blocks, 256, 0, c.s>>>(dm, count, w.u32a, (float*)nullptr, 0.f, q);
  else if (d->r64) k_part_apply<1, double><<<blocks, 256, 0, c.s>>>(dm, count, nullptr, w.f64b, (double)d->eps, q);
  else k_part_apply<1, float><<<blocks, 256, 0, c.s>>>(dm, count, nullptr, w.f32b, d->eps, q);
  CK(cudaGetLastError());
  if (d->app != 2) d->launches++;
  if (tmp) CK(cudaFreeAsync(tmp, c.s));
  CKS(read_ctl(g, c.s));
  return ATOS_OK;
}

extern "C" atos_status atos_part_finish(atos_graph g, void* out, atos_stats* st) {
  LaunchCtx c;
  CKS(part_ctx(g, c));
  DistState* d = g->dist;
  Workspace& w = g->ws;
  const int64_t n = g->n;
  if (n && !out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "out == NULL");
  CKS(read_ctl(g, c.s));
  w.dirty = std::min<uint64_t>(w.h_ctl->tail.v, w.cap);
  if (n) {
    if (d->app == 0) {
      CKS(copy_out(out, w.u32a, (size_t)n * sizeof(uint32_t), c.s));
    } else if (d->app == 2) {
      CKS(copy_out(out, d->gc_color + g->v_begin, (size_t)n * sizeof(int32_t), c.s));
    } else {
      k_f64_to_f32<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.f64a, w.f32a, n);
      CK(cudaGetLastError());
      CKS(copy_out(out, w.f32a, (size_t)n * sizeof(float), c.s));
    }
  }
  CK(cudaStreamSynchronize(c.s));
  if (st) {
    std::memset(st, 0, sizeof *st);
    st->struct_size = sizeof(atos_stats);
    st->ms = d->ms;
    st->kernel_ms = d->kernel_ms;
    st->kernel_launches = d->launches;
    st->chunk_tasks = (int64_t)w.h_ctl->chunk_done.v;
    st->tasks_popped = (int64_t)w.h_ctl->stats[0].v - st->chunk_tasks;
    st->tasks_pushed = (int64_t)w.h_ctl->stats[1].v;
    st->edges_processed = (int64_t)w.h_ctl->stats[2].v;
    st->rounds = d->rounds;
    st->queue_high_water = (int64_t)w.h_ctl->high_water.v;
    st->bytes_sent = d->bytes_sent;
    st->trace_records = (int64_t)w.h_ctl->trace_count.v;
  }
  d->app = -1;
  return ATOS_OK;
}
