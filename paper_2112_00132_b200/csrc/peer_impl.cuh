// peer_impl.cuh — asynchronous multi-partition BFS / PageRank over peer
// memory ("asynchronous execution across
// frontiers": workers loop with no global synchronisation).
//
// The 1-D vertex partition of §8e, but with NO exchange rounds: partition p
// (its CSR rows, per-vertex state and task queue) lives in the memory of
// device d_p, and a worker of partition p that relaxes an edge into a vertex
// owned by partition o updates o's state IN PLACE (atomicMin / atomicAdd on a
// peer pointer) and pushes the activated vertex straight onto o's queue
// (warp-aggregated atomicAdd on o's tail + slot stores into o's ring, again
// through peer pointers).  Every queue keeps the single-GPU protocol
// (device.cuh); termination is global: an idle worker reads every
// partition's `processed` (acquire) THEN every `tail`, and quits when the sums
// are equal.  (Sum_p processed_p <= Sum_p tail_p holds at all times — a task's
// pushes, local or remote, are reserved before its own processed increment —
// and both sums only grow, so equal sums read in that order mean quiescence
// at the last processed read, the argument of device.cuh's a7.)
//
// Placement:
//  * several devices (one per partition, peer access enabled between every
//    pair): one persistent kernel per device, launched on all devices before
//    any is waited for — kernels on distinct GPUs run concurrently;
//  * one device for every partition (how this build is exercised: gpurun
//    offers one B200): ONE persistent kernel whose blocks are split into P
//    groups, block b serving partition b / blocks_per_part — kernels that
//    wait on one another must never be separate launches on one GPU
//    (nothing makes them co-resident), one launch over all partitions is.
// Workers are warps (the paper's persist-32) with FETCH-sized pops and
// int4 column loads (engine.cuh warp_batch); residues are fp64 (the
// partitions do not see global in-degrees, so no hub tags: R34).
#pragma once

namespace atos {

constexpr int PEER_MAX = 8;

struct PeerSet {
  int P;
  int blocks_per_part;            // one-device launch: block b serves partition b / blocks_per_part
  int64_t base[PEER_MAX + 1];     // partition p owns global ids [base[p], base[p+1])
  Queue q[PEER_MAX];              // each partition's queue (ring + control block on its device)
  GraphView g[PEER_MAX];          // off shifted by -base[p] (off[v] is valid for owned global v), global cols
};

__device__ __forceinline__ int peer_owner(const PeerSet* ps, uint32_t w) {
  int o = 0;
#pragma unroll
  for (int k = 1; k < PEER_MAX; ++k) o += (k < ps->P && (int64_t)w >= ps->base[k]) ? 1 : 0;
  return o;
}

// Warp-aggregated push of each activated vertex onto its OWNER's queue: one
// atomicAdd on each destination's tail per warp step.
struct PeerSink {
  const PeerSet* ps;
  uint64_t deadline;  // the pushing worker's watchdog deadline
  template <int U>
  __device__ __forceinline__ uint32_t warp_push_multi(const bool (&pred)[U], const uint32_t (&item)[U]) const {
    int o[U];
    unsigned any = 0;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      o[k] = pred[k] ? peer_owner(ps, item[k]) : -1;
      any |= __ballot_sync(FULL_MASK, pred[k]);
    }
    if (!any) return 0;
    uint32_t total = 0;
    for (int d = 0; d < ps->P; ++d) {
      unsigned m[U];
      uint32_t cnt = 0;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        m[k] = __ballot_sync(FULL_MASK, o[k] == d);
        cnt += __popc(m[k]);
      }
      if (!cnt) continue;
      Queue q = ps->q[d];
      q.deadline = deadline;
      unsigned long long base = 0;
      if (lane_id() == 0) {
        base = atomicAdd(reinterpret_cast<unsigned long long*>(&q.ctl->tail.v), (unsigned long long)cnt);
        red_add_relaxed_s64(&q.ctl->count.v, (int64_t)cnt);
      }
      base = __shfl_sync(FULL_MASK, base, 0);
      const unsigned lt = lanemask_lt();
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (o[k] == d) q_store_slot(q, base + __popc(m[k] & lt), item[k]);
        base += __popc(m[k]);
      }
      total += cnt;
    }
    return total;
  }
  __device__ __forceinline__ uint32_t warp_push(bool pred, uint32_t item) const {
    const bool p[1] = {pred};
    const uint32_t it[1] = {item};
    return warp_push_multi<1>(p, it);
  }
};

// BFS (Alg. 2) over peer state: dist / done of partition o at dist[o] (shifted
// by -base[o], so dist[o][w] is owned global vertex w).
struct PeerBfsApp {
  static constexpr bool kWindow = false;
  const PeerSet* ps;
  uint32_t* dist[PEER_MAX];
  uint32_t* done[PEER_MAX];
  using Payload = uint32_t;
  using Probe = uint32_t;
  using Raw = uint32_t;
  __device__ __forceinline__ uint32_t item_of(uint32_t w) const { return w; }
  __device__ __forceinline__ bool chunk_current(uint32_t, Payload) const { return true; }
  // expand owned v at its current depth d (R3) unless already expanded at <= d (R25)
  __device__ __forceinline__ bool begin(uint32_t v, const GraphView& g, int64_t& e0, int64_t& e1, Payload& p) const {
    const int me = peer_owner(ps, v);
    e0 = ld_nc_s64(g.off + v);
    e1 = ld_nc_s64(g.off + v + 1);
    const uint32_t d = ld_relaxed_u32(dist[me] + v);
    p = d + 1u;
    if (e0 == e1) return false;
    return atomicMin(done[me] + v, d) > d;
  }
  __device__ __forceinline__ Probe probe(uint32_t, uint32_t) const { return 0xFFFFFFFFu; }
  __device__ __forceinline__ Raw issue(Payload nd, uint32_t w, Probe) const {
    return atomicMin(dist[peer_owner(ps, w)] + w, nd);  // local or peer memory
  }
  __device__ __forceinline__ bool decide(Payload nd, uint32_t, Probe, Raw old) const { return nd < old; }
  __device__ __forceinline__ bool edge(Payload nd, uint32_t w, uint32_t t) const { return decide(nd, w, t, issue(nd, w, t)); }
};

// Push PageRank (Alg. 4) over peer state, fp64 residues and ranks.
struct PeerPrApp {
  static constexpr bool kWindow = false;
  const PeerSet* ps;
  double* res[PEER_MAX];
  double* rank[PEER_MAX];
  double alpha, eps;
  using Payload = double;
  using Probe = uint32_t;
  using Raw = double;
  __device__ __forceinline__ uint32_t item_of(uint32_t w) const { return w; }
  __device__ __forceinline__ bool chunk_current(uint32_t, Payload) const { return true; }
  __device__ __forceinline__ bool begin(uint32_t v, const GraphView& g, int64_t& e0, int64_t& e1, Payload& p) const {
    const int me = peer_owner(ps, v);
    e0 = ld_nc_s64(g.off + v);
    e1 = ld_nc_s64(g.off + v + 1);
    const double r = atomic_take(res[me] + v);
    if (r == 0.0) return false;
    red_add_cold(rank[me] + v, r);
    if (e1 == e0) return false;  // dangling: rank keeps the residue (R5)
    p = alpha * r / (double)(e1 - e0);
    return true;
  }
  __device__ __forceinline__ Probe probe(uint32_t, uint32_t) const { return 0u; }
  __device__ __forceinline__ Raw issue(Payload c, uint32_t w, Probe) const {
    return atomicAdd(res[peer_owner(ps, w)] + w, c);  // local or peer memory
  }
  // threshold crossing (R6, R7)
  __device__ __forceinline__ bool decide(Payload c, uint32_t, Probe, Raw old) const {
    return old <= eps && old + c > eps;
  }
  __device__ __forceinline__ bool edge(Payload c, uint32_t w, uint32_t t) const { return decide(c, w, t, issue(c, w, t)); }
};

// Global quiescence / abort over every partition (see the header comment).
__device__ __forceinline__ uint32_t peer_pop_or_quit(const PeerSet* ps, const Queue& q, uint32_t want,
                                                     uint64_t& first, uint64_t& hw) {
  unsigned ns = 0;
  for (;;) {
    uint64_t qlen = 0;
    const uint32_t n = q_try_pop(q, want, first, qlen);
    if (n) {
      if (qlen > hw) hw = qlen;
      return n;
    }
    uint64_t sp = 0, st = 0;
    bool dead = q_timed_out(q);
    for (int k = 0; k < ps->P; ++k) {
      sp += ld_acquire_u64(&ps->q[k].ctl->processed.v);
      dead |= ld_relaxed_u64(&ps->q[k].ctl->abort.v) != 0;
    }
    for (int k = 0; k < ps->P; ++k) st += ld_relaxed_u64(&ps->q[k].ctl->tail.v);
    if (sp == st || dead) return 0;
    if (ns) __nanosleep(ns);
    ns = ns == 0 ? 32 : (ns < q.backoff_ns ? ns * 2 : ns);
  }
}

constexpr int PEER_THREADS = 256;

// part >= 0: this launch serves one partition (one kernel per device);
// part < 0: block b serves partition b / ps->blocks_per_part (one device).
template <class App>
__global__ void __launch_bounds__(PEER_THREADS) k_peer(App app, const PeerSet* __restrict__ ps, int F, int part) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int p = part >= 0 ? part : min((int)blockIdx.x / ps->blocks_per_part, ps->P - 1);
  Queue q = ps->q[p];
  q_arm(q);
  const GraphView g = ps->g[p];
  const PeerSink sink{ps, q.deadline};
  LocalStats st;
  uint32_t* stage = reinterpret_cast<uint32_t*>(smem) + (size_t)(threadIdx.x >> 5) * (uint32_t)F;
  for (;;) {
    uint64_t first = 0;
    uint32_t n = 0;
    if (lane_id() == 0) n = peer_pop_or_quit(ps, q, (uint32_t)F, first, st.hw);
    n = __shfl_sync(FULL_MASK, n, 0);
    first = __shfl_sync(FULL_MASK, first, 0);
    if (n == 0) break;
    stage_items(q, first, n, stage);  // every claimed slot read before any push
    StageSrc src{stage};
    warp_batch(app, g, src, sink, n, st);
    __syncwarp();
    if (lane_id() == 0) {
      st.popped += n;
      q_done(q, n);
    }
  }
  st.flush(q);
}

// ---- init kernels (timed, a2)
__global__ void k_peer_ring_fill(uint64_t* ring, int64_t n, int64_t base) {  // all owned ids in id order
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    ring[i] = (1ull << 32) | (uint64_t)(uint32_t)(base + i);
}
// R4 seeding: residue[w] += (1-a) a / deg(v) for every edge v -> w of partition p (w's owner's memory)
__global__ void k_peer_pr_seed(PeerPrApp app, const PeerSet* __restrict__ ps, int p, double coef) {
  const GraphView g = ps->g[p];
  const int64_t b = ps->base[p], e = ps->base[p + 1];
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = b + wid; v < e; v += nw) {
    const int64_t e0 = g.off[v], e1 = g.off[v + 1];
    const double c = coef / (double)(e1 - e0);
    for (int64_t k = e0 + lane_id(); k < e1; k += 32) {
      const uint32_t w = (uint32_t)g.col[k] & VID_MASK;
      red_add_hot(app.res[peer_owner(ps, w)] + w, c);
    }
  }
}

}  // namespace atos

// ------------------------------------------------------------------ host side

struct PeerPart {
  int device = 0;
  int sms = 0;
  int64_t n = 0, m = 0;
  int64_t* off = nullptr;   // local rows [0, n]
  int32_t* col = nullptr;   // global ids, 16-B padded
  uint64_t* ring = nullptr;
  uint64_t cap = 0;
  QueueCtl* ctl = nullptr;
  QueueCtl* h_ctl = nullptr;
  uint32_t* u32a = nullptr;  // BFS dist
  uint32_t* u32b = nullptr;  // BFS done
  double* f64a = nullptr;    // PR rank
  double* f64b = nullptr;    // PR residue
  float* f32 = nullptr;      // PR output staging
  PeerSet* d_ps = nullptr;   // this device's copy of the peer set
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[2] = {nullptr, nullptr};
};

struct PeerState {
  int P = 0;
  bool one_device = true;
  int64_t base[PEER_MAX + 1] = {};
  PeerPart part[PEER_MAX];
};

static void peer_free(PeerState* ps) {
  if (!ps) return;
  int cur = 0;
  cudaGetDevice(&cur);
  for (int p = 0; p < ps->P; ++p) {
    PeerPart& x = ps->part[p];
    cudaSetDevice(x.device);
    cudaFree(x.off);
    cudaFree(x.col);
    cudaFree(x.ring);
    cudaFree(x.ctl);
    cudaFreeHost(x.h_ctl);
    cudaFree(x.u32a);
    cudaFree(x.u32b);
    cudaFree(x.f64a);
    cudaFree(x.f64b);
    cudaFree(x.f32);
    cudaFree(x.d_ps);
    if (x.stream) cudaStreamDestroy(x.stream);
    for (auto& e : x.ev)
      if (e) cudaEventDestroy(e);
  }
  cudaSetDevice(cur);
  delete ps;
}

#define CKP(x)                                                                                               \
  do {                                                                                                       \
    cudaError_t e_ = (x);                                                                                    \
    if (e_ != cudaSuccess) {                                                                                 \
      cudaSetDevice(cur);                                                                                    \
      return atos_set_error(e_ == cudaErrorMemoryAllocation ? ATOS_ERR_OUT_OF_MEMORY : ATOS_ERR_CUDA,       \
                            "%s: %s", #x, cudaGetErrorString(e_));                                           \
    }                                                                                                        \
  } while (0)

extern "C" atos_status atos_graph_create_peer(int32_t parts, const int32_t* devices, const int64_t* off,
                                              const int32_t* col, int64_t n, int64_t m, uint32_t flags,
                                              atos_graph* out) {
  if (!out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "out == NULL");
  *out = nullptr;
  if (parts < 1 || parts > PEER_MAX) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "parts %d not in [1, %d]", parts, PEER_MAX);
  if (n < parts || m < 0 || !off || (m > 0 && !col))
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bad n / m / pointers (n must be >= parts)");
  if (n >= (int64_t)VID_MASK) return atos_set_error(ATOS_ERR_UNSUPPORTED, "n >= 2^30 - 1 (R37)");
  if (flags & (ATOS_GRAPH_DEVICE_PTRS | ATOS_GRAPH_BORROW))
    return atos_set_error(ATOS_ERR_UNSUPPORTED, "peer graphs copy host CSR arrays");
  int cur = 0;
  CK(cudaGetDevice(&cur));
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  std::vector<int64_t> hoff(off, off + n + 1);
  if (hoff[0] != 0 || hoff[n] != m) return atos_set_error(ATOS_ERR_INVALID_GRAPH, "off[0] != 0 or off[n] != m");
  if (flags & ATOS_GRAPH_VALIDATE) {
    for (int64_t v = 0; v < n; ++v)
      if (hoff[v + 1] < hoff[v]) return atos_set_error(ATOS_ERR_INVALID_GRAPH, "offsets not monotone");
    for (int64_t e = 0; e < m; ++e)
      if (col[e] < 0 || col[e] >= n) return atos_set_error(ATOS_ERR_INVALID_GRAPH, "column out of range");
  }
  PeerState* st = new PeerState();
  st->P = parts;
  for (int p = 0; p <= parts; ++p) st->base[p] = (int64_t)p * n / parts;
  for (int p = 0; p < parts; ++p) {
    const int d = devices ? devices[p] : cur;
    if (d < 0 || d >= ndev) { peer_free(st); return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "device %d", d); }
    st->part[p].device = d;
    if (d != st->part[0].device) st->one_device = false;
  }
  // either every partition on one device (one launch over all of them) or one partition per device
  // (one launch per device): two launches that wait on each other must never share a GPU
  for (int p = 0; p < parts && !st->one_device; ++p)
    for (int o = p + 1; o < parts; ++o)
      if (st->part[p].device == st->part[o].device) {
        peer_free(st);
        return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "devices: all equal or all distinct");
      }
  // peer access between every pair of distinct devices
  for (int p = 0; p < parts && !st->one_device; ++p)
    for (int o = 0; o < parts; ++o) {
      const int a = st->part[p].device, b = st->part[o].device;
      if (a == b) continue;
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, a, b);
      if (!ok) { peer_free(st); return atos_set_error(ATOS_ERR_UNSUPPORTED, "no peer access %d -> %d", a, b); }
      cudaSetDevice(a);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        cudaSetDevice(cur);
        peer_free(st);
        return atos_set_error(ATOS_ERR_CUDA, "cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
      }
      cudaGetLastError();
    }
  atos_graph g = new atos_graph_s();
  g->n = n;
  g->m = m;
  g->global_n = n;
  g->device = cur;
  g->peer = st;
  for (int p = 0; p < parts; ++p) {
    PeerPart& x = st->part[p];
    CKP(cudaSetDevice(x.device));
    CKP(cudaDeviceGetAttribute(&x.sms, cudaDevAttrMultiProcessorCount, x.device));
    const int64_t b = st->base[p], e = st->base[p + 1];
    x.n = e - b;
    x.m = hoff[e] - hoff[b];
    std::vector<int64_t> lo(x.n + 1);
    for (int64_t v = 0; v <= x.n; ++v) lo[v] = hoff[b + v] - hoff[b];
    CKP(cudaMalloc(&x.off, (x.n + 1) * sizeof(int64_t)));
    CKP(cudaMemcpy(x.off, lo.data(), (x.n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    const int64_t ccap = (x.m + 3) / 4 * 4 + 4;
    CKP(cudaMalloc(&x.col, ccap * sizeof(int32_t)));
    CKP(cudaMemset(x.col, 0, ccap * sizeof(int32_t)));
    if (x.m) CKP(cudaMemcpy(x.col, col + hoff[b], x.m * sizeof(int32_t), cudaMemcpyHostToDevice));
    x.cap = 1024;
    while (x.cap < 2 * (uint64_t)x.n) x.cap <<= 1;
    CKP(cudaMalloc(&x.ring, x.cap * sizeof(uint64_t)));
    CKP(cudaMalloc(&x.ctl, sizeof(QueueCtl)));
    CKP(cudaMallocHost(&x.h_ctl, sizeof(QueueCtl)));
    CKP(cudaMalloc(&x.d_ps, sizeof(PeerSet)));
    CKP(cudaStreamCreateWithFlags(&x.stream, cudaStreamNonBlocking));
    for (auto& ev : x.ev) CKP(cudaEventCreate(&ev));
  }
  CKP(cudaSetDevice(cur));
  *out = g;
  return ATOS_OK;
}

// One peer-set image (device pointers of every partition), copied to every device.
static atos_status peer_publish(PeerState* st, double timeout_s) {
  int cur = 0;
  CK(cudaGetDevice(&cur));
  PeerSet h{};
  h.P = st->P;
  h.blocks_per_part = 1;
  for (int p = 0; p <= st->P; ++p) h.base[p] = st->base[p];
  for (int p = 0; p < st->P; ++p) {
    const PeerPart& x = st->part[p];
    Queue q{};
    q.ring = x.ring;
    q.mask = x.cap - 1;
    q.log2cap = 0;
    while ((1ull << q.log2cap) < x.cap) ++q.log2cap;
    q.ctl = x.ctl;
    q.backoff_ns = ATOS_BACKOFF_NS;
    q.timeout_ns = timeout_s > 0 ? (uint64_t)(timeout_s * 1e9) : 0;
    h.q[p] = q;
    h.g[p] = GraphView{x.off - st->base[p], x.col, st->base[st->P], (x.m + 3) / 4 * 4 + 4};
  }
  for (int p = 0; p < st->P; ++p) {
    CKP(cudaSetDevice(st->part[p].device));
    CKP(cudaMemcpy(st->part[p].d_ps, &h, sizeof h, cudaMemcpyHostToDevice));
  }
  CKP(cudaSetDevice(cur));
  return ATOS_OK;
}

template <class App>
static atos_status peer_launch(PeerState* st, const App& app, int F, int per_sm_cap, atos_stats* stats,
                               int64_t* launches) {
  int cur = 0;
  CK(cudaGetDevice(&cur));
  const size_t smem = (size_t)(PEER_THREADS / 32) * F * sizeof(uint32_t);
  if (smem > 227 * 1024) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "fetch_size %d too large for warp workers", F);
  auto kern = k_peer<App>;
  if (st->one_device) {
    PeerPart& x0 = st->part[0];
    CKP(cudaSetDevice(x0.device));
    CKP(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CKP(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PEER_THREADS, smem));
    per_sm = std::max(1, std::min(per_sm, per_sm_cap));
    // every partition gets an equal share of the resident grid (all blocks co-resident)
    const int bpp = std::max(1, per_sm * x0.sms / st->P);
    CKP(cudaMemcpy(reinterpret_cast<char*>(x0.d_ps) + offsetof(PeerSet, blocks_per_part), &bpp, sizeof bpp,
                   cudaMemcpyHostToDevice));
    CKP(cudaEventRecord(x0.ev[0], x0.stream));
    kern<<<bpp * st->P, PEER_THREADS, smem, x0.stream>>>(app, x0.d_ps, F, -1);
    CKP(cudaGetLastError());
    CKP(cudaEventRecord(x0.ev[1], x0.stream));
    CKP(cudaStreamSynchronize(x0.stream));
    *launches += 1;
  } else {
    // one persistent kernel per device, all launched before any is waited for
    for (int p = 0; p < st->P; ++p) {
      PeerPart& x = st->part[p];
      CKP(cudaSetDevice(x.device));
      CKP(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0;
      CKP(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PEER_THREADS, smem));
      per_sm = std::max(1, std::min(per_sm, per_sm_cap));
      App a = app;
      a.ps = x.d_ps;  // owner lookups read this device's copy
      CKP(cudaEventRecord(x.ev[0], x.stream));
      kern<<<per_sm * x.sms, PEER_THREADS, smem, x.stream>>>(a, x.d_ps, F, p);
      CKP(cudaGetLastError());
      CKP(cudaEventRecord(x.ev[1], x.stream));
      *launches += 1;
    }
    for (int p = 0; p < st->P; ++p) {
      CKP(cudaSetDevice(st->part[p].device));
      CKP(cudaStreamSynchronize(st->part[p].stream));
    }
  }
  // control blocks: abort codes and statistics of every partition
  uint64_t abort = 0;
  for (int p = 0; p < st->P; ++p) {
    PeerPart& x = st->part[p];
    CKP(cudaSetDevice(x.device));
    CKP(cudaMemcpy(x.h_ctl, x.ctl, sizeof(QueueCtl), cudaMemcpyDeviceToHost));
    if (x.h_ctl->abort.v) abort = x.h_ctl->abort.v;
    if (stats) {
      stats->tasks_popped += (int64_t)x.h_ctl->stats[0].v;
      stats->tasks_pushed += (int64_t)x.h_ctl->stats[1].v;
      stats->edges_processed += (int64_t)x.h_ctl->stats[2].v;
      stats->queue_high_water = std::max<int64_t>(stats->queue_high_water, (int64_t)x.h_ctl->high_water.v);
    }
  }
  if (stats) {
    float ms = 0;
    for (int p = 0; p < (st->one_device ? 1 : st->P); ++p) {
      float t = 0;
      CKP(cudaSetDevice(st->part[p].device));
      CKP(cudaEventElapsedTime(&t, st->part[p].ev[0], st->part[p].ev[1]));
      ms = std::max(ms, t);
    }
    stats->kernel_ms = ms;
  }
  CKP(cudaSetDevice(cur));
  if (abort == ABORT_OVERFLOW) return atos_set_error(ATOS_ERR_QUEUE_OVERFLOW, "a partition's task queue overflowed");
  if (abort == ABORT_TIMEOUT) return atos_set_error(ATOS_ERR_TIMEOUT, "device watchdog fired");
  if (abort) return atos_set_error(ATOS_ERR_CUDA, "unknown abort code %llu", (unsigned long long)abort);
  return check_failures();
}

static atos_status peer_bfs(atos_graph g, int64_t src, const atos_config& cfg, uint32_t* depth_out, atos_stats* stats) {
  PeerState* st = g->peer;
  if (src < 0 || src >= g->n) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "src %lld not in [0, %lld)", (long long)src, (long long)g->n);
  if (!depth_out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "depth_out == NULL");
  int cur = 0;
  CK(cudaGetDevice(&cur));
  const auto t0 = std::chrono::steady_clock::now();
  PeerBfsApp app{};
  for (int p = 0; p < st->P; ++p) {
    PeerPart& x = st->part[p];
    CKP(cudaSetDevice(x.device));
    if (!x.u32a) CKP(cudaMalloc(&x.u32a, std::max<int64_t>(1, x.n) * sizeof(uint32_t)));
    if (!x.u32b) CKP(cudaMalloc(&x.u32b, std::max<int64_t>(1, x.n) * sizeof(uint32_t)));
    app.dist[p] = x.u32a - st->base[p];
    app.done[p] = x.u32b - st->base[p];
  }
  CKS(peer_publish(st, cfg.timeout_s));
  int64_t launches = 0;
  for (int p = 0; p < st->P; ++p) {
    PeerPart& x = st->part[p];
    CKP(cudaSetDevice(x.device));
    const bool own = src >= st->base[p] && src < st->base[p + 1];
    k_bfs_init<<<grid_for(x.n, 256, x.sms), 256, 0, x.stream>>>(x.u32a, x.u32b, nullptr, x.n,
                                                                 own ? src - st->base[p] : -1);
    CKP(cudaMemsetAsync(x.ring, 0, x.cap * sizeof(uint64_t), x.stream));
    k_ctl_init<<<1, 1, 0, x.stream>>>(x.ctl, own ? 1 : 0, x.ring, own ? src : -1);
    CKP(cudaGetLastError());
    CKP(cudaStreamSynchronize(x.stream));
    launches += 2;
  }
  app.ps = st->part[0].d_ps;  // one device; per-device launches substitute their own copy
  const atos_status s = peer_launch(st, app, cfg.fetch_size, 64, stats, &launches);
  if (s != ATOS_OK) { cudaSetDevice(cur); return s; }
  for (int p = 0; p < st->P; ++p) {
    PeerPart& x = st->part[p];
    CKP(cudaSetDevice(x.device));
    if (x.n) CKP(cudaMemcpy(depth_out + st->base[p], x.u32a, x.n * sizeof(uint32_t), cudaMemcpyDefault));
  }
  CKP(cudaSetDevice(cur));
  if (stats) {
    stats->ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    stats->kernel_launches = launches;
    stats->rounds = 0;
  }
  return ATOS_OK;
}

static atos_status peer_pagerank(atos_graph g, float alpha, float eps, const atos_config& cfg, float* rank_out,
                                 atos_stats* stats) {
  PeerState* st = g->peer;
  if (!rank_out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "rank_out == NULL");
  int cur = 0;
  CK(cudaGetDevice(&cur));
  const auto t0 = std::chrono::steady_clock::now();
  PeerPrApp app{};
  app.alpha = alpha;
  app.eps = eps;
  for (int p = 0; p < st->P; ++p) {
    PeerPart& x = st->part[p];
    CKP(cudaSetDevice(x.device));
    if (!x.f64a) CKP(cudaMalloc(&x.f64a, std::max<int64_t>(1, x.n) * sizeof(double)));
    if (!x.f64b) CKP(cudaMalloc(&x.f64b, std::max<int64_t>(1, x.n) * sizeof(double)));
    if (!x.f32) CKP(cudaMalloc(&x.f32, std::max<int64_t>(1, x.n) * sizeof(float)));
    app.rank[p] = x.f64a - st->base[p];
    app.res[p] = x.f64b - st->base[p];
  }
  CKS(peer_publish(st, cfg.timeout_s));
  app.ps = st->part[0].d_ps;
  int64_t launches = 0;
  for (int p = 0; p < st->P; ++p) {  // rank = 1 - a, residue = 0
    PeerPart& x = st->part[p];
    CKP(cudaSetDevice(x.device));
    k_fill<double><<<grid_for(x.n, 256, x.sms), 256, 0, x.stream>>>(x.f64a, x.n, 1.0 - (double)alpha);
    k_fill<double><<<grid_for(x.n, 256, x.sms), 256, 0, x.stream>>>(x.f64b, x.n, 0.0);
    CKP(cudaGetLastError());
    CKP(cudaStreamSynchronize(x.stream));
    launches += 2;
  }
  for (int p = 0; p < st->P; ++p) {  // R4 seeding into the owners' residues (peer atomics)
    PeerPart& x = st->part[p];
    CKP(cudaSetDevice(x.device));
    PeerPrApp a = app;
    a.ps = x.d_ps;
    k_peer_pr_seed<<<grid_for(x.n * 32, 256, x.sms), 256, 0, x.stream>>>(a, x.d_ps, p,
                                                                        (1.0 - (double)alpha) * (double)alpha);
    CKP(cudaGetLastError());
    launches++;
  }
  for (int p = 0; p < st->P; ++p) {  // every vertex queued in id order
    PeerPart& x = st->part[p];
    CKP(cudaSetDevice(x.device));
    CKP(cudaStreamSynchronize(x.stream));
    CKP(cudaMemsetAsync(x.ring, 0, x.cap * sizeof(uint64_t), x.stream));
    k_peer_ring_fill<<<grid_for(x.n, 256, x.sms), 256, 0, x.stream>>>(x.ring, x.n, st->base[p]);
    k_ctl_init<<<1, 1, 0, x.stream>>>(x.ctl, (uint64_t)x.n, x.ring, -1);
    CKP(cudaGetLastError());
    CKP(cudaStreamSynchronize(x.stream));
    launches += 2;
  }
  const atos_status s = peer_launch(st, app, cfg.fetch_size, 64, stats, &launches);
  if (s != ATOS_OK) { cudaSetDevice(cur); return s; }
  double maxres = 0;
  for (int p = 0; p < st->P; ++p) {
    PeerPart& x = st->part[p];
    CKP(cudaSetDevice(x.device));
    k_f64_to_f32<<<grid_for(x.n, 256, x.sms), 256, 0, x.stream>>>(x.f64a, x.f32, x.n);
    CKP(cudaGetLastError());
    CKP(cudaStreamSynchronize(x.stream));
    if (x.n) CKP(cudaMemcpy(rank_out + st->base[p], x.f32, x.n * sizeof(float), cudaMemcpyDefault));
    if (stats) {
      std::vector<double> r(x.n);
      if (x.n) CKP(cudaMemcpy(r.data(), x.f64b, x.n * sizeof(double), cudaMemcpyDeviceToHost));
      for (double v : r) maxres = std::max(maxres, v);
    }
    launches++;
  }
  CKP(cudaSetDevice(cur));
  if (stats) {
    stats->ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    stats->kernel_launches = launches;
    stats->max_residue = maxres;
  }
  return ATOS_OK;
}
