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
  __device__ __forceinline__ Probe probe(uint32_t w, uint32_t) const {
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
  __device__ __forceinline__ bool edge(Payload nd, uint32_t w, uint32_t tag) const { return commit(nd, w, probe(w, tag)); }
};

// PageRank on a partition: contributions to remote vertices accumulate in
// racc (global n, fp64: many small adds onto one growing sum, R30) and are
// flushed as messages at the end of every round.  Partitioned graphs keep fp64
// residues (R34: their columns carry no hub tags — in-degrees are global).
template <class R>
struct PrPartAppT {
  static constexpr bool kWindow = false;
  double* rank;
  R* res;
  R alpha, eps;
  uint32_t vb, ve;
  double* racc;
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
  __device__ __forceinline__ Probe probe(uint32_t, uint32_t) const { return 0; }
  __device__ __forceinline__ Raw issue(Payload c, uint32_t w, Probe) const {
    if (local(w)) return atom_add_hot(res + (w - vb), c);
    red_add_hot(racc + w, (double)c);
    return R(0);
  }
  __device__ __forceinline__ bool decide(Payload c, uint32_t w, Probe, Raw old) const {
    return local(w) && old <= eps && add_rn(old, c) > eps;
  }
  __device__ __forceinline__ bool commit(Payload c, uint32_t w, Probe p) const { return decide(c, w, p, issue(c, w, p)); }
  __device__ __forceinline__ bool edge(Payload c, uint32_t w, uint32_t) const { return commit(c, w, 0); }
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
  __device__ __forceinline__ Probe probe(uint32_t, uint32_t) const { return 0; }
  __device__ __forceinline__ Raw issue(Payload c, uint32_t w, Probe) const {
    if (w >= vb && w < ve) atomicAdd(res + (w - vb), c);
    else atomicAdd(racc + w, c);
    return 0;
  }
  __device__ __forceinline__ bool decide(Payload, uint32_t, Probe, Raw) const { return false; }
  __device__ __forceinline__ bool commit(Payload c, uint32_t w, Probe p) const { return decide(c, w, p, issue(c, w, p)); }
  __device__ __forceinline__ bool edge(Payload c, uint32_t w, uint32_t) const { return commit(c, w, 0); }
};

// Flush remote PR accumulations of destination r's range into messages: only
// those above `eps` in a regular round — a smaller amount cannot re-activate
// its target on its own and keeps accumulating at the sender — and every
// non-zero one in a closing round, so no mass is stranded.  A message carries fp32 bits; the
// fp64 remainder of that rounding stays in racc for a later round, except in
// a closing round (it is < 2^-24 of the message).
__global__ void k_pr_flush(double* racc, int64_t b0, int64_t b1, int r, Outbox out, float eps, int flush_all) {
  for (int64_t w = b0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < b1; w += (int64_t)gridDim.x * blockDim.x) {
    const double v = racc[w];
    if (flush_all ? v != 0.0 : v > (double)eps) {
      const float f = (float)v;
      racc[w] = flush_all ? 0.0 : v - (double)f;
      out.put(r, ((uint64_t)(uint32_t)(w - b0) << 32) | (uint64_t)__float_as_uint(f));
    }
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
        const int r = owner_of(bounds, world, (uint32_t)g.col[e] & VID_MASK);
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
      const uint32_t u = (uint32_t)g.col[e] & VID_MASK;
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

// ------------------------------------------------ round bookkeeping kernels
// Discrete rounds on a partition: DevRound {h, t} is the superstep snapshot.
// Before a round: h = t (everything before the previous snapshot's end is
// consumed), t = tail (messages applied and pushes since are the next superstep).
__global__ void k_round_snap(DevRound* r, const QueueCtl* ctl) {
  r->h = r->t;
  r->t = *(volatile const uint64_t*)&ctl->tail.v;
  r->next = 0;
  r->rounds++;
}
// After a discrete round: every position < t is consumed (later pushes —
// applied messages — check ring wrap-around against it).
__global__ void k_round_head(const DevRound* r, QueueCtl* ctl) { ctl->head.v = r->t; }

// This rank's round vector (rounds.h): messages per destination, pending
// local tasks (discrete: not-yet-processed queue positions; persistent: none
// — it ran to local quiescence), abort code, outbox overflow flag.
__global__ void k_round_vec(const unsigned long long* cnt, int world, const QueueCtl* ctl, const DevRound* r,
                            int64_t* rv) {
  for (int i = threadIdx.x; i < world; i += blockDim.x) rv[i] = (int64_t)cnt[i];
  if (threadIdx.x == 0) {
    const uint64_t tail = *(volatile const uint64_t*)&ctl->tail.v;
    rv[world] = r ? (int64_t)(tail - r->t) : 0;
    rv[world + 1] = (int64_t)*(volatile const uint64_t*)&ctl->abort.v;
    rv[world + 2] = (int64_t)(cnt[world] & 0xFFFFFFFFull);
  }
}

// largest colour of the owned vertices (partitioned colouring) into out[0]
__global__ void k_max_color_i64(const int32_t* color, int64_t n, int64_t* out) {
  int m = -1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) m = max(m, color[i]);
  for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(FULL_MASK, m, d));
  if (lane_id() == 0) atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)(int64_t)(m + 1));
}

}  // namespace atos


// ======================================================= communicators (host)
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy already mapped in
// the process — torch's — if there is one), so libatos.so has no link-time
// NCCL dependency and reports ATOS_ERR_NCCL when it is missing.
#include <dlfcn.h>
#include <nccl.h>

#include "rounds.h"

namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    api.why = std::string("dlopen libnccl.so.2: ") + dlerror();
    return api;
  }
  bool all = true;
  auto sym = [&](auto& f, const char* name) {
    f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
    if (!f) all = false;
  };
  sym(api.GetUniqueId, "ncclGetUniqueId");
  sym(api.CommInitRank, "ncclCommInitRank");
  sym(api.CommDestroy, "ncclCommDestroy");
  sym(api.AllGather, "ncclAllGather");
  sym(api.Send, "ncclSend");
  sym(api.Recv, "ncclRecv");
  sym(api.GroupStart, "ncclGroupStart");
  sym(api.GroupEnd, "ncclGroupEnd");
  sym(api.GetErrorString, "ncclGetErrorString");
  api.ok = all;
  if (!all) api.why = "libnccl.so.2 lacks a required symbol";
  return api;
}
}  // namespace

#define NCK(call)                                                                                     \
  do {                                                                                                \
    ncclResult_t r_ = (call);                                                                         \
    if (r_ != ncclSuccess)                                                                            \
      return atos_set_error(ATOS_ERR_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call,                 \
                            nccl_api().GetErrorString ? nccl_api().GetErrorString(r_) : "?");         \
  } while (0)

struct atos_comm_s {
  int rank = 0, world = 1, device = 0;
  ncclComm_t nccl = nullptr;
  atos_rounds::HostExchange host;
  int64_t* d_buf = nullptr;  // NCCL: device staging of gathered round vectors
  size_t d_cap = 0;
};

// NCCL exchange over device buffers on the call's stream (NVLink / NVSwitch).
struct NcclExchange : atos_rounds::Exchange {
  atos_comm c = nullptr;
  cudaStream_t s = nullptr;
  bool on_device() const override { return true; }
  atos_status gather(const int64_t* vec, int K, int64_t* M) override {
    NcclApi& A = nccl_api();
    const size_t need = (size_t)world * (size_t)K;
    if (c->d_cap < need) {
      cudaFree(c->d_buf);
      c->d_buf = nullptr;
      c->d_cap = 0;
      CK(cudaMalloc(&c->d_buf, need * sizeof(int64_t)));
      c->d_cap = need;
    }
    NCK(A.AllGather(vec, c->d_buf, (size_t)K, ncclInt64, c->nccl, s));
    CK(cudaMemcpyAsync(M, c->d_buf, need * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));  // the round's one host synchronisation
    return ATOS_OK;
  }
  atos_status alltoallv(const uint64_t* send, const int64_t* soff, const int64_t* scnt, uint64_t* recv,
                        const int64_t* roff, const int64_t* rcnt) override {
    NcclApi& A = nccl_api();
    NCK(A.GroupStart());
    for (int r = 0; r < world; ++r) {
      if (r == rank) continue;
      if (scnt[r]) NCK(A.Send(send + soff[r], (size_t)scnt[r], ncclUint64, r, c->nccl, s));
      if (rcnt[r]) NCK(A.Recv(recv + roff[r], (size_t)rcnt[r], ncclUint64, r, c->nccl, s));
    }
    NCK(A.GroupEnd());
    return ATOS_OK;
  }
};

extern "C" atos_status atos_comm_unique_id(uint8_t id_out[128]) {
  if (!id_out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "id_out == NULL");
  NcclApi& A = nccl_api();
  if (!A.ok) return atos_set_error(ATOS_ERR_NCCL, "%s", A.why.c_str());
  ncclUniqueId id;
  NCK(A.GetUniqueId(&id));
  std::memcpy(id_out, id.internal, 128);
  return ATOS_OK;
}

extern "C" atos_status atos_comm_init(int32_t rank, int32_t world, const uint8_t id[128], atos_comm* out) {
  if (!out || !id || world < 1 || rank < 0 || rank >= world)
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bad communicator arguments");
  *out = nullptr;
  NcclApi& A = nccl_api();
  if (!A.ok) return atos_set_error(ATOS_ERR_NCCL, "%s", A.why.c_str());
  atos_comm c = new (std::nothrow) atos_comm_s();
  if (!c) return atos_set_error(ATOS_ERR_OUT_OF_MEMORY, "host allocation");
  c->rank = rank;
  c->world = world;
  CK(cudaGetDevice(&c->device));
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  ncclResult_t r = A.CommInitRank(&c->nccl, world, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return atos_set_error(ATOS_ERR_NCCL, "ncclCommInitRank: %s", A.GetErrorString(r));
  }
  *out = c;
  return ATOS_OK;
}

extern "C" atos_status atos_comm_init_host(int32_t rank, int32_t world, atos_allgather_fn ag, atos_alltoallv_fn a2a,
                                           void* user, atos_comm* out) {
  if (!out || !ag || !a2a || world < 1 || rank < 0 || rank >= world)
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bad communicator arguments");
  *out = nullptr;
  atos_comm c = new (std::nothrow) atos_comm_s();
  if (!c) return atos_set_error(ATOS_ERR_OUT_OF_MEMORY, "host allocation");
  c->rank = rank;
  c->world = world;
  (void)cudaGetDevice(&c->device);
  (void)cudaGetLastError();
  c->host.rank = rank;
  c->host.world = world;
  c->host.ag = ag;
  c->host.a2a = a2a;
  c->host.user = user;
  c->host.errf = atos_set_error;
  *out = c;
  return ATOS_OK;
}

extern "C" atos_status atos_comm_info(atos_comm c, int32_t* rank, int32_t* world) {
  if (!c) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "NULL communicator");
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  return ATOS_OK;
}

extern "C" atos_status atos_comm_destroy(atos_comm c) {
  if (!c) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "NULL communicator");
  if (c->nccl) nccl_api().CommDestroy(c->nccl);
  cudaFree(c->d_buf);
  delete c;
  return ATOS_OK;
}

// The exchange object of a communicator for one call on stream s.
struct ExchangeRef {
  NcclExchange nx;
  atos_rounds::Exchange* ex = nullptr;
  ExchangeRef(atos_comm c, cudaStream_t s) {
    if (c->nccl) {
      nx.c = c;
      nx.s = s;
      nx.rank = c->rank;
      nx.world = c->world;
      nx.errf = atos_set_error;
      ex = &nx;
    } else {
      ex = &c->host;
    }
  }
};

// ======================================================= partitioned graphs
struct DistState {
  int world = 1, rank = 0;
  atos_comm comm = nullptr;
  std::vector<int64_t> bounds;
  int64_t* d_bounds = nullptr;
  int64_t* d_seg = nullptr;
  std::vector<int64_t> seg;
  uint64_t* outbox = nullptr;
  uint64_t* inbox = nullptr;
  int64_t inbox_cap = 0;
  unsigned long long* d_cnt = nullptr;  // [world] messages per destination + overflow flag
  int64_t* d_rv = nullptr;              // round vector (rounds.h), world + 3
  DevRound* d_round = nullptr;          // discrete supersteps
  uint32_t* sent_min = nullptr;
  double* racc = nullptr;       // PageRank: accumulated contributions to remote vertices (global ids)
  int32_t* gc_color = nullptr;  // colouring: replica of all N colours
  uint8_t* gc_chg = nullptr;    // colouring: local vertex changed colour this round
  uint8_t* gc_gchg = nullptr;   // colouring: ghost changed this round (global ids)
};

void dist_free(atos_graph g) {
  if (!g || !g->dist) return;
  DistState* d = g->dist;
  cudaFree(d->d_bounds);
  cudaFree(d->d_seg);
  pool_free(d->outbox);
  pool_free(d->inbox);
  cudaFree(d->d_cnt);
  cudaFree(d->d_rv);
  cudaFree(d->d_round);
  pool_free(d->sent_min);
  pool_free(d->racc);
  pool_free(d->gc_color);
  pool_free(d->gc_chg);
  pool_free(d->gc_gchg);
  delete d;
  g->dist = nullptr;
}

extern "C" atos_status atos_graph_create_partitioned(atos_comm comm, int64_t global_n, int64_t v_begin, int64_t v_end,
                                                     const int64_t* off, const int32_t* col, int64_t m, uint32_t flags,
                                                     atos_graph* out) {
  if (!out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "out == NULL");
  *out = nullptr;
  if (!comm) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "NULL communicator");
  const int world = comm->world, rank = comm->rank;
  // all-gather every rank's range first (collective: every rank takes part even with bad arguments)
  const bool args_ok = global_n >= 0 && m >= 0 && off && (m == 0 || col) && 0 <= v_begin && v_begin <= v_end &&
                       v_end <= global_n;
  std::vector<int64_t> M((size_t)world * 3);
  {
    int64_t mine[3] = {v_begin, v_end, args_ok ? 1 : 0};
    ExchangeRef xr(comm, nullptr);
    int64_t* vec = mine;
    int64_t* dvec = nullptr;
    if (xr.ex->on_device()) {
      CK(cudaMalloc(&dvec, sizeof mine));
      CK(cudaMemcpy(dvec, mine, sizeof mine, cudaMemcpyHostToDevice));
      vec = dvec;
    }
    const atos_status s = xr.ex->gather(vec, 3, M.data());
    cudaFree(dvec);
    CKS(s);
  }
  std::vector<int64_t> bounds(world + 1, 0);
  bool tiled = true;
  for (int r = 0; r < world; ++r) {
    tiled = tiled && M[r * 3 + 2] == 1 && M[r * 3] == (r ? M[(r - 1) * 3 + 1] : 0);
    bounds[r + 1] = M[r * 3 + 1];
  }
  tiled = tiled && bounds[world] == global_n;
  if (!tiled)
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "partition ranges do not tile [0, global_n) in rank order "
                          "(or a rank passed bad arguments)");
  if (global_n >= (int64_t)VID_MASK) return atos_set_error(ATOS_ERR_UNSUPPORTED, "global_n >= 2^30-1 (R37)");
  const int64_t n = v_end - v_begin;
  atos_graph g = new (std::nothrow) atos_graph_s();
  if (!g) return atos_set_error(ATOS_ERR_OUT_OF_MEMORY, "host allocation");
  auto fail = [&](atos_status st) {
    graph_free(g);
    return st;
  };
  atos_status s = graph_init_common(g, off, col, n, m, flags & ~(uint32_t)ATOS_GRAPH_BORROW, global_n);
  if (s != ATOS_OK) return fail(s);
  g->global_n = global_n;
  g->v_begin = v_begin;
  g->v_end = v_end;
  DistState* d = new (std::nothrow) DistState();
  if (!d) return fail(atos_set_error(ATOS_ERR_OUT_OF_MEMORY, "host allocation"));
  g->dist = d;
  d->world = world;
  d->rank = rank;
  d->comm = comm;
  d->bounds = bounds;
  // outbox segment r: room for 2x destination r's vertex count (BFS sends each
  // remote vertex once per improvement; PR flushes each at most once per round;
  // colouring sends each changed vertex once per round)
  d->seg.assign(world + 1, 0);
  for (int r = 0; r < world; ++r) d->seg[r + 1] = d->seg[r] + (r == rank ? 0 : 2 * (bounds[r + 1] - bounds[r]) + 1024);
  if (cudaMalloc(&d->d_bounds, (world + 1) * sizeof(int64_t)) != cudaSuccess ||
      cudaMalloc(&d->d_seg, (world + 1) * sizeof(int64_t)) != cudaSuccess ||
      pool_malloc(&d->outbox, std::max<int64_t>(d->seg[world], 1) * sizeof(uint64_t)) != cudaSuccess ||
      cudaMalloc(&d->d_cnt, (world + 1) * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&d->d_rv, (world + 3) * sizeof(int64_t)) != cudaSuccess ||
      cudaMalloc(&d->d_round, sizeof(DevRound)) != cudaSuccess)
    return fail(atos_set_error(ATOS_ERR_OUT_OF_MEMORY, "partition buffers"));
  CK(cudaMemcpy(d->d_bounds, bounds.data(), (world + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d->d_seg, d->seg.data(), (world + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
  *out = g;
  return ATOS_OK;
}

// One rank's local work of a partitioned call (rounds.h Engine).
struct PartEngine : atos_rounds::Engine {
  enum { BFS = 0, PR = 1, GC = 2 };
  LaunchCtx* c = nullptr;
  atos_graph g = nullptr;
  DistState* d = nullptr;
  int app = 0;
  float alpha = 0.85f, eps = 1e-6f;
  bool disc = false;
  bool on_device() const override { return true; }

  Outbox outbox_view() const {
    return Outbox{d->outbox, d->d_seg, d->d_cnt, reinterpret_cast<unsigned int*>(d->d_cnt + d->world)};
  }
  Queue queue() const { return make_queue(g, c->cfg, (uint32_t)app); }

  // discrete: one superstep over the device-side snapshot [h, t) with the fixed persistent-size grid
  template <class P, class A, int W>
  atos_status superstep_w(const A& a) {
    auto kern = k_discrete_dev<P, A, W>;
    const int F = c->cfg.fetch_size, T = clamp_threads(W, F, c->cfg.cta_threads);
    const size_t smem = worker_smem_bytes<P>(W, F, T);
    if (smem > 227 * 1024) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "fetch_size %d needs %zu B shared memory", F, smem);
    CKS(set_smem(kern, smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem));
    const unsigned blocks = (unsigned)std::max(1, per_sm) * (unsigned)g->sms;
    k_round_snap<<<1, 1, 0, c->s>>>(d->d_round, g->ws.ctl);
    kern<<<blocks, T, smem, c->s>>>(a, c->gv, queue(), F, d->d_round);
    k_round_head<<<1, 1, 0, c->s>>>(d->d_round, g->ws.ctl);
    CK(cudaGetLastError());
    c->launches += 3;
    return ATOS_OK;
  }
  template <class P, class A>
  atos_status superstep(const A& a) {
    switch (c->cfg.worker) {
      case ATOS_WORKER_THREAD: return superstep_w<P, A, W_THREAD>(a);
      case ATOS_WORKER_WARP: return superstep_w<P, A, W_WARP>(a);
      default: return superstep_w<P, A, W_CTA>(a);
    }
  }
  template <class P, class A>
  atos_status local(const A& a) {
    return disc ? superstep<P>(a) : run_persistent<P>(*c, a, queue());
  }

  atos_status local_round(int flush_all) override {
    Workspace& w = g->ws;
    const uint32_t vb = (uint32_t)g->v_begin, ve = (uint32_t)g->v_end;
    const Outbox ob = outbox_view();
    CK(cudaMemsetAsync(d->d_cnt, 0, (d->world + 1) * sizeof(unsigned long long), c->s));
    if (app == GC) {
      CKS((local<GcPolicy<GC_UBER>>(GcApp{d->gc_color, w.u32a, vb, ve, d->gc_chg})));
      if (g->n) {
        k_gc_pack<<<fill_blocks(g->n, g->sms), 256, 0, c->s>>>(c->gv, d->gc_color, d->gc_chg, vb, d->d_bounds,
                                                                d->world, d->rank, ob);
        c->launches++;
      }
    } else if (app == BFS) {
      CKS(local<EdgeMapPolicy<BfsPartApp>>(BfsPartApp{w.u32a, w.u32b, d->sent_min, c->cfg.bfs_filter, vb, ve,
                                                      d->d_bounds, d->world, ob}));
    } else {
      CKS(local<EdgeMapPolicy<PrPartAppT<double>>>(
          PrPartAppT<double>{w.f64a, w.f64b, (double)alpha, (double)eps, vb, ve, d->racc}));
    }
    if (app == PR) {
      for (int r = 0; r < d->world; ++r) {
        if (r == d->rank || d->bounds[r + 1] == d->bounds[r]) continue;
        k_pr_flush<<<fill_blocks(d->bounds[r + 1] - d->bounds[r], g->sms), 256, 0, c->s>>>(
            d->racc, d->bounds[r], d->bounds[r + 1], r, ob, eps, flush_all);
        c->launches++;
      }
    }
    k_round_vec<<<1, 32, 0, c->s>>>(d->d_cnt, d->world, w.ctl, disc ? d->d_round : nullptr, d->d_rv);
    c->launches++;
    CK(cudaGetLastError());
    return ATOS_OK;
  }
  const int64_t* round_vector() override { return d->d_rv; }
  const uint64_t* outbox() override { return d->outbox; }
  const int64_t* outbox_seg() override { return d->seg.data(); }
  atos_status inbox(int64_t cap, uint64_t** p) override {
    if (cap > d->inbox_cap) {
      pool_free(d->inbox);
      d->inbox = nullptr;
      d->inbox_cap = 0;
      const int64_t want = std::max<int64_t>(cap, std::max<int64_t>(1024, 2 * d->inbox_cap));
      CK(pool_malloc(&d->inbox, (size_t)want * sizeof(uint64_t)));
      d->inbox_cap = want;
    }
    *p = d->inbox;
    return ATOS_OK;
  }
  atos_status apply(int64_t count) override {
    if (!count) return ATOS_OK;
    Workspace& w = g->ws;
    Queue q = queue();
    const int blocks = fill_blocks(count, g->sms);
    const uint64_t* dm = d->inbox;
    if (app == GC) {
      k_gc_apply<<<blocks, 256, 0, c->s>>>(dm, count, d->gc_color, d->gc_gchg, 1);
      if (g->n)
        k_gc_ghost_scan<<<fill_blocks(g->n * 32, g->sms), 256, 0, c->s>>>(c->gv, d->gc_color, d->gc_gchg, w.u32a,
                                                                           (uint32_t)g->v_begin, q);
      k_gc_apply<<<blocks, 256, 0, c->s>>>(dm, count, nullptr, d->gc_gchg, 0);
      c->launches += g->n ? 3 : 2;
    } else if (app == BFS) {
      k_part_apply<0, float><<<blocks, 256, 0, c->s>>>(dm, count, w.u32a, (float*)nullptr, 0.f, q);
      c->launches++;
    } else {
      k_part_apply<1, double><<<blocks, 256, 0, c->s>>>(dm, count, nullptr, w.f64b, (double)eps, q);
      c->launches++;
    }
    CK(cudaGetLastError());
    return ATOS_OK;
  }
  atos_status to_host(void* dst, const void* src, size_t bytes) override {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    return ATOS_OK;
  }
  atos_status to_engine(void* dst, const void* src, size_t bytes) override {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->s));
    CK(cudaStreamSynchronize(c->s));
    return ATOS_OK;
  }
};

// Local state of a partitioned call (a2, timed with the rounds).
static atos_status part_init(PartEngine& e, int64_t src) {
  LaunchCtx& c = *e.c;
  atos_graph g = e.g;
  DistState* d = e.d;
  Workspace& w = g->ws;
  const int64_t n = g->n, N = g->global_n, n1 = std::max<int64_t>(n, 1), N1 = std::max<int64_t>(N, 1);
  CKS(ws_prepare(g, c.cfg, n, (e.app == PartEngine::GC ? 4 : 2) * (uint64_t)n1, true, c.s));
  if (e.app >= 1 && (uint64_t)n > w.cap) return atos_set_error(ATOS_ERR_QUEUE_OVERFLOW, "queue_capacity < n");
  if (e.app == PartEngine::BFS) {
    CKS(ensure(w.u32a, w.u32a_n, (size_t)n1));
    CKS(ensure(w.u32b, w.u32b_n, (size_t)n1));
    if (!d->sent_min) CK(pool_malloc(&d->sent_min, (size_t)N1 * sizeof(uint32_t)));
  } else if (e.app == PartEngine::GC) {
    CKS(ensure(w.u32a, w.u32a_n, (size_t)n1));
    if (!d->gc_color) CK(pool_malloc(&d->gc_color, (size_t)N1 * sizeof(int32_t)));
    if (!d->gc_gchg) {
      CK(pool_malloc(&d->gc_gchg, (size_t)N1));
      CK(cudaMemsetAsync(d->gc_gchg, 0, (size_t)N1, c.s));
    }
    if (!d->gc_chg) CK(pool_malloc(&d->gc_chg, (size_t)n1));
  } else {
    CKS(ensure(w.f32a, w.f32a_n, (size_t)n1));
    CKS(ensure(w.f64a, w.f64a_n, (size_t)n1));
    CKS(ensure(w.f64b, w.f64b_n, (size_t)n1));  // fp64 residues (R34)
    if (!d->racc) CK(pool_malloc(&d->racc, (size_t)N1 * sizeof(double)));
  }
  CK(cudaEventRecord(w.ev[0], c.s));
  CKS(ring_reset(w, c.s));
  CK(cudaMemsetAsync(d->d_round, 0, sizeof(DevRound), c.s));
  if (e.app == PartEngine::BFS) {
    const bool mine = src >= g->v_begin && src < g->v_end;
    k_bfs_init<<<fill_blocks(n1, g->sms), 256, 0, c.s>>>(w.u32a, w.u32b, nullptr, n, mine ? src - g->v_begin : -1);
    k_fill<uint32_t><<<fill_blocks(N1, g->sms), 256, 0, c.s>>>(d->sent_min, N, 0xFFFFFFFFu);
    k_ctl_init<<<1, 1, 0, c.s>>>(w.ctl, mine ? 1 : 0, w.ring, mine ? src - g->v_begin : -1);
    c.launches += 3;
  } else if (e.app == PartEngine::GC) {
    // replica colours -1, pend = 1 (every vertex has its initial ASSIGN queued), ASSIGN(v) in id order (R22)
    CK(cudaMemsetAsync(d->gc_chg, 0, (size_t)n1, c.s));
    k_fill<int32_t><<<fill_blocks(N1, g->sms), 256, 0, c.s>>>(d->gc_color, N, -1);
    k_fill<uint32_t><<<fill_blocks(n1, g->sms), 256, 0, c.s>>>(w.u32a, n, 1u);
    k_ctl_init<<<1, 1, 0, c.s>>>(w.ctl, (uint64_t)n, w.ring, -1);
    if (n) k_ring_prefill<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.ring, n, 0u);
    c.launches += n ? 4 : 3;
  } else {
    CK(cudaMemsetAsync(d->racc, 0, (size_t)N * sizeof(double), c.s));
    k_fill<double><<<fill_blocks(n1, g->sms), 256, 0, c.s>>>(w.f64a, n, 1.0 - (double)e.alpha);
    k_ctl_init<<<1, 1, 0, c.s>>>(w.ctl, (uint64_t)n, w.ring, -1);
    c.launches += 2;
    if (n) {
      k_ring_prefill<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.ring, n, 0u);
      // R30: local seeding sums accumulate in the fp64 residues; remote ones in racc (fp64)
      k_fill<double><<<fill_blocks(n1, g->sms), 256, 0, c.s>>>(w.f64b, n, 0.0);
      PrPartInitAppT<double> ia{w.f64b, d->racc, (1.0 - (double)e.alpha) * (double)e.alpha, (uint32_t)g->v_begin,
                                (uint32_t)g->v_end};
      LaunchCtx ci = c;
      ci.cfg.worker = ATOS_WORKER_CTA;
      CKS((bsp_step_w<EdgeMapPolicy<PrPartInitAppT<double>>, PrPartInitAppT<double>, W_CTA>(
          ci, ia, nullptr, (uint64_t)n, nullptr, nullptr, 256, nullptr)));
      c.launches += 3;
    }
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(w.ev[1], c.s));
  return ATOS_OK;
}

// A partitioned atos_bfs / atos_pagerank / atos_color: init, the round loop, outputs.
static atos_status part_call(LaunchCtx& c, int app, int64_t src, float alpha, float eps, void* out,
                             int32_t* ncolors_out, atos_stats* st) {
  atos_graph g = c.g;
  DistState* d = g->dist;
  if (c.cfg.kernel == ATOS_KERNEL_BSP)
    return atos_set_error(ATOS_ERR_UNSUPPORTED, "partitioned runs use the persistent or discrete kernel");
  if (app == PartEngine::GC && d->world > 64) return atos_set_error(ATOS_ERR_UNSUPPORTED, "partitioned colouring: world > 64");
  if (g->n && !out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "output == NULL");
  PartEngine e;
  e.c = &c;
  e.g = g;
  e.d = d;
  e.app = app;
  e.alpha = alpha;
  e.eps = eps;
  e.disc = c.cfg.kernel == ATOS_KERNEL_DISCRETE;
  CKS(part_init(e, src));
  ExchangeRef xr(d->comm, c.s);
  atos_rounds::RoundStats rs;
  CKS(atos_rounds::run_rounds(*xr.ex, e, app == PartEngine::PR, c.cfg.timeout_s, rs, atos_set_error));
  Workspace& w = g->ws;
  const int64_t n = g->n;
  if (n) {
    if (app == PartEngine::BFS) {
      CKS(copy_out(out, w.u32a, (size_t)n * sizeof(uint32_t), c.s));
    } else if (app == PartEngine::GC) {
      CKS(copy_out(out, d->gc_color + g->v_begin, (size_t)n * sizeof(int32_t), c.s));
    } else {
      k_f64_to_f32<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.f64a, w.f32a, n);
      c.post_launches++;
      CK(cudaGetLastError());
      CKS(copy_out(out, w.f32a, (size_t)n * sizeof(float), c.s));
    }
  }
  int64_t colors = 0;
  if (app == PartEngine::GC) {
    // global colour count: max over ranks of the owned vertices' largest colour + 1
    CK(cudaMemsetAsync(d->d_rv, 0, sizeof(int64_t), c.s));
    if (n) k_max_color_i64<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(d->gc_color + g->v_begin, n, d->d_rv);
    c.post_launches++;
    std::vector<int64_t> M(d->world);
    if (xr.ex->on_device()) {
      CKS(xr.ex->gather(d->d_rv, 1, M.data()));
    } else {
      int64_t mine = 0;
      CKS(e.to_host(&mine, d->d_rv, sizeof(int64_t)));
      CKS(xr.ex->gather(&mine, 1, M.data()));
    }
    for (int64_t v : M) colors = std::max(colors, v);
    if (ncolors_out) *ncolors_out = (int32_t)colors;
  }
  CK(cudaEventRecord(w.ev[2], c.s));
  CKS(read_ctl(g, c.s));
  w.dirty = std::max<uint64_t>(std::min<uint64_t>(w.h_ctl->tail.v, w.cap), w.dirty_rest);
  if (st) {
    float ms = 0, kms = 0;
    CK(cudaEventElapsedTime(&ms, w.ev[0], w.ev[2]));
    CK(cudaEventElapsedTime(&kms, w.ev[1], w.ev[2]));
    st->ms = ms;
    st->kernel_ms = kms;
    st->kernel_launches = c.launches + c.post_launches;
    st->chunk_tasks = (int64_t)w.h_ctl->chunk_done.v;
    st->tasks_popped = (int64_t)w.h_ctl->stats[0].v - st->chunk_tasks;
    st->tasks_pushed = (int64_t)w.h_ctl->stats[1].v;
    st->edges_processed = (int64_t)w.h_ctl->stats[2].v;
    st->rounds = rs.rounds;
    st->queue_high_water = (int64_t)w.h_ctl->high_water.v;
    st->bytes_sent = rs.bytes_sent;
    st->trace_records = (int64_t)w.h_ctl->trace_count.v;
    st->num_colors = (int32_t)colors;
  }
  return ATOS_OK;
}
