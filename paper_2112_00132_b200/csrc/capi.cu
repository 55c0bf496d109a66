// capi.cu — the C ABI of libatos.so (include/atos.h): graph handles,
// workspaces, the persistent / discrete / BSP drivers for BFS, PageRank and
// colouring, timing and statistics.  Every function returns atos_status and
// records a detail string on error; nothing here aborts the process.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdarg>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/atos.h"
#include "kernels.cuh"
#include "capi_internal.h"

using namespace atos;

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

atos_status atos_set_error(atos_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

#define CK(call)                                                                                          \
  do {                                                                                                    \
    cudaError_t e_ = (call);                                                                              \
    if (e_ != cudaSuccess) {                                                                              \
      (void)cudaGetLastError();                                                                           \
      return atos_set_error(e_ == cudaErrorMemoryAllocation ? ATOS_ERR_OUT_OF_MEMORY : ATOS_ERR_CUDA,   \
                            "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));           \
    }                                                                                                     \
  } while (0)

#define CKS(call)                        \
  do {                                   \
    atos_status s_ = (call);             \
    if (s_ != ATOS_OK) return s_;        \
  } while (0)

// ------------------------------------------------------------------ HBM pool
// Graph-lifetime arrays (CSR, queue ring, per-vertex state) come from a
// PRIVATE stream-ordered memory pool per device (cudaMemPoolCreate) that keeps
// up to kPoolRetainBytes of freed HBM mapped: a create/destroy cycle of the
// same graph (the e2e loop, a serving process) reuses it instead of paying
// cudaMalloc/cudaFree (measured 24-100 ms per RMAT-24 create).  The device's
// default pool — shared with every other library in the process — is left
// alone, and atos_pool_trim() hands retained memory back.  Allocations and
// frees are ordered on a library-owned stream: an allocation is completed
// before it is returned (so any caller stream may use it); a free needs no
// wait, because every entry point is synchronous — no work on the array is
// outstanding when a handle is destroyed or a workspace regrows.
static constexpr uint64_t kPoolRetainBytes = 32ull << 30;  // 18% of a B200; 8 GB measured trims of 155-460 ms per destroy in the e2e loop

struct DevPool {
  cudaMemPool_t pool = nullptr;
  cudaStream_t stream = nullptr;
};

static cudaError_t dev_pool(DevPool** out) {
  static DevPool pools[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  DevPool& d = pools[dev];
  if (!d.pool) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if ((e = cudaMemPoolCreate(&pool, &props)) != cudaSuccess) return e;
    uint64_t thr = kPoolRetainBytes;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    cudaStream_t s = nullptr;
    if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess) return e;
    d.stream = s;
    d.pool = pool;
  }
  *out = &d;
  return cudaSuccess;
}

static cudaError_t pool_malloc(void** p, size_t bytes) {
  DevPool* d = nullptr;
  cudaError_t e = dev_pool(&d);
  if (e != cudaSuccess) return e;
  e = cudaMallocFromPoolAsync(p, bytes, d->pool, d->stream);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(d->stream);
}

template <class T>
static cudaError_t pool_malloc(T** p, size_t bytes) { return pool_malloc(reinterpret_cast<void**>(p), bytes); }

static void pool_free(void* p) {
  if (!p) return;
  DevPool* d = nullptr;
  if (dev_pool(&d) == cudaSuccess) cudaFreeAsync(p, d->stream);
  (void)cudaGetLastError();
}

extern "C" atos_status atos_pool_trim(uint64_t keep_bytes) {
  DevPool* d = nullptr;
  cudaError_t e = dev_pool(&d);
  if (e == cudaSuccess) e = cudaStreamSynchronize(d->stream);
  if (e == cudaSuccess) e = cudaMemPoolTrimTo(d->pool, (size_t)keep_bytes);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return atos_set_error(ATOS_ERR_CUDA, "atos_pool_trim: %s", cudaGetErrorString(e));
  }
  return ATOS_OK;
}

extern "C" atos_status atos_pool_reserved(uint64_t* bytes) {
  if (!bytes) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bytes == NULL");
  DevPool* d = nullptr;
  cudaError_t e = dev_pool(&d);
  uint64_t v = 0;
  if (e == cudaSuccess) e = cudaMemPoolGetAttribute(d->pool, cudaMemPoolAttrReservedMemCurrent, &v);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    return atos_set_error(ATOS_ERR_CUDA, "atos_pool_reserved: %s", cudaGetErrorString(e));
  }
  *bytes = v;
  return ATOS_OK;
}

extern "C" const char* atos_status_string(atos_status s) {
  switch (s) {
    case ATOS_OK: return "ATOS_OK";
    case ATOS_ERR_INVALID_ARGUMENT: return "ATOS_ERR_INVALID_ARGUMENT";
    case ATOS_ERR_INVALID_GRAPH: return "ATOS_ERR_INVALID_GRAPH";
    case ATOS_ERR_OUT_OF_MEMORY: return "ATOS_ERR_OUT_OF_MEMORY";
    case ATOS_ERR_CUDA: return "ATOS_ERR_CUDA";
    case ATOS_ERR_NCCL: return "ATOS_ERR_NCCL";
    case ATOS_ERR_QUEUE_OVERFLOW: return "ATOS_ERR_QUEUE_OVERFLOW";
    case ATOS_ERR_TIMEOUT: return "ATOS_ERR_TIMEOUT";
    case ATOS_ERR_UNSUPPORTED: return "ATOS_ERR_UNSUPPORTED";
  }
  return "ATOS_ERR_UNKNOWN";
}
extern "C" const char* atos_last_error(void) { return g_last_error.c_str(); }
extern "C" const char* atos_version(void) { return "atos-b200 1.0 sm_100a"; }

extern "C" void atos_config_default(atos_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->struct_size = sizeof(atos_config);
  c->kernel = ATOS_KERNEL_PERSISTENT;
  c->worker = ATOS_WORKER_CTA;
  c->cta_threads = 256;
  c->fetch_size = 256;
  c->num_blocks = 0;
  c->bfs_filter = 1;
  c->pr_activation = 0;
  c->check_size = 32;
  c->gc_literal = 0;
  c->pr_residue_fp64 = 0;
  c->adaptive_fetch = 1;
  c->device_loop = 0;
  c->queue_capacity = 0;
  c->timeout_s = 0.0;
  c->stream = nullptr;
  c->stage_edges = 0;  // off: measured slower on RMAT-24 (the staging smem costs L1 the probes use)
  c->sink_defer = 1;
  c->pr_defer_degree = 0;
  c->pr_defer_factor = 4;
  c->pr_hub_check = 4;
  c->hub_split = -1;
}

#ifndef ATOS_BACKOFF_NS
#define ATOS_BACKOFF_NS 256  // idle-poll backoff cap (ns) of queue poppers
#endif

static atos_status check_failures();

// asynchronous peer-memory partitions (peer_impl.cuh)
struct PeerState;
static atos_status peer_bfs(atos_graph g, int64_t src, const atos_config& cfg, uint32_t* depth_out, atos_stats* st);
static atos_status peer_pagerank(atos_graph g, float alpha, float eps, const atos_config& cfg, float* rank_out,
                                 atos_stats* st);
static void peer_free(PeerState* ps);

static atos_status check_config(const atos_config* c) {
  if (c->struct_size != sizeof(atos_config))
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "atos_config.struct_size %u != %zu (use atos_config_default)",
                          c->struct_size, sizeof(atos_config));
  if (c->kernel < 0 || c->kernel > 2) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bad kernel %d", c->kernel);
  if (c->worker < 0 || c->worker > 2) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "bad worker %d", c->worker);
  if (c->cta_threads < 32 || c->cta_threads > 1024 || c->cta_threads % 32)
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "cta_threads %d not a multiple of 32 in [32,1024]", c->cta_threads);
  if (c->fetch_size < 1 || c->fetch_size > (1 << 16))
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "fetch_size %d not in [1, 65536]", c->fetch_size);
  if (c->num_blocks < 0) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "num_blocks < 0");
  if (c->queue_capacity < 0) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "queue_capacity < 0");
  if (!(c->timeout_s >= 0)) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "timeout_s < 0");
  if (c->pr_activation != 0 && c->pr_activation != 1)
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "pr_activation must be 0 or 1");
  if (c->trace && c->trace_capacity < 0) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "trace_capacity < 0");
  if (c->stage_edges < -1 || c->stage_edges > (1 << 20))
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "stage_edges %d not in [-1, 2^20]", c->stage_edges);
  if (c->hub_split < -1 || c->hub_split > 1)
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "hub_split %d not in {-1, 0, 1}", c->hub_split);
  if (c->pr_hub_check < 0 || c->pr_hub_check > (1 << 20))
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "pr_hub_check %d not in [0, 2^20]", c->pr_hub_check);
  if (c->pr_activation == 1 && c->check_size < 1)
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "check_size < 1");
  return ATOS_OK;
}

// ------------------------------------------------------------------ graph
__global__ void k_validate(const int64_t* off, const int32_t* col, int64_t n, int64_t m, int64_t col_bound,
                           unsigned int* bad, bool cols) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = tid; v < n; v += stride)
    if (off[v + 1] < off[v]) atomicOr(bad, 1u);
  for (int64_t e = tid; cols && e < m; e += stride)
    if (col[e] < 0 || (int64_t)col[e] >= col_bound) atomicOr(bad, 2u);
  if (tid == 0 && (off[0] != 0 || off[n] != m)) atomicOr(bad, 4u);
}
// One pass over a freshly uploaded chunk of columns [e0, e1): the range check
// of ATOS_GRAPH_VALIDATE (bad |= 2) and/or the in-degree count of R34's hub
// tagging (in-range targets only; a bad column fails the create anyway).
__global__ void k_col_pass(const int32_t* col, int64_t e0, int64_t e1, int64_t n, int64_t col_bound,
                           uint32_t* indeg, unsigned int* bad) {
  bool ok = true;
  for (int64_t e = e0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = col[e];
    const bool in = c >= 0 && (int64_t)c < col_bound;
    ok &= in;
    if (indeg && in && (int64_t)c < n) atomicAdd(indeg + c, 1u);
  }
  if (bad && !ok) atomicOr(bad, 2u);
}
__global__ void k_max_degree(const int64_t* off, int64_t n, unsigned long long* out) {
  unsigned long long m = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)(off[v + 1] - off[v]));
  for (int d = 16; d; d >>= 1) m = max(m, __shfl_xor_sync(FULL_MASK, m, d));
  if (lane_id() == 0) atomicMax(out, m);
}

static int grid_for(int64_t work, int threads, int sms) {
  int64_t b = (work + threads - 1) / threads;
  int64_t cap = (int64_t)sms * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

static atos_status device_sms(int* sms) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
  return ATOS_OK;
}

// L2 set-aside for evict_last (persisting) lines: the per-vertex state the
// edge loop hits at random (BFS dist, PR residue) is accessed with an
// evict_last policy, which only persists within this carve-out (default 0;
// measured 51% atomic misses on a 64 MB residue array without it).
static void l2_carveout(int device) {
  int max_persist = 0;
  if (cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device) == cudaSuccess &&
      max_persist > 0) {
    size_t cur = 0;
    if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) == cudaSuccess && cur < (size_t)max_persist)
      (void)cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist);
    (void)cudaGetLastError();
  }
}

// Upload of a library-owned CSR copy, then ONE pass over the columns
// (k_col_pass): the VALIDATE range check fused with the in-degree count R34's
// hub tags need.  A whole-graph copy (col_bound == n, m > 0) leaves the
// in-degrees in g->d_indeg for the tagging.  (A pipelined variant — columns in
// 128 MB chunks on a second stream with the pass over each landed chunk —
// made create 2-3 ms shorter but the PageRank kernel that later runs on the
// uploaded graph 2.3% slower, 160.5 -> 164.1 ms, in same-box A/B runs, so it
// was dropped: profiles/r02_e2e_breakdown.md.)
static atos_status upload_csr(atos_graph g, const int64_t* off, const int32_t* col, bool dev_ptrs,
                              int64_t col_bound, bool validate) {
  const int64_t n = g->n, m = g->m;
  const cudaMemcpyKind kind = dev_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyDefault;
  const bool count = col_bound == n && m > 0;
  CK(cudaMalloc(&g->d_scratch, 256));
  CK(cudaMemset(g->d_scratch, 0, 256));
  if (count) {
    CK(pool_malloc(&g->d_indeg, (size_t)n * sizeof(uint32_t)));
    CK(cudaMemset(g->d_indeg, 0, (size_t)n * sizeof(uint32_t)));
  }
  CK(cudaMemcpy(g->d_off, off, (size_t)(n + 1) * sizeof(int64_t), kind));
  if (m) CK(cudaMemcpy(g->d_col, col, (size_t)m * sizeof(int32_t), kind));
  if (m && (validate || count))
    k_col_pass<<<grid_for(m, 256, g->sms), 256>>>(g->d_col, 0, m, n, col_bound, count ? g->d_indeg : nullptr,
                                                  validate ? reinterpret_cast<unsigned int*>(g->d_scratch) : nullptr);
  CK(cudaGetLastError());
  return ATOS_OK;
}

atos_status graph_init_common(atos_graph g, const int64_t* off, const int32_t* col, int64_t n, int64_t m,
                              uint32_t flags, int64_t col_bound) {
  if (col_bound < 0) col_bound = n;
  g->n = n;
  g->m = m;
  g->symmetric = (flags & ATOS_GRAPH_SYMMETRIC) != 0;
  CK(cudaGetDevice(&g->device));
  CKS(device_sms(&g->sms));
  const bool dev_ptrs = flags & ATOS_GRAPH_DEVICE_PTRS;
  const bool borrow = dev_ptrs && (flags & ATOS_GRAPH_BORROW) && (((uintptr_t)col & 15) == 0);
  if (borrow) {
    g->d_off = const_cast<int64_t*>(off);
    g->d_col = const_cast<int32_t*>(col);
    g->col_cap = m;
    g->owned = false;
  } else {
    CK(pool_malloc(&g->d_off, (size_t)(n + 1) * sizeof(int64_t)));
    g->col_cap = ((m + 3) & ~(int64_t)3) + 4;  // padded: 16-B bulk copies may overrun a list's end
    CK(pool_malloc(&g->d_col, (size_t)g->col_cap * sizeof(int32_t)));
    CK(cudaMemset(g->d_col + m, 0, (size_t)(g->col_cap - m) * sizeof(int32_t)));  // the pad only
    g->owned = true;
    CKS(upload_csr(g, off, col, dev_ptrs, col_bound, (flags & ATOS_GRAPH_VALIDATE) != 0));
  }
  l2_carveout(g->device);
  if (!g->d_scratch) {
    CK(cudaMalloc(&g->d_scratch, 256));
    CK(cudaMemset(g->d_scratch, 0, 256));
  }
  if (flags & ATOS_GRAPH_VALIDATE) {
    unsigned int* bad = reinterpret_cast<unsigned int*>(g->d_scratch);
    // owned copies had their columns checked chunk by chunk during the upload (k_col_pass)
    k_validate<<<grid_for(std::max(n, m), 256, g->sms), 256>>>(g->d_off, g->d_col, n, m, col_bound, bad, !g->owned);
    unsigned int hbad = 0;
    CK(cudaMemcpy(&hbad, bad, sizeof hbad, cudaMemcpyDeviceToHost));
    if (hbad)
      return atos_set_error(ATOS_ERR_INVALID_GRAPH, "CSR validation failed (code %u: 1=non-monotone offsets, "
                            "2=column out of range, 4=off[0]!=0 or off[n]!=m)", hbad);
  }
  unsigned long long* md = reinterpret_cast<unsigned long long*>(g->d_scratch) + 2;
  if (n) k_max_degree<<<grid_for(n, 256, g->sms), 256>>>(g->d_off, n, md);
  unsigned long long hmd = 0;
  CK(cudaMemcpy(&hmd, md, sizeof hmd, cudaMemcpyDeviceToHost));
  g->max_degree = (int64_t)hmd;
  // dangling-vertex bitmap (R29): a property of the immutable CSR, like the max degree
  if (!g->d_sink) CK(pool_malloc(&g->d_sink, (size_t)std::max<int64_t>(1, (n + 31) / 32) * sizeof(uint32_t)));
  if (n) k_sink_bitmap<<<grid_for(n, 256, g->sms), 256>>>(g->d_off, n, g->d_sink);
  // Hub tags (R34): a library-owned CSR of a whole graph gets bit 31 set on
  // every column entry whose target has in-degree >= HUB_IN_DEG, plus a hub
  // bitmap.  (Borrowed columns are the caller's and partitioned graphs only
  // know local edges: neither is tagged, and PageRank keeps fp64 residues.)
  if (g->owned && col_bound == n && m > 0) {
    uint32_t* indeg = g->d_indeg;  // counted during the upload (upload_csr)
    g->d_indeg = nullptr;
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(g->d_scratch) + 4;
    CK(cudaMemset(cnt, 0, sizeof(unsigned long long)));
    if (!g->d_hub) CK(pool_malloc(&g->d_hub, (size_t)((n + 31) / 32) * sizeof(uint32_t)));
    k_hub_bitmap<<<grid_for(n, 256, g->sms), 256>>>(indeg, n, HUB_IN_DEG, g->d_hub, cnt);
    unsigned long long hubs = 0;
    CK(cudaMemcpy(&hubs, cnt, sizeof hubs, cudaMemcpyDeviceToHost));
    g->num_hubs = (int64_t)hubs;
    // the in-degree array (n words) is dead once the hub bitmap exists: it holds the interleaved tag map
    k_tag_map<<<grid_for((n + 15) / 16, 256, g->sms), 256>>>(g->d_hub, g->d_sink, n, indeg);
    k_tag_hubs<<<grid_for((m + 3) / 4, 256, g->sms), 256>>>(g->d_col, m, n, indeg);
    if (hubs) {  // R35: the hubs a PageRank sweep may activate (dangling hubs are absorbed at the end, R29)
      CK(pool_malloc(&g->d_hub_list, (size_t)hubs * sizeof(uint32_t)));
      CK(cudaMemset(cnt, 0, sizeof(unsigned long long)));
      k_hub_list<<<grid_for(n, 256, g->sms), 256>>>(g->d_hub, g->d_off, n, g->d_hub_list, cnt);
      unsigned long long nl = 0;
      CK(cudaMemcpy(&nl, cnt, sizeof nl, cudaMemcpyDeviceToHost));
      g->num_hub_list = (int64_t)nl;
    }
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    pool_free(indeg);
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return check_failures();
}

// Per-run control blocks (device QueueCtl, its pinned host mirror, the BSP
// counter, the timing events) are recycled across graph handles: a handle's
// first call would otherwise pay cudaMalloc + cudaMallocHost + event creation,
// and its destroy the matching frees (measured: ~6 ms of the first BFS on a
// fresh handle in the e2e loop).  Keyed by device; at most kCtlCache kept.
struct CtlBlock {
  int device;
  QueueCtl* ctl;
  QueueCtl* h_ctl;
  unsigned long long* fcount;
  cudaEvent_t ev[4];
};
static std::mutex g_ctl_mu;
static std::vector<CtlBlock> g_ctl_cache;
constexpr size_t kCtlCache = 16;

static atos_status ctl_acquire(Workspace& w, int device) {
  {
    std::lock_guard<std::mutex> lk(g_ctl_mu);
    for (size_t i = 0; i < g_ctl_cache.size(); ++i)
      if (g_ctl_cache[i].device == device) {
        const CtlBlock b = g_ctl_cache[i];
        g_ctl_cache.erase(g_ctl_cache.begin() + (std::ptrdiff_t)i);
        w.ctl = b.ctl;
        w.h_ctl = b.h_ctl;
        w.fcount = b.fcount;
        for (int k = 0; k < 4; ++k) w.ev[k] = b.ev[k];
        return ATOS_OK;
      }
  }
  CK(cudaMalloc(&w.ctl, sizeof(QueueCtl)));
  CK(cudaMallocHost(&w.h_ctl, sizeof(QueueCtl)));
  for (auto& e : w.ev) CK(cudaEventCreate(&e));
  CK(cudaMalloc(&w.fcount, 4 * sizeof(unsigned long long)));
  return ATOS_OK;
}

static void ctl_release(Workspace& w, int device) {
  if (!w.ctl || !w.h_ctl || !w.fcount || !w.ev[0] || !w.ev[1] || !w.ev[2] || !w.ev[3]) {
    cudaFree(w.ctl);
    cudaFree(w.fcount);
    if (w.h_ctl) cudaFreeHost(w.h_ctl);
    for (auto& e : w.ev)
      if (e) cudaEventDestroy(e);
    return;
  }
  {
    std::lock_guard<std::mutex> lk(g_ctl_mu);
    if (g_ctl_cache.size() < kCtlCache) {
      g_ctl_cache.push_back(CtlBlock{device, w.ctl, w.h_ctl, w.fcount, {w.ev[0], w.ev[1], w.ev[2], w.ev[3]}});
      return;
    }
  }
  cudaFree(w.ctl);
  cudaFree(w.fcount);
  cudaFreeHost(w.h_ctl);
  for (auto& e : w.ev) cudaEventDestroy(e);
}

static void graph_free(atos_graph g) {
  if (!g) return;
  if (g->peer) {
    peer_free(g->peer);
    delete g;
    return;
  }
  if (g->owned) {
    pool_free(g->d_off);
    pool_free(g->d_col);
  }
  cudaFree(g->d_scratch);
  pool_free(g->d_sink);
  pool_free(g->d_hub);
  pool_free(g->d_indeg);
  pool_free(g->d_hub_list);
  Workspace& w = g->ws;
  pool_free(w.ring);
  pool_free(w.u32a);
  pool_free(w.u32b);
  pool_free(w.u16a);
  pool_free(w.f32a);
  pool_free(w.f32b);
  pool_free(w.f64a);
  pool_free(w.f64b);
  pool_free(w.front[0]);
  pool_free(w.front[1]);
  pool_free(w.chunks);
  cudaFree(w.devround);
  dist_free(g);
  ctl_release(w, g->device);
  delete g;
}

extern "C" atos_status atos_graph_create(const int64_t* off, const int32_t* col, int64_t n, int64_t m, uint32_t flags,
                                         atos_graph* out) {
  if (!out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "out == NULL");
  *out = nullptr;
  if (n < 0 || m < 0) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "n < 0 or m < 0");
  if (!off || (m > 0 && !col)) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "NULL CSR pointer");
  if (n >= (int64_t)VID_MASK)
    return atos_set_error(ATOS_ERR_UNSUPPORTED, "n >= 2^30-1 (bits 30-31 of a column entry are tags, R37)");
  atos_graph g = new (std::nothrow) atos_graph_s();
  if (!g) return atos_set_error(ATOS_ERR_OUT_OF_MEMORY, "host allocation");
  atos_status s = graph_init_common(g, off, col, n, m, flags, n);
  if (s != ATOS_OK) {
    graph_free(g);
    return s;
  }
  *out = g;
  return ATOS_OK;
}

extern "C" atos_status atos_graph_destroy(atos_graph g) {
  if (!g) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "NULL graph");
  graph_free(g);
  return ATOS_OK;
}

extern "C" atos_status atos_graph_info(atos_graph g, int64_t* n, int64_t* m, int64_t* maxd) {
  if (!g) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "NULL graph");
  if (n) *n = g->global_n ? g->global_n : g->n;
  if (m) *m = g->m;
  if (maxd) *maxd = g->max_degree;
  return ATOS_OK;
}

// ------------------------------------------------------------------ workspace
template <class T>
static atos_status ensure(T*& p, size_t& have, size_t want_elems) {
  if (p && have >= want_elems) return ATOS_OK;
  pool_free(p);
  p = nullptr;
  have = 0;
  CK(pool_malloc(&p, std::max<size_t>(want_elems, 1) * sizeof(T)));
  have = want_elems;
  return ATOS_OK;
}

static uint64_t pow2_at_least(uint64_t x, uint64_t floor_cap = 1024) {
  uint64_t c = floor_cap;
  while (c < x) c <<= 1;
  return c;
}

atos_status ws_prepare(atos_graph g, const atos_config& cfg, int64_t n_local, uint64_t default_cap, bool need_ring,
                       cudaStream_t s) {
  Workspace& w = g->ws;
  if (!w.ctl) CKS(ctl_acquire(w, g->device));
  if (need_ring) {
    uint64_t cap = cfg.queue_capacity > 0 ? pow2_at_least((uint64_t)cfg.queue_capacity, 32) : pow2_at_least(default_cap);
    // The ring is allocated for the largest capacity asked so far and each run
    // uses its first `cap` slots (BFS and PageRank alternate 2n and 16n on one
    // handle: no reallocation per call).  `dirty` = leading slots that may hold
    // tags; a run clears the ones it will use, the rest stay recorded.
    if (cap > w.ring_slots) {
      pool_free(w.ring);
      w.ring = nullptr;
      CK(pool_malloc(&w.ring, cap * sizeof(uint64_t)));
      w.ring_slots = cap;
      w.clear = cap;
      w.dirty_rest = 0;
    } else {
      w.clear = std::min<uint64_t>(w.dirty, cap);
      w.dirty_rest = w.dirty > cap ? w.dirty : 0;
    }
    w.cap = cap;
    w.dirty = w.ring_slots;  // unknown until this run finishes cleanly (finish_stats narrows it)
  }
  (void)n_local;
  return ATOS_OK;
}

// Zero the ring slots the last run used (w.clear, set by ws_prepare), on the
// call's stream INSIDE the timed region (after ev[0]): a clean ring is part of
// every run's init (a2).
static atos_status ring_reset(Workspace& w, cudaStream_t s) {
  if (w.ring && w.clear) CK(cudaMemsetAsync(w.ring, 0, w.clear * sizeof(uint64_t), s));
  w.clear = 0;
  return ATOS_OK;
}

static Queue make_queue(atos_graph g, const atos_config& cfg, uint32_t kind) {
  Queue q{};
  q.ring = g->ws.ring;
  q.mask = g->ws.cap - 1;
  q.log2cap = 0;
  while ((1ull << q.log2cap) < g->ws.cap) q.log2cap++;
  q.ctl = g->ws.ctl;
  q.deadline = 0;
  q.timeout_ns = cfg.timeout_s > 0 ? (uint64_t)(cfg.timeout_s * 1e9) : 0;
  q.head_floor = 0;
  q.trace_kind = kind;
  q.backoff_ns = ATOS_BACKOFF_NS;
  q.trace = reinterpret_cast<TraceRec*>(cfg.trace);
  q.trace_cap = cfg.trace ? (uint64_t)cfg.trace_capacity : 0;
  return q;
}

// Checked builds (-DATOS_CHECKED, device.cuh chk): report and clear the first
// failed bounds check of the last kernels.  Product builds: always OK.
static atos_status check_failures() {
#ifdef ATOS_CHECKED
  {
    CheckRec r{};
    CK(cudaMemcpyFromSymbol(&r, g_atos_check, sizeof r));
    if (r.hit) {
      const CheckRec z{};
      CK(cudaMemcpyToSymbol(g_atos_check, &z, sizeof z));
      const char* names[] = {"engine.cuh", "gc.cuh", "cta_ws.cuh", "cta_ws2.cuh", "kernels.cuh", "dist_impl.cuh",
                             "device.cuh"};
      const char* f = "?";
      for (const char* nm : names)
        if (chk_fhash(nm) == r.file) f = nm;
      return atos_set_error(ATOS_ERR_CUDA, "bounds check failed at %s:%u (index %lld, bound %lld)", f, r.line,
                            r.value, r.bound);
    }
  }
#endif
  return ATOS_OK;
}

// Read back the control block; translate abort codes.
static atos_status read_ctl(atos_graph g, cudaStream_t s) {
  CK(cudaMemcpyAsync(g->ws.h_ctl, g->ws.ctl, sizeof(QueueCtl), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint64_t ab = g->ws.h_ctl->abort.v;
  if (ab == ABORT_OVERFLOW)
    return atos_set_error(ATOS_ERR_QUEUE_OVERFLOW, "task queue overflow (capacity %llu); retry with a larger "
                          "queue_capacity", (unsigned long long)g->ws.cap);
  if (ab == ABORT_TIMEOUT) return atos_set_error(ATOS_ERR_TIMEOUT, "device watchdog fired");
  if (ab) return atos_set_error(ATOS_ERR_CUDA, "unknown abort code %llu", (unsigned long long)ab);
  return check_failures();
}

// ------------------------------------------------------------------ launchers
struct LaunchCtx {
  atos_graph g;
  atos_config cfg;
  cudaStream_t s;
  GraphView gv;
  int64_t launches = 0;       // every kernel launched by the call up to the run's end
  int64_t post_launches = 0;  // launched after the run (reductions, conversions)
  int64_t rounds = 0;
  bool split = true;  // hub chunk splitting (R24) for persistent CTA edge-map workers
  std::chrono::steady_clock::time_point t0;
};

template <class K>
static atos_status set_smem(K kern, size_t smem) {
  if (smem > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return ATOS_OK;
}

// Warp/thread workers stage their claimed items in shared memory (4 B per item,
// FETCH per warp worker, 32*FETCH per thread-worker warp); shrink the block so
// the staging buffer fits in 227 KB.  CTA workers keep cta_threads.
static int clamp_threads(int W, int F, int T, bool ws = false) {
  if (W == W_CTA) return ws ? std::min(T, CTA_MAX_THREADS) : T;
  const size_t per_warp = (W == W_WARP ? (size_t)F : 32 * (size_t)F) * 4;
  int max_warps = (int)((227 * 1024) / per_warp);
  if (max_warps < 1) max_warps = 1;
  return std::min(T, max_warps * 32);
}

// Staged column elements per batch buffer: `req` (>0: as requested, -1: auto)
// rounded to a multiple of 4, bounded so per_sm CTAs still fit in the SM's
// shared memory with `l1_keep` bytes left to L1 (the BFS probes and PR
// residue atomics go through it).
static int stage_capacity(int req, int per_sm, size_t base_smem) {
  if (req == 0) return 0;
  const size_t sm_total = 228 * 1024, per_block_reserved = 1024, l1_keep = 64 * 1024;
  const size_t budget = (sm_total - l1_keep) / (size_t)per_sm;
  if (budget <= base_smem + per_block_reserved) return 0;
  size_t fit = (budget - base_smem - per_block_reserved) / (NBUF * 4);
  size_t want = req > 0 ? (size_t)req : 4096;
  size_t S = std::min(fit, want) & ~(size_t)3;
  return S >= 256 ? (int)S : 0;
}

template <class P, class App, int W>
static atos_status run_persistent_w(LaunchCtx& c, const App& app, const Queue& q) {
  auto kern = k_persistent<P, App, W>;
  const int F = c.cfg.fetch_size, T = clamp_threads(W, F, c.cfg.cta_threads, P::kWarpSpecialised);
  Queue qq = q;
  // R24 hub chunk tasks: only if some vertex is a hub; the table has one
  // 16-B entry per ring slot (device.cuh, Chunk; indexed by pos & mask), so it
  // cannot overflow.  Like the ring it is kept at the largest capacity seen.
  if (W == W_CTA && P::kSplit && c.split && c.g->max_degree > SPLIT_DEG) {
    Workspace& w = c.g->ws;
    if (w.chunk_cap < w.cap) {
      pool_free(w.chunks);
      w.chunks = nullptr;
      w.chunk_cap = 0;
      CK(pool_malloc(&w.chunks, w.cap * sizeof(Chunk)));
      w.chunk_cap = w.cap;
    }
    qq.chunks = w.chunks;
  }
  size_t smem = worker_smem_bytes<P>(W, F, T, true);
  if (smem > 227 * 1024) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "fetch_size %d x cta_threads %d needs %zu B shared memory (> 227 KB)", F, c.cfg.cta_threads, smem);
  constexpr int agents = AgentsTrait<App>::value;
  if (W == W_CTA && P::kWarpSpecialised && T < 32 * (agents + 1))
    return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "persistent CTA workers of this app need cta_threads >= %d "
                          "(%d queue-agent warp(s) + workers)", 32 * (agents + 1), agents);
  CKS(set_smem(kern, smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem));
  if (W == W_CTA && P::kWarpSpecialised && per_sm >= 1) {
    // Column staging (TMA bulk copies into each batch buffer): the capacity
    // that keeps the register-limited CTAs per SM resident, minus an L1 share.
    const int S = stage_capacity(c.cfg.stage_edges, per_sm, smem);
    if (S > 0) {
      qq.stage_cap = (uint32_t)S;
      smem = worker_smem_bytes<P>(W, F, T, true, S);
      CKS(set_smem(kern, smem));
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem));
    }
  }
  if (per_sm < 1) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "kernel cannot be resident with %d threads", T);
  int blocks = per_sm * c.g->sms;
  if (c.cfg.num_blocks > 0) blocks = std::min(blocks, c.cfg.num_blocks);  // persistent: <= resident maximum
  if (c.cfg.adaptive_fetch) qq.workers = (uint32_t)(W == W_CTA ? blocks : blocks * (T / 32));
  kern<<<blocks, T, smem, c.s>>>(app, c.gv, qq, F);
  CK(cudaGetLastError());
  c.launches++;
  return ATOS_OK;
}

template <class P, class App>
static atos_status run_persistent(LaunchCtx& c, const App& app, const Queue& q) {
  switch (c.cfg.worker) {
    case ATOS_WORKER_THREAD: return run_persistent_w<P, App, W_THREAD>(c, app, q);
    case ATOS_WORKER_WARP: return run_persistent_w<P, App, W_WARP>(c, app, q);
    default: return run_persistent_w<P, App, W_CTA>(c, app, q);
  }
}

static atos_status host_timeout(LaunchCtx& c) {
  if (c.cfg.timeout_s > 0) {
    double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - c.t0).count();
    if (el > c.cfg.timeout_s) return atos_set_error(ATOS_ERR_TIMEOUT, "host watchdog: %.1f s", el);
  }
  return ATOS_OK;
}

// Discrete scheduler: one launch per round over the queue snapshot [h, t).
template <class P, class App, int W>
static atos_status run_discrete_w(LaunchCtx& c, const App& app, Queue q, uint64_t t0, uint64_t h0 = 0,
                                  int64_t max_rounds = -1, uint64_t* h_end = nullptr) {
  auto kern = k_discrete<P, App, W>;
  const int F = c.cfg.fetch_size, T = clamp_threads(W, F, c.cfg.cta_threads);
  const size_t smem = worker_smem_bytes<P>(W, F, T);
  if (smem > 227 * 1024) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "fetch_size %d x cta_threads %d needs %zu B shared memory (> 227 KB)", F, c.cfg.cta_threads, smem);
  CKS(set_smem(kern, smem));
  const uint64_t chunk = (W == W_CTA) ? (uint64_t)F : (W == W_WARP ? (uint64_t)F : 32ull * (uint64_t)F);
  const uint64_t per_block = (W == W_CTA) ? 1 : (uint64_t)(T / 32);
  uint64_t h = h0, t = t0;
  uint64_t* h_tail = &c.g->ws.h_ctl->tail.v;
  while (h < t && max_rounds-- != 0) {
    const uint64_t workers = (t - h + chunk - 1) / chunk;
    uint64_t blocks = (workers + per_block - 1) / per_block;
    blocks = std::min<uint64_t>(blocks, 1u << 30);
    q.head_floor = t;
    kern<<<(unsigned)blocks, T, smem, c.s>>>(app, c.gv, q, h, t, F);
    CK(cudaGetLastError());
    c.launches++;
    c.rounds++;
    // one device->host crossing per round: the new tail and the abort flag
    CK(cudaMemcpyAsync(h_tail, &c.g->ws.ctl->tail.v, sizeof(uint64_t), cudaMemcpyDeviceToHost, c.s));
    CK(cudaMemcpyAsync(&c.g->ws.h_ctl->abort.v, &c.g->ws.ctl->abort.v, sizeof(uint64_t), cudaMemcpyDeviceToHost, c.s));
    CK(cudaStreamSynchronize(c.s));
    if (c.g->ws.h_ctl->abort.v) break;
    CKS(host_timeout(c));
    h = t;
    t = *h_tail;
  }
  if (h_end) *h_end = h;
  return ATOS_OK;
}

// Discrete strategy with the round loop on the device: a CUDA graph whose
// WHILE node repeats {one round over [h, t) with a fixed grid, round-end
// kernel that advances [h, t) and sets the condition}.
template <class P, class App, int W>
static atos_status run_discrete_graph_w(LaunchCtx& c, const App& app, Queue q, uint64_t t0, uint64_t* h_end) {
  auto kern = k_discrete_dev<P, App, W>;
  const int F = c.cfg.fetch_size, T = clamp_threads(W, F, c.cfg.cta_threads);
  const size_t smem = worker_smem_bytes<P>(W, F, T);
  if (smem > 227 * 1024) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "fetch_size %d x cta_threads %d needs %zu B shared memory (> 227 KB)", F, c.cfg.cta_threads, smem);
  CKS(set_smem(kern, smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem));
  const unsigned blocks = (unsigned)std::max(1, per_sm) * (unsigned)c.g->sms;
  Workspace& w = c.g->ws;
  if (!w.devround) CK(cudaMalloc(&w.devround, sizeof(DevRound)));
  DevRound r0{0, t0, 0, 0};
  CK(cudaMemcpyAsync(w.devround, &r0, sizeof r0, cudaMemcpyHostToDevice, c.s));
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  atos_status st = ATOS_OK;
  do {
    if (cudaGraphCreate(&graph, 0) != cudaSuccess) { st = atos_set_error(ATOS_ERR_CUDA, "cudaGraphCreate"); break; }
    cudaGraphConditionalHandle hnd;
    if (cudaGraphConditionalHandleCreate(&hnd, graph, t0 > 0 ? 1u : 0u, cudaGraphCondAssignDefault) != cudaSuccess) {
      st = atos_set_error(ATOS_ERR_CUDA, "cudaGraphConditionalHandleCreate");
      break;
    }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hnd;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    if (cudaGraphAddNode(&cn, graph, nullptr, 0, &cp) != cudaSuccess) {
      st = atos_set_error(ATOS_ERR_CUDA, "cudaGraphAddNode(conditional): %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    GraphView gv = c.gv;
    int Fv = F;
    DevRound* rp = w.devround;
    void* a1[] = {(void*)&app, (void*)&gv, (void*)&q, (void*)&Fv, (void*)&rp};
    cudaKernelNodeParams k1 = {};
    k1.func = (void*)kern;
    k1.gridDim = dim3(blocks);
    k1.blockDim = dim3(T);
    k1.sharedMemBytes = (unsigned)smem;
    k1.kernelParams = a1;
    cudaGraphNode_t n1, n2;
    DevRound* rw = w.devround;
    const QueueCtl* ctl = w.ctl;
    void* a2[] = {(void*)&rw, (void*)&ctl, (void*)&hnd};
    cudaKernelNodeParams k2 = {};
    k2.func = (void*)k_round_end;
    k2.gridDim = dim3(1);
    k2.blockDim = dim3(1);
    k2.kernelParams = a2;
    if (cudaGraphAddKernelNode(&n1, body, nullptr, 0, &k1) != cudaSuccess ||
        cudaGraphAddKernelNode(&n2, body, &n1, 1, &k2) != cudaSuccess) {
      st = atos_set_error(ATOS_ERR_CUDA, "cudaGraphAddKernelNode: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
      st = atos_set_error(ATOS_ERR_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    if (cudaGraphLaunch(exec, c.s) != cudaSuccess) {
      st = atos_set_error(ATOS_ERR_CUDA, "cudaGraphLaunch: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
  } while (0);
  (void)cudaGetLastError();
  if (st == ATOS_OK) {
    DevRound r1{};
    CK(cudaMemcpyAsync(&r1, w.devround, sizeof r1, cudaMemcpyDeviceToHost, c.s));
    CK(cudaStreamSynchronize(c.s));
    c.rounds += (int64_t)r1.rounds;
    c.launches += 2 * (int64_t)r1.rounds;
    if (h_end) *h_end = r1.h;
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  return st;
}

template <class P, class App>
static atos_status run_discrete(LaunchCtx& c, const App& app, const Queue& q, uint64_t t0, uint64_t h0 = 0,
                                int64_t max_rounds = -1, uint64_t* h_end = nullptr) {
  if (c.cfg.device_loop && max_rounds < 0 && h0 == 0) {
    switch (c.cfg.worker) {
      case ATOS_WORKER_THREAD: return run_discrete_graph_w<P, App, W_THREAD>(c, app, q, t0, h_end);
      case ATOS_WORKER_WARP: return run_discrete_graph_w<P, App, W_WARP>(c, app, q, t0, h_end);
      default: return run_discrete_graph_w<P, App, W_CTA>(c, app, q, t0, h_end);
    }
  }
  switch (c.cfg.worker) {
    case ATOS_WORKER_THREAD: return run_discrete_w<P, App, W_THREAD>(c, app, q, t0, h0, max_rounds, h_end);
    case ATOS_WORKER_WARP: return run_discrete_w<P, App, W_WARP>(c, app, q, t0, h0, max_rounds, h_end);
    default: return run_discrete_w<P, App, W_CTA>(c, app, q, t0, h0, max_rounds, h_end);
  }
}

// One BSP step over an explicit frontier (in == nullptr: all vertices).
template <class P, class App, int W>
static atos_status bsp_step_w(LaunchCtx& c, const App& app, const uint32_t* in, uint64_t count, uint32_t* out,
                              unsigned long long* out_count, int F, QueueCtl* ctl) {
  if (count == 0) return ATOS_OK;
  auto kern = k_bsp<P, App, W>;
  const int T = c.cfg.cta_threads;
  const size_t smem = (W == W_CTA) ? P::smem_bytes(F) : 0;
  if (smem > 227 * 1024) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "fetch_size %d x cta_threads %d needs %zu B shared memory (> 227 KB)", F, c.cfg.cta_threads, smem);
  CKS(set_smem(kern, smem));
  const uint64_t chunk = (W == W_CTA) ? (uint64_t)F : (W == W_WARP ? (uint64_t)F : 32ull * (uint64_t)F);
  const uint64_t per_block = (W == W_CTA) ? 1 : (uint64_t)(T / 32);
  const uint64_t workers = (count + chunk - 1) / chunk;
  uint64_t blocks = std::min<uint64_t>((workers + per_block - 1) / per_block, 1u << 30);
  kern<<<(unsigned)blocks, T, smem, c.s>>>(app, c.gv, in, count, out, out_count, ctl, F);
  CK(cudaGetLastError());
  c.launches++;
  return ATOS_OK;
}

template <class P, class App>
static atos_status bsp_step(LaunchCtx& c, const App& app, const uint32_t* in, uint64_t count, uint32_t* out,
                            unsigned long long* out_count) {
  const int F = c.cfg.fetch_size;
  switch (c.cfg.worker) {
    case ATOS_WORKER_THREAD: return bsp_step_w<P, App, W_THREAD>(c, app, in, count, out, out_count, F, c.g->ws.ctl);
    case ATOS_WORKER_WARP: return bsp_step_w<P, App, W_WARP>(c, app, in, count, out, out_count, F, c.g->ws.ctl);
    default: return bsp_step_w<P, App, W_CTA>(c, app, in, count, out, out_count, F, c.g->ws.ctl);
  }
}

static atos_status bsp_read_count(LaunchCtx& c, unsigned long long* dcount, uint64_t& out) {
  CK(cudaMemcpyAsync(&c.g->ws.h_ctl->aux[3].v, dcount, sizeof(uint64_t), cudaMemcpyDeviceToHost, c.s));
  CK(cudaStreamSynchronize(c.s));
  out = c.g->ws.h_ctl->aux[3].v;
  c.rounds++;
  return host_timeout(c);
}

static int fill_blocks(int64_t n, int sms) { return grid_for(n, 256, sms); }
// k_pr_seed: 8 resident CTAs per SM, at most one per merge-path tile
static int seed_blocks(atos_graph g) {
  const int64_t tiles = (g->n + g->m + SEED_D - 1) / SEED_D;
  return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)g->sms * 8));
}

// Output copy: host or device destination (UVA).
static atos_status copy_out(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (!bytes) return ATOS_OK;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
  return ATOS_OK;
}

static atos_status finish_stats(LaunchCtx& c, atos_stats* st, bool bsp) {
  Workspace& w = c.g->ws;
  CK(cudaEventRecord(w.ev[2], c.s));
  CKS(read_ctl(c.g, c.s));
  if (!bsp) w.dirty = std::max<uint64_t>(std::min<uint64_t>(w.h_ctl->tail.v, w.cap), w.dirty_rest);
  if (st) {
    float ms = 0, kms = 0;
    CK(cudaEventElapsedTime(&ms, w.ev[0], w.ev[2]));
    CK(cudaEventElapsedTime(&kms, w.ev[1], w.ev[2]));
    st->ms = ms;
    st->kernel_ms = kms;
    st->kernel_launches = c.launches + c.post_launches;
    st->chunk_tasks = (int64_t)w.h_ctl->chunk_done.v;
    st->trace_records = (int64_t)w.h_ctl->trace_count.v;
    st->tasks_popped = (int64_t)w.h_ctl->stats[0].v - st->chunk_tasks;
    st->tasks_pushed = (int64_t)w.h_ctl->stats[1].v;
    st->edges_processed = (int64_t)w.h_ctl->stats[2].v;
    st->rounds = c.rounds;
    st->queue_high_water = bsp ? (int64_t)w.h_ctl->high_water.v : (int64_t)w.h_ctl->high_water.v;
  }
#ifdef ATOS_WAIT_PROF
  {
    const QueueCtl* h = w.h_ctl;
    fprintf(stderr, "ATOS_PROF Mcycles agent: wait_free %.1f pop %.1f prep %.1f | workers: wait_ready %.1f steps %.1f exit %.1f\n",
            h->prof[0].v * 1e-6, h->prof[1].v * 1e-6, h->prof[2].v * 1e-6, h->prof[3].v * 1e-6, h->prof[4].v * 1e-6,
            h->prof[5].v * 1e-6);
    if (h->prof[9].v)
      fprintf(stderr, "ATOS_PROF step cycles: %.0f steps, col %.0f, probe+atomic+decide %.0f, push %.0f (mean per step)\n",
              (double)h->prof[9].v, (double)h->prof[6].v / h->prof[9].v, (double)h->prof[7].v / h->prof[9].v,
              (double)h->prof[8].v / h->prof[9].v);
  }
#endif
  return ATOS_OK;
}

static atos_status begin_call(atos_graph g, const atos_config* cfg_in, LaunchCtx& c, atos_stats* st) {
  if (!g) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "NULL graph");
  if (cfg_in) c.cfg = *cfg_in;
  else atos_config_default(&c.cfg);
  CKS(check_config(&c.cfg));
  if (st) {
    if (st->struct_size != 0 && st->struct_size != sizeof(atos_stats))
      return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "atos_stats.struct_size mismatch");
    std::memset(st, 0, sizeof *st);
    st->struct_size = sizeof(atos_stats);
  }
  c.g = g;
  c.s = reinterpret_cast<cudaStream_t>(c.cfg.stream);
  c.gv = GraphView{g->d_off, g->d_col, g->n, g->col_cap};
  c.t0 = std::chrono::steady_clock::now();
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev != g->device) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "current device %d != graph device %d", dev, g->device);
  return ATOS_OK;
}

// ------------------------------------------------------------------ BFS
// partitioned graphs (dist_impl.cuh): the whole multi-round run
static atos_status part_call(LaunchCtx& c, int app, int64_t src, float alpha, float eps, void* out,
                             int32_t* ncolors_out, atos_stats* st);

extern "C" atos_status atos_bfs(atos_graph g, int64_t src, const atos_config* cfg, uint32_t* depth_out, atos_stats* st) {
  LaunchCtx c;
  CKS(begin_call(g, cfg, c, st));
  if (g->peer) return peer_bfs(g, src, c.cfg, depth_out, st);
  if (g->dist) {
    if (src < 0 || src >= g->global_n)
      return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "src %lld not in [0, %lld)", (long long)src, (long long)g->global_n);
    return part_call(c, 0, src, 0.f, 0.f, depth_out, nullptr, st);
  }
  const int64_t n = g->n;
  if (n == 0) return ATOS_OK;
  if (src < 0 || src >= n) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "src %lld not in [0, %lld)", (long long)src, (long long)n);
  if (!depth_out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "depth_out == NULL");
  Workspace& w = g->ws;
  const bool bsp = c.cfg.kernel == ATOS_KERNEL_BSP;
  CKS(ws_prepare(g, c.cfg, n, 2 * (uint64_t)n, !bsp, c.s));
  CKS(ensure(w.u32a, w.u32a_n, (size_t)n));
  CKS(ensure(w.u16a, w.u16a_n, (size_t)n));
  if (bsp) {
    CKS(ensure(w.front[0], w.front_n[0], (size_t)n));
    CKS(ensure(w.front[1], w.front_n[1], (size_t)n));
  }
  CK(cudaEventRecord(w.ev[0], c.s));
  CKS(ring_reset(w, c.s));
  // a2: init (timed)
  k_bfs_init<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.u32a, nullptr, w.u16a, n, src);
  k_ctl_init<<<1, 1, 0, c.s>>>(w.ctl, bsp ? 0 : 1, w.ring, bsp ? -1 : src);
  CK(cudaGetLastError());
  c.launches += 2;
  CK(cudaEventRecord(w.ev[1], c.s));
  BfsApp app{w.u32a, w.u16a, c.cfg.bfs_filter, c.cfg.sink_defer ? g->d_sink : nullptr,
             g->d_hub != nullptr ? 1u : 0u};
  c.split = c.cfg.hub_split != 0;  // R24: on by default for BFS
  using P = EdgeMapPolicy<BfsApp>;
  if (c.cfg.kernel == ATOS_KERNEL_PERSISTENT) {
    CKS(run_persistent<P>(c, app, make_queue(g, c.cfg, 0)));
  } else if (c.cfg.kernel == ATOS_KERNEL_DISCRETE) {
    CKS(run_discrete<P>(c, app, make_queue(g, c.cfg, 0), 1));
  } else {
    // Alg. 1: double-buffered frontiers
    uint32_t h_src = (uint32_t)src;
    CK(cudaMemcpyAsync(w.front[0], &h_src, sizeof h_src, cudaMemcpyHostToDevice, c.s));
    uint64_t cnt = 1;
    int cur = 0;
    while (cnt > 0) {
      CK(cudaMemsetAsync(w.fcount, 0, sizeof(unsigned long long), c.s));
      CKS(bsp_step<P>(c, app, w.front[cur], cnt, w.front[cur ^ 1], w.fcount));
      CKS(bsp_read_count(c, w.fcount, cnt));
      cur ^= 1;
    }
  }
  CKS(finish_stats(c, st, bsp));
  CKS(copy_out(depth_out, w.u32a, (size_t)n * sizeof(uint32_t), c.s));
  CK(cudaStreamSynchronize(c.s));
  return ATOS_OK;
}

// ------------------------------------------------------------------ PageRank
// rs: residue storage (R34) — fp32 with fp64 hubs (res64 = the seeding sums
// array) on a tagged graph, or all-fp64 (R = double).
template <class R>
static atos_status pagerank_run(LaunchCtx& c, Residues<R> rs, double* rank, float alpha, float eps) {
  atos_graph g = c.g;
  Workspace& w = g->ws;
  const int64_t n = g->n;
  const bool bsp = c.cfg.kernel == ATOS_KERNEL_BSP;
  CK(cudaEventRecord(w.ev[0], c.s));
  CKS(ring_reset(w, c.s));
  // a2: rank = 1 - alpha ; residue seeded by one synchronous push (R4) ; all vertices enqueued
  k_fill<double><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(rank, n, 1.0 - (double)alpha);
  // R30: the seeding sums accumulate in fp64 (w.f64b: the hub residues, or every residue when R = double)
  // and are rounded once to fp32 for non-hubs: fp32 adds of one repeated c = (1-a)a/deg(v) onto a hub's
  // growing sum round with correlated errors (measured: RMAT-27's hub 4.8e-4 of max x* low)
  const bool f32 = !std::is_same<R, double>::value;
  k_ctl_init<<<1, 1, 0, c.s>>>(w.ctl, bsp ? 0 : (uint64_t)n, w.ring, -1);
  if constexpr (std::is_same<R, float>::value) {
    // tagged graph: fp32 sums for non-hubs, fp64 at hubs (k_pr_seed<true>)
    k_fill<float><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(rs.res, n, 0.f);
    k_zero_hubs<<<fill_blocks((n + 31) / 32, g->sms), 256, 0, c.s>>>(rs.hub, n, rs.res64, rs.r2);
    k_pr_seed<true><<<seed_blocks(g), SEED_T, 0, c.s>>>(g->d_off, (const uint32_t*)g->d_col, n, g->m, rs.res, rs.res64, rs.r2,
                                                        (1.0 - (double)alpha) * (double)alpha);
  } else {
    double* acc = w.f64b;  // every residue fp64: the sums are the residues
    k_fill<double><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(acc, n, 0.0);
    k_pr_seed<false><<<seed_blocks(g), SEED_T, 0, c.s>>>(g->d_off, (const uint32_t*)g->d_col, n, g->m, nullptr, acc, 0,
                                                         (1.0 - (double)alpha) * (double)alpha);
  }
  if (!bsp) k_ring_prefill<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.ring, n, 0u);
  // R29: sink deferral for the threshold-activated queue strategies
  const bool sinks = c.cfg.sink_defer && !bsp && c.cfg.pr_activation == 0;
  const uint32_t* sink_bits = sinks ? g->d_sink : nullptr;
  CK(cudaGetLastError());
  c.launches += (bsp ? 4 : 5) + (f32 ? 1 : 0);  // fills, ctl, seeding, (hub zeroing), ring
  CK(cudaEventRecord(w.ev[1], c.s));
  // R31: hub deferral only where the queue agent runs (persistent CTA workers) and ids leave bit 30 free
  const bool dfr = c.cfg.pr_defer_degree > 0 && c.cfg.kernel == ATOS_KERNEL_PERSISTENT &&
                   c.cfg.worker == ATOS_WORKER_CTA && n <= (int64_t)DEFER_BIT;
  c.split = c.cfg.hub_split == 1;  // R33: off by default for PageRank
  PrAppT<R> app{rank, rs, (R)alpha, (R)eps, sink_bits, g->d_hub != nullptr ? 1u : 0u,
                dfr ? (uint32_t)c.cfg.pr_defer_degree : 0u,
                (R)eps * (R)std::max(1, c.cfg.pr_defer_factor), nullptr, 0u, 0u, nullptr};
  // R35: sweep-activated hubs where the batch-closing warp runs (persistent CTA workers, fp32 residues
  // with fp64 hubs, threshold activation elsewhere)
  if constexpr (std::is_same<R, float>::value) {
    if (rs.res64 && g->num_hub_list > 0 && c.cfg.pr_hub_check > 0 && c.cfg.pr_activation == 0 &&
        c.cfg.kernel == ATOS_KERNEL_PERSISTENT && c.cfg.worker == ATOS_WORKER_CTA) {
      PrAppT<float, true> hs{rank, rs, alpha, eps, sink_bits, app.sink_tagged, app.defer_deg, app.defer_res,
                             g->d_hub_list,
                             (uint32_t)g->num_hub_list, (uint32_t)c.cfg.pr_hub_check, w.u32a};
      k_hub_mark<<<fill_blocks(g->num_hub_list, g->sms), 256, 0, c.s>>>(g->d_hub_list, g->num_hub_list, w.u32a);
      CK(cudaGetLastError());
      c.launches++;
      CKS((run_persistent<EdgeMapPolicy<PrAppT<float, true>>>(c, hs, make_queue(g, c.cfg, 1))));
      if (sinks) {
        k_pr_absorb_sinks<R><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(sink_bits, rs, rank, n);
        CK(cudaGetLastError());
        c.launches++;
      }
      return ATOS_OK;
    }
  }
  if (c.cfg.pr_activation == 1) {
    if constexpr (std::is_same<R, float>::value) {
      // f1: Alg. 4's Check_Size window activation; every vertex starts queued
      k_fill<uint32_t><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.u32a, n, 1u);
      PrWindowAppT<float> wapp{rank, rs, w.u32a, alpha, eps, n, c.cfg.check_size};
      CKS(run_persistent<EdgeMapPolicy<PrWindowAppT<float>>>(c, wapp, make_queue(g, c.cfg, 1)));
      return ATOS_OK;
    }
  }
  if (c.cfg.kernel == ATOS_KERNEL_PERSISTENT || c.cfg.kernel == ATOS_KERNEL_DISCRETE) {
    if (c.cfg.kernel == ATOS_KERNEL_PERSISTENT)
      CKS(run_persistent<EdgeMapPolicy<PrAppT<R>>>(c, app, make_queue(g, c.cfg, 1)));
    else
      CKS(run_discrete<EdgeMapPolicy<PrAppT<R>>>(c, app, make_queue(g, c.cfg, 1), (uint64_t)n));
    if (sinks) {
      k_pr_absorb_sinks<R><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(sink_bits, rs, rank, n);
      CK(cudaGetLastError());
      c.launches++;
    }
  } else {
    // Alg. 3: push kernel over the frontier, then filter kernel over all vertices
    PrBspAppT<R> bapp{app};
    uint64_t cnt = (uint64_t)n;
    const uint32_t* in = nullptr;  // first frontier: all vertices
    int cur = 0;
    while (cnt > 0) {
      CKS(bsp_step<EdgeMapPolicy<PrBspAppT<R>>>(c, bapp, in, cnt, nullptr, nullptr));
      CK(cudaMemsetAsync(w.fcount, 0, sizeof(unsigned long long), c.s));
      k_pr_filter<R><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(rs, n, (R)eps, w.front[cur], w.fcount);
      CK(cudaGetLastError());
      c.launches++;
      CKS(bsp_read_count(c, w.fcount, cnt));
      in = w.front[cur];
      cur ^= 1;
    }
  }
  return ATOS_OK;
}

extern "C" atos_status atos_pagerank(atos_graph g, float alpha, float eps, const atos_config* cfg, float* rank_out,
                                     atos_stats* st) {
  LaunchCtx c;
  CKS(begin_call(g, cfg, c, st));
  if (!(alpha > 0.f && alpha < 1.f)) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "alpha not in (0,1)");
  if (!(eps > 0.f)) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "eps <= 0 or NaN");
  if (g->peer) {
    if (c.cfg.pr_activation == 1)
      return atos_set_error(ATOS_ERR_UNSUPPORTED, "Check_Size window activation is not built for peer graphs");
    return peer_pagerank(g, alpha, eps, c.cfg, rank_out, st);
  }
  if (g->dist) {
    if (c.cfg.pr_activation == 1)
      return atos_set_error(ATOS_ERR_UNSUPPORTED, "Check_Size window activation is not built for partitioned graphs");
    return part_call(c, 1, 0, alpha, eps, rank_out, nullptr, st);
  }
  const int64_t n = g->n;
  if (n == 0) return ATOS_OK;
  if (!rank_out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "rank_out == NULL");
  if (c.cfg.pr_activation == 1 && (c.cfg.kernel != ATOS_KERNEL_PERSISTENT || c.cfg.worker != ATOS_WORKER_CTA ||
                                   c.cfg.pr_residue_fp64 || !g->d_hub))
    return atos_set_error(ATOS_ERR_UNSUPPORTED,
                          "Check_Size window activation is built for persistent CTA workers with fp32 residues "
                          "(a library-owned CSR)");
  Workspace& w = g->ws;
  const bool bsp = c.cfg.kernel == ATOS_KERNEL_BSP;
  // R34: fp32 residues need the hub tags; an untagged (borrowed) graph keeps every residue in fp64
  const bool r64 = c.cfg.pr_residue_fp64 != 0 || !g->d_hub;
  // at most 2 live copies per vertex (initial + one threshold crossing), so 2n slots suffice (R16);
  // auto capacity is larger — min(16n, 2^28) slots (2 GB at RMAT-24) — so a run's ~12n pushes
  // rarely wrap: a push to a position of lap 0 needs no load of its slot (q_wait_free), measured
  // -1.8% PageRank time on RMAT-24 (profiles/r02_agents.md)
  const uint64_t pr_cap = std::max<uint64_t>(2 * (uint64_t)n, std::min<uint64_t>(16 * (uint64_t)n, 1ull << 28));
  CKS(ws_prepare(g, c.cfg, n, pr_cap, !bsp, c.s));
  if (!bsp && (uint64_t)n > w.cap)
    return atos_set_error(ATOS_ERR_QUEUE_OVERFLOW, "queue_capacity %llu < n = %lld initial tasks",
                          (unsigned long long)w.cap, (long long)n);
  CKS(ensure(w.f32a, w.f32a_n, (size_t)n));
  CKS(ensure(w.f64a, w.f64a_n, (size_t)n));
  CKS(ensure(w.u32a, w.u32a_n, (size_t)n));  // queued flags (window activation f1; hubs R35)
  // fp64 residues: all of them (untagged / pr_residue_fp64), or the hubs' in two replicas (R34, R38)
  CKS(ensure(w.f64b, w.f64b_n, (size_t)n * (r64 ? 1 : ATOS_HUB_REPLICAS)));
  if (!r64) CKS(ensure(w.f32b, w.f32b_n, (size_t)n));
  if (bsp) {
    CKS(ensure(w.front[0], w.front_n[0], (size_t)n));
    CKS(ensure(w.front[1], w.front_n[1], (size_t)n));
  }
  double* rank = w.f64a;
  const Residues<double> rs64{w.f64b, nullptr, nullptr, 0};
  const Residues<float> rs32{w.f32b, w.f64b, g->d_hub, n};  // hub residues: ATOS_HUB_REPLICAS replicas n apart (R38)
  if (r64) CKS(pagerank_run<double>(c, rs64, rank, alpha, eps));
  else CKS(pagerank_run<float>(c, rs32, rank, alpha, eps));
  c.post_launches = st ? 2 : 1;
  CKS(finish_stats(c, st, bsp));
  if (st) {
    unsigned int* mb = reinterpret_cast<unsigned int*>(g->d_scratch) + 8;
    CK(cudaMemsetAsync(mb, 0, sizeof(unsigned int), c.s));
    if (r64) k_max_res<double><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(rs64, n, mb);
    else k_max_res<float><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(rs32, n, mb);
    unsigned int hb = 0;
    CK(cudaMemcpyAsync(&hb, mb, sizeof hb, cudaMemcpyDeviceToHost, c.s));
    CK(cudaStreamSynchronize(c.s));
    float f;
    std::memcpy(&f, &hb, sizeof f);
    st->max_residue = f;
  }
  k_f64_to_f32<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(rank, w.f32a, n);
  CK(cudaGetLastError());
  CKS(copy_out(rank_out, w.f32a, (size_t)n * sizeof(float), c.s));
  CK(cudaStreamSynchronize(c.s));
  return ATOS_OK;
}

// ------------------------------------------------------------------ colouring
extern "C" atos_status atos_color(atos_graph g, const atos_config* cfg, int32_t* color_out, int32_t* ncolors_out,
                                  atos_stats* st) {
  LaunchCtx c;
  CKS(begin_call(g, cfg, c, st));
  if (g->peer) return atos_set_error(ATOS_ERR_UNSUPPORTED, "colouring is not built for peer graphs (f2: BFS, PageRank)");
  if (!g->symmetric) return atos_set_error(ATOS_ERR_INVALID_GRAPH, "atos_color needs ATOS_GRAPH_SYMMETRIC");
  if (c.cfg.gc_literal) return atos_set_error(ATOS_ERR_UNSUPPORTED, "paper-literal colouring (livelocks, R13) not built");
  if (ncolors_out) *ncolors_out = 0;
  if (g->dist) return part_call(c, 2, 0, 0.f, 0.f, color_out, ncolors_out, st);
  const int64_t n = g->n;
  if (n == 0) return ATOS_OK;
  if (!color_out) return atos_set_error(ATOS_ERR_INVALID_ARGUMENT, "color_out == NULL");
  Workspace& w = g->ws;
  const bool bsp = c.cfg.kernel == ATOS_KERNEL_BSP;
  CKS(ws_prepare(g, c.cfg, n, 4 * (uint64_t)n, !bsp, c.s));
  CKS(ensure(w.u32a, w.u32a_n, (size_t)n));  // pend flags
  CKS(ensure(reinterpret_cast<float*&>(w.f32a), w.f32a_n, (size_t)n));
  int32_t* color = reinterpret_cast<int32_t*>(w.f32a);
  uint32_t* pend = w.u32a;
  if (!bsp && (uint64_t)n > w.cap)
    return atos_set_error(ATOS_ERR_QUEUE_OVERFLOW, "queue_capacity %llu < n = %lld initial tasks",
                          (unsigned long long)w.cap, (long long)n);
  if (bsp) {
    CKS(ensure(w.front[0], w.front_n[0], (size_t)n));
    CKS(ensure(w.front[1], w.front_n[1], (size_t)n));
  }
  CK(cudaEventRecord(w.ev[0], c.s));
  CKS(ring_reset(w, c.s));
  k_fill<int32_t><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(color, n, -1);
  k_fill<uint32_t><<<fill_blocks(n, g->sms), 256, 0, c.s>>>(pend, n, 1u);
  k_ctl_init<<<1, 1, 0, c.s>>>(w.ctl, bsp ? 0 : (uint64_t)n, w.ring, -1);
  if (!bsp) k_ring_prefill<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(w.ring, n, 0u);  // ASSIGN(v), id order (R22)
  CK(cudaGetLastError());
  c.launches += bsp ? 3 : 4;
  CK(cudaEventRecord(w.ev[1], c.s));
  GcApp app{color, pend};
  if (c.cfg.kernel == ATOS_KERNEL_PERSISTENT) {
    CKS(run_persistent<GcPolicy<GC_UBER>>(c, app, make_queue(g, c.cfg, 2)));
  } else if (c.cfg.kernel == ATOS_KERNEL_DISCRETE) {
    CKS(run_discrete<GcPolicy<GC_UBER>>(c, app, make_queue(g, c.cfg, 2), (uint64_t)n));
  } else {
    // Alg. 5: assign kernel then conflict-detect kernel over the frontier
    uint64_t cnt = (uint64_t)n;
    const uint32_t* in = nullptr;
    int cur = 0;
    while (cnt > 0) {
      CKS(bsp_step<GcPolicy<GC_BSP_ASSIGN>>(c, app, in, cnt, nullptr, nullptr));
      CK(cudaMemsetAsync(w.fcount, 0, sizeof(unsigned long long), c.s));
      CKS(bsp_step<GcPolicy<GC_BSP_DETECT>>(c, app, in, cnt, w.front[cur], w.fcount));
      CKS(bsp_read_count(c, w.fcount, cnt));
      in = w.front[cur];
      cur ^= 1;
    }
  }
  c.post_launches = 1;
  CKS(finish_stats(c, st, bsp));
  int* mx = reinterpret_cast<int*>(g->d_scratch) + 12;
  CK(cudaMemsetAsync(mx, 0xFF, sizeof(int), c.s));
  k_max_s32<<<fill_blocks(n, g->sms), 256, 0, c.s>>>(color, n, mx);
  int hmx = -1;
  CK(cudaMemcpyAsync(&hmx, mx, sizeof hmx, cudaMemcpyDeviceToHost, c.s));
  CKS(copy_out(color_out, color, (size_t)n * sizeof(int32_t), c.s));
  CK(cudaStreamSynchronize(c.s));
  if (ncolors_out) *ncolors_out = hmx + 1;
  if (st) st->num_colors = hmx + 1;
  return ATOS_OK;
}

#include "dist_impl.cuh"
#include "peer_impl.cuh"
