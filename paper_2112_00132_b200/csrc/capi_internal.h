// capi_internal.h — host-side structures shared by capi.cu and dist.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/atos.h"
#include "device.cuh"

struct Workspace {
  uint64_t* ring = nullptr;
  uint64_t cap = 0;
  uint64_t dirty = 0;  // ring slots that may hold non-zero tags
  uint64_t clear = 0;  // slots the next run zeroes in its timed init (ring_reset)
  uint64_t ring_slots = 0;  // allocated slots (>= cap, the capacity of the current run)
  uint64_t dirty_rest = 0;  // dirty slots beyond the current run's capacity (kept for later runs)
  atos::QueueCtl* ctl = nullptr;
  atos::QueueCtl* h_ctl = nullptr;  // pinned mirror
  uint32_t* u32a = nullptr;         // BFS dist / GC pend
  size_t u32a_n = 0;
  uint32_t* u32b = nullptr;         // BFS done (expanded-at-depth)
  size_t u32b_n = 0;
  uint16_t* u16a = nullptr;         // BFS near (2-byte dist mirror for the edge filter)
  size_t u16a_n = 0;
  float* f32a = nullptr;  // PR rank / GC colour
  size_t f32a_n = 0;
  float* f32b = nullptr;  // PR residue
  size_t f32b_n = 0;
  double* f64a = nullptr;  // PR rank (fp64 accumulation)
  size_t f64a_n = 0;
  double* f64b = nullptr;  // PR: fp64 residues (all with pr_residue_fp64 / untagged graphs; hubs otherwise, R34)
  size_t f64b_n = 0;
  uint32_t* front[2] = {nullptr, nullptr};
  size_t front_n[2] = {0, 0};
  unsigned long long* fcount = nullptr;
  atos::Chunk* chunks = nullptr;  // hub chunk table
  struct atos::DevRound* devround = nullptr;  // device-driven discrete rounds
  uint64_t chunk_cap = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

struct DistState;  // dist_impl.cuh
struct PeerState;  // peer_impl.cuh

struct atos_graph_s {
  int64_t n = 0;  // local vertex count (== global n when not partitioned)
  int64_t m = 0;
  int64_t max_degree = 0;
  int64_t* d_off = nullptr;
  int32_t* d_col = nullptr;
  int64_t col_cap = 0;  // readable elements of d_col
  uint32_t* d_sink = nullptr;  // bit v = (deg(v) == 0), built at create (R29)
  uint32_t* d_indeg = nullptr;  // in-degrees counted during the upload, freed after tagging
  uint32_t* d_hub = nullptr;   // bit v = in-degree >= HUB_IN_DEG; columns carry HUB_TAG (R34); nullptr = untagged
  int64_t num_hubs = 0;
  uint32_t* d_hub_list = nullptr;  // hub vertex ids with out-degree > 0 (R35 sweep activation)
  int64_t num_hub_list = 0;
  void* d_scratch = nullptr;
  bool owned = false;
  bool symmetric = false;
  int device = 0;
  int sms = 0;
  Workspace ws;
  // multi-GPU partition (dist_impl.cuh)
  int64_t global_n = 0, v_begin = 0, v_end = 0;
  DistState* dist = nullptr;
  // asynchronous peer-memory partitions (peer_impl.cuh)
  PeerState* peer = nullptr;
};

atos_status atos_set_error(atos_status s, const char* fmt, ...);
atos_status graph_init_common(atos_graph g, const int64_t* off, const int32_t* col, int64_t n, int64_t m,
                              uint32_t flags, int64_t col_bound);
atos_status ws_prepare(atos_graph g, const atos_config& cfg, int64_t n_local, uint64_t default_cap, bool need_ring,
                       cudaStream_t s);
void dist_free(atos_graph g);
