/*
 * atos.h — C ABI of the B200-native Atos hot path (libatos.so).
 *
 * Atos (arxiv 2112.00132, "A Task-Parallel GPU Dynamic Scheduling Framework for
 * Dynamic Irregular Computations"): persistent workers pop chunks of frontier
 * vertices from ONE shared device task queue, expand their CSR neighbour
 * lists, apply a relaxed-dependency update and push newly activated vertices
 * back onto the same queue with no frontier barrier (PAPER.md P:237-256,
 * Listing "SPMD code of each thread worker").  Citations: P:n = PAPER.md line n,
 * S:n = SPEC.md line n, R# = reading number in DESIGN.md §3.
 *
 * Conventions for every entry point
 *  - Returns atos_status; never aborts or exits the process.  On error a
 *    thread-local detail string is available from atos_last_error().
 *  - Calls are synchronous: outputs are complete when the call returns.
 *  - One call at a time per graph handle; distinct handles used from distinct
 *    host threads on distinct streams are independent.
 *  - Vertex ids are 32-bit: n must be < 2^30 - 1 (bits 30-31 of a column entry are tags, R37; bit 31 tags colouring CHECK
 *    tasks, R10).  Edge offsets are 64-bit.
 *  - Output buffers are caller-allocated with n entries and may live in host
 *    or device memory (detected with cudaPointerGetAttributes).  They are fully
 *    written on ATOS_OK and unspecified on error.
 */
#ifndef ATOS_H_
#define ATOS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ATOS_OK = 0,
  ATOS_ERR_INVALID_ARGUMENT = 1, /* bad n/m/src/alpha/eps/config field                */
  ATOS_ERR_INVALID_GRAPH = 2,    /* CSR failed validation, or colouring a non-symmetric graph */
  ATOS_ERR_OUT_OF_MEMORY = 3,    /* device or host allocation failed                 */
  ATOS_ERR_CUDA = 4,             /* CUDA runtime error (detail in atos_last_error)   */
  ATOS_ERR_NCCL = 5,             /* NCCL error or NCCL library not loadable          */
  ATOS_ERR_QUEUE_OVERFLOW = 6,   /* more live tasks than queue_capacity */
  ATOS_ERR_TIMEOUT = 7,          /* device watchdog fired (timeout_s exceeded)        */
  ATOS_ERR_UNSUPPORTED = 8       /* e.g. n >= 2^30-1, or an option not built          */
} atos_status;

typedef struct atos_graph_s* atos_graph; /* opaque; owns (or borrows) a device CSR */

/* Kernel strategy, P:318-325 ("persistent" vs "discrete"); BSP = Alg. 1/3/5. */
typedef enum { ATOS_KERNEL_PERSISTENT = 0, ATOS_KERNEL_DISCRETE = 1, ATOS_KERNEL_BSP = 2 } atos_kernel;
/* Worker size: a worker is one thread, one warp or one CTA. */
typedef enum { ATOS_WORKER_THREAD = 0, ATOS_WORKER_WARP = 1, ATOS_WORKER_CTA = 2 } atos_worker;

/* atos_graph_create flags */
enum {
  ATOS_GRAPH_DEVICE_PTRS = 1, /* row_offsets / col_indices are device pointers          */
  ATOS_GRAPH_BORROW = 2,      /* with DEVICE_PTRS: zero-copy, caller keeps them alive;   */
                              /*   the library never writes them (no hub tags, R34)      */
  ATOS_GRAPH_VALIDATE = 4,    /* check off[0]==0, off[n]==m, monotone, cols in range     */
  ATOS_GRAPH_SYMMETRIC = 8    /* caller asserts the graph is undirected (needed by atos_color) */
};

/* Scheduler configuration (the paper's launch* arguments). */
typedef struct {
  uint32_t struct_size;   /* sizeof(atos_config); set by atos_config_default (ABI versioning) */
  int32_t kernel;         /* atos_kernel                                                      */
  int32_t worker;         /* atos_worker                                                      */
  int32_t cta_threads;    /* numThread: threads per CTA, multiple of 32 in [32, 1024]   */
  int32_t fetch_size;     /* FETCH_SIZE: tasks popped per worker per pop, >= 1         */
  int32_t num_blocks;     /* numBlock: persistent grid; 0 = resident maximum           */
  int32_t bfs_filter;     /* 1: read dist[w] before atomicMin (skip if not improving)         */
  int32_t pr_activation;  /* 0: threshold crossing (R6, default); 1: Check_Size window */
  int32_t check_size;     /* Alg. 4 Check_Size; used when pr_activation == 1          */
  int32_t gc_literal;     /* 1: paper-literal Alg. 6 (both endpoints recolour) — ablation only */
  int32_t pr_residue_fp64; /* 1: PageRank residues in fp64 (rank is always fp64-accumulated)   */
  int32_t adaptive_fetch; /* 1 (default): pop min(FETCH, ceil(queued / workers)) items         */
  int32_t device_loop;    /* discrete kernel: 1 = rounds driven by a CUDA-graph WHILE node    */
  int64_t queue_capacity; /* ring slots; 0 = auto (power of two >= 2n); rounded up to pow2     */
  double timeout_s;       /* device watchdog deadline in seconds; 0 = none                    */
  void* stream;           /* cudaStream_t to run on; NULL = legacy default stream             */
  void* trace;            /* optional device buffer of atos_trace_rec (timeline);  */
  int64_t trace_capacity; /*   records; one per processed batch; extra records are dropped    */
  int32_t stage_edges;    /* persistent CTA workers: column-list staging per batch buffer via   */
                          /*   TMA bulk copies, in edges; 0 = off (default), -1 =   */
                          /*   auto (largest that keeps occupancy and 64 KB of L1 per SM)       */
  int32_t sink_defer;     /* 1 (default): never push a dangling (out-degree 0) vertex (R29).     */
                          /*   BFS: its depth is already final in dist[] (its task expands no   */
                          /*   edge).  PageRank (threshold activation): its task is rank += exch */
                          /*   (res) with no other effect, applied once after quiescence.       */
  int32_t pr_defer_degree; /* PageRank, persistent CTA workers: a popped vertex with >= this many */
                          /*   out-edges and residue < pr_defer_factor * eps is re-queued once   */
                          /*   instead of expanded (R31); 0 = off                                 */
  int32_t pr_defer_factor;
  int32_t hub_split;      /* persistent CTA workers: split a popped vertex with > 2048 edges into  */
                          /*   1024-edge chunk tasks (R24).  -1 = app default (BFS on, PageRank  */
                          /*   off: R33), 0 = off, 1 = on                                         */
  int32_t pr_hub_check;   /* PageRank, persistent CTA workers with fp32 residues: hub targets    */
                          /*   (in-degree >= 2048) take fire-and-forget fp64 adds and are      */
                          /*   activated by sweeps — this many hubs checked per processed batch */
                          /*   (R35; default 4); 0 = threshold crossing at hubs too (R34)      */
} atos_config;

/* One timeline record per batch processed by a persistent/discrete worker:
 * %globaltimer at batch end, items in the batch, edges expanded, SM id.
 * Sorted by t_ns they give cumulative work vs time (the paper's normalized
 * throughput plots).  The number written is stats.trace_records. */
typedef struct {
  uint64_t t_ns;
  uint32_t items;
  uint32_t edges;
  uint32_t sm;
  uint32_t kind; /* 0 = BFS, 1 = PageRank, 2 = colouring */
} atos_trace_rec;

/* Per-call statistics (P:818 overwork, P:908 normalized throughput). */
typedef struct {
  uint32_t struct_size;
  double ms;                /* device time of init + run (CUDA events on cfg->stream)     */
  double kernel_ms;         /* device time of the hot-path kernels alone (sum)            */
  int64_t kernel_launches;  /* every kernel this call launched (init + hot path + reductions) */
  int64_t tasks_popped;     /* vertex / colour tasks processed (excludes chunk tasks)     */
  int64_t tasks_pushed;     /* items pushed after init                                    */
  int64_t edges_processed;  /* edge visits (BFS relax attempts, PR edge pushes, GC scans) */
  int64_t rounds;           /* discrete/BSP rounds, multi-GPU exchange rounds             */
  int64_t queue_high_water; /* max observed (tail - head)                                 */
  int64_t bytes_sent;       /* multi-GPU: payload bytes sent by this rank                 */
  int32_t num_colors;       /* atos_color: colours used                                   */
  int32_t _pad;
  double max_residue;       /* atos_pagerank: max residue at return (must be <= eps)      */
  int64_t chunk_tasks;      /* hub edge-chunk tasks processed (persistent CTA workers)    */
  int64_t trace_records;    /* timeline records produced (may exceed trace_capacity)       */
} atos_stats;

/* Fill *cfg with defaults: persistent, CTA worker, 256 threads, fetch 256,
 * resident-maximum grid, filter on, threshold activation, auto capacity. */
void atos_config_default(atos_config* cfg);

/* Build a graph handle from CSR: row_offsets int64[n+1], col_indices int32[m]
 * (P:427 vertex.neighbors; S:26-37 invariants).  Copies to the device unless
 * ATOS_GRAPH_BORROW|ATOS_GRAPH_DEVICE_PTRS.  A copied CSR gets hub tags (bit
 * 31 of a column entry = its target's in-degree is >= 2048, R34; internal to
 * the library).  m may exceed 2^31.  n == 0 is allowed.  Errors: INVALID_ARGUMENT (n<0, m<0, NULL pointers with m>0, out==NULL),
 * UNSUPPORTED (n >= 2^30-1), INVALID_GRAPH (with VALIDATE), OUT_OF_MEMORY, CUDA. */
atos_status atos_graph_create(const int64_t* row_offsets, const int32_t* col_indices, int64_t n,
                              int64_t m, uint32_t flags, atos_graph* out);
atos_status atos_graph_destroy(atos_graph g);
/* n, m and max out-degree of a handle (any pointer may be NULL). */
atos_status atos_graph_info(atos_graph g, int64_t* n, int64_t* m, int64_t* max_degree);

/* Speculative BFS (Alg. 2; BSP: Alg. 1).
 * depth_out[v] = hop distance from src, 0xFFFFFFFF if unreachable;
 * bit-exact with serial BFS for every configuration.  cfg NULL = defaults;
 * stats may be NULL.  Errors: INVALID_ARGUMENT (src not in [0,n)), QUEUE_OVERFLOW,
 * TIMEOUT, CUDA. */
atos_status atos_bfs(atos_graph g, int64_t src, const atos_config* cfg, uint32_t* depth_out,
                     atos_stats* stats);

/* Push PageRank (async: Alg. 4; BSP: Alg. 3) with
 * damping alpha (the paper's lambda) and threshold eps: unnormalised ranks,
 * fixed point x = (1-alpha) 1 + alpha P x (R4, R5, R8).  On return every
 * residue is <= eps and 0 <= x^* - rank <= eps x^* / (1-alpha), up to the
 * residues' rounding: fp32 residues, except fp64 at hub vertices (in-degree
 * >= 2048, tagged at graph create, R34) — rounding stays below 2048 2^-25 of
 * each rank (R36) — or fp64 everywhere with cfg->pr_residue_fp64, on a graph
 * created with ATOS_GRAPH_BORROW, and on partitioned / peer graphs.  With
 * persistent CTA workers hub targets take fire-and-forget fp64 adds and are
 * activated by sweeps (cfg->pr_hub_check, R35); the run ends only after a
 * clean sweep of every hub, so the residue bound holds at every vertex.  Ranks accumulate in
 * fp64 and are returned as float.  rank_out: float[n].  Errors:
 * INVALID_ARGUMENT (alpha not in (0,1), eps <= 0 or NaN), QUEUE_OVERFLOW,
 * TIMEOUT, CUDA; UNSUPPORTED for Check_Size window activation outside
 * persistent CTA workers with fp32 residues. */
atos_status atos_pagerank(atos_graph g, float alpha, float eps, const atos_config* cfg,
                          float* rank_out, atos_stats* stats);

/* Speculative greedy colouring (async uberkernel: Alg. 6; BSP:
 * Alg. 5) with the max-id tie-break and pending-flag dedupe (R12,
 * R13).  Requires a graph created with ATOS_GRAPH_SYMMETRIC (else
 * INVALID_GRAPH).  color_out: int32[n], a proper colouring with
 * color[v] <= deg(v); *num_colors_out = max colour + 1 (may be NULL). */
atos_status atos_color(atos_graph g, const atos_config* cfg, int32_t* color_out,
                       int32_t* num_colors_out, atos_stats* stats);

const char* atos_status_string(atos_status s);
const char* atos_last_error(void);
/* Library version string, e.g. "atos-b200 1.0 sm_100a". */
const char* atos_version(void);

/* ---------------- multi-GPU (one process per GPU, 1-D vertex partition) ---------------- */
/* BFS and PageRank shard by a 1-D vertex split — rank r owns the
 * contiguous global ids [v_begin_r, v_end_r) (callers permute ids first: a
 * block split of RMAT is 3.4x edge-imbalanced).  atos_bfs / atos_pagerank /
 * atos_color on a partitioned handle run the WHOLE multi-round computation
 * inside the library (the worker loop of P:251-256 "until the stop condition",
 * with remote activations batched per round):
 *   - each round every rank runs the single-GPU queue kernel on its own
 *     vertices (persistent: to local quiescence; discrete: one superstep) on
 *     cfg->stream; updates of remote vertices go to a per-destination outbox;
 *   - the ranks exchange one round vector each (messages per destination,
 *     pending local tasks, abort/overflow flags) with an all-gather — the
 *     round's only host synchronisation — then the messages with an
 *     all-to-all (NCCL send/recv on device buffers over NVLink/NVSwitch, or the
 *     host callbacks of atos_comm_init_host), applied by the receiver;
 *   - a round with no message and no pending task on any rank ends the run
 *     (PageRank: after one closing round that flushes every remaining remote
 *     contribution); an error on any rank fails the call on EVERY rank.
 * Every rank must make the same call (same src / alpha / eps / cfg->kernel).
 * Messages are (uint64)(dest_local_id << 32 | payload), payload = BFS depth,
 * PageRank contribution (f32 bits) or colour.  BFS sends a remote vertex once
 * per improvement (per-rank sent_min filter); PageRank accumulates remote
 * contributions per destination in fp64 and sends those above eps (R28);
 * colouring (ATOS_GRAPH_SYMMETRIC, world <= 64) keeps a replica of
 * all colours and sends a changed colour once per round to every rank owning
 * a neighbour; the receiver re-ASSIGNs a local v that now shares a colour with
 * a smaller changed neighbour (R13 across ranks). */
typedef struct atos_comm_s* atos_comm; /* opaque communicator */

/* NCCL unique id (128 bytes) for atos_comm_init: one rank creates it and the
 * caller distributes it to the others.  Errors: NCCL (libnccl.so.2 not
 * loadable, or NCCL failed). */
atos_status atos_comm_unique_id(uint8_t id_out[128]);
/* NCCL communicator of rank `rank` of `world` on the current device (one
 * process per GPU).  Collective: every rank must call it.  NCCL is loaded at
 * run time (dlopen "libnccl.so.2": the copy already in the process, e.g.
 * torch's, if any).  Errors: INVALID_ARGUMENT, NCCL. */
atos_status atos_comm_init(int32_t rank, int32_t world, const uint8_t id[128], atos_comm* out);
/* Communicator whose exchanges are done by caller callbacks on HOST memory
 * (e.g. a gloo process group; the library stages device buffers through
 * pinned host memory).  Both callbacks are collective over the `world` ranks
 * and return 0 on success (anything else fails the call with ATOS_ERR_NCCL):
 *   allgather(user, send, recv, bytes): recv = every rank's `bytes` bytes of
 *     send, in rank order (world * bytes);
 *   alltoallv(user, send, send_bytes, recv, recv_bytes): send holds world
 *     packed segments in rank order, send_bytes[r] of them for rank r; recv
 *     receives recv_bytes[r] bytes from rank r, packed in rank order. */
typedef int (*atos_allgather_fn)(void* user, const void* send, void* recv, int64_t bytes);
typedef int (*atos_alltoallv_fn)(void* user, const void* send, const int64_t* send_bytes, void* recv,
                                 const int64_t* recv_bytes);
atos_status atos_comm_init_host(int32_t rank, int32_t world, atos_allgather_fn allgather,
                                atos_alltoallv_fn alltoallv, void* user, atos_comm* out);
/* Rank / world of a communicator (either pointer may be NULL). */
atos_status atos_comm_info(atos_comm c, int32_t* rank, int32_t* world);
/* Destroy a communicator (after every graph using it is destroyed). */
atos_status atos_comm_destroy(atos_comm c);

/* This rank's partition: it owns global vertices [v_begin, v_end) of a graph
 * with global_n vertices.  local_row_offsets int64[v_end - v_begin + 1]
 * starting at 0, col_global int32[local_m] GLOBAL ids (host or device per
 * ATOS_GRAPH_DEVICE_PTRS; copied; VALIDATE and SYMMETRIC honoured, BORROW
 * ignored).  Collective over `c` (the ranks' ranges are all-gathered and must
 * tile [0, global_n) in rank order, else INVALID_ARGUMENT on every rank).
 * atos_bfs(src = GLOBAL id), atos_pagerank and atos_color on the handle write
 * the results of the owned vertices (v_end - v_begin entries); stats->rounds
 * = exchange rounds, stats->bytes_sent = message bytes this rank sent. */
atos_status atos_graph_create_partitioned(atos_comm c, int64_t global_n, int64_t v_begin, int64_t v_end,
                                          const int64_t* local_row_offsets, const int32_t* col_global,
                                          int64_t local_m, uint32_t flags, atos_graph* out);

/* ---------------- asynchronous peer-memory partitions ----------------
 * The same 1-D vertex split as above, but with no exchange rounds (PAPER.md
 * P:99): partition p = global ids [p*n/parts, (p+1)*n/parts) (callers
 * permute first) keeps its CSR rows, per-vertex state and task queue on
 * devices[p]; a worker relaxing an edge into another partition's vertex
 * updates that vertex's state in place (atomicMin / fp64 atomicAdd through a
 * peer pointer) and pushes it onto the owner's queue (remote warp-aggregated
 * push); termination = equal sums of every queue's processed and tail
 * counters (read in that order).  devices NULL = every partition on the
 * current device, run as ONE persistent kernel whose blocks are split among
 * the partitions; otherwise devices must be pairwise distinct with peer
 * access (one persistent kernel per device, launched together).  Host CSR
 * only (copied); VALIDATE honoured.  atos_bfs / atos_pagerank (threshold
 * activation, fp64 residues, warp workers of FETCH_SIZE; kernel / worker
 * fields ignored) write all n outputs; atos_color returns UNSUPPORTED.
 * Errors: INVALID_ARGUMENT (parts not in [1, 8], n < parts, devices neither
 * all equal nor all distinct), UNSUPPORTED (no peer access, device pointers,
 * n >= 2^30-1), INVALID_GRAPH, OUT_OF_MEMORY, CUDA. */
atos_status atos_graph_create_peer(int32_t parts, const int32_t* devices, const int64_t* row_offsets,
                                   const int32_t* col_indices, int64_t n, int64_t m, uint32_t flags,
                                   atos_graph* out);

/* Graph-lifetime device memory comes from a private stream-ordered pool that
 * keeps up to 32 GB of freed memory mapped for reuse by the next graph
 * (DESIGN §5).  atos_pool_trim releases all but keep_bytes of it to the
 * device; atos_pool_reserved reports what the pool currently holds. */
atos_status atos_pool_trim(uint64_t keep_bytes);
atos_status atos_pool_reserved(uint64_t* bytes);

#ifdef __cplusplus
}
#endif
#endif /* ATOS_H_ */
