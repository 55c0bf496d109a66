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
 *  - Vertex ids are 32-bit: n must be < 2^31 - 1 (bit 31 tags colouring CHECK
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
  ATOS_ERR_UNSUPPORTED = 8       /* e.g. n >= 2^31-1, or an option not built          */
} atos_status;

typedef struct atos_graph_s* atos_graph; /* opaque; owns (or borrows) a device CSR */

/* Kernel strategy, P:318-325 ("persistent" vs "discrete"); BSP = Alg. 1/3/5. */
typedef enum { ATOS_KERNEL_PERSISTENT = 0, ATOS_KERNEL_DISCRETE = 1, ATOS_KERNEL_BSP = 2 } atos_kernel;
/* Worker size: a worker is one thread, one warp or one CTA. */
typedef enum { ATOS_WORKER_THREAD = 0, ATOS_WORKER_WARP = 1, ATOS_WORKER_CTA = 2 } atos_worker;

/* atos_graph_create flags */
enum {
  ATOS_GRAPH_DEVICE_PTRS = 1, /* row_offsets / col_indices are device pointers          */
  ATOS_GRAPH_BORROW = 2,      /* with DEVICE_PTRS: zero-copy, caller keeps them alive    */
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
  int32_t hub_split;      /* persistent CTA workers: split a popped vertex with > 4096 edges into  */
                          /*   2048-edge chunk tasks (R24).  -1 = app default (BFS on, PageRank  */
                          /*   off: R33), 0 = off, 1 = on                                         */
  int32_t _pad0;
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
 * ATOS_GRAPH_BORROW|ATOS_GRAPH_DEVICE_PTRS.  m may exceed 2^31.  n == 0 is
 * allowed.  Errors: INVALID_ARGUMENT (n<0, m<0, NULL pointers with m>0, out==NULL),
 * UNSUPPORTED (n >= 2^31-1), INVALID_GRAPH (with VALIDATE), OUT_OF_MEMORY, CUDA. */
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
 * residue is <= eps and 0 <= x^* - rank <= eps x^* / (1-alpha), up to fp32 rounding.
 * rank_out: float[n].  Errors: INVALID_ARGUMENT (alpha not in (0,1), eps <= 0 or
 * NaN), QUEUE_OVERFLOW, TIMEOUT, CUDA. */
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
/* BFS and PageRank shard by a 1-D vertex split (callers permute
 * vertex ids first: a block split of RMAT is 3.4x edge-imbalanced).  Each rank
 * runs the same persistent queue kernel on its own vertices to LOCAL
 * quiescence; activations of remote vertices are batched per round into one
 * message buffer grouped by destination rank; the caller exchanges the buffers
 * with an all-to-all (torch.distributed -> NCCL over NVLink/NVSwitch) and
 * applies what it received; the run ends when a round sends no message on any
 * rank (an all-reduce).  A message is (uint64)(dest_local_id << 32 | payload),
 * payload = BFS depth (u32) or PageRank residue contribution (f32 bits).
 * BFS: a remote vertex is sent at most once per improvement (per-rank
 * sent_min filter).  PageRank: remote contributions are accumulated per
 * destination vertex; a round sends those above eps, and the run closes with
 * a flush-all round (no mass is stranded).  Colouring (app 2, SURVEY §8f row
 * f4; needs ATOS_GRAPH_SYMMETRIC, world <= 64): each rank colours its vertices
 * with Alg. 6 against a replica of all colours; a message is
 * (uint64)(global_id << 32 | colour), sent once per round to every rank owning
 * a neighbour of a vertex whose colour changed; the receiver re-ASSIGNs a
 * local v that now shares a colour with a smaller changed neighbour (R13 across
 * ranks).  The run ends after a round in which no rank sent anything. */

/* Partitioned graph for rank `rank` of `world`: it owns global vertices
 * [bounds[rank], bounds[rank+1]) (bounds: host int64[world+1], bounds[0] = 0,
 * bounds[world] = global_n).  local_row_offsets int64[n_local+1] starting at 0,
 * col_global int32[local_m] global ids.  Copies like atos_graph_create (flags:
 * DEVICE_PTRS / VALIDATE honoured; BORROW ignored). */
atos_status atos_graph_create_partitioned(int64_t global_n, int32_t world, int32_t rank,
                                          const int64_t* bounds, const int64_t* local_row_offsets,
                                          const int32_t* col_global, int64_t local_m, uint32_t flags,
                                          atos_graph* out);
/* Start a partitioned run: app 0 = BFS from global vertex src (alpha/eps
 * ignored), app 1 = PageRank(alpha, eps) (src ignored), app 2 = greedy
 * colouring (src/alpha/eps ignored; INVALID_GRAPH without SYMMETRIC).
 * Initialises local state (timed into the first round's stats). */
atos_status atos_part_begin(atos_graph g, int32_t app, int64_t src, float alpha, float eps,
                            const atos_config* cfg);
/* One exchange round: run the local queue kernel — persistent: to local
 * quiescence; discrete (cfg.kernel): one superstep over the current snapshot —
 * then gather the round's outgoing messages.  send_counts: host
 * int64[world + 1]: messages per destination ([rank] is 0) and, at [world],
 * local tasks still queued (0 for persistent).  PageRank sends only remote accumulations above
 * eps unless flush_all != 0 (a closing round: everything is sent); the caller
 * ends a PageRank run only after a flush_all round in which no rank sent. */
atos_status atos_part_run(atos_graph g, int32_t flush_all, int64_t* send_counts);
/* Copy the round's messages, grouped by destination rank in rank order, to
 * dst (host or device, capacity cap messages; cap >= sum(send_counts)). */
atos_status atos_part_pack(atos_graph g, uint64_t* dst, int64_t cap);
/* Apply received messages (host or device buffer of `count` uint64):
 * BFS atomicMin + push on improvement; PageRank atomicAdd + push on an
 * eps crossing; colouring: ghost colour update, then every local vertex in
 * conflict with a smaller changed ghost is re-ASSIGNed. */
atos_status atos_part_apply(atos_graph g, const uint64_t* msgs, int64_t count);
/* Finish: write the local results (BFS: uint32 depth, PageRank: float rank, colouring: int32 colour;
 * n_local = bounds[rank+1]-bounds[rank] entries, host or device) and the
 * accumulated statistics (rounds = exchange rounds; bytes_sent = message bytes). */
atos_status atos_part_finish(atos_graph g, void* out, atos_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* ATOS_H_ */
