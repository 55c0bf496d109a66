/* c_partitioned_bfs.c — TEST PROGRAM: a plain C caller of libatos.so runs a
 * partitioned BFS through atos_bfs alone (include/atos.h, multi-GPU).
 *   world 1: one rank over an NCCL communicator (atos_comm_unique_id / _init);
 *   world 2: two forked processes sharing the GPU, exchanging through
 *            atos_comm_init_host callbacks over a socket pair.
 * usage: cbfs <world> <n> <m> <dir>; reads dir/off.bin (int64[n+1]) and
 * dir/col.bin (int32[m]), BFS from global vertex 0, writes dir/depth<r>.bin. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/socket.h>
#include <sys/wait.h>
#include <unistd.h>

#include "atos.h"

static int g_sock = -1, g_me = 0;

static int io_all(int write_, void* p, int64_t n) {
  char* c = (char*)p;
  while (n > 0) {
    ssize_t k = write_ ? write(g_sock, c, (size_t)n) : read(g_sock, c, (size_t)n);
    if (k <= 0) return 1;
    c += k;
    n -= k;
  }
  return 0;
}
/* ordered exchange with the peer (rank 0 sends first): no deadlock on full socket buffers */
static int xchg(const void* s, int64_t sb, void* r, int64_t rb) {
  if (g_me == 0) return io_all(1, (void*)s, sb) || io_all(0, r, rb);
  return io_all(0, r, rb) || io_all(1, (void*)s, sb);
}
static int ag(void* user, const void* send, void* recv, int64_t bytes) {
  (void)user;
  memcpy((char*)recv + g_me * bytes, send, (size_t)bytes);
  return xchg(send, bytes, (char*)recv + (1 - g_me) * bytes, bytes);
}
static int a2a(void* user, const void* send, const int64_t* sb, void* recv, const int64_t* rb) {
  (void)user;
  const int peer = 1 - g_me;
  const int64_t so_me = g_me ? sb[0] : 0, so_peer = peer ? sb[0] : 0;
  const int64_t ro_me = g_me ? rb[0] : 0, ro_peer = peer ? rb[0] : 0;
  memcpy((char*)recv + ro_me, (const char*)send + so_me, (size_t)sb[g_me]);
  return xchg((const char*)send + so_peer, sb[peer], (char*)recv + ro_peer, rb[peer]);
}

static int run_rank(int world, int me, int64_t n, int64_t m, const char* dir) {
  char path[4096];
  int64_t* off = (int64_t*)malloc((size_t)(n + 1) * 8);
  int32_t* col = (int32_t*)malloc((size_t)(m ? m : 1) * 4);
  snprintf(path, sizeof path, "%s/off.bin", dir);
  FILE* f = fopen(path, "rb");
  if (!f || fread(off, 8, (size_t)n + 1, f) != (size_t)n + 1) return 2;
  fclose(f);
  snprintf(path, sizeof path, "%s/col.bin", dir);
  f = fopen(path, "rb");
  if (!f || fread(col, 4, (size_t)m, f) != (size_t)m) return 2;
  fclose(f);
  atos_comm comm = NULL;
  atos_status s;
  if (world == 1) {
    uint8_t id[128];
    if ((s = atos_comm_unique_id(id)) || (s = atos_comm_init(0, 1, id, &comm))) goto fail;
  } else if ((s = atos_comm_init_host(me, world, ag, a2a, NULL, &comm))) {
    goto fail;
  }
  {
    const int64_t vb = me * n / world, ve = (me + 1) * n / world, nl = ve - vb;
    int64_t* lo = (int64_t*)malloc((size_t)(nl + 1) * 8);
    for (int64_t v = 0; v <= nl; ++v) lo[v] = off[vb + v] - off[vb];
    atos_graph g = NULL;
    if ((s = atos_graph_create_partitioned(comm, n, vb, ve, lo, col + off[vb], lo[nl], ATOS_GRAPH_VALIDATE, &g)))
      goto fail;
    uint32_t* depth = (uint32_t*)malloc((size_t)(nl ? nl : 1) * 4);
    atos_config cfg;
    atos_config_default(&cfg);
    cfg.timeout_s = 120;
    atos_stats st;
    memset(&st, 0, sizeof st);
    if ((s = atos_bfs(g, 0, &cfg, depth, &st))) goto fail;
    snprintf(path, sizeof path, "%s/depth%d.bin", dir, me);
    f = fopen(path, "wb");
    if (!f || fwrite(depth, 4, (size_t)nl, f) != (size_t)nl) return 3;
    fclose(f);
    printf("rank %d: %lld rounds, %lld bytes sent\n", me, (long long)st.rounds, (long long)st.bytes_sent);
    atos_graph_destroy(g);
    atos_comm_destroy(comm);
  }
  return 0;
fail:
  fprintf(stderr, "rank %d: %s: %s\n", me, atos_status_string(s), atos_last_error());
  return 1;
}

int main(int argc, char** argv) {
  if (argc != 5) return 64;
  const int world = atoi(argv[1]);
  const int64_t n = atoll(argv[2]), m = atoll(argv[3]);
  if (world == 1) return run_rank(1, 0, n, m, argv[4]);
  if (world != 2) return 64;
  int sv[2];
  if (socketpair(AF_UNIX, SOCK_STREAM, 0, sv)) return 65;
  pid_t kids[2];
  for (int r = 0; r < 2; ++r) {  /* fork before any CUDA call */
    kids[r] = fork();
    if (kids[r] == 0) {
      g_me = r;
      g_sock = sv[r];
      close(sv[1 - r]);
      _exit(run_rank(2, r, n, m, argv[4]));
    }
  }
  int rc = 0;
  for (int r = 0; r < 2; ++r) {
    int stt = 0;
    waitpid(kids[r], &stt, 0);
    if (!WIFEXITED(stt) || WEXITSTATUS(stt)) rc = 1;
  }
  return rc;
}
