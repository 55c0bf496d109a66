// dist.cu — multi-GPU BFS / PageRank over a 1-D vertex partition.
#include "capi_internal.h"

atos_status dist_bfs(atos_graph, int64_t, const atos_config*, uint32_t*, atos_stats*) {
  return atos_set_error(ATOS_ERR_UNSUPPORTED, "multi-GPU BFS not built yet");
}
atos_status dist_pagerank(atos_graph, float, float, const atos_config*, float*, atos_stats*) {
  return atos_set_error(ATOS_ERR_UNSUPPORTED, "multi-GPU PageRank not built yet");
}
void dist_free(atos_graph) {}
extern "C" atos_status atos_comm_unique_id(uint8_t*) { return atos_set_error(ATOS_ERR_UNSUPPORTED, "not built"); }
extern "C" atos_status atos_comm_init(int32_t, int32_t, const uint8_t*, atos_comm* out) {
  if (out) *out = nullptr;
  return atos_set_error(ATOS_ERR_UNSUPPORTED, "not built");
}
extern "C" atos_status atos_comm_destroy(atos_comm) { return atos_set_error(ATOS_ERR_UNSUPPORTED, "not built"); }
extern "C" atos_status atos_graph_create_partitioned(atos_comm, int64_t, int64_t, int64_t, const int64_t*,
                                                     const int32_t*, int64_t, uint32_t, atos_graph* out) {
  if (out) *out = nullptr;
  return atos_set_error(ATOS_ERR_UNSUPPORTED, "not built");
}
