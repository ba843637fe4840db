// stubs.cu — entry points whose device implementation is not in this build
// yet.  They fail loudly (no CPU fallback).
#include "engine.cuh"

extern "C" {
static int not_yet(const char* what) {
  gg::set_last_error(std::string(what) + ": not implemented in this build");
  return GG_ERR_ENGINE;
}
int gg_sssp_delta(const gg_graph*, int64_t, const gg_binding*, int32_t, const gg_exec*, uint64_t*,
                  gg_stats*) { return not_yet("gg_sssp_delta"); }
int gg_cc(const gg_graph*, const gg_binding*, int32_t, const gg_exec*, int32_t*, gg_stats*) {
  return not_yet("gg_cc");
}
int gg_bc(const gg_graph*, const int64_t*, int64_t, const gg_binding*, const gg_exec*, double*,
          gg_stats*) { return not_yet("gg_bc"); }
int gg_nccl_unique_id(char*) { return not_yet("gg_nccl_unique_id"); }
int gg_comm_init(int32_t, int32_t, int32_t, const char*, gg_comm**) { return not_yet("gg_comm_init"); }
int gg_comm_destroy(gg_comm*) { return not_yet("gg_comm_destroy"); }
int gg_pagerank_dist(gg_comm*, const gg_graph*, int64_t, double, double, double*, gg_stats*) {
  return not_yet("gg_pagerank_dist");
}
}
