// stubs.cu — entry points whose device implementation is not in this build
// yet.  They fail loudly (no CPU fallback).
#include "engine.cuh"

extern "C" {
static int not_yet(const char* what) {
  gg::set_last_error(std::string(what) + ": not implemented in this build");
  return GG_ERR_ENGINE;
}
int gg_nccl_unique_id(char*) { return not_yet("gg_nccl_unique_id"); }
int gg_comm_init(int32_t, int32_t, int32_t, const char*, gg_comm**) { return not_yet("gg_comm_init"); }
int gg_comm_destroy(gg_comm*) { return not_yet("gg_comm_destroy"); }
int gg_pagerank_dist(gg_comm*, const gg_graph*, int64_t, double, double, double*, gg_stats*) {
  return not_yet("gg_pagerank_dist");
}
}
