// bfs.cu — algos.bfs (reference algos.py:101-135) on the device.
//
// parent[source] = source, -1 unreached; each round is one edgeset.apply with
// the BFS functor (push CAS / pull owner store, filter parent[v] == -1) under
// the bound schedule or hybrid switch, input frontier recycled (reuse=True),
// loop until the output frontier is empty (engine.fused_loop).
#include "engine.cuh"

namespace gg {

void bfs_fused(Runtime& rt, const gg_binding& b, int32_t* parent, int32_t source);

void bfs_run(const Graph& g, int64_t source, const gg_binding& b, bool fusion, Runtime& rt,
             int32_t* parents_out) {
  if (source < 0 || source >= g.V)
    fail(GG_ERR_VALUE, strf("invalid source %lld for graph with %lld vertices", (long long)source,
                            (long long)g.V));
  check_binding(b);
  DeviceGuard guard(g.dev);
  cudaStream_t st = rt.stream;
  DevBuf<int32_t> parent(g.V);
  GG_CUDA(cudaMemsetAsync(parent.p, 0xff, g.V * sizeof(int32_t), st));
  int32_t src32 = (int32_t)source;
  GG_CUDA(cudaMemcpyAsync(parent.p + source, &src32, 4, cudaMemcpyHostToDevice, st));
  if (fusion) {
    bfs_fused(rt, b, parent.p, src32);
    GG_CUDA(cudaMemcpyAsync(parents_out, parent.p, g.V * sizeof(int32_t), cudaMemcpyDefault, st));
    GG_CUDA(cudaStreamSynchronize(st));
    return;
  }
  std::unique_ptr<Frontier> frontier = rt.new_frontier(&src32, 1);
  gg_udf_state ust{parent.p, nullptr, 0};
  while (frontier_size(&rt, frontier.get()) > 0) {
    rt.edge_begin();
    std::unique_ptr<Frontier> out = edgeset_apply(&rt, UDF_BFS, ust, true, &frontier, b, true, true);
    rt.edge_end();
    frontier = std::move(out);
    rt.stats.rounds += 1;
  }
  GG_CUDA(cudaMemcpyAsync(parents_out, parent.p, g.V * sizeof(int32_t), cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gg
