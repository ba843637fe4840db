// bfs.cu — algos.bfs (reference algos.py:101-135) on the device.
//
// parent[source] = source, -1 unreached; each round is one edgeset.apply with
// the BFS functor (push CAS / pull owner store, filter parent[v] == -1) under
// the bound schedule or hybrid switch, input frontier recycled (reuse=True),
// loop until the output frontier is empty (engine.fused_loop).
#include "engine.cuh"
#include <cstdio>
#include <cstdlib>

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
  // a device result buffer on this device is the working array (no copy)
  cudaPointerAttributes at{};
  bool direct = false;
  if (cudaPointerGetAttributes(&at, parents_out) == cudaSuccess)
    direct = at.type == cudaMemoryTypeDevice && at.device == g.dev;
  else
    cudaGetLastError();
  DevBuf<int32_t> scratch;
  if (!direct) scratch.alloc(g.V);
  struct { int32_t* p; } parent{direct ? parents_out : scratch.p};
  auto finish = [&] {
    if (!direct)
      GG_CUDA(cudaMemcpyAsync(parents_out, parent.p, g.V * sizeof(int32_t), cudaMemcpyDefault, st));
    GG_CUDA(cudaStreamSynchronize(st));
  };
  GG_CUDA(cudaMemsetAsync(parent.p, 0xff, g.V * sizeof(int32_t), st));
  int32_t src32 = (int32_t)source;
  GG_CUDA(cudaMemcpyAsync(parent.p + source, &src32, 4, cudaMemcpyHostToDevice, st));
  if (fusion) {
    bfs_fused(rt, b, parent.p, src32);
    finish();
    return;
  }
  std::unique_ptr<Frontier> frontier = rt.new_frontier(&src32, 1);
  gg_udf_state ust{parent.p, nullptr, 0};
  static const bool trace = getenv("GG_ROUND_TRACE") != nullptr;
  std::vector<int64_t> sizes;
  while (frontier_size(&rt, frontier.get()) > 0) {
    if (trace) sizes.push_back(frontier_size(&rt, frontier.get()));
    rt.edge_begin();
    std::unique_ptr<Frontier> out = edgeset_apply(&rt, UDF_BFS, ust, true, &frontier, b, true, true);
    rt.edge_end();
    frontier = std::move(out);
    rt.stats.rounds += 1;
  }
  if (trace) {  // per-round input size, direction and edge-phase time
    const size_t base = rt.edge_events.size() - sizes.size();
    for (size_t i = 0; i < sizes.size(); ++i) {
      auto& ev = rt.edge_events[base + i];
      GG_CUDA(cudaEventSynchronize(ev.second));
      float ms = 0;
      GG_CUDA(cudaEventElapsedTime(&ms, ev.first, ev.second));
      fprintf(stderr, "bfs round %zu: |in| %lld %s %.3f ms\n", i, (long long)sizes[i],
              rt.stats.direction_log[rt.stats.direction_log.size() - sizes.size() + i] == GG_PUSH ? "push" : "pull", ms);
    }
  }
  finish();
}

}  // namespace gg
