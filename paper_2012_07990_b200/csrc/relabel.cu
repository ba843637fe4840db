// relabel.cu — locality relabelling of a graph for the frontier algorithms
// (CC, BC, BFS): the same graph with vertices renumbered by degree,
// descending (stable), cached on the Graph like the PageRank layout.
//
// GG_RELABEL_DEAL=P deals the ranks over P id ranges (rl_dealt below)
// instead of numbering them densely, so the hottest vertices do not share
// cache lines (measured for CC; BC, the default user, is best dense).
//
// Why: Graph500 Kronecker inputs permute vertex ids, so the per-vertex state
// those algorithms gather per arc (label[dst] in the CC hook, depth / sigma /
// delta in BC) is read at uniformly random positions of arrays as large as
// the L2 (Kronecker-25: 134 MB of labels), and every hook round streams
// ~26 GB of DRAM for ~4.7 GB of algorithmic bytes
// (profiles/r01/ncu_cc_lb_warp_efficiency.txt).  Arc endpoints follow the
// degree distribution, so numbering hubs first packs the hot states into a
// prefix that stays L2-resident.
//
// The relabelled graph keeps every arc in COO order (src -> newid[src],
// dst -> newid[dst]); its CSR views are built the same way as the
// original's (stable by source), so each adjacency list keeps the original
// arc order and every order-dependent statistic (pull early-exit scan
// counts, frontier sizes, rounds) is unchanged.  Results are mapped back to
// the original ids on the way out: canonical CC labels are recomputed as
// each component's minimum ORIGINAL id (algos.py:304-307), BFS parents and
// BC scores are permuted back.  The reference has no such step: it is a
// layout choice, like the EdgeBlocking layout.
#include "graph.cuh"
#include "engine.cuh"
#include <cub/device/device_radix_sort.cuh>

namespace gg {

struct Relabel {
  std::unique_ptr<Graph> g;       // the graph in new ids
  DevBuf<int32_t> newid, order;   // old -> new, new -> old
  int64_t deal = 1;               // id ranges the degree ranks are dealt over
  double prep_ms = 0;
};

__global__ void k_rl_deg(const int32_t* s, int64_t E, uint32_t* deg) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31); base < E; base += stride) {
    const int64_t e = base + lane_id();
    const int32_t u = e < E ? s[e] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, u);  // hubs and source-sorted runs add once
    if (u >= 0 && lane_id() == __ffs(grp) - 1) atomicAdd(deg + u, (uint32_t)__popc(grp));
  }
}
__global__ void k_rl_keys(const uint32_t* deg, int64_t V, uint32_t* key, int32_t* ids) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    key[v] = ~deg[v];  // descending degree, ties by id (stable sort)
    ids[v] = (int32_t)v;
  }
}
// rank r (0 = highest degree) -> new id: ranks dealt round-robin over P
// contiguous id ranges (range p holds ranks p, p+P, p+2P, ...; the first
// V % P ranges hold one more).  P = 1 is the plain degree order.  With P > 1
// the hottest vertices land in different 128-byte lines (and L2 slices):
// measured, the dense order packs the top hubs' labels into a few lines that
// every hook round reads ~10^7 times each, and those lines' L2 slices, not
// DRAM, became the bound (CC 121 -> 63 GTEPS on Kronecker-25).
__device__ __forceinline__ int64_t rl_dealt(int64_t r, int64_t V, int64_t P) {
  const int64_t p = r % P, q = V / P, x = V % P;
  return p * q + (p < x ? p : x) + r / P;
}
__global__ void k_rl_inverse(const int32_t* order_rank, int64_t V, int64_t P, int32_t* newid, int32_t* order) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < V; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nid = rl_dealt(r, V, P);
    const int32_t o = order_rank[r];
    newid[o] = (int32_t)nid;
    order[nid] = o;
  }
}
__global__ void k_rl_map(const int32_t* in, int64_t n, const int32_t* newid, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = newid[in[i]];
}

static std::shared_ptr<Relabel> build_relabel(const Graph& g) {
  NvtxRange nvtx("gg.relabel.build");
  const int dev = g.dev;
  const int64_t V = g.V, E = g.E;
  if (!g.has_coo) fail(GG_ERR_ENGINE, "graph COO view was dropped");
  const double t0 = now_ms();
  auto R = std::make_shared<Relabel>();
  R->order.alloc(std::max<int64_t>(V, 1));
  R->newid.alloc(std::max<int64_t>(V, 1));
  {
    DevBuf<uint32_t> deg(std::max<int64_t>(V, 1)), key(std::max<int64_t>(V, 1)), key2(std::max<int64_t>(V, 1));
    DevBuf<int32_t> ids(std::max<int64_t>(V, 1));
    deg.zero();
    if (E) k_rl_deg<<<grid_for(E, 256, dev), 256>>>(g.coo_src.p, E, deg.p);
    k_rl_keys<<<grid_for(V, 256, dev), 256>>>(deg.p, V, key.p, ids.p);
    GG_LAUNCH_CHECK();
    DevBuf<int32_t> by_rank(std::max<int64_t>(V, 1));
    size_t temp = 0;
    GG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, key.p, key2.p, ids.p, by_rank.p, V));
    DevBuf<uint8_t> tb(std::max<size_t>(temp, 1));
    GG_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, temp, key.p, key2.p, ids.p, by_rank.p, V));
    int64_t P = 1;  // dense degree order (BC: 44.9 GTEPS hybrid vs 31.4 dealt over 1024 ranges)
    if (const char* e = getenv("GG_RELABEL_DEAL")) P = std::max<int64_t>(1, atoll(e));
    if (P > V) P = std::max<int64_t>(V, 1);
    R->deal = P;
    k_rl_inverse<<<grid_for(V, 256, dev), 256>>>(by_rank.p, V, P, R->newid.p, R->order.p);
    GG_LAUNCH_CHECK();
  }
  DevBuf<int32_t> s(E), d(E);
  DevBuf<uint32_t> w;
  if (E) {
    k_rl_map<<<grid_for(E, 256, dev), 256>>>(g.coo_src.p, E, R->newid.p, s.p);
    k_rl_map<<<grid_for(E, 256, dev), 256>>>(g.coo_dst.p, E, R->newid.p, d.p);
    GG_LAUNCH_CHECK();
  }
  if (g.weighted) {
    w.alloc(E);
    if (E) GG_CUDA(cudaMemcpyAsync(w.p, g.coo_w.p, E * 4, cudaMemcpyDeviceToDevice, 0));
  }
  R->g = graph_adopt_coo(dev, V, std::move(s), std::move(d), std::move(w), g.weighted, g.symmetric);
  R->g->ensure_out();  // the frontier algorithms' view: built here, not inside a timed query
  if (!g.symmetric) R->g->ensure_in();
  GG_CUDA(cudaDeviceSynchronize());
  R->prep_ms = now_ms() - t0;
  return R;
}

// Cached per graph; callers hold the shared_ptr for the whole query.
std::shared_ptr<Relabel> relabel_for(const Graph& gc) {
  Graph& g = const_cast<Graph&>(gc);
  std::lock_guard<std::mutex> lk(g.mu);
  auto cur = std::static_pointer_cast<Relabel>(g.relabel);
  if (cur) return cur;
  auto R = build_relabel(g);
  g.relabel = R;
  return R;
}

const Graph* relabel_graph(const Relabel& R) { return R.g.get(); }
double relabel_prep_ms(const Relabel& R) { return R.prep_ms; }

// Policy: GG_RELABEL=0 / 1 forces it; by default only BC relabels (graphs
// of >= 2^20 vertices).  Measured on Kronecker-25 / RMAT-24,
// with the level-bitmap filters: BC ETWC 22.3 -> 29.8 GTEPS, TWC 24.0 -> 34.6,
// hybrid 30.9 -> 44.9 (dense order; dealt over 1024 ranges: 22.9 / 25.2 /
// 31.4); CC loses
// (ETWC 121 -> 31..63: the hubs' adjacency lists cluster into a few CTAs of
// the vertex-partitioned balancers, and dense numbering makes the hub labels'
// L2 slices the bound), DO-BFS on RMAT-24 (natural ids already hub-first)
// changes by -20..+7% with the deal width.
bool relabel_wanted(const Graph& g, int algo) {
  if (const char* e = getenv("GG_RELABEL")) return atoi(e) != 0;
  if (algo != kRelabelBc) return false;
  return g.V >= (int64_t(1) << 20);
}

int32_t relabel_vertex(const Relabel& R, int64_t v) {
  int32_t h = 0;
  GG_CUDA(cudaMemcpy(&h, R.newid.p + v, 4, cudaMemcpyDeviceToHost));
  return h;
}

// ---- results back to the original ids ----
__global__ void k_rl_cc_first(const int32_t* lab, const int32_t* order, int64_t V, int32_t* first) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = lab[v], o = order[v];
    if (o < *((volatile int32_t*)first + l)) atomicMin(first + l, o);  // read first: giant components
  }
}
__global__ void k_rl_cc_out(const int32_t* lab, const int32_t* first, const int32_t* order, int64_t V,
                            int32_t* out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    out[order[v]] = first[lab[v]];
}
__global__ void k_rl_parents(const int32_t* par, const int32_t* order, int64_t V, int32_t* out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = par[v];
    out[order[v]] = p < 0 ? p : order[p];
  }
}
__global__ void k_rl_scatter_f64(const double* x, const int32_t* order, int64_t V, double* out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    out[order[v]] = x[v];
}

// labels_new: any component labelling in new ids (device); writes canonical
// labels (component's minimum original id) to `out` (host or device)
void relabel_cc_out(const Relabel& R, const int32_t* labels_new, int32_t* out, cudaStream_t st) {
  const int64_t V = R.g->V;
  const int dev = R.g->dev;
  DevBuf<int32_t> first(std::max<int64_t>(V, 1)), res(std::max<int64_t>(V, 1));
  GG_CUDA(cudaMemsetAsync(first.p, 0x7f, std::max<int64_t>(V, 1) * 4, st));
  k_rl_cc_first<<<grid_for(V, 256, dev), 256, 0, st>>>(labels_new, R.order.p, V, first.p);
  k_rl_cc_out<<<grid_for(V, 256, dev), 256, 0, st>>>(labels_new, first.p, R.order.p, V, res.p);
  GG_LAUNCH_CHECK();
  count_launch(2);
  if (V) GG_CUDA(cudaMemcpyAsync(out, res.p, V * 4, cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
}
void relabel_parents_out(const Relabel& R, const int32_t* par_new, int32_t* out, cudaStream_t st) {
  const int64_t V = R.g->V;
  DevBuf<int32_t> res(std::max<int64_t>(V, 1));
  k_rl_parents<<<grid_for(V, 256, R.g->dev), 256, 0, st>>>(par_new, R.order.p, V, res.p);
  GG_LAUNCH_CHECK();
  count_launch();
  if (V) GG_CUDA(cudaMemcpyAsync(out, res.p, V * 4, cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
}
void relabel_scores_out(const Relabel& R, const double* x_new, double* out, cudaStream_t st) {
  const int64_t V = R.g->V;
  DevBuf<double> res(std::max<int64_t>(V, 1));
  k_rl_scatter_f64<<<grid_for(V, 256, R.g->dev), 256, 0, st>>>(x_new, R.order.p, V, res.p);
  GG_LAUNCH_CHECK();
  count_launch();
  if (V) GG_CUDA(cudaMemcpyAsync(out, res.p, V * 8, cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gg
