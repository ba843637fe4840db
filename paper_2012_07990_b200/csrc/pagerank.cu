// pagerank.cu — algos.pagerank (reference algos.py:163-208) on the device.
//
// Per iteration (reference semantics):
//   dm      = sum(rank[v] for out_deg(v) == 0)         (pre-update rank)
//   contrib = rank / out_deg (0 for dangling)
//   acc[dst] += contrib[src]  over the schedule's edge traversal
//   rank'   = (1-d)/n + d*dm/n + d*acc ;  l1 = sum|rank' - rank| ; acc = 0
// The stop test runs before each body with l1 = inf initially
// (algos.py:178, 204-205), so tolerance <= 0 gives exactly max_iters rounds.
//
// Device layout: rank f64[V], acc f64[V], contrib CT[V] (CT = f64, or f32
// when requested), per-iteration scalars f64[2*(iters+1)] (dm, l1) so that
// no host synchronisation is needed between rounds unless tolerance > 0.
// The vertex pass fuses: rank update, L1, next dangling mass, next contrib
// and the acc reset (one read of acc/rank/deg, one write of rank/contrib/acc).
#include "prtile.cuh"
#include "apply.cuh"
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

namespace gg {

// rank_0 = 1/n (algos.py:178), or the given vector (a resumed power
// iteration: gg_pagerank_resume, the observed loop of pagerank(on_iteration))
template <class CT>
__global__ void __launch_bounds__(256) k_pr_init(const int64_t* off, int64_t V, double* rank,
                                                 CT* contrib, double* acc, double* dm0, const double* init) {
  double dm = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = off[v + 1] - off[v];
    const double r0 = init ? init[v] : 1.0 / (double)V;
    rank[v] = r0;
    acc[v] = 0.0;
    contrib[v] = d ? (CT)(r0 / (double)d) : (CT)0;
    if (!d) dm += r0;
  }
  dm = block_sum(dm);
  if (threadIdx.x == 0 && dm != 0.0) atomicAdd(dm0, dm);
}

// Vertex pass of iteration `it` (algos.py:192-198 fused with :184-189 of it+1).
template <class CT>
__device__ __forceinline__ void pr_update_range(const int64_t* off, int64_t V, double* rank,
                                                CT* contrib, double* acc, double* scal, int64_t it,
                                                double damping, int64_t v0, int64_t stride) {
  const double n = (double)V;
  const double base = (1.0 - damping) / n + damping * scal[2 * it] / n;
  double l1 = 0, dm = 0;
  for (int64_t v = v0; v < V; v += stride) {
    int64_t d = __ldg(off + v + 1) - __ldg(off + v);
    double nv = base + damping * acc[v];
    l1 += fabs(nv - rank[v]);
    rank[v] = nv;
    acc[v] = 0.0;
    if (d) contrib[v] = (CT)(nv / (double)d);
    else dm += nv;
  }
  l1 = block_sum(l1);
  dm = block_sum(dm);
  if (threadIdx.x == 0) {
    if (l1 != 0.0) atomicAdd(scal + 2 * it + 1, l1);
    if (dm != 0.0) atomicAdd(scal + 2 * (it + 1), dm);
  }
}

template <class CT>
__global__ void __launch_bounds__(256) k_pr_update(const int64_t* off, int64_t V, double* rank,
                                                   CT* contrib, double* acc, double* scal,
                                                   int64_t it, double damping) {
  pr_update_range(off, V, rank, contrib, acc, scal, it, damping,
                  blockIdx.x * (int64_t)blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

// ---------------------------------------------------------------------------
// Fused loop (engine.fused_loop with fusion=True, engine.py:639-662): the
// whole while-loop is one cooperative launch; rounds are separated by grid
// barriers and the stop test is evaluated on the device.
// Edge phase: EDGE_ONLY (flat, or blocked with a barrier per segment), PULL
// (thread per destination, register accumulation) or PUSH (thread per source).
// ---------------------------------------------------------------------------
template <class CT>
struct PrFusedArgs {
  CsrView out, in;
  CooView coo;
  const int64_t* seg_end;
  int64_t nseg;
  int mode;  // 0 edge-only, 1 blocked, 2 pull, 3 push
  double* rank;
  CT* contrib;
  double* acc;
  double* scal;
  int64_t max_iters;
  double tol, damping;
  int64_t* iters_out;
};

template <class CT>
__global__ void __launch_bounds__(256) k_pr_fused(PrFusedArgs<CT> a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t V = a.out.V;
  OpPr<CT> op{a.acc, a.contrib};
  OutBuilder none{};
  none.mode = OUT_NONE;
  int64_t it = 0;
  double l1 = INFINITY;
  while (!(it >= a.max_iters || l1 < a.tol)) {
    if (a.mode == 0 || a.mode == 1) {
      EdgeArgs<OpPr<CT>> ea{a.coo, InView{-1}, op, none, 0};
      if (a.mode == 0) {
        edge_range(ea, 0, a.coo.E, tid, nth);
      } else {
        int64_t lo = 0;
        for (int64_t s = 0; s < a.nseg; ++s) {
          edge_range(ea, lo, a.seg_end[s], tid, nth);
          lo = a.seg_end[s];
          grid.sync();
        }
      }
    } else if (a.mode == 2) {
      for (int64_t v = tid; v < V; v += nth) {
        double s = 0;
        for (int64_t e = a.in.off[v]; e < a.in.off[v + 1]; ++e) s += (double)__ldg(a.contrib + __ldg(a.in.nbr + e));
        a.acc[v] += s;
      }
    } else {
      for (int64_t u = tid; u < V; u += nth) {
        double c = (double)a.contrib[u];
        for (int64_t e = a.out.off[u]; e < a.out.off[u + 1]; ++e) atomicAdd(a.acc + __ldg(a.out.nbr + e), c);
      }
    }
    grid.sync();
    pr_update_range(a.out.off, V, a.rank, a.contrib, a.acc, a.scal, it, a.damping, tid, nth);
    grid.sync();
    l1 = *((volatile double*)a.scal + 2 * it + 1);
    ++it;
  }
  if (tid == 0) *a.iters_out = it;
}

template <class CT>
static int64_t pagerank_pull_wm(const Graph& g, bool fusion, int64_t max_iters, double tol,
                                double damping, double* rank, CT* contrib0, double* scal,
                                Runtime& rt) {
  const int64_t V = g.V;
  const int dev = g.dev;
  cudaStream_t st = rt.stream;
  std::shared_ptr<PullPlan> plan_hold = pull_plan_for(g, kPieceEdges);
  PullPlan* plan = plan_hold.get();
  CsrView in = g.in_view();
  DevBuf<CT> contrib1(V);
  DevBuf<double> hubsum(V);
  hubsum.zero(st);
  DevBuf<int32_t> outdeg(V);
  k_outdeg<<<grid_for(V, 256, dev), 256, 0, st>>>(g.out_view().off, V, outdeg.p);
  GG_LAUNCH_CHECK();
  count_launch();
  PrPullArgs<CT> a{plan->voff.p, plan->vowner.p, plan->nvrows / 32, in.nbr, contrib0, contrib1.p,
                   rank, outdeg.p, hubsum.p, plan->hubs.p, plan->nhubs, scal, V, damping};
  int64_t it = 0;
  if (!fusion) {
    double l1 = INFINITY;
    const unsigned grid = (unsigned)sm_count(dev) * 8;
    const unsigned hgrid = grid_for(plan->nhubs, 256, dev);
    while (!(it >= max_iters || l1 < tol)) {
      a.contrib = (it & 1) ? contrib1.p : contrib0;
      a.contrib_next = (it & 1) ? contrib0 : contrib1.p;
      rt.edge_begin();
      k_pr_pull<CT><<<grid, 256, 0, st>>>(a, it);
      rt.edge_end();
      if (plan->nhubs) k_pr_pull_hubs<CT><<<hgrid, 256, 0, st>>>(a, it);
      GG_LAUNCH_CHECK();
      count_launch(plan->nhubs ? 2 : 1);
      rt.stats.dispatch_count += 1;
      rt.stats.direction_log.push_back(GG_PULL);
      ++it;
      if (tol > 0.0) {
        GG_CUDA(cudaMemcpyAsync(&l1, scal + 2 * (it - 1) + 1, 8, cudaMemcpyDeviceToHost, st));
        GG_CUDA(cudaStreamSynchronize(st));
      }
    }
  } else {
    DevBuf<int64_t> iters(1);
    int per_sm = 0;
    GG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_pr_pull_fused<CT>,
                                                          256, 0));
    CT* c0 = contrib0;
    CT* c1 = contrib1.p;
    int64_t* ip = iters.p;
    void* args[] = {&a, &c0, &c1, &max_iters, &tol, &ip};
    rt.edge_begin();
    GG_CUDA(cudaLaunchCooperativeKernel((const void*)k_pr_pull_fused<CT>, per_sm * sm_count(dev), 256,
                                        args, 0, st));
    rt.edge_end();
    count_launch();
    GG_CUDA(cudaMemcpyAsync(&it, iters.p, 8, cudaMemcpyDeviceToHost, st));
    GG_CUDA(cudaStreamSynchronize(st));
    rt.stats.dispatch_count += 1;
    for (int64_t k = 0; k < it; ++k) rt.stats.direction_log.push_back(GG_PULL);
  }
  rt.stats.rounds += it;
  rt.stats.edges_traversed += it * g.E;
  return it;
}

// ---------------------------------------------------------------------------
// PULL + STRICT: exact edge balance as merge-path tiles over CSR-in (rows
// split by a tile boundary are combined through an f64 add and finished in
// the crossing pass).  Same kernel as the EdgeBlocking path, minus the
// blocking (no renumbering, no source segments): the ablation baseline.
// ---------------------------------------------------------------------------
static __global__ void k_tile_starts_g(const int64_t* roff, int64_t nrows, int64_t ntiles, int64_t* trow,
                                       int64_t* tedge) {
  const int64_t ne = roff[nrows];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t d = t * (int64_t)kTile;
    if (d > nrows + ne) d = nrows + ne;
    int64_t lo = 0, hi = nrows;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (roff[mid + 1] + mid < d) lo = mid + 1; else hi = mid;
    }
    trow[t] = lo;
    tedge[t] = d - lo;
  }
}

static TilePlan* csr_tiles_for(const Graph& gc) {
  Graph& g = const_cast<Graph&>(gc);
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.pr_tiles) return static_cast<TilePlan*>(g.pr_tiles.get());
  CsrView in = g.in_view();
  const int dev = g.dev;
  auto tp = std::make_shared<TilePlan>();
  tp->nrows = g.V;
  tp->ntiles = (g.V + g.E + kTile - 1) / kTile;
  tp->tile_row.alloc(tp->ntiles + 1);
  tp->tile_edge.alloc(tp->ntiles + 1);
  k_tile_starts_g<<<grid_for(tp->ntiles + 1, 256, dev), 256>>>(in.off, g.V, tp->ntiles, tp->tile_row.p,
                                                                tp->tile_edge.p);
  GG_LAUNCH_CHECK();
  DevBuf<uint8_t> mark(g.V + 1);
  mark.zero();
  if (tp->ntiles > 1)
    k_mark_cross<<<grid_for(tp->ntiles, 256, dev), 256>>>(in.off, tp->tile_row.p, tp->tile_edge.p,
                                                          tp->ntiles, 0, g.V, mark.p);
  GG_LAUNCH_CHECK();
  tp->cross.alloc(g.V + 1);
  DevBuf<unsigned long long> n(1);
  cub::CountingInputIterator<int32_t> it((int32_t)0);
  size_t temp = 0;
  GG_CUDA(cub::DeviceSelect::Flagged(nullptr, temp, it, mark.p, tp->cross.p, n.p, g.V));
  DevBuf<uint8_t> tb(temp);
  GG_CUDA(cub::DeviceSelect::Flagged(tb.p, temp, it, mark.p, tp->cross.p, n.p, g.V));
  unsigned long long h = 0;
  GG_CUDA(cudaMemcpy(&h, n.p, 8, cudaMemcpyDeviceToHost));
  tp->ncross = (int64_t)h;
  g.pr_tiles = tp;
  return tp.get();
}

template <class CT>
static __global__ void __launch_bounds__(kTileThreads) k_pr_tiles_fused(TileArgs<CT> a, CT* c0, CT* c1,
                                                                        const int32_t* cross,
                                                                        int64_t ncross, int64_t max_iters,
                                                                        double tol, int64_t* iters_out) {
  __shared__ double s_val[kTile];
  __shared__ int32_t s_rend[kTile + 1];
  __shared__ double s_rowsum[kTile + 1];
  cg::grid_group grid = cg::this_grid();
  a.coherent = 1;
  int64_t it = 0;
  double l1 = INFINITY;
  while (!(it >= max_iters || l1 < tol)) {
    a.contrib = (it & 1) ? c1 : c0;
    a.contrib_next = (it & 1) ? c0 : c1;
    pr_tiles<CT, 0>(a, it, s_val, s_rend, s_rowsum);
    grid.sync();
    pr_crossing(a, it, cross, ncross);
    grid.sync();
    l1 = *((volatile double*)a.scal + 2 * it + 1);
    ++it;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *iters_out = it;
}

template <class CT>
static int64_t pagerank_pull_tiles(const Graph& g, bool fusion, int64_t max_iters, double tol,
                                   double damping, double* rank, CT* contrib0, double* scal,
                                   Runtime& rt) {
  const int64_t V = g.V;
  const int dev = g.dev;
  cudaStream_t st = rt.stream;
  TilePlan* tp = csr_tiles_for(g);
  CsrView in = g.in_view();
  DevBuf<CT> contrib1(V);
  DevBuf<double> hubsum(V);
  hubsum.zero(st);
  DevBuf<int32_t> outdeg(V);
  k_outdeg<<<grid_for(V, 256, dev), 256, 0, st>>>(g.out_view().off, V, outdeg.p);
  GG_LAUNCH_CHECK();
  count_launch();
  TileArgs<CT> a{};
  a.roff = in.off;
  a.owner = nullptr;
  a.row_base = 0;
  a.src = in.nbr;
  a.tile_row = tp->tile_row.p;
  a.tile_edge = tp->tile_edge.p;
  a.ntiles = tp->ntiles;
  a.rank = rank;
  a.outdeg = outdeg.p;
  a.acc = hubsum.p;
  a.hubsum = hubsum.p;
  a.scal = scal;
  a.V = V;
  a.damping = damping;
  int64_t it = 0;
  if (!fusion) {
    double l1 = INFINITY;
    const unsigned grid = (unsigned)sm_count(dev) * 5;
    const unsigned cgrid = grid_for(tp->ncross, 256, dev);
    while (!(it >= max_iters || l1 < tol)) {
      a.contrib = (it & 1) ? contrib1.p : contrib0;
      a.contrib_next = (it & 1) ? contrib0 : contrib1.p;
      rt.edge_begin();
      k_pr_tiles<CT, 0><<<grid, kTileThreads, 0, st>>>(a, it);
      if (tp->ncross) k_pr_crossing<CT><<<cgrid, 256, 0, st>>>(a, it, tp->cross.p, tp->ncross);
      rt.edge_end();
      GG_LAUNCH_CHECK();
      count_launch(tp->ncross ? 2 : 1);
      rt.stats.dispatch_count += 1;
      rt.stats.direction_log.push_back(GG_PULL);
      ++it;
      if (tol > 0.0) {
        GG_CUDA(cudaMemcpyAsync(&l1, scal + 2 * (it - 1) + 1, 8, cudaMemcpyDeviceToHost, st));
        GG_CUDA(cudaStreamSynchronize(st));
      }
    }
  } else {
    DevBuf<int64_t> iters(1);
    int blocks = max_coop_blocks((const void*)k_pr_tiles_fused<CT>, kTileThreads, dev);
    CT* c0 = contrib0;
    CT* c1 = contrib1.p;
    const int32_t* cr = tp->cross.p;
    int64_t nc = tp->ncross;
    int64_t* ip = iters.p;
    void* args[] = {&a, &c0, &c1, &cr, &nc, &max_iters, &tol, &ip};
    rt.edge_begin();
    GG_CUDA(cudaLaunchCooperativeKernel((const void*)k_pr_tiles_fused<CT>, blocks, kTileThreads, args, 0,
                                        st));
    rt.edge_end();
    count_launch();
    GG_CUDA(cudaMemcpyAsync(&it, iters.p, 8, cudaMemcpyDeviceToHost, st));
    GG_CUDA(cudaStreamSynchronize(st));
    rt.stats.dispatch_count += 1;
    for (int64_t k = 0; k < it; ++k) rt.stats.direction_log.push_back(GG_PULL);
  }
  rt.stats.rounds += it;
  rt.stats.edges_traversed += it * g.E;
  return it;
}

template <class CT>
static void pagerank_impl(const Graph& g, const gg_binding& b, bool fusion, const gg_exec* cfg,
                          int64_t max_iters, double tol, double damping, double* ranks_out,
                          Runtime& rt, const double* init) {
  const int64_t V = g.V;
  const int dev = g.dev;
  cudaStream_t st = rt.stream;
  g.ensure_out();  // out-degrees
  const int64_t iters_cap = max_iters > 0 ? max_iters : 0;
  DevBuf<double> rank(V), acc(V), scal(2 * (iters_cap + 2));
  DevBuf<CT> contrib(V);
  scal.zero(st);
  k_pr_init<CT><<<grid_for(V, 256, dev), 256, 0, st>>>(g.out_off.p, V, rank.p, contrib.p, acc.p, scal.p, init);
  GG_LAUNCH_CHECK();
  count_launch();
  const gg_schedule& s = b.s1;
  int64_t it = 0;
  if (s.direction == GG_PULL && s.load_balance == GG_LB_WM) {
    pagerank_pull_wm<CT>(g, fusion, max_iters, tol, damping, rank.p, contrib.p, scal.p, rt);
  } else if (s.direction == GG_PULL && s.load_balance == GG_LB_STRICT) {
    pagerank_pull_tiles<CT>(g, fusion, max_iters, tol, damping, rank.p, contrib.p, scal.p, rt);
  } else if (!fusion) {
    double l1 = INFINITY;
    gg_udf_state ust{acc.p, contrib.p, 0};
    const int udf = sizeof(CT) == 8 ? UDF_PR : UDF_PR32;
    while (!(it >= max_iters || l1 < tol)) {
      rt.edge_begin();
      edgeset_apply(&rt, udf, ust, false, nullptr, b, false, false);
      rt.edge_end();
      k_pr_update<CT><<<grid_for(V, 256, dev), 256, 0, st>>>(g.out_off.p, V, rank.p, contrib.p, acc.p,
                                                             scal.p, it, damping);
      GG_LAUNCH_CHECK();
      count_launch();
      ++it;
      rt.stats.rounds += 1;
      if (tol > 0.0) {
        GG_CUDA(cudaMemcpyAsync(&l1, scal.p + 2 * (it - 1) + 1, 8, cudaMemcpyDeviceToHost, st));
        GG_CUDA(cudaStreamSynchronize(st));
      }
    }
  } else {
    PrFusedArgs<CT> a{};
    a.out = g.out_view();
    if (s.load_balance != GG_LB_EDGE_ONLY && s.direction == GG_PULL) a.in = g.in_view();
    a.coo = g.coo_view();
    if (s.load_balance == GG_LB_EDGE_ONLY) {
      a.mode = 0;
      if (s.blocking) {
        int64_t n = s.blocking_size > 0 ? s.blocking_size : default_blocking_size(g);
        Blocked* bl = blocked_for(const_cast<Graph&>(g), n);
        a.coo = CooView{bl->src.p, bl->dst.p, nullptr, bl->E};
        a.seg_end = bl->seg_end.p;
        a.nseg = bl->nseg;
        a.mode = 1;
      } else if (!g.has_coo) {
        fail(GG_ERR_ENGINE, "graph COO view was dropped");
      }
    } else {
      a.mode = s.direction == GG_PULL ? 2 : 3;
    }
    a.rank = rank.p;
    a.contrib = contrib.p;
    a.acc = acc.p;
    a.scal = scal.p;
    a.max_iters = max_iters;
    a.tol = tol;
    a.damping = damping;
    DevBuf<int64_t> iters(1);
    a.iters_out = iters.p;
    int per_sm = 0;
    GG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_pr_fused<CT>, 256, 0));
    void* args[] = {&a};
    rt.edge_begin();
    GG_CUDA(cudaLaunchCooperativeKernel((const void*)k_pr_fused<CT>, per_sm * sm_count(dev), 256, args,
                                        0, st));
    rt.edge_end();
    count_launch();
    GG_CUDA(cudaMemcpyAsync(&it, iters.p, 8, cudaMemcpyDeviceToHost, st));
    GG_CUDA(cudaStreamSynchronize(st));
    rt.stats.dispatch_count += 1;
    rt.stats.rounds += it;
    rt.stats.edges_traversed += it * g.E;
    for (int64_t k = 0; k < it; ++k) rt.stats.direction_log.push_back(s.direction);
  }
  GG_CUDA(cudaMemcpyAsync(ranks_out, rank.p, V * sizeof(double), cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------------------
// ExecConfig(deterministic=True) (runtime.py:26-50, :167): the reference then
// runs every dispatch inline in worker order, so PageRank's floating-point
// sums follow one fixed order.  Here the same operations in the same order:
// acc[d] summed from 0.0 over d's in-arcs in COO order (the CSR-in is a stable
// sort of the COO by destination: the order the reference's EDGE_ONLY
// apply -- blocked or not, blocking.py:78-113 is stable -- and its PULL
// apply visit them); the dangling mass and the L1 summed sequentially in
// vertex order (algos.py:184-198); every multiply, divide and add rounded
// separately (__d*_rn: no FMA contraction, which the compiler would
// otherwise apply to base + damping * acc).  The ranks are then bitwise equal
// to the reference's for EDGE_ONLY (+ BLOCKED) and PULL schedules; PUSH
// schedules, whose reference order follows the load balancer's source
// order, get the same reproducible COO-order sums.  One thread carries each
// sequential sum: a correctness mode, not a fast one.
// ---------------------------------------------------------------------------
__global__ void k_prd_contrib(const int64_t* out_off, int64_t V, const double* rank, double* contrib) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = out_off[v + 1] - out_off[v];
    contrib[v] = d ? __ddiv_rn(rank[v], (double)d) : 0.0;  // rank[v] / d (algos.py:186-188)
  }
}
// the dangling mass, sequentially in vertex order (algos.py:184-185)
__global__ void k_prd_dangling(const int64_t* out_off, int64_t V, const double* rank, double* dm) {
  double m = 0.0;
  for (int64_t v = 0; v < V; ++v)
    if (out_off[v + 1] == out_off[v]) m = __dadd_rn(m, rank[v]);
  *dm = m;
}
// acc[d] in COO order: thread per destination walks its in-arcs in order
__global__ void k_prd_acc(const int64_t* in_off, const int32_t* in_nbr, int64_t V, const double* contrib,
                          double* acc) {
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < V; d += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int64_t e = in_off[d], e1 = in_off[d + 1]; e < e1; ++e) a = __dadd_rn(a, contrib[in_nbr[e]]);
    acc[d] = a;
  }
}
// rank' = base + damping * acc (algos.py:189-196), L1 sequentially in vertex order
__global__ void k_prd_update(int64_t V, const double* acc, double* rank, double* nv_tmp, const double* dm,
                             double damping) {
  const double n = (double)V;
  const double base = __dadd_rn(__ddiv_rn(__dsub_rn(1.0, damping), n), __ddiv_rn(__dmul_rn(damping, *dm), n));
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    nv_tmp[v] = __dadd_rn(base, __dmul_rn(damping, acc[v]));
}
__global__ void k_prd_l1(int64_t V, const double* nv, const double* rank, double* l1) {
  double s = 0.0;
  for (int64_t v = 0; v < V; ++v) s = __dadd_rn(s, fabs(__dsub_rn(nv[v], rank[v])));
  *l1 = s;
}

static void pagerank_deterministic(const Graph& g, const gg_binding& b, int64_t max_iters, double tol,
                                   double damping, double* ranks_out, Runtime& rt, const double* init) {
  const int64_t V = g.V;
  const int dev = g.dev;
  cudaStream_t st = rt.stream;
  CsrView out = g.out_view();
  CsrView in = g.in_view();
  DevBuf<double> rank(V), nv(V), contrib(V), acc(V), sc(2);
  if (init) {
    GG_CUDA(cudaMemcpyAsync(rank.p, init, V * 8, cudaMemcpyDeviceToDevice, st));
  } else {
    std::vector<double> r0(V, 1.0 / (double)V);  // [1.0 / n] * n (algos.py:176)
    GG_CUDA(cudaMemcpyAsync(rank.p, r0.data(), V * 8, cudaMemcpyHostToDevice, st));
    GG_CUDA(cudaStreamSynchronize(st));
  }
  const unsigned grid = grid_for(V, 256, dev);
  int64_t it = 0;
  double l1 = INFINITY;
  while (!(it >= max_iters || l1 < tol)) {  // stop test before each body (engine.py:659-661)
    k_prd_dangling<<<1, 1, 0, st>>>(out.off, V, rank.p, sc.p);
    k_prd_contrib<<<grid, 256, 0, st>>>(out.off, V, rank.p, contrib.p);
    rt.edge_begin();
    k_prd_acc<<<grid, 256, 0, st>>>(in.off, in.nbr, V, contrib.p, acc.p);
    rt.edge_end();
    k_prd_update<<<grid, 256, 0, st>>>(V, acc.p, rank.p, nv.p, sc.p, damping);
    k_prd_l1<<<1, 1, 0, st>>>(V, nv.p, rank.p, sc.p + 1);
    GG_LAUNCH_CHECK();
    count_launch(5);
    std::swap(rank, nv);
    ++it;
    rt.stats.rounds += 1;
    rt.stats.dispatch_count += 1;
    rt.stats.edges_traversed += g.E;
    rt.stats.direction_log.push_back(b.s1.direction);
    GG_CUDA(cudaMemcpyAsync(&l1, sc.p + 1, 8, cudaMemcpyDeviceToHost, st));
    GG_CUDA(cudaStreamSynchronize(st));
  }
  GG_CUDA(cudaMemcpyAsync(ranks_out, rank.p, V * sizeof(double), cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
}

template <class CT>
int64_t pagerank_blocked(const Graph& g, const gg_schedule& s, bool fusion, int64_t max_iters,
                         double tol, double damping, double* ranks_out, Runtime& rt,
                         const double* init = nullptr);

void pagerank_run(const Graph& g, const gg_binding& b, bool fusion, const gg_exec* cfg,
                  int64_t max_iters, double tol, double damping, double* ranks_out, Runtime& rt,
                  bool fp32_contrib, const double* init_ranks) {
  if (g.V == 0) fail(GG_ERR_VALUE, "empty graph");
  if (b.is_hybrid)
    fail(GG_ERR_SCHEDULE, "label 's0:s1' of pagerank takes a SimpleGPUSchedule (hybrid direction "
                          "switching applies to bfs/bc)");
  check_binding(b);
  DeviceGuard guard(g.dev);
  if (cfg && cfg->deterministic) {  // fixed summation order, bitwise the reference's (see above)
    if (init_ranks) {
      DevBuf<double> ini(g.V);
      GG_CUDA(cudaMemcpyAsync(ini.p, init_ranks, g.V * 8, cudaMemcpyDefault, rt.stream));
      pagerank_deterministic(g, b, max_iters, tol, damping, ranks_out, rt, ini.p);
    } else {
      pagerank_deterministic(g, b, max_iters, tol, damping, ranks_out, rt, nullptr);
    }
    return;
  }
  if (b.s1.load_balance == GG_LB_EDGE_ONLY && b.s1.blocking) {
    if (fp32_contrib)
      pagerank_blocked<float>(g, b.s1, fusion, max_iters, tol, damping, ranks_out, rt, init_ranks);
    else
      pagerank_blocked<double>(g, b.s1, fusion, max_iters, tol, damping, ranks_out, rt, init_ranks);
    return;
  }
  if (fp32_contrib)
    pagerank_impl<float>(g, b, fusion, cfg, max_iters, tol, damping, ranks_out, rt, init_ranks);
  else
    pagerank_impl<double>(g, b, fusion, cfg, max_iters, tol, damping, ranks_out, rt, init_ranks);
}

}  // namespace gg
