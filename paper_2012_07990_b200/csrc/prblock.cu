// prblock.cu — PageRank under the EdgeBlocking schedule (EDGE_ONLY + BLOCKED)
// on B200.
//
// The reference's Alg. 1/2 (blocking.py:78-186) groups edges into segments
// of N *destinations* so that the per-edge atomic updates stay in cache.  On
// B200 per-edge L2 atomics are the bottleneck (measured ~185 G ops/s for an
// L2-resident window, profiles/r01/microbench_atomics_gathers.txt) while
// L2-resident gathers run at ~280 G/s and DRAM-random gathers at ~41 G/s.
// So the B200 blocking confines the *random* side of the gather formulation
// to the L2 instead:
//
//   preprocessing (once per graph and window, cached):
//     1. renumber vertices by out-degree, descending (hot sources first);
//     2. segment k = sources [k*Ns, (k+1)*Ns), Ns*sizeof(contrib) sized to a
//        fraction of the queried L2 (blocking_size overrides Ns);
//     3. stable sort of all edges by (segment, destination, source): inside
//        a segment each destination's in-edges are contiguous;
//     4. virtual rows per segment (long rows split into hub pieces), every
//        segment padded to whole 32-row warp chunks.  Segment 0 (the hot
//        sources, ~94% of RMAT-27 edges) lists *every* destination.
//   per iteration (Alg. 2: segments in order, a barrier between them):
//     cold segments k = 1..K-1: warp-per-32-rows gather from the segment's
//       L2-resident contrib window, row sums added to acc[dst];
//     hot segment 0 last: gather + acc + fused vertex update (rank, L1,
//       dangling mass, next contrib) and acc reset; hub pass finishes split rows.
// All per-vertex state lives in the renumbered id space; ranks are permuted
// back on output.  Results equal the reference's up to f64 summation order.
#include "prpull.cuh"
#include "apply.cuh"
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

namespace gg {

struct PrBlockLayout {
  int64_t ns = 0, K = 0, V = 0, E = 0, hub_t = 0, nvrows = 0, nhubs = 0;
  int ct_bytes = 0;
  DevBuf<int32_t> newid, order, outdeg, src, vowner, hubs;
  DevBuf<int64_t> voff;
  std::vector<int64_t> seg_chunk;  // K+1 boundaries in 32-row chunks; segment 0 first
  double prep_ms = 0;
};

static int nbits(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b ? b : 1;
}

__global__ void k_neg_deg(const int64_t* off, int64_t V, uint32_t* key, int32_t* ids) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    key[v] = ~(uint32_t)(off[v + 1] - off[v]);
    ids[v] = (int32_t)v;
  }
}
__global__ void k_relabel_tables(const int32_t* order, const int64_t* off, int64_t V, int32_t* newid,
                                 int32_t* outdeg_new) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t o = order[i];
    newid[o] = (int32_t)i;
    outdeg_new[i] = (int32_t)(off[o + 1] - off[o]);
  }
}
__global__ void k_edge_keys(const int32_t* s, const int32_t* d, int64_t E, const int32_t* newid,
                            int64_t ns, int nvb, uint64_t* key) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t nu = (uint32_t)newid[s[e]], nv = (uint32_t)newid[d[e]];
    uint64_t k = nu / (uint64_t)ns;
    key[e] = (k << (32 + nvb)) | (nv << 32) | nu;
  }
}
__global__ void k_split_keys(const uint64_t* key, int64_t E, int nvb, int32_t* src, int32_t* dst_hot,
                             int64_t E0) {
  const uint64_t mask = (1ULL << nvb) - 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = key[e];
    src[e] = (int32_t)(k & 0xffffffffULL);
    if (e < E0) dst_hot[e] = (int32_t)((k >> 32) & mask);
  }
}
struct IsCold {
  const uint64_t* key;
  int shift;
  __device__ __forceinline__ bool operator()(int64_t e) const { return (key[e] >> shift) != 0; }
};
__global__ void k_count_hot(const uint64_t* key, int64_t E, int shift, unsigned long long* n) {
  unsigned long long c = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x)
    c += (key[e] >> shift) == 0;
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(n, c);
}
// cold run starts: positions e in [E0, E) where (segment, dst) changes
struct RunStart {
  const uint64_t* key;
  int64_t E0;
  __device__ __forceinline__ bool operator()(int64_t e) const {
    return e == E0 || (key[e] >> 32) != (key[e - 1] >> 32);
  }
};
__global__ void k_pieces(const int64_t* start, int64_t n, int64_t end, int64_t hub_t, int64_t* pieces,
                         int min1) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    int64_t len = (p + 1 < n ? start[p + 1] : end) - start[p];
    int64_t q = (len + hub_t - 1) / hub_t;
    pieces[p] = q < 1 ? (min1 ? 1 : 0) : q;
  }
}
// hot rows: row v = destination v, edges [off0[v], off0[v+1])
__global__ void k_fill_hot(const int64_t* off0, int64_t V, const int64_t* vstart, int64_t hub_t,
                           int64_t* voff, int32_t* vowner, int32_t* hubs, unsigned long long* nh) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = off0[v], len = off0[v + 1] - lo, s = vstart[v];
    if (len > hub_t) {
      int64_t np = (len + hub_t - 1) / hub_t;
      for (int64_t k = 0; k < np; ++k) {
        voff[s + k] = lo + k * hub_t;
        vowner[s + k] = ~(int32_t)v;
      }
      hubs[atomicAdd(nh, 1ULL)] = (int32_t)v;
    } else {
      voff[s] = lo;
      vowner[s] = (int32_t)v;
    }
  }
}
// cold rows: pair p = (segment, dst) run starting at start[p]
__global__ void k_fill_cold(const int64_t* start, const uint64_t* key, int64_t n, int64_t E,
                            const int64_t* vstart, const int64_t* seg_first_vs,
                            const int64_t* seg_base, int nvb, int64_t hub_t, int64_t* voff,
                            int32_t* vowner) {
  const uint64_t mask = (1ULL << nvb) - 1;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = start[p];
    const int64_t len = (p + 1 < n ? start[p + 1] : E) - lo;
    const uint64_t k = key[lo] >> (32 + nvb);
    const int32_t dst = (int32_t)((key[lo] >> 32) & mask);
    const int64_t row = seg_base[k] + (vstart[p] - seg_first_vs[k]);
    const int64_t np = (len + hub_t - 1) / hub_t;
    for (int64_t q = 0; q < np; ++q) {
      voff[row + q] = lo + q * hub_t;
      vowner[row + q] = np > 1 ? ~dst : dst;
    }
  }
}
__global__ void k_fill_pad(int64_t* voff, int32_t* vowner, int64_t r0, int64_t r1, int64_t edge) {
  for (int64_t r = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < r1;
       r += (int64_t)gridDim.x * blockDim.x) {
    voff[r] = edge;
    vowner[r] = INT32_MIN;
  }
}

template <class T>
static T dget(const T* p) {
  T h;
  GG_CUDA(cudaMemcpy(&h, p, sizeof(T), cudaMemcpyDeviceToHost));
  return h;
}

static std::shared_ptr<PrBlockLayout> build_layout(const Graph& g, int64_t ns, int ct_bytes) {
  const int dev = g.dev;
  const int64_t V = g.V, E = g.E;
  if (!g.has_coo) fail(GG_ERR_ENGINE, "graph COO view was dropped");
  CsrView out = g.out_view();
  auto L = std::make_shared<PrBlockLayout>();
  double t0 = now_ms();
  L->ns = ns;
  L->K = (V + ns - 1) / ns;
  L->V = V;
  L->E = E;
  L->ct_bytes = ct_bytes;
  L->hub_t = kPieceEdges;
  const int nvb = nbits((uint64_t)(V > 1 ? V - 1 : 1));
  const int kb = nbits((uint64_t)(L->K > 1 ? L->K - 1 : 1));
  if (32 + nvb + kb > 64) fail(GG_ERR_VALUE, "EdgeBlocking layout: too many segments for this graph");
  // 1. out-degree renumbering (stable, descending)
  {
    DevBuf<uint32_t> key(V), key2(V);
    DevBuf<int32_t> ids(V);
    L->order.alloc(V);
    k_neg_deg<<<grid_for(V, 256, dev), 256>>>(out.off, V, key.p, ids.p);
    size_t temp = 0;
    GG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, key.p, key2.p, ids.p, L->order.p, V));
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, temp, key.p, key2.p, ids.p, L->order.p, V));
    L->newid.alloc(V);
    L->outdeg.alloc(V);
    k_relabel_tables<<<grid_for(V, 256, dev), 256>>>(L->order.p, out.off, V, L->newid.p, L->outdeg.p);
    GG_LAUNCH_CHECK();
  }
  // 2-3. (segment, dst, src) keys, sorted
  DevBuf<uint64_t> keys(E);
  {
    DevBuf<uint64_t> k0(E);
    k_edge_keys<<<grid_for(E, 256, dev), 256>>>(g.coo_src.p, g.coo_dst.p, E, L->newid.p, ns, nvb, k0.p);
    GG_LAUNCH_CHECK();
    size_t temp = 0;
    GG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp, k0.p, keys.p, E, 0, 32 + nvb + kb));
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceRadixSort::SortKeys(tb.p, temp, k0.p, keys.p, E, 0, 32 + nvb + kb));
  }
  const int shift = 32 + nvb;
  DevBuf<unsigned long long> cnt(1);
  cnt.zero();
  k_count_hot<<<grid_for(E, 256, dev), 256>>>(keys.p, E, shift, cnt.p);
  GG_LAUNCH_CHECK();
  const int64_t E0 = (int64_t)dget(cnt.p);
  // 4a. sources + hot destination offsets
  L->src.alloc(E);
  DevBuf<int64_t> off0(V + 1);
  {
    DevBuf<int32_t> dh(E0 > 0 ? E0 : 1);
    k_split_keys<<<grid_for(E, 256, dev), 256>>>(keys.p, E, nvb, L->src.p, dh.p, E0);
    GG_LAUNCH_CHECK();
    offsets_from_sorted(dev, dh.p, E0, V, off0.p, 0);
  }
  // 4b. hot virtual rows
  DevBuf<int64_t> hpieces(V), hvstart(V);
  k_pieces<<<grid_for(V, 256, dev), 256>>>(off0.p, V, E0, L->hub_t, hpieces.p, 1);
  // (k_pieces computes len from consecutive starts; off0 has V+1 entries so
  // start[p+1] is off0[v+1] and `end` is unused for v < V)
  size_t temp = 0;
  GG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, hpieces.p, hvstart.p, V));
  {
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, temp, hpieces.p, hvstart.p, V));
  }
  const int64_t hot_rows = dget(hvstart.p + V - 1) + dget(hpieces.p + V - 1);
  const int64_t R0 = (hot_rows + 31) / 32 * 32;
  // 4c. cold pairs
  const int64_t Ec = E - E0;
  DevBuf<int64_t> pstart(Ec > 0 ? Ec : 1);
  DevBuf<unsigned long long> npairs(1);
  npairs.zero();
  int64_t P = 0;
  if (Ec > 0) {
    cub::CountingInputIterator<int64_t> it(E0);
    RunStart pred{keys.p, E0};
    temp = 0;
    GG_CUDA(cub::DeviceSelect::If(nullptr, temp, it, pstart.p, npairs.p, Ec, pred));
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceSelect::If(tb.p, temp, it, pstart.p, npairs.p, Ec, pred));
    P = (int64_t)dget(npairs.p);
  }
  DevBuf<int64_t> cpieces(P > 0 ? P : 1), cvstart(P > 0 ? P : 1);
  std::vector<int64_t> seg_first_pair(L->K + 1, P), seg_rows(L->K, 0);
  std::vector<int64_t> seg_base(L->K + 1, 0), seg_first_vs(L->K, 0), seg_end_edge(L->K, E);
  if (P > 0) {
    k_pieces<<<grid_for(P, 256, dev), 256>>>(pstart.p, P, E, L->hub_t, cpieces.p, 1);
    temp = 0;
    GG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, cpieces.p, cvstart.p, P));
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, temp, cpieces.p, cvstart.p, P));
    // segment of every pair start (host: K is small) -> first pair per segment
    std::vector<int64_t> hstart(P);
    GG_CUDA(cudaMemcpy(hstart.data(), pstart.p, P * 8, cudaMemcpyDeviceToHost));
    std::vector<int64_t> hvs(P), hpc(P);
    GG_CUDA(cudaMemcpy(hvs.data(), cvstart.p, P * 8, cudaMemcpyDeviceToHost));
    GG_CUDA(cudaMemcpy(hpc.data(), cpieces.p, P * 8, cudaMemcpyDeviceToHost));
    // binary search the segment boundaries through the sorted keys
    auto seg_of_edge = [&](int64_t e) { return (int64_t)(dget(keys.p + e) >> shift); };
    for (int64_t k = 1; k < L->K; ++k) {
      int64_t lo = 0, hi = P;  // first pair with segment >= k
      while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (seg_of_edge(hstart[mid]) < k) lo = mid + 1; else hi = mid;
      }
      seg_first_pair[k] = lo;
    }
    seg_first_pair[0] = 0;
    for (int64_t k = 1; k < L->K; ++k) {
      const int64_t a = seg_first_pair[k];
      const int64_t bb = (k + 1 < L->K) ? seg_first_pair[k + 1] : P;
      seg_first_vs[k] = a < P ? hvs[a] : (P ? hvs[P - 1] + hpc[P - 1] : 0);
      const int64_t end_vs = bb < P ? hvs[bb] : (hvs[P - 1] + hpc[P - 1]);
      seg_rows[k] = end_vs - seg_first_vs[k];
      seg_end_edge[k] = bb < P ? hstart[bb] : E;
    }
  }
  // row layout: [hot R0][seg1 padded]...[segK-1 padded]
  seg_base[0] = 0;
  seg_base[1] = R0;
  for (int64_t k = 1; k < L->K; ++k) seg_base[k + 1] = seg_base[k] + (seg_rows[k] + 31) / 32 * 32;
  L->nvrows = seg_base[L->K];
  L->voff.alloc(L->nvrows + 1);
  L->vowner.alloc(L->nvrows + 1);
  L->hubs.alloc(V);
  DevBuf<unsigned long long> nh(1);
  nh.zero();
  k_fill_hot<<<grid_for(V, 256, dev), 256>>>(off0.p, V, hvstart.p, L->hub_t, L->voff.p, L->vowner.p,
                                             L->hubs.p, nh.p);
  k_fill_pad<<<grid_for(R0 - hot_rows + 1, 256, dev), 256>>>(L->voff.p, L->vowner.p, hot_rows, R0, E0);
  GG_LAUNCH_CHECK();
  if (P > 0) {
    DevBuf<int64_t> d_sfv(L->K), d_base(L->K + 1);
    GG_CUDA(cudaMemcpy(d_sfv.p, seg_first_vs.data(), L->K * 8, cudaMemcpyHostToDevice));
    GG_CUDA(cudaMemcpy(d_base.p, seg_base.data(), (L->K + 1) * 8, cudaMemcpyHostToDevice));
    k_fill_cold<<<grid_for(P, 256, dev), 256>>>(pstart.p, keys.p, P, E, cvstart.p, d_sfv.p, d_base.p, nvb,
                                                L->hub_t, L->voff.p, L->vowner.p);
    GG_LAUNCH_CHECK();
    for (int64_t k = 1; k < L->K; ++k) {
      const int64_t r0 = seg_base[k] + seg_rows[k], r1 = seg_base[k + 1];
      if (r1 > r0)
        k_fill_pad<<<grid_for(r1 - r0, 256, dev), 256>>>(L->voff.p, L->vowner.p, r0, r1, seg_end_edge[k]);
    }
    GG_LAUNCH_CHECK();
  }
  k_fill_pad<<<1, 32>>>(L->voff.p, L->vowner.p, L->nvrows, L->nvrows + 1, E);
  GG_LAUNCH_CHECK();
  L->nhubs = (int64_t)dget(nh.p);
  L->seg_chunk.resize(L->K + 1);
  for (int64_t k = 0; k <= L->K; ++k) L->seg_chunk[k] = seg_base[k] / 32;
  GG_CUDA(cudaDeviceSynchronize());
  L->prep_ms = now_ms() - t0;
  return L;
}

// cached on the graph (one layout per (window, contrib width))
static PrBlockLayout* layout_for(const Graph& gc, int64_t ns, int ct_bytes) {
  Graph& g = const_cast<Graph&>(gc);
  std::lock_guard<std::mutex> lk(g.mu);
  auto* cur = static_cast<PrBlockLayout*>(g.pr_block.get());
  if (cur && cur->ns == ns && cur->ct_bytes == ct_bytes) return cur;
  g.pr_block.reset();  // free the previous layout before building another
  auto L = build_layout(g, ns, ct_bytes);
  g.pr_block = L;
  return L.get();
}

int64_t pr_block_window(const Graph& g, int ct_bytes, int64_t blocking_size) {
  if (blocking_size > 0) return blocking_size;
  int64_t ns = l2_bytes(g.dev) * 3 / 8 / ct_bytes;  // ~3/8 of L2 holds one window
  if (ns < 1) ns = 1;
  return ns < g.V ? ns : (g.V > 0 ? g.V : 1);
}

double pr_block_prep_ms(const Graph& g, int64_t blocking_size, int ct_bytes) {
  PrBlockLayout* L = layout_for(g, pr_block_window(g, ct_bytes, blocking_size), ct_bytes);
  return L->prep_ms;
}

template <class CT>
static __global__ void __launch_bounds__(256) k_prb_init(const int32_t* outdeg, int64_t V, double* rank,
                                                         CT* contrib, double* dm0) {
  const double r0 = 1.0 / (double)V;
  double dm = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t d = outdeg[v];
    rank[v] = r0;
    contrib[v] = d ? (CT)(r0 / (double)d) : (CT)0;
    if (!d) dm += r0;
  }
  dm = block_sum(dm);
  if (threadIdx.x == 0 && dm != 0.0) atomicAdd(dm0, dm);
}

__global__ void k_unpermute(const double* rank_new, const int32_t* newid, int64_t V, double* out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x)
    out[v] = rank_new[newid[v]];
}

template <class CT>
static __global__ void __launch_bounds__(256) k_prb_fused(PrPullArgs<CT> a, CT* c0, CT* c1,
                                                          const int64_t* seg_chunk, int64_t K,
                                                          int64_t max_iters, double tol,
                                                          int64_t* iters_out) {
  __shared__ double s_acc[8 * 32];
  cg::grid_group grid = cg::this_grid();
  a.coherent = 1;
  int64_t it = 0;
  double l1 = INFINITY;
  while (!(it >= max_iters || l1 < tol)) {
    a.contrib = (it & 1) ? c1 : c0;
    a.contrib_next = (it & 1) ? c0 : c1;
    for (int64_t k = 1; k < K; ++k) {
      pr_pull_chunks<CT, 1>(a, it, s_acc, seg_chunk[k], seg_chunk[k + 1]);
      grid.sync();
    }
    pr_pull_chunks<CT, 2>(a, it, s_acc, seg_chunk[0], seg_chunk[1]);
    grid.sync();
    pr_pull_hubs(a, it);
    grid.sync();
    l1 = *((volatile double*)a.scal + 2 * it + 1);
    ++it;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *iters_out = it;
}

template <class CT>
int64_t pagerank_blocked(const Graph& g, const gg_schedule& s, bool fusion, int64_t max_iters,
                         double tol, double damping, double* ranks_out, Runtime& rt) {
  const int dev = g.dev;
  const int64_t V = g.V;
  cudaStream_t st = rt.stream;
  PrBlockLayout* L = layout_for(g, pr_block_window(g, sizeof(CT), s.blocking_size), sizeof(CT));
  const int64_t iters_cap = max_iters > 0 ? max_iters : 0;
  DevBuf<double> rank(V), acc(V), scal(2 * (iters_cap + 2));
  DevBuf<CT> c0(V), c1(V);
  scal.zero(st);
  acc.zero(st);
  k_prb_init<CT><<<grid_for(V, 256, dev), 256, 0, st>>>(L->outdeg.p, V, rank.p, c0.p, scal.p);
  GG_LAUNCH_CHECK();
  count_launch();
  PrPullArgs<CT> a{L->voff.p, L->vowner.p, L->nvrows / 32, L->src.p, c0.p, c1.p, rank.p,
                   L->outdeg.p, acc.p, L->hubs.p, L->nhubs, scal.p, V, damping};
  int64_t it = 0;
  if (!fusion) {
    double l1 = INFINITY;
    const unsigned grid = (unsigned)sm_count(dev) * 8;
    const unsigned hgrid = grid_for(L->nhubs, 256, dev);
    while (!(it >= max_iters || l1 < tol)) {
      a.contrib = (it & 1) ? c1.p : c0.p;
      a.contrib_next = (it & 1) ? c0.p : c1.p;
      rt.edge_begin();
      for (int64_t k = 1; k < L->K; ++k) {
        if (L->seg_chunk[k + 1] > L->seg_chunk[k]) {
          k_pr_seg<CT, 1><<<grid, 256, 0, st>>>(a, it, L->seg_chunk[k], L->seg_chunk[k + 1]);
          count_launch();
        }
      }
      k_pr_seg<CT, 2><<<grid, 256, 0, st>>>(a, it, L->seg_chunk[0], L->seg_chunk[1]);
      count_launch();
      if (L->nhubs) {
        k_pr_pull_hubs<CT><<<hgrid, 256, 0, st>>>(a, it);
        count_launch();
      }
      rt.edge_end();
      GG_LAUNCH_CHECK();
      rt.stats.dispatch_count += 1;
      rt.stats.direction_log.push_back(s.direction);
      ++it;
      if (tol > 0.0) {
        GG_CUDA(cudaMemcpyAsync(&l1, scal.p + 2 * (it - 1) + 1, 8, cudaMemcpyDeviceToHost, st));
        GG_CUDA(cudaStreamSynchronize(st));
      }
    }
  } else {
    DevBuf<int64_t> iters(1), segc(L->K + 1);
    GG_CUDA(cudaMemcpyAsync(segc.p, L->seg_chunk.data(), (L->K + 1) * 8, cudaMemcpyHostToDevice, st));
    int blocks = max_coop_blocks((const void*)k_prb_fused<CT>, 256, dev);
    CT* p0 = c0.p;
    CT* p1 = c1.p;
    const int64_t* sc = segc.p;
    int64_t K = L->K;
    int64_t* ip = iters.p;
    void* args[] = {&a, &p0, &p1, &sc, &K, &max_iters, &tol, &ip};
    rt.edge_begin();
    GG_CUDA(cudaLaunchCooperativeKernel((const void*)k_prb_fused<CT>, blocks, 256, args, 0, st));
    rt.edge_end();
    count_launch();
    it = dget(iters.p);
    rt.stats.dispatch_count += 1;
    for (int64_t k = 0; k < it; ++k) rt.stats.direction_log.push_back(s.direction);
  }
  rt.stats.rounds += it;
  rt.stats.edges_traversed += it * g.E;
  DevBuf<double> outv(V);
  k_unpermute<<<grid_for(V, 256, dev), 256, 0, st>>>(rank.p, L->newid.p, V, outv.p);
  GG_LAUNCH_CHECK();
  count_launch();
  GG_CUDA(cudaMemcpyAsync(ranks_out, outv.p, V * 8, cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
  return it;
}

template int64_t pagerank_blocked<double>(const Graph&, const gg_schedule&, bool, int64_t, double,
                                          double, double*, Runtime&);
template int64_t pagerank_blocked<float>(const Graph&, const gg_schedule&, bool, int64_t, double,
                                         double, double*, Runtime&);

}  // namespace gg
