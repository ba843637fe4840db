// graph.cu — device graph construction, synthetic generators and EdgeBlocking
// preprocessing (Alg. 1).
//
// Reference anchors:
//   Graph.from_coo / _build_csr    graphio.py:58-81, 95-102 (stable counting sort)
//   _symmetrize                    graphio.py:118-140 (first occurrence wins)
//   block_edges                    blocking.py:78-113 (stable partition by dst // n)
//   default_blocking_size          blocking.py:63-66 (2 MiB budget -> here: queried L2)
#include "graph.cuh"
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_reduce.cuh>

namespace gg {

static int bits_for(uint64_t maxval) {
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

__global__ void k_iota_u32(uint32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (uint32_t)i;
}

template <class T>
__global__ void k_gather(const T* __restrict__ in, const uint32_t* __restrict__ perm, T* out,
                         int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[perm[i]];
}

__global__ void k_check_range(const int32_t* a, int64_t n, int64_t lim, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t x = a[i];
    if (x < 0 || x >= lim) { *bad = 1; return; }
  }
}

__global__ void k_check_sorted(const int32_t* a, int64_t n, int* unsorted) {
  for (int64_t i = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (a[i - 1] > a[i]) { *unsorted = 1; return; }
}

// off[k] = first index i with sorted[i] >= k, for k in [0, nkeys]: a count
// per key (runs of the sorted keys add once, warp-aggregated) and an
// exclusive scan.  (The first version let each element fill the offsets of
// the empty keys before it: one thread then wrote every trailing empty key --
// ~10^7 of them in a degree-ordered graph, 23 ms.)
__global__ void k_key_counts(const int32_t* sorted, int64_t n, unsigned long long* cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31); base < n; base += stride) {
    const int64_t i = base + lane_id();
    const int32_t k = i < n ? sorted[i] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, k);
    if (k >= 0 && lane_id() == __ffs(grp) - 1) atomicAdd(cnt + k, (unsigned long long)__popc(grp));
  }
}

void offsets_from_sorted(int dev, const int32_t* sorted, int64_t n, int64_t nkeys, int64_t* off,
                         cudaStream_t s) {
  DevBuf<unsigned long long> cnt(nkeys + 1);
  GG_CUDA(cudaMemsetAsync(cnt.p, 0, (nkeys + 1) * sizeof(unsigned long long), s));
  if (n) k_key_counts<<<grid_for(n, 256, dev), 256, 0, s>>>(sorted, n, cnt.p);
  GG_LAUNCH_CHECK();
  size_t temp = 0;
  GG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, cnt.p, (unsigned long long*)off, nkeys + 1, s));
  DevBuf<uint8_t> tb(std::max<size_t>(temp, 1));
  GG_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, temp, cnt.p, (unsigned long long*)off, nkeys + 1, s));
  count_launch(2);
}

void stable_order(int dev, const int32_t* keys, int64_t n, int64_t key_limit, DevBuf<uint32_t>& perm,
                  DevBuf<int32_t>* sorted_keys, cudaStream_t s) {
  DevBuf<uint32_t> iota(n);
  perm.alloc(n);
  k_iota_u32<<<grid_for(n, 256, dev), 256, 0, s>>>(iota.p, n);
  GG_LAUNCH_CHECK();
  DevBuf<int32_t> tmp_keys;
  int32_t* kout;
  if (sorted_keys) {
    sorted_keys->alloc(n);
    kout = sorted_keys->p;
  } else {
    tmp_keys.alloc(n);
    kout = tmp_keys.p;
  }
  int end_bit = bits_for((uint64_t)(key_limit > 0 ? key_limit - 1 : 0));
  size_t temp = 0;
  GG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t*)keys, (uint32_t*)kout,
                                          iota.p, perm.p, n, 0, end_bit, s));
  DevBuf<uint8_t> tb(temp);
  GG_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, temp, (const uint32_t*)keys, (uint32_t*)kout,
                                          iota.p, perm.p, n, 0, end_bit, s));
  count_launch(4);
}

// One CSR view: stable order of (keys -> values).
static void build_csr(int dev, int64_t V, int64_t E, const int32_t* keys, const int32_t* vals,
                      const uint32_t* w, bool weighted, DevBuf<int64_t>& off, DevBuf<int32_t>& nbr,
                      DevBuf<uint32_t>& wout, cudaStream_t s) {
  off.alloc(V + 1);
  nbr.alloc(E);
  if (weighted) wout.alloc(E);
  DevBuf<int> flag(1);
  flag.zero(s);
  if (E > 1) {
    k_check_sorted<<<grid_for(E, 256, dev), 256, 0, s>>>(keys, E, flag.p);
    GG_LAUNCH_CHECK();
  }
  int unsorted = 0;
  GG_CUDA(cudaMemcpyAsync(&unsorted, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  GG_CUDA(cudaStreamSynchronize(s));
  if (!unsorted) {
    // already in key order (edge-list-file order): identity permutation
    GG_CUDA(cudaMemcpyAsync(nbr.p, vals, E * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    if (weighted) GG_CUDA(cudaMemcpyAsync(wout.p, w, E * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    offsets_from_sorted(dev, keys, E, V, off.p, s);
    return;
  }
  DevBuf<uint32_t> perm;
  DevBuf<int32_t> sorted;
  stable_order(dev, keys, E, V, perm, &sorted, s);
  k_gather<int32_t><<<grid_for(E, 256, dev), 256, 0, s>>>(vals, perm.p, nbr.p, E);
  GG_LAUNCH_CHECK();
  if (weighted) {
    k_gather<uint32_t><<<grid_for(E, 256, dev), 256, 0, s>>>(w, perm.p, wout.p, E);
    GG_LAUNCH_CHECK();
  }
  offsets_from_sorted(dev, sorted.p, E, V, off.p, s);
}

__global__ void k_max_degree(const int64_t* off, int64_t V, unsigned long long* mx) {
  unsigned long long m = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V; v += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)(off[v + 1] - off[v]));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0 && m) atomicMax(mx, m);
}

void Graph::ensure_out() const {
  Graph& g = const_cast<Graph&>(*this);
  std::lock_guard<std::mutex> lk(g.view_mu);
  if (g.has_out) return;
  if (!g.has_coo) fail(GG_ERR_ENGINE, "graph COO view was dropped before CSR-out was built");
  DeviceGuard guard(g.dev);
  build_csr(g.dev, g.V, g.E, g.coo_src.p, g.coo_dst.p, g.coo_w.p, g.weighted, g.out_off, g.out_nbr,
            g.out_w, 0);
  {
    DevBuf<unsigned long long> mx(1);
    mx.zero();
    k_max_degree<<<grid_for(g.V, 256, g.dev), 256>>>(g.out_off.p, g.V, mx.p);
    GG_LAUNCH_CHECK();
    unsigned long long h = 0;
    GG_CUDA(cudaMemcpy(&h, mx.p, 8, cudaMemcpyDeviceToHost));
    g.max_out_degree = (int64_t)h;
  }
  GG_CUDA(cudaStreamSynchronize(0));
  g.has_out = true;
}

void Graph::ensure_in() const {
  Graph& g = const_cast<Graph&>(*this);
  std::lock_guard<std::mutex> lk(g.view_mu);
  if (g.has_in) return;
  if (!g.has_coo) fail(GG_ERR_ENGINE, "graph COO view was dropped before CSR-in was built");
  DeviceGuard guard(g.dev);
  build_csr(g.dev, g.V, g.E, g.coo_dst.p, g.coo_src.p, g.coo_w.p, g.weighted, g.in_off, g.in_nbr,
            g.in_w, 0);
  GG_CUDA(cudaStreamSynchronize(0));
  g.has_in = true;
}

static void build_views(Graph& g, cudaStream_t s) {
  // views are lazy; nothing to do eagerly
  (void)g;
  (void)s;
}

std::unique_ptr<Graph> graph_adopt_coo(int dev, int64_t V, DevBuf<int32_t>&& src,
                                       DevBuf<int32_t>&& dst, DevBuf<uint32_t>&& w, bool weighted,
                                       bool symmetric) {
  auto g = std::make_unique<Graph>();
  g->dev = dev;
  g->V = V;
  g->E = (int64_t)src.n;
  g->coo_src = std::move(src);
  g->coo_dst = std::move(dst);
  g->weighted = weighted;
  if (weighted) g->coo_w = std::move(w);
  g->symmetric = symmetric;
  build_views(*g, 0);
  return g;
}

std::unique_ptr<Graph> graph_from_device_coo(int dev, int64_t V, int64_t E, const int32_t* src,
                                             const int32_t* dst, const uint32_t* w, bool symmetric) {
  if (V < 0 || E < 0) fail(GG_ERR_VALUE, "negative graph size");
  if (V > INT32_MAX) fail(GG_ERR_VALUE, "vertex ids must fit int32");
  if (E >= (int64_t)UINT32_MAX) fail(GG_ERR_VALUE, "edge count must be < 2^32");
  cudaStream_t s = 0;
  DevBuf<int32_t> s_(E), d_(E);
  DevBuf<uint32_t> w_;
  if (E) {
    GG_CUDA(cudaMemcpyAsync(s_.p, src, E * 4, cudaMemcpyDefault, s));
    GG_CUDA(cudaMemcpyAsync(d_.p, dst, E * 4, cudaMemcpyDefault, s));
  }
  if (w) {
    w_.alloc(E);
    if (E) GG_CUDA(cudaMemcpyAsync(w_.p, w, E * 4, cudaMemcpyDefault, s));
  }
  DevBuf<int> bad(1);
  bad.zero(s);
  if (E) {
    k_check_range<<<grid_for(E, 256, dev), 256, 0, s>>>(s_.p, E, V, bad.p);
    k_check_range<<<grid_for(E, 256, dev), 256, 0, s>>>(d_.p, E, V, bad.p);
    GG_LAUNCH_CHECK();
  }
  int hbad = 0;
  GG_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  GG_CUDA(cudaStreamSynchronize(s));
  if (hbad) fail(GG_ERR_VALUE, strf("vertex id out of range [0, %lld)", (long long)V));
  s_.n = E; d_.n = E;  // keep exact element counts for empty graphs
  w_.n = w ? E : 0;
  auto g = std::make_unique<Graph>();
  g->dev = dev;
  g->V = V;
  g->E = E;
  g->coo_src = std::move(s_);
  g->coo_dst = std::move(d_);
  g->weighted = w != nullptr;
  if (w) g->coo_w = std::move(w_);
  g->symmetric = symmetric;
  build_views(*g, s);
  return g;
}

// ---------------------------------------------------------------------------
// Synthetic generators (SURVEY §8d inputs).  Counter-based hashing makes every
// edge a pure function of (seed, index): reproducible across runs and hosts.
// ---------------------------------------------------------------------------
__global__ void k_rmat(int scale, int64_t E, uint32_t ta, uint32_t tab, uint32_t tabc, uint64_t seed,
                       int32_t* src, int32_t* dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t s = 0, d = 0;
    uint64_t h = 0;
    for (int l = 0; l < scale; ++l) {
      if ((l & 1) == 0) h = mix64(seed ^ mix64((uint64_t)i * 64 + l));
      uint32_t r = (l & 1) ? (uint32_t)(h >> 32) : (uint32_t)h;
      uint32_t bs = r >= tab, bd = (r >= ta && r < tab) || r >= tabc;
      s = (s << 1) | bs;
      d = (d << 1) | bd;
    }
    src[i] = (int32_t)s;
    dst[i] = (int32_t)d;
  }
}

__global__ void k_weights(uint32_t* w, int64_t E, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = 1u + (uint32_t)(mix64(seed ^ mix64((uint64_t)i ^ 0x5bd1e995ULL)) % 1000ULL);
}

// 4-neighbour grid, CSR order: for u=(r,c) arcs to up, left, right, down.
__global__ void k_grid_deg(int64_t side, int64_t* deg) {
  int64_t V = side * side;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < V;
       u += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = u / side, c = u % side;
    deg[u] = (r > 0) + (c > 0) + (c < side - 1) + (r < side - 1);
  }
}
__global__ void k_grid_arcs(int64_t side, const int64_t* off, int32_t* src, int32_t* dst) {
  int64_t V = side * side;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < V;
       u += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = u / side, c = u % side, e = off[u];
    if (r > 0) { src[e] = (int32_t)u; dst[e++] = (int32_t)(u - side); }
    if (c > 0) { src[e] = (int32_t)u; dst[e++] = (int32_t)(u - 1); }
    if (c < side - 1) { src[e] = (int32_t)u; dst[e++] = (int32_t)(u + 1); }
    if (r < side - 1) { src[e] = (int32_t)u; dst[e++] = (int32_t)(u + side); }
  }
}

__global__ void k_hash_keys(uint64_t* k, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    k[i] = mix64(seed ^ mix64((uint64_t)i + 0x2545F4914F6CDD1DULL));
}
__global__ void k_invert(const int32_t* order, int64_t n, int32_t* newid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    newid[order[i]] = (int32_t)i;
}
__global__ void k_relabel(int32_t* a, int64_t n, const int32_t* newid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = newid[a[i]];
}

// symmetrize: candidate 2i = (u,v), 2i+1 = (v,u); position order = emission order
__global__ void k_sym_candidates(const int32_t* src, const int32_t* dst, int64_t E, uint64_t* key,
                                 uint32_t* pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t u = (uint32_t)src[i], v = (uint32_t)dst[i];
    key[2 * i] = (u << 32) | v;
    key[2 * i + 1] = (v << 32) | u;
    pos[2 * i] = (uint32_t)(2 * i);
    pos[2 * i + 1] = (uint32_t)(2 * i + 1);
  }
}
__global__ void k_first_flags(const uint64_t* key, int64_t n, uint8_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}
__global__ void k_sym_emit(const uint64_t* key_by_pos, const uint32_t* pos, int64_t n,
                           const uint32_t* w_in, int32_t* src, int32_t* dst, uint32_t* w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = key_by_pos[i];
    src[i] = (int32_t)(k >> 32);
    dst[i] = (int32_t)(k & 0xffffffffULL);
    if (w) w[i] = w_in[pos[i] >> 1];
  }
}

static int64_t count_from_device(const unsigned long long* p) {
  unsigned long long h = 0;
  GG_CUDA(cudaMemcpy(&h, p, sizeof(h), cudaMemcpyDeviceToHost));
  return (int64_t)h;
}

// graphio._symmetrize on the device: each arc and its mirror once, first
// occurrence (in emission order 2i, 2i+1) wins and fixes the weight.
static void symmetrize(int dev, int64_t V, DevBuf<int32_t>& src, DevBuf<int32_t>& dst,
                       DevBuf<uint32_t>& w, bool weighted) {
  const int64_t E = (int64_t)src.n, n = 2 * E;
  if (n >= (int64_t)UINT32_MAX) fail(GG_ERR_VALUE, "symmetrize: too many arcs");
  DevBuf<uint64_t> key(n), key2(n);
  DevBuf<uint32_t> pos(n), pos2(n);
  k_sym_candidates<<<grid_for(E, 256, dev), 256>>>(src.p, dst.p, E, key.p, pos.p);
  GG_LAUNCH_CHECK();
  int kb = 32 + bits_for((uint64_t)(V > 0 ? V - 1 : 0));
  size_t temp = 0;
  GG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, key.p, key2.p, pos.p, pos2.p, n, 0, kb));
  {
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, temp, key.p, key2.p, pos.p, pos2.p, n, 0, kb));
  }
  // unique-first: keep the smallest position of every (a,b)
  DevBuf<uint8_t> flag(n);
  k_first_flags<<<grid_for(n, 256, dev), 256>>>(key2.p, n, flag.p);
  GG_LAUNCH_CHECK();
  DevBuf<unsigned long long> nsel(1);
  temp = 0;
  GG_CUDA(cub::DeviceSelect::Flagged(nullptr, temp, pos2.p, flag.p, pos.p, nsel.p, n));
  {
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceSelect::Flagged(tb.p, temp, pos2.p, flag.p, pos.p, nsel.p, n));
  }
  temp = 0;
  GG_CUDA(cub::DeviceSelect::Flagged(nullptr, temp, key2.p, flag.p, key.p, nsel.p, n));
  {
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceSelect::Flagged(tb.p, temp, key2.p, flag.p, key.p, nsel.p, n));
  }
  const int64_t m = count_from_device(nsel.p);
  flag.release();
  // back to emission order
  int pb = bits_for((uint64_t)(n - 1));
  temp = 0;
  GG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, pos.p, pos2.p, key.p, key2.p, m, 0, pb));
  {
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, temp, pos.p, pos2.p, key.p, key2.p, m, 0, pb));
  }
  DevBuf<int32_t> ns(m), nd(m);
  DevBuf<uint32_t> nw;
  if (weighted) nw.alloc(m);
  k_sym_emit<<<grid_for(m, 256, dev), 256>>>(key2.p, pos2.p, m, weighted ? w.p : nullptr, ns.p, nd.p,
                                             weighted ? nw.p : nullptr);
  GG_LAUNCH_CHECK();
  GG_CUDA(cudaDeviceSynchronize());
  ns.n = m; nd.n = m;
  src = std::move(ns);
  dst = std::move(nd);
  if (weighted) { nw.n = m; w = std::move(nw); }
}

static void permute_ids(int dev, int64_t V, uint64_t seed, DevBuf<int32_t>& src, DevBuf<int32_t>& dst) {
  DevBuf<uint64_t> k(V), k2(V);
  DevBuf<int32_t> ids(V), order(V), newid(V);
  k_hash_keys<<<grid_for(V, 256, dev), 256>>>(k.p, V, seed);
  k_iota_u32<<<grid_for(V, 256, dev), 256>>>((uint32_t*)ids.p, V);
  size_t temp = 0;
  GG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, k.p, k2.p, ids.p, order.p, V));
  DevBuf<uint8_t> tb(temp);
  GG_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, temp, k.p, k2.p, ids.p, order.p, V));
  k_invert<<<grid_for(V, 256, dev), 256>>>(order.p, V, newid.p);
  k_relabel<<<grid_for(src.n, 256, dev), 256>>>(src.p, (int64_t)src.n, newid.p);
  k_relabel<<<grid_for(dst.n, 256, dev), 256>>>(dst.p, (int64_t)dst.n, newid.p);
  GG_LAUNCH_CHECK();
}

// Reorder COO by source (stable), like an edge-list file sorted by source.
static void sort_by_source(int dev, int64_t V, DevBuf<int32_t>& src, DevBuf<int32_t>& dst,
                           DevBuf<uint32_t>& w, bool weighted) {
  const int64_t E = (int64_t)src.n;
  DevBuf<uint32_t> perm;
  DevBuf<int32_t> sorted;
  stable_order(dev, src.p, E, V, perm, &sorted, 0);
  DevBuf<int32_t> nd(E);
  k_gather<int32_t><<<grid_for(E, 256, dev), 256>>>(dst.p, perm.p, nd.p, E);
  if (weighted) {
    DevBuf<uint32_t> nw(E);
    k_gather<uint32_t><<<grid_for(E, 256, dev), 256>>>(w.p, perm.p, nw.p, E);
    GG_LAUNCH_CHECK();
    w = std::move(nw);
  }
  GG_LAUNCH_CHECK();
  src = std::move(sorted);
  dst = std::move(nd);
}

std::unique_ptr<Graph> generate_graph(int dev, int kind, int scale, int edge_factor, double a,
                                      double b, double c, uint64_t seed, int flags) {
  DeviceGuard guard(dev);
  int64_t V = 0, E = 0;
  DevBuf<int32_t> src, dst;
  DevBuf<uint32_t> w;
  const bool weighted = flags & 4;
  if (kind == 0 || kind == 1) {
    if (scale < 1 || scale > 30) fail(GG_ERR_VALUE, "scale must be in [1, 30]");
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0) fail(GG_ERR_VALUE, "bad RMAT probabilities");
    V = (int64_t)1 << scale;
    E = V * (int64_t)edge_factor;
    src.alloc(E);
    dst.alloc(E);
    const double s32 = 4294967296.0;
    auto th = [&](double p) { double t = p * s32; return (uint32_t)(t >= s32 ? 4294967295.0 : t); };
    k_rmat<<<grid_for(E, 256, dev, 16), 256>>>(scale, E, th(a), th(a + b), th(a + b + c), seed,
                                               src.p, dst.p);
    GG_LAUNCH_CHECK();
  } else if (kind == 2) {
    const int64_t side = scale;  // scale = side length for grids
    if (side < 1 || side * side > INT32_MAX) fail(GG_ERR_VALUE, "bad grid side");
    V = side * side;
    DevBuf<int64_t> deg(V), off(V + 1);
    k_grid_deg<<<grid_for(V, 256, dev), 256>>>(side, deg.p);
    size_t temp = 0;
    GG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, deg.p, off.p, V));
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, temp, deg.p, off.p, V));
    E = 4 * side * (side - 1);
    src.alloc(E);
    dst.alloc(E);
    k_grid_arcs<<<grid_for(V, 256, dev), 256>>>(side, off.p, src.p, dst.p);
    GG_LAUNCH_CHECK();
  } else {
    fail(GG_ERR_VALUE, "unknown generator kind");
  }
  if (weighted) {
    w.alloc(E);
    k_weights<<<grid_for(E, 256, dev), 256>>>(w.p, E, seed ^ 0xA5A5A5A5ULL);
    GG_LAUNCH_CHECK();
  }
  if ((flags & 2) || kind == 1) permute_ids(dev, V, seed ^ 0x77ULL, src, dst);
  bool sym = false;
  if (flags & 1) {
    symmetrize(dev, V, src, dst, w, weighted);
    sym = true;
  }
  if (flags & 8) sort_by_source(dev, V, src, dst, w, weighted);
  GG_CUDA(cudaDeviceSynchronize());
  return graph_adopt_coo(dev, V, std::move(src), std::move(dst), std::move(w), weighted, sym);
}

// ---------------------------------------------------------------------------
// EdgeBlocking, Alg. 1 (blocking.py:78-113) on the device.
// ---------------------------------------------------------------------------
__global__ void k_segment_keys(const int32_t* dst, int64_t E, int64_t n, int32_t* seg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x)
    seg[i] = (int32_t)(dst[i] / n);
}

int64_t default_blocking_size(const Graph& g) {
  // Half the L2 holds one segment's destination data (fp64 accumulators);
  // the rest is left to the streamed edges.  Reference: 2 MiB / 8 B.
  int64_t n = l2_bytes(g.dev) / 2 / 8;
  if (n < 1) n = 1;
  return n < g.V ? n : (g.V > 0 ? g.V : 1);
}

// Sidecar install (blocking.load_blocked, blocking.py:200-217, straight to the
// device): validates the layout against the graph -- segment ends, every
// edge inside its segment, and the edge multiset (order-free hash sum) --
// then caches it as blocked_for(g, n) would have built it.
__global__ void k_seg_check(const int32_t* dst, const int64_t* seg_end, int64_t nseg, int64_t E, int64_t n,
                            int* bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = dst[e] / n;
    const int64_t lo = s ? seg_end[s - 1] : 0;
    if (s >= nseg || e < lo || e >= seg_end[s]) *bad = 1;
  }
}
__global__ void k_edge_hash(const int32_t* src, const int32_t* dst, const uint32_t* w, int64_t E,
                            unsigned long long* h) {
  unsigned long long acc = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    acc += mix64(((uint64_t)(uint32_t)src[e] << 32) ^ (uint32_t)dst[e] ^ ((uint64_t)(w ? w[e] : 0u) << 17));
  acc = warp_sum(acc);
  if (lane_id() == 0) atomicAdd(h, acc);
}

Blocked* blocked_install(Graph& g, int64_t n, int64_t nseg, const int64_t* seg_end, const int32_t* src,
                         const int32_t* dst, const uint32_t* w) {
  if (n < 1) fail(GG_ERR_VALUE, "vertices per segment must be >= 1");
  if (g.V == 0) fail(GG_ERR_VALUE, "empty graph");
  if (!g.has_coo) fail(GG_ERR_ENGINE, "graph COO view was dropped");
  if (nseg != (g.V + n - 1) / n) fail(GG_ERR_VALUE, "sidecar segment count does not match the graph");
  if ((w != nullptr) != g.weighted) fail(GG_ERR_VALUE, "sidecar weights do not match the graph");
  for (int64_t s = 0; s < nseg; ++s)
    if (seg_end[s] < (s ? seg_end[s - 1] : 0) || seg_end[s] > g.E)
      fail(GG_ERR_VALUE, "sidecar segment ends are not monotone");
  if (nseg && seg_end[nseg - 1] != g.E) fail(GG_ERR_VALUE, "sidecar edge count does not match the graph");
  DeviceGuard guard(g.dev);
  double t0 = now_ms();
  auto b = std::make_unique<Blocked>();
  b->n = n;
  b->E = g.E;
  b->nseg = nseg;
  b->seg_end.alloc(nseg);
  b->src.alloc(g.E);
  b->dst.alloc(g.E);
  GG_CUDA(cudaMemcpy(b->seg_end.p, seg_end, nseg * 8, cudaMemcpyDefault));
  GG_CUDA(cudaMemcpy(b->src.p, src, g.E * 4, cudaMemcpyDefault));
  GG_CUDA(cudaMemcpy(b->dst.p, dst, g.E * 4, cudaMemcpyDefault));
  if (w) {
    b->w.alloc(g.E);
    GG_CUDA(cudaMemcpy(b->w.p, w, g.E * 4, cudaMemcpyDefault));
  }
  DevBuf<int> bad(1);
  bad.zero();
  DevBuf<unsigned long long> h(2);
  h.zero();
  if (g.E) {
    k_check_range<<<grid_for(g.E, 256, g.dev), 256>>>(b->src.p, g.E, g.V, bad.p);
    k_check_range<<<grid_for(g.E, 256, g.dev), 256>>>(b->dst.p, g.E, g.V, bad.p);
    k_seg_check<<<grid_for(g.E, 256, g.dev), 256>>>(b->dst.p, b->seg_end.p, nseg, g.E, n, bad.p);
    k_edge_hash<<<grid_for(g.E, 256, g.dev), 256>>>(b->src.p, b->dst.p, w ? b->w.p : nullptr, g.E, h.p);
    k_edge_hash<<<grid_for(g.E, 256, g.dev), 256>>>(g.coo_src.p, g.coo_dst.p, g.weighted ? g.coo_w.p : nullptr,
                                                    g.E, h.p + 1);
    GG_LAUNCH_CHECK();
  }
  int hb = 0;
  unsigned long long hh[2];
  GG_CUDA(cudaMemcpy(&hb, bad.p, 4, cudaMemcpyDeviceToHost));
  GG_CUDA(cudaMemcpy(hh, h.p, 16, cudaMemcpyDeviceToHost));
  if (hb) fail(GG_ERR_VALUE, "sidecar edges are out of range or outside their segments");
  if (hh[0] != hh[1]) fail(GG_ERR_VALUE, "sidecar edges are not the graph's edges");
  b->prep_ms = now_ms() - t0;
  std::lock_guard<std::mutex> lk(g.mu);
  Blocked* raw = b.get();
  g.blocked[n] = std::move(b);
  return raw;
}

Blocked* blocked_for(Graph& g, int64_t n) {
  if (n < 1) fail(GG_ERR_VALUE, "vertices per segment must be >= 1");
  if (g.V == 0) fail(GG_ERR_VALUE, "empty graph");
  if (!g.has_coo) fail(GG_ERR_ENGINE, "graph COO view was dropped");
  std::lock_guard<std::mutex> lk(g.mu);
  auto it = g.blocked.find(n);
  if (it != g.blocked.end()) return it->second.get();
  DeviceGuard guard(g.dev);
  double t0 = now_ms();
  auto b = std::make_unique<Blocked>();
  b->n = n;
  b->E = g.E;
  b->nseg = (g.V + n - 1) / n;
  DevBuf<int32_t> seg(g.E);
  k_segment_keys<<<grid_for(g.E, 256, g.dev), 256>>>(g.coo_dst.p, g.E, n, seg.p);
  GG_LAUNCH_CHECK();
  DevBuf<uint32_t> perm;
  DevBuf<int32_t> sorted;
  stable_order(g.dev, seg.p, g.E, b->nseg, perm, &sorted, 0);
  seg.release();
  b->src.alloc(g.E);
  b->dst.alloc(g.E);
  k_gather<int32_t><<<grid_for(g.E, 256, g.dev), 256>>>(g.coo_src.p, perm.p, b->src.p, g.E);
  k_gather<int32_t><<<grid_for(g.E, 256, g.dev), 256>>>(g.coo_dst.p, perm.p, b->dst.p, g.E);
  if (g.weighted) {
    b->w.alloc(g.E);
    k_gather<uint32_t><<<grid_for(g.E, 256, g.dev), 256>>>(g.coo_w.p, perm.p, b->w.p, g.E);
  }
  GG_LAUNCH_CHECK();
  // inclusive segment ends = exclusive offsets shifted by one
  DevBuf<int64_t> off(b->nseg + 1);
  offsets_from_sorted(g.dev, sorted.p, g.E, b->nseg, off.p, 0);
  b->seg_end.alloc(b->nseg);
  GG_CUDA(cudaMemcpy(b->seg_end.p, off.p + 1, b->nseg * sizeof(int64_t), cudaMemcpyDeviceToDevice));
  GG_CUDA(cudaDeviceSynchronize());
  b->prep_ms = now_ms() - t0;
  Blocked* raw = b.get();
  g.blocked[n] = std::move(b);
  return raw;
}

}  // namespace gg
