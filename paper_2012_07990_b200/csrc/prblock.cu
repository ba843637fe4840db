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
//   preprocessing (once per graph and window, cached; prblock build_layout):
//     1. out-degree histogram of the COO (warp-aggregated atomics) and a
//        renumbering by out-degree, descending (hot sources first);
//     2. segment k = sources [k*Ns, (k+1)*Ns), Ns*sizeof(contrib) sized to a
//        fraction of the queried L2 (blocking_size overrides Ns);
//     3. stable radix sort of the edges by (segment, destination) with the
//        source as payload (32-bit keys when they fit): inside a segment each
//        destination's in-edges are contiguous, in COO order;
//   per iteration (Alg. 2: segments in order, a barrier between them):
//     cold segments k = 1..K-1: edge-parallel gather from the segment's
//       L2-resident contrib window, destination runs reduced in registers
//       (warp segmented scan), one f64 add per run;
//     hot segment 0 last: the same with the hottest sources' contributions
//       staged in shared memory (128 KB; the rest of the array stays L1,
//       which stages the in-flight gather lines); then the vertex pass.
// All per-vertex state lives in the renumbered id space; ranks are permuted
// back on output.  Results equal the reference's up to f64 summation order.
#include "prtile.cuh"  // block_sum
#include "apply.cuh"
#include "prdist.cuh"
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

namespace gg {

// Destination partition of a multi-GPU run: this rank owns the
// renumbered destinations [lo, hi); P == 1 owns everything.
struct PrPart {
  int P = 1, r = 0;
};

struct PrBlockLayout {
  int64_t ns = 0, ns_cold = 0, K = 0, V = 0, E = 0;  // hot window, cold windows
  int ct_bytes = 0;
  int P = 1, r = 0;
  int64_t lo = 0, hi = 0;                            // owned destinations (renumbered ids)
  std::vector<int64_t> bounds;                       // P+1 partition bounds (renumbered ids)
  DevBuf<int32_t> newid, order, outdeg, src;         // src: renumbered sources, blocked order
  DevBuf<int32_t> dst;                               // local destination of every blocked edge
  std::vector<int64_t> seg_edge;                     // K+1 edge boundaries (segment 0 = hot)
  double prep_ms = 0;
  int64_t vloc() const { return hi - lo; }
  // per-run work buffers, kept across calls (cudaMalloc/cudaFree of GB-sized
  // buffers per call would dominate short runs)
  DevBuf<double> w_rank, w_acc, w_scal, w_out;
  DevBuf<uint8_t> w_c0, w_c1;
  std::mutex w_mu;
};

static int nbits(uint64_t x) {
  int b = 0;
  while (b < 64 && (x >> b)) ++b;
  return b ? b : 1;
}

// out-degree histogram; lanes holding the same source (runs in source-sorted
// input, hubs in any order) add once per group
__global__ void k_outdeg_hist(const int32_t* s, int64_t E, uint32_t* deg) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31); base < E; base += stride) {
    const int64_t e = base + lane_id();
    const int32_t u = e < E ? s[e] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, u);
    if (u >= 0 && lane_id() == __ffs(grp) - 1) atomicAdd(deg + u, (uint32_t)__popc(grp));
  }
}
__global__ void k_neg_deg(const uint32_t* deg, int64_t V, uint32_t* key, int32_t* ids) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    key[v] = ~deg[v];
    ids[v] = (int32_t)v;
  }
}
__global__ void k_relabel_tables(const int32_t* order, const uint32_t* deg, int64_t V, int32_t* newid,
                                 int32_t* outdeg_new) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t o = order[i];
    newid[o] = (int32_t)i;
    outdeg_new[i] = (int32_t)deg[o];
  }
}
// key = (source segment, local destination), payload = renumbered source;
// edges whose destination another rank owns get segment K (sorted last).
template <class KT>
__global__ void k_edge_keys(const int32_t* s, const int32_t* d, int64_t E, const int32_t* newid,
                            int64_t ns, int64_t ns_cold, int nvb, int64_t lo, int64_t hi, uint64_t K, KT* key,
                            int32_t* val) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t nu = newid[s[e]];
    const int64_t nv = newid[d[e]];
    val[e] = nu;
    if (nv < lo || nv >= hi) {
      key[e] = (KT)(K << nvb);
      continue;
    }
    // segment 0 = the hot window [0, ns); then cold windows of ns_cold sources
    const uint64_t seg = (uint64_t)nu < (uint64_t)ns ? 0 : 1 + ((uint64_t)nu - ns) / (uint64_t)ns_cold;
    key[e] = (KT)((seg << nvb) | (uint64_t)(nv - lo));
  }
}
template <class KT>
__global__ void k_owned_flags(const KT* key, int64_t E, uint64_t K, int nvb, uint8_t* flags) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
    flags[e] = ((uint64_t)key[e] >> nvb) < K;
}
template <class KT>
__global__ void k_count_hot(const KT* key, int64_t E, int shift, unsigned long long* n) {
  unsigned long long c = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x)
    c += ((uint64_t)key[e] >> shift) == 0;
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(n, c);
}
template <class KT>
__global__ void k_dst_of_keys(const KT* key, int64_t E, int nvb, int32_t* dst) {
  const uint64_t mask = (1ULL << nvb) - 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = (int32_t)((uint64_t)key[e] & mask);
}
// first edge of each segment (segments are sorted): seg_edge[k] = lower bound
template <class KT>
__global__ void k_seg_bounds(const KT* key, int64_t E, int shift, int64_t K, int64_t* seg_edge) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k > K) return;
  int64_t a = 0, b = E;
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if ((int64_t)((uint64_t)key[mid] >> shift) < k) a = mid + 1; else b = mid;
  }
  seg_edge[k] = a;
}
// in-degree per renumbered vertex (partition balance)
__global__ void k_indeg_new(const int32_t* d, int64_t E, const int32_t* newid, unsigned long long* cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + newid[d[e]], 1ULL);
}
// bounds[r] = first renumbered v (rounded down to a multiple of 32, so the
// vertex pass keeps 16-byte alignment) with in_off[v] >= r*E/P
__global__ void k_part_bounds(const unsigned long long* in_off, int64_t V, int P, int64_t* bounds) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > P) return;
  if (r == 0) { bounds[0] = 0; return; }
  if (r == P) { bounds[r] = V; return; }
  const unsigned long long E = in_off[V];
  const unsigned long long target = (unsigned long long)((unsigned __int128)E * r / P);
  int64_t lo = 0, hi = V;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (in_off[mid] < target) lo = mid + 1; else hi = mid;
  }
  bounds[r] = lo & ~int64_t(31);
}
template <class T>
static T dget(const T* p) {
  T h;
  GG_CUDA(cudaMemcpy(&h, p, sizeof(T), cudaMemcpyDeviceToHost));
  return h;
}


template <class KT>
static void sort_edges(const Graph& g, PrBlockLayout* L, int nvb, int kb, int64_t E) {
  const int dev = g.dev;
  const int64_t Eall = g.E;
  const int shift = nvb;
  DevBuf<KT> keys(std::max<int64_t>(E, 1));
  {
    DevBuf<KT> k0(Eall);
    DevBuf<int32_t> v0(Eall);
    k_edge_keys<KT><<<grid_for(Eall, 256, dev), 256>>>(g.coo_src.p, g.coo_dst.p, Eall, L->newid.p, L->ns,
                                                       L->ns_cold, nvb,
                                                       L->lo, L->hi, (uint64_t)L->K, k0.p, v0.p);
    GG_LAUNCH_CHECK();
    DevBuf<KT> k1;
    DevBuf<int32_t> v1;
    KT* kin = k0.p;
    int32_t* vin = v0.p;
    if (E < Eall) {
      // a partitioned run keeps only the edges into its own destinations
      // (order-preserving, so the stable sort's ties stay in COO order): the
      // layout and the sort scale with the rank's E, not the graph's
      k1.alloc(std::max<int64_t>(E, 1));
      v1.alloc(std::max<int64_t>(E, 1));
      DevBuf<uint8_t> flags(Eall);
      DevBuf<unsigned long long> nsel(1);
      k_owned_flags<KT><<<grid_for(Eall, 256, dev), 256>>>(k0.p, Eall, (uint64_t)L->K, nvb, flags.p);
      GG_LAUNCH_CHECK();
      size_t t1 = 0, t2 = 0;
      GG_CUDA(cub::DeviceSelect::Flagged(nullptr, t1, k0.p, flags.p, k1.p, nsel.p, Eall));
      GG_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, v0.p, flags.p, v1.p, nsel.p, Eall));
      DevBuf<uint8_t> tb(std::max(t1, t2));
      GG_CUDA(cub::DeviceSelect::Flagged(tb.p, t1, k0.p, flags.p, k1.p, nsel.p, Eall));
      GG_CUDA(cub::DeviceSelect::Flagged(tb.p, t2, v0.p, flags.p, v1.p, nsel.p, Eall));
      kin = k1.p;
      vin = v1.p;
    }
    L->src.alloc(std::max<int64_t>(E, 1));  // payload: renumbered sources in (segment, destination) order
    size_t temp = 0;
    GG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, kin, keys.p, vin, L->src.p, E, 0, nvb + kb));
    DevBuf<uint8_t> tb(std::max<size_t>(temp, 1));
    GG_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, temp, kin, keys.p, vin, L->src.p, E, 0, nvb + kb));
  }
  L->src.n = E;
  L->dst.alloc(E);
  k_dst_of_keys<KT><<<grid_for(E, 256, dev), 256>>>(keys.p, E, nvb, L->dst.p);
  DevBuf<int64_t> se(L->K + 1);
  k_seg_bounds<KT><<<(unsigned)((L->K + 1 + 127) / 128), 128>>>(keys.p, E, shift, L->K, se.p);
  GG_LAUNCH_CHECK();
  L->seg_edge.resize(L->K + 1);
  GG_CUDA(cudaMemcpy(L->seg_edge.data(), se.p, (L->K + 1) * 8, cudaMemcpyDeviceToHost));
  L->seg_edge[L->K] = E;
}

static std::shared_ptr<PrBlockLayout> build_layout(const Graph& g, int64_t ns, int ct_bytes, PrPart part) {
  NvtxRange nvtx("gg.pr_block.build_layout");
  const int dev = g.dev;
  const int64_t V = g.V, Eall = g.E;
  if (!g.has_coo) fail(GG_ERR_ENGINE, "graph COO view was dropped");
  auto L = std::make_shared<PrBlockLayout>();
  double t0 = now_ms();
  L->ns = ns;
  // cold windows: GG_PR_COLD_WINDOW16 sixteenths of L2 (default: the hot size)
  L->ns_cold = ns;
  if (const char* e = getenv("GG_PR_COLD_WINDOW16"))
    L->ns_cold = std::max<int64_t>(1, l2_bytes(g.dev) * std::max(1, atoi(e)) / 16 / ct_bytes);
  L->K = V > ns ? 1 + (V - ns + L->ns_cold - 1) / L->ns_cold : 1;
  L->V = V;
  L->ct_bytes = ct_bytes;
  L->P = part.P;
  L->r = part.r;
  // 1. out-degree renumbering (stable, descending), from a COO histogram
  {
    DevBuf<uint32_t> deg(V), key(V), key2(V);
    DevBuf<int32_t> ids(V);
    deg.zero();
    k_outdeg_hist<<<grid_for(Eall, 256, dev), 256>>>(g.coo_src.p, Eall, deg.p);
    L->order.alloc(V);
    k_neg_deg<<<grid_for(V, 256, dev), 256>>>(deg.p, V, key.p, ids.p);
    GG_LAUNCH_CHECK();
    if (getenv("GG_PR_NO_RELABEL")) GG_CUDA(cudaMemset(key.p, 0, V * sizeof(uint32_t)));  // ablation
    size_t temp = 0;
    GG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, key.p, key2.p, ids.p, L->order.p, V));
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceRadixSort::SortPairs(tb.p, temp, key.p, key2.p, ids.p, L->order.p, V));
    L->newid.alloc(V);
    L->outdeg.alloc(V);
    k_relabel_tables<<<grid_for(V, 256, dev), 256>>>(L->order.p, deg.p, V, L->newid.p, L->outdeg.p);
    GG_LAUNCH_CHECK();
  }
  // 1b. destination partition in the renumbered id space, balanced by in-edges
  L->bounds.assign(part.P + 1, 0);
  L->bounds[part.P] = V;
  int64_t E = Eall;  // edges this rank keeps
  if (part.P > 1) {
    DevBuf<unsigned long long> cnt(V + 1), off(V + 1);
    cnt.zero();
    k_indeg_new<<<grid_for(Eall, 256, dev), 256>>>(g.coo_dst.p, Eall, L->newid.p, cnt.p);
    GG_LAUNCH_CHECK();
    size_t temp = 0;
    GG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, cnt.p, off.p, V + 1));
    DevBuf<uint8_t> tb(temp);
    GG_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, temp, cnt.p, off.p, V + 1));
    DevBuf<int64_t> db(part.P + 1);
    k_part_bounds<<<1, 256>>>(off.p, V, part.P, db.p);
    GG_LAUNCH_CHECK();
    GG_CUDA(cudaMemcpy(L->bounds.data(), db.p, (part.P + 1) * 8, cudaMemcpyDeviceToHost));
    const int64_t elo = (int64_t)dget(off.p + L->bounds[part.r]);
    const int64_t ehi = (int64_t)dget(off.p + L->bounds[part.r + 1]);
    E = ehi - elo;
  }
  L->lo = L->bounds[part.r];
  L->hi = L->bounds[part.r + 1];
  L->E = E;
  const int64_t Vl = L->hi - L->lo;
  const int nvb = nbits((uint64_t)(Vl > 1 ? Vl - 1 : 1));
  const int kb = nbits((uint64_t)L->K);  // segment K marks edges of other ranks
  if (nvb + kb > 64) fail(GG_ERR_VALUE, "EdgeBlocking layout: too many segments for this graph");
  // 2-3. (segment, destination) keys with the source as payload, stably sorted
  if (nvb + kb <= 32)
    sort_edges<uint32_t>(g, L.get(), nvb, kb, E);
  else
    sort_edges<uint64_t>(g, L.get(), nvb, kb, E);
  GG_CUDA(cudaDeviceSynchronize());
  L->prep_ms = now_ms() - t0;
  return L;
}

// cached on the graph (one layout per (window, contrib width, partition)).
// Callers hold the returned shared_ptr for the whole query: a concurrent
// query on the same graph that needs another layout replaces the cache
// entry, and the old layout (its buffers and its w_mu) lives until its last
// user returns.
static std::shared_ptr<PrBlockLayout> layout_for(const Graph& gc, int64_t ns, int ct_bytes,
                                                 PrPart part = PrPart()) {
  Graph& g = const_cast<Graph&>(gc);
  std::lock_guard<std::mutex> lk(g.mu);
  auto cur = std::static_pointer_cast<PrBlockLayout>(g.pr_block);
  if (cur && cur->ns == ns && cur->ct_bytes == ct_bytes && cur->P == part.P && cur->r == part.r) return cur;
  cur.reset();
  g.pr_block.reset();  // drop the cache's reference before building another
  auto L = build_layout(g, ns, ct_bytes, part);
  g.pr_block = L;
  return L;
}

int64_t pr_block_window(const Graph& g, int ct_bytes, int64_t blocking_size) {
  if (blocking_size > 0) return blocking_size;
  if (const char* e = getenv("GG_PR_ONE_SEGMENT"))  // A/B: every edge in the hot kernel
    if (atoi(e) != 0) return g.V > 0 ? g.V : 1;
  // one source window in a fraction of the queried L2 (default 6/16; the
  // rest holds the streamed edges and the destination accumulators);
  // GG_PR_WINDOW16 overrides the sixteenths
  int64_t frac16 = 6;
  if (const char* e = getenv("GG_PR_WINDOW16")) frac16 = std::max(1, std::min(16, atoi(e)));
  int64_t ns = l2_bytes(g.dev) * frac16 / 16 / ct_bytes;
  if (ns < 1) ns = 1;
  // the sort key (segment | destination) must fit 64 bits, with one
  // spare segment id for a partitioned run's foreign edges: widen the window
  // when a small L2 share would need too many segments
  const int nvb = nbits((uint64_t)(g.V > 1 ? g.V - 1 : 1));
  while (nvb + nbits((uint64_t)((g.V + ns - 1) / ns)) > 64) ns *= 2;
  return ns < g.V ? ns : (g.V > 0 ? g.V : 1);
}

double pr_block_prep_ms(const Graph& g, int64_t blocking_size, int ct_bytes) {
  return layout_for(g, pr_block_window(g, ct_bytes, blocking_size), ct_bytes)->prep_ms;
}

// rank_0 = 1/n, or a given vector in original ids (order: renumbered -> original)
template <class CT>
static __global__ void __launch_bounds__(256) k_prb_init(const int32_t* outdeg, int64_t V, double* rank,
                                                         CT* contrib, double* dm0, const double* init,
                                                         const int32_t* order) {
  double dm = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < V;
       v += (int64_t)gridDim.x * blockDim.x) {
    const double r0 = init ? init[order[v]] : 1.0 / (double)V;
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

// ---------------------------------------------------------------------------
// Edge phase (EDGE_ONLY semantics, Alg. 2): for one segment, every warp takes
// kU*32 consecutive blocked edges per step -- coalesced (src, dst) loads, kU
// independent gathers per lane, then a warp segmented scan keyed by the
// (sorted) destination so each destination run issues ONE f64 add to acc.
// ---------------------------------------------------------------------------
constexpr int kE = 8;  // consecutive blocked edges per lane (two 16-byte loads per array)

// Load one lane's kE consecutive edges [my, my+kE) clipped to [e0, e1);
// dst = -1 marks a dead slot.
__device__ __forceinline__ void pr_load_edges(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                              int64_t my, int64_t e0, int64_t e1, int32_t (&su)[kE],
                                              int32_t (&dv)[kE]) {
  if (my + kE <= e1 && my >= e0) {
    const int4* s4 = reinterpret_cast<const int4*>(src + my);
    const int4* d4 = reinterpret_cast<const int4*>(dst + my);
    int4 a0 = __ldcs(s4), a1 = __ldcs(s4 + 1), b0 = __ldcs(d4), b1 = __ldcs(d4 + 1);
    su[0] = a0.x; su[1] = a0.y; su[2] = a0.z; su[3] = a0.w;
    su[4] = a1.x; su[5] = a1.y; su[6] = a1.z; su[7] = a1.w;
    dv[0] = b0.x; dv[1] = b0.y; dv[2] = b0.z; dv[3] = b0.w;
    dv[4] = b1.x; dv[5] = b1.y; dv[6] = b1.z; dv[7] = b1.w;
  } else {
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      const int64_t e = my + q;
      const bool live = e >= e0 && e < e1;
      su[q] = live ? __ldcs(src + e) : 0;
      dv[q] = live ? __ldcs(dst + e) : -1;
    }
  }
}

// Gather + reduce one warp step (kE*32 edges).  Invariant: destinations are
// nondecreasing over [e0, e1) (one segment), so equal destinations are
// contiguous across lanes -- the segmented scan relies on it (a launch over
// several segments would break it: measured and rejected, it was also
// slower).  Runs of equal destination
// inside a lane are summed in registers; runs crossing lanes are joined by ONE
// warp segmented scan per step; each destination run issues one f64 add.
// kSmem: sources < nhot are read from the CTA's shared-memory copy of the
// hottest contributions (degree-renumbered ids: hot = small).
// Gather flavours for the hot kernel (GG_PR_GATHER): 0 ld.global.nc (default),
// 1 ld.global.cg (L2 only), 2 ld.global.nc.L1::no_allocate.
// kLoad 3: sources past the hot window (`cold_from`) are gathered with an
// L2 evict-first policy, so one-shot cold lines do not push the hot window
// out of L2 (one-segment layout, GG_PR_ONE_SEGMENT)
__device__ __forceinline__ double ld_evict_first(const double* p) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_evict_first(const float* p) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}

template <int kLoad>
__device__ __forceinline__ double ld_gather(const double* p) {
  if (kLoad == 1) return __ldcg(p);
  if (kLoad == 2) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
  }
  return __ldg(p);
}
template <int kLoad>
__device__ __forceinline__ float ld_gather(const float* p) {
  if (kLoad == 1) return __ldcg(p);
  if (kLoad == 2) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
  }
  return __ldg(p);
}

template <class CT, bool kSmem, int kLoad = 0>
__device__ __forceinline__ void pr_reduce_step(const int32_t (&su)[kE], const int32_t (&dv)[kE], const CT* contrib,
                                               double* acc, int coherent, const CT* s_hot, int32_t nhot,
                                               int32_t cold_from = INT32_MAX) {
  const int lane = lane_id();
  double v[kE];
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    if (kSmem)
      v[q] = dv[q] < 0 ? 0.0
             : su[q] < nhot ? (double)s_hot[su[q]]
             : kLoad == 3 ? (double)(su[q] >= cold_from ? ld_evict_first(contrib + su[q]) : __ldg(contrib + su[q]))
             : (double)ld_gather<kLoad>(contrib + su[q]);
    else
      v[q] = dv[q] < 0 ? 0.0 : (double)(coherent ? ld_fresh(contrib + su[q]) : __ldg(contrib + su[q]));
  }
  // in-lane runs: head run (may continue the previous lane), complete middle
  // runs (emitted here), tail run (joined across lanes by the scan)
  int head_d = dv[0];
  double head = 0.0, run = 0.0;
  int run_d = dv[0];
  bool has_head = false;
#pragma unroll
  for (int q = 0; q < kE; ++q) {
    if (dv[q] != run_d) {
      if (!has_head) {
        head = run;
        has_head = true;
      } else if (run_d >= 0) {
        atomicAdd(acc + run_d, run);
      }
      run = 0.0;
      run_d = dv[q];
    }
    run += v[q];
  }
  // segmented inclusive scan of tails (destinations nondecreasing in lane)
  int td = run_d;
  double tv = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_up_sync(0xffffffffu, tv, o);
    int dd = __shfl_up_sync(0xffffffffu, td, o);
    if (lane >= o && dd == td) tv += t;
  }
  const int prev_td = __shfl_up_sync(0xffffffffu, td, 1);
  const double prev_tv = __shfl_up_sync(0xffffffffu, tv, 1);
  const int next_head = __shfl_down_sync(0xffffffffu, head_d, 1);
  if (has_head && head_d >= 0) {
    double h = head;
    if (lane > 0 && prev_td == head_d) h += prev_tv;
    atomicAdd(acc + head_d, h);
  }
  // my tail is emitted by me unless the next lane continues it
  if (td >= 0 && (lane == 31 || next_head != td)) atomicAdd(acc + td, tv);
}

// Edge phase (EDGE_ONLY semantics, Alg. 2) over blocked edges [e0, e1) of one
// segment: warps stride over kE*32-edge steps; the next step's edges are
// loaded (registers) before the current step's gathers, so the DRAM latency
// of the edge stream overlaps the L2 latency of the gathers.
template <class CT, bool kSmem = false, bool kPrefetch = true, int kLoad = 0>
__device__ __forceinline__ void pr_edges_seg(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                             int64_t e0, int64_t e1, const CT* contrib, double* acc,
                                             int coherent, const CT* s_hot = nullptr, int32_t nhot = 0,
                                             int32_t cold_from = INT32_MAX) {
  const int lane = lane_id();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t start = e0 & ~int64_t(kE - 1);  // 32-byte aligned start
  const int64_t stride = nwarps * 32 * kE;
  int64_t base = start + warp * 32 * kE;
  if (base >= e1) return;
  int32_t su[kE], dv[kE];
  pr_load_edges(src, dst, base + lane * kE, e0, e1, su, dv);
  for (; base < e1; base += stride) {
    if (!kPrefetch) {
      if (base != start + warp * 32 * kE) pr_load_edges(src, dst, base + lane * kE, e0, e1, su, dv);
      pr_reduce_step<CT, kSmem, kLoad>(su, dv, contrib, acc, coherent, s_hot, nhot, cold_from);
      continue;
    }
    int32_t nsu[kE], ndv[kE];
    pr_load_edges(src, dst, base + stride + lane * kE, e0, e1, nsu, ndv);  // dead past e1
    pr_reduce_step<CT, kSmem, kLoad>(su, dv, contrib, acc, coherent, s_hot, nhot, cold_from);
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      su[q] = nsu[q];
      dv[q] = ndv[q];
    }
  }
}

// All cold segments in ONE launch (Alg. 2 without the barrier between
// segments): the segments' warp steps are concatenated in segment order and
// dealt to warps cyclically, so the grid sweeps segment 1, then 2, ...
// together (the L2 window moves as in the per-segment launches) while the
// warps that finish a segment early start the next one instead of idling at
// the launch boundary.  A step never straddles two segments, so the
// destination order inside a step -- the segmented scan's invariant -- holds.
constexpr int kMaxColdSegs = 48;
struct ColdSegs {
  int64_t a[kMaxColdSegs];  // 8-aligned first edge (steps start here)
  int64_t e0[kMaxColdSegs], e1[kMaxColdSegs];
  int64_t s0[kMaxColdSegs + 1];  // first global step of each segment; s0[n] = total
  int n;
};
__device__ __forceinline__ void cold_step(const ColdSegs& cs, int64_t s, int64_t& base, int64_t& e0, int64_t& e1) {
  int k = 0;
  while (k + 1 < cs.n && s >= cs.s0[k + 1]) ++k;
  base = cs.a[k] + (s - cs.s0[k]) * (32 * kE);
  e0 = cs.e0[k];
  e1 = cs.e1[k];
}
template <class CT>
static __global__ void __launch_bounds__(256) k_pr_edges_cold(const int32_t* __restrict__ src,
                                                            const int32_t* __restrict__ dst, const __grid_constant__ ColdSegs cs,
                                                            const CT* contrib, double* acc) {
  const int lane = lane_id();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total = cs.s0[cs.n];
  int64_t s = warp;
  if (s >= total) return;
  int64_t base, e0, e1;
  cold_step(cs, s, base, e0, e1);
  int32_t su[kE], dv[kE];
  pr_load_edges(src, dst, base + lane * kE, e0, e1, su, dv);
  for (; s < total; s += nwarps) {
    int32_t nsu[kE], ndv[kE];
    const int64_t sn = s + nwarps;
    if (sn < total) {
      int64_t nb, n0, n1;
      cold_step(cs, sn, nb, n0, n1);
      pr_load_edges(src, dst, nb + lane * kE, n0, n1, nsu, ndv);
    } else {
#pragma unroll
      for (int q = 0; q < kE; ++q) {
        nsu[q] = 0;
        ndv[q] = -1;
      }
    }
    pr_reduce_step<CT, false>(su, dv, contrib, acc, 0, nullptr, 0);
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      su[q] = nsu[q];
      dv[q] = ndv[q];
    }
  }
}

template <class CT, bool kPrefetch, int kMinBlocks = 1>
static __global__ void __launch_bounds__(256, kMinBlocks) k_pr_edges(const int32_t* src, const int32_t* dst,
                                                                     int64_t e0, int64_t e1, const CT* contrib,
                                                                     double* acc) {
  pr_edges_seg<CT, false, kPrefetch>(src, dst, e0, e1, contrib, acc, 0);
}

// Hot segment: the first `nhot` (highest out-degree) sources' contributions
// are staged once per CTA in shared memory; their gathers leave the L1TEX
// line pipeline and the L2 (the two bounds of this kernel, ~1 line/clk/SM)
// for the shared-memory banks.
template <class CT, int kThreads, int kMinBlocks, int kLoad = 0>
static __global__ void __launch_bounds__(kThreads, kMinBlocks) k_pr_edges_hot(const int32_t* src, const int32_t* dst,
                                                                             int64_t e0, int64_t e1, const CT* contrib,
                                                                             double* acc, int32_t nhot,
                                                                             int32_t cold_from = INT32_MAX) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  CT* s_hot = reinterpret_cast<CT*>(s_raw);
  const int n4 = (int)((int64_t)nhot * sizeof(CT) / 16);
  for (int i = threadIdx.x; i < n4; i += blockDim.x)
    reinterpret_cast<int4*>(s_raw)[i] = __ldg(reinterpret_cast<const int4*>(contrib) + i);
  for (int i = n4 * (16 / (int)sizeof(CT)) + threadIdx.x; i < nhot; i += blockDim.x) s_hot[i] = __ldg(contrib + i);
  __syncthreads();
  pr_edges_seg<CT, true, true, kLoad>(src, dst, e0, e1, contrib, acc, 0, s_hot, nhot, cold_from);
}

// Peer contribution buffers of a partitioned run with the fused all-gather:
// the vertex pass stores every owned next-contribution into each peer's
// buffer over NVLink (P2P stores into IPC-mapped memory), so no separate
// all-gather runs (prdist.cuh).  Same global indexing on every rank.
constexpr int kMaxPeers = 15;
template <class CT>
struct PeerSet {
  CT* p[kMaxPeers];
  int n;
};

// vertex pass: rank' = base + d*acc, L1, next dangling mass, next contrib, acc reset.
// 4 consecutive vertices per thread with 16-byte loads/stores (restrict ->
// all loads of a group are issued before any store).
template <class CT, bool kRank = true>
__device__ __forceinline__ void pr_vertex_one(int64_t v, const int32_t* __restrict__ outdeg,
                                              double* __restrict__ rank, CT* __restrict__ contrib_next,
                                              double* __restrict__ acc, double base, double damping,
                                              double& l1, double& dm, const PeerSet<CT>& peers) {
  const double nv = base + damping * acc[v];
  acc[v] = 0.0;
  if (kRank) {
    l1 += fabs(nv - rank[v]);
    rank[v] = nv;
  }
  const int32_t od = outdeg[v];
  if (od) {
    const CT c = (CT)(nv / (double)od);
    contrib_next[v] = c;
    for (int k = 0; k < peers.n; ++k) peers.p[k][v] = c;
  } else {
    dm += nv;
  }
}

// kRank = false (tolerance 0 and not the last iteration): the L1 only feeds
// the stop test, which tolerance 0 never passes, and the rank vector is only
// read back after the last iteration -- so rank is neither read nor written
// (16 of the 44 bytes per vertex); the contributions and the dangling mass
// come from the new value as always.
template <class CT, bool kRank = true>
__device__ __forceinline__ void pr_vertex_pass(int64_t V, const int32_t* __restrict__ outdeg,
                                               double* __restrict__ rank, CT* __restrict__ contrib_next,
                                               double* __restrict__ acc, double* scal, int64_t it,
                                               double damping, int64_t nglob, const PeerSet<CT>& peers) {
  const double n = (double)nglob;
  const double base = (1.0 - damping) / n + damping * scal[2 * it] / n;
  double l1 = 0, dm = 0;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t V4 = V & ~int64_t(3);
  for (int64_t v = tid * 4; v < V4; v += nth * 4) {
    const int4 od = __ldcs(reinterpret_cast<const int4*>(outdeg + v));
    const double2 a0 = __ldcs(reinterpret_cast<const double2*>(acc + v));
    const double2 a1 = __ldcs(reinterpret_cast<const double2*>(acc + v + 2));
    double2 r0 = make_double2(0.0, 0.0), r1 = r0;
    if (kRank) {
      r0 = __ldcs(reinterpret_cast<const double2*>(rank + v));
      r1 = __ldcs(reinterpret_cast<const double2*>(rank + v + 2));
    }
    const double nv[4] = {base + damping * a0.x, base + damping * a0.y, base + damping * a1.x,
                          base + damping * a1.y};
    const double rv[4] = {r0.x, r0.y, r1.x, r1.y};
    const int dg[4] = {od.x, od.y, od.z, od.w};
    CT c[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (kRank) l1 += fabs(nv[q] - rv[q]);
      if (dg[q]) c[q] = (CT)(nv[q] / (double)dg[q]);
      else { c[q] = (CT)0; dm += nv[q]; }
    }
    __stcs(reinterpret_cast<double2*>(acc + v), make_double2(0.0, 0.0));
    __stcs(reinterpret_cast<double2*>(acc + v + 2), make_double2(0.0, 0.0));
    if (kRank) {
      __stcs(reinterpret_cast<double2*>(rank + v), make_double2(nv[0], nv[1]));
      __stcs(reinterpret_cast<double2*>(rank + v + 2), make_double2(nv[2], nv[3]));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (dg[q]) contrib_next[v + q] = c[q];  // dangling entries are never gathered
    for (int k = 0; k < peers.n; ++k) {      // fused all-gather: one vector store per peer
      if (sizeof(CT) == 8) {
        double2* d = reinterpret_cast<double2*>(peers.p[k] + v);
        d[0] = make_double2((double)c[0], (double)c[1]);
        d[1] = make_double2((double)c[2], (double)c[3]);
      } else {
        *reinterpret_cast<float4*>(peers.p[k] + v) =
            make_float4((float)c[0], (float)c[1], (float)c[2], (float)c[3]);
      }
    }
  }
  for (int64_t v = V4 + tid; v < V; v += nth)
    pr_vertex_one<CT, kRank>(v, outdeg, rank, contrib_next, acc, base, damping, l1, dm, peers);
  if (peers.n) __threadfence_system();  // peer stores visible before the exchange's barrier
  l1 = block_sum(l1);
  dm = block_sum(dm);
  if (threadIdx.x == 0) {
    if (l1 != 0.0) atomicAdd(scal + 2 * it + 1, l1);
    if (dm != 0.0) atomicAdd(scal + 2 * (it + 1), dm);
  }
}

template <class CT, bool kRank = true>
static __global__ void __launch_bounds__(256) k_pr_vertex(int64_t V, int64_t nglob, PeerSet<CT> peers,
                                                          const int32_t* outdeg, double* rank,
                                                          CT* contrib_next, double* acc, double* scal,
                                                          int64_t it, double damping) {
  pr_vertex_pass<CT, kRank>(V, outdeg, rank, contrib_next, acc, scal, it, damping, nglob, peers);
}

// Whole loop in one cooperative launch (kernel fusion on "s0").
template <class CT>
static __global__ void __launch_bounds__(256) k_prb_fused(const int32_t* src, const int32_t* dst,
                                                          const int64_t* seg_edge, int64_t K, int64_t V,
                                                          const int32_t* outdeg, double* rank, CT* c0, CT* c1,
                                                          double* acc, double* scal, int64_t max_iters,
                                                          double tol, double damping, int64_t* iters_out) {
  cg::grid_group grid = cg::this_grid();
  int64_t it = 0;
  double l1 = INFINITY;
  while (!(it >= max_iters || l1 < tol)) {
    const CT* cur = (it & 1) ? c1 : c0;
    CT* nxt = (it & 1) ? c0 : c1;
    for (int64_t k = 1; k <= K; ++k) {  // cold segments, then the hot one
      const int64_t s = k == K ? 0 : k;
      pr_edges_seg<CT>(src, dst, seg_edge[s], seg_edge[s + 1], cur, acc, 1);
      grid.sync();
    }
    PeerSet<CT> none;
    none.n = 0;
    pr_vertex_pass<CT>(V, outdeg, rank, nxt, acc, scal, it, damping, V, none);
    grid.sync();
    l1 = *((volatile double*)scal + 2 * it + 1);
    ++it;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *iters_out = it;
}

// ---------------------------------------------------------------------------
// Host side.  One PrRank is one destination partition's state; a single-GPU
// run is one PrRank with no exchange, a multi-GPU run one PrRank per process
// with an NCCL exchange (dist.cu), and the virtual-rank test mode P PrRanks
// on one device with a copy exchange.
// ---------------------------------------------------------------------------
struct HotCfg {
  int32_t nhot = 0;
  int per_sm = 1;
  bool prefetch = true;
  int gather = 0;
  int32_t cold_from = INT32_MAX;  // one-segment layout: first source past the L2 window
  int cold_minb = 0;              // cold-segment kernel register cap (GG_PR_COLD_MINB)
  bool cold_one = false;          // all cold segments in one launch (GG_PR_COLD_ONE)
  unsigned grid = 0, hot_grid = 0;
};

template <class CT>
static HotCfg hot_cfg(int dev, const PrBlockLayout* L) {
  // shared-memory hot-source cache for the hot segment: the top `nhot`
  // sources (as many as fit next to the CTA).  GG_PR_HOT=0 disables it,
  // GG_PR_HOT_THREADS picks 1024x1 (default) or 512x2 CTAs per SM,
  // GG_PR_NHOT caps the cached count, GG_PR_PREFETCH=0 drops the register
  // prefetch of the next edge step.
  HotCfg h;
  int smem_max = 0;
  GG_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const char* hot_env = getenv("GG_PR_HOT");
  const bool hot_on = !(hot_env && atoi(hot_env) == 0);
  const char* thr_env = getenv("GG_PR_HOT_THREADS");
  h.per_sm = thr_env && atoi(thr_env) == 512 ? 2 : 1;
  // at most 128 KB per SM: the rest of the 256 KB L1/shared array stays L1,
  // which stages the in-flight gather lines (measured: 227 KB of cache halves
  // the kernel's gather rate; 128 KB gives the best time at f32 and f64)
  int cap_kb = 128;
  if (const char* e = getenv("GG_PR_HOT_KB")) cap_kb = std::max(4, atoi(e));
  int smem_per_cta = std::min(smem_max - 2048, cap_kb * 1024) / h.per_sm;
  int64_t nhot64 = std::min<int64_t>(smem_per_cta / (int)sizeof(CT), L->ns);
  if (const char* nh = getenv("GG_PR_NHOT")) nhot64 = std::min<int64_t>(nhot64, atoll(nh));
  nhot64 &= ~int64_t(3);
  h.nhot = hot_on && nhot64 >= 1024 ? (int32_t)nhot64 : 0;
  if (h.nhot) {
    const void* fn = h.per_sm == 2 ? (const void*)k_pr_edges_hot<CT, 512, 2> : (const void*)k_pr_edges_hot<CT, 1024, 1>;
    GG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, h.nhot * (int)sizeof(CT)));
  }
  const char* pf_env = getenv("GG_PR_PREFETCH");
  h.prefetch = !(pf_env && atoi(pf_env) == 0);
  if (const char* ge = getenv("GG_PR_GATHER")) h.gather = std::max(0, std::min(2, atoi(ge)));
  if (L->K == 1 && L->V > 1) {  // one segment: evict-first gathers past the L2-sized window
    const int64_t w = l2_bytes(dev) * 6 / 16 / (int64_t)sizeof(CT);
    if (w < L->V) {
      h.cold_from = (int32_t)w;
      h.gather = 3;
      if (h.nhot && h.per_sm == 1)
        GG_CUDA(cudaFuncSetAttribute((const void*)k_pr_edges_hot<CT, 1024, 1, 3>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, h.nhot * (int)sizeof(CT)));
    }
  }
  if (h.nhot && h.per_sm == 1 && h.gather) {
    const void* fn = h.gather == 1 ? (const void*)k_pr_edges_hot<CT, 1024, 1, 1> : (const void*)k_pr_edges_hot<CT, 1024, 1, 2>;
    GG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, h.nhot * (int)sizeof(CT)));
  }
  // cold segments: GG_PR_COLD_MINB = 4 / 5 / 6 / 8 caps registers for that
  // many resident CTAs per SM (0: the compiler's choice); the grid
  // is GG_PR_COLD_GRID CTAs per SM (default 8)
  // default 4: caps the prefetching kernel at 63 registers (no spill) so 4
  // CTAs fit per SM instead of 3 at 75 registers (cold phase -6%, measured)
  h.cold_minb = 4;
  if (const char* e = getenv("GG_PR_COLD_MINB")) h.cold_minb = atoi(e);
  if (const char* e = getenv("GG_PR_COLD_ONE")) h.cold_one = atoi(e) != 0;
  int per = 8;
  if (const char* e = getenv("GG_PR_COLD_GRID")) per = std::max(1, atoi(e));
  h.grid = (unsigned)sm_count(dev) * per;
  h.hot_grid = (unsigned)sm_count(dev) * h.per_sm;
  return h;
}

template <class CT>
struct PrRank {
  PrBlockLayout* L = nullptr;
  HotCfg hc;
  int dev = 0;
  int64_t V = 0;
  double *rank = nullptr, *acc = nullptr, *scal = nullptr, *outv = nullptr;
  CT *c0 = nullptr, *c1 = nullptr;
  int launches = 0;

  // buffers: the layout's cached work buffers (rank/contrib full V, acc Vloc)
  void bind(PrBlockLayout* lay, int device, int64_t iters_cap) {
    L = lay;
    dev = device;
    V = L->V;
    if (L->w_rank.n < (size_t)V) {
      L->w_rank.alloc(V);
      L->w_out.alloc(V);
      L->w_c0.alloc(V * sizeof(CT));
      L->w_c1.alloc(V * sizeof(CT));
    }
    if (L->w_acc.n < (size_t)std::max<int64_t>(L->vloc(), 1)) L->w_acc.alloc(std::max<int64_t>(L->vloc(), 1));
    if (L->w_scal.n < (size_t)(2 * (iters_cap + 2))) L->w_scal.alloc(2 * (iters_cap + 2));
    rank = L->w_rank.p;
    acc = L->w_acc.p;
    scal = L->w_scal.p;
    outv = L->w_out.p;
    c0 = reinterpret_cast<CT*>(L->w_c0.p);
    c1 = reinterpret_cast<CT*>(L->w_c1.p);
    hc = hot_cfg<CT>(dev, L);
  }
  // rank_0 = 1/n, contrib_0, dangling mass_0 over ALL vertices (identical on
  // every rank, so no exchange precedes the first iteration)
  void init(int64_t iters_cap, cudaStream_t st, const double* init_ranks = nullptr) {
    GG_CUDA(cudaMemsetAsync(scal, 0, 2 * (iters_cap + 2) * sizeof(double), st));
    GG_CUDA(cudaMemsetAsync(acc, 0, std::max<int64_t>(L->vloc(), 1) * sizeof(double), st));
    k_prb_init<CT><<<grid_for(V, 256, dev), 256, 0, st>>>(L->outdeg.p, V, rank, c0, scal, init_ranks, L->order.p);
    GG_LAUNCH_CHECK();
    ++launches;
  }
  CT* cur(int64_t it) const { return (it & 1) ? c1 : c0; }
  CT* nxt(int64_t it) const { return (it & 1) ? c0 : c1; }
  // Alg. 2: segments in order, cold first, the hot one last
  Runtime* rt_top = nullptr;  // records the hot-segment launches (dominant kernel)
  // which: 0 = every segment (cold ones first, the hot one last),
  //        1 = only the hot segment, 2 = only the cold segments
  void edges(int64_t it, cudaStream_t st, int which = 0) {
    NvtxRange nvtx("gg.pr_block.edge_phase");
    const CT* c = cur(it);
    bool cold_done = false;
    if (hc.cold_one && which != 1 && hc.prefetch) {
      ColdSegs cs;
      cs.n = 0;
      int64_t steps = 0;
      for (int64_t k = 1; k < L->K && cs.n < kMaxColdSegs; ++k) {
        const int64_t e0 = L->seg_edge[k], e1 = L->seg_edge[k + 1];
        if (e1 <= e0) continue;
        const int64_t a = e0 & ~int64_t(kE - 1);
        cs.a[cs.n] = a;
        cs.e0[cs.n] = e0;
        cs.e1[cs.n] = e1;
        cs.s0[cs.n] = steps;
        steps += (e1 - a + 32 * kE - 1) / (32 * kE);
        ++cs.n;
      }
      cs.s0[cs.n] = steps;
      if (L->K - 1 <= kMaxColdSegs) {
        cold_done = true;
        if (cs.n > 0) {
          k_pr_edges_cold<CT><<<hc.grid, 256, 0, st>>>(L->src.p, L->dst.p, cs, c, acc);
          ++launches;
        }
      }
    }
    for (int64_t k = 1; k <= L->K; ++k) {
      const int64_t sg = k == L->K ? 0 : k;
      if ((which == 1 && sg != 0) || (which == 2 && sg == 0)) continue;
      if (cold_done && sg != 0) continue;
      const int64_t e0 = L->seg_edge[sg], e1 = L->seg_edge[sg + 1];
      if (e1 <= e0) continue;
      cudaEvent_t ta = nullptr, tb = nullptr;
      if (sg == 0 && rt_top) {
        GG_CUDA(cudaEventCreate(&ta));
        GG_CUDA(cudaEventCreate(&tb));
        GG_CUDA(cudaEventRecord(ta, st));
        rt_top->top_edges = e1 - e0;
      }
      if (sg == 0 && hc.nhot > 0 && hc.per_sm == 2)
        k_pr_edges_hot<CT, 512, 2><<<hc.hot_grid, 512, hc.nhot * sizeof(CT), st>>>(L->src.p, L->dst.p, e0, e1, c,
                                                                                  acc, hc.nhot);
      else if (sg == 0 && hc.nhot > 0 && hc.gather == 1)
        k_pr_edges_hot<CT, 1024, 1, 1><<<hc.hot_grid, 1024, hc.nhot * sizeof(CT), st>>>(L->src.p, L->dst.p, e0,
                                                                                       e1, c, acc, hc.nhot);
      else if (sg == 0 && hc.nhot > 0 && hc.gather == 3)
        k_pr_edges_hot<CT, 1024, 1, 3><<<hc.hot_grid, 1024, hc.nhot * sizeof(CT), st>>>(L->src.p, L->dst.p, e0,
                                                                                       e1, c, acc, hc.nhot,
                                                                                       hc.cold_from);
      else if (sg == 0 && hc.nhot > 0 && hc.gather == 2)
        k_pr_edges_hot<CT, 1024, 1, 2><<<hc.hot_grid, 1024, hc.nhot * sizeof(CT), st>>>(L->src.p, L->dst.p, e0,
                                                                                       e1, c, acc, hc.nhot);
      else if (sg == 0 && hc.nhot > 0)
        k_pr_edges_hot<CT, 1024, 1><<<hc.hot_grid, 1024, hc.nhot * sizeof(CT), st>>>(L->src.p, L->dst.p, e0, e1,
                                                                                    c, acc, hc.nhot);
      else if (hc.prefetch)
      {
        if (hc.cold_minb == 4)
          k_pr_edges<CT, true, 4><<<hc.grid, 256, 0, st>>>(L->src.p, L->dst.p, e0, e1, c, acc);
        else if (hc.cold_minb == 5)
          k_pr_edges<CT, true, 5><<<hc.grid, 256, 0, st>>>(L->src.p, L->dst.p, e0, e1, c, acc);
        else if (hc.cold_minb == 6)
          k_pr_edges<CT, true, 6><<<hc.grid, 256, 0, st>>>(L->src.p, L->dst.p, e0, e1, c, acc);
        else if (hc.cold_minb == 8)
          k_pr_edges<CT, true, 8><<<hc.grid, 256, 0, st>>>(L->src.p, L->dst.p, e0, e1, c, acc);
        else
          k_pr_edges<CT, true><<<hc.grid, 256, 0, st>>>(L->src.p, L->dst.p, e0, e1, c, acc);
      }
      else
        k_pr_edges<CT, false><<<hc.grid, 256, 0, st>>>(L->src.p, L->dst.p, e0, e1, c, acc);
      if (ta) {
        GG_CUDA(cudaEventRecord(tb, st));
        rt_top->top_record(ta, tb);
      }
      ++launches;
    }
    GG_LAUNCH_CHECK();
  }
  // owned destinations [lo, hi): rank', L1 partial, next dangling partial,
  // next contrib slice, acc reset
  // fused all-gather: the peers' contribution buffers (same parity layout)
  std::vector<CT*> peer_c0, peer_c1;
  // track_rank: the L1 / rank vector are needed (tolerance > 0, or the last
  // iteration); see pr_vertex_pass
  void vertex(int64_t it, double damping, cudaStream_t st, bool track_rank = true) {
    NvtxRange nvtx("gg.pr_block.vertex_pass");
    const int64_t lo = L->lo, n = L->vloc();
    PeerSet<CT> ps;
    ps.n = (int)peer_c0.size();
    for (int k = 0; k < ps.n; ++k) ps.p[k] = ((it & 1) ? peer_c0[k] : peer_c1[k]) + lo;
    if (n > 0 && track_rank)
      k_pr_vertex<CT, true><<<grid_for(n, 256, dev), 256, 0, st>>>(n, V, ps, L->outdeg.p + lo, rank + lo,
                                                                   nxt(it) + lo, acc, scal, it, damping);
    else if (n > 0)
      k_pr_vertex<CT, false><<<grid_for(n, 256, dev), 256, 0, st>>>(n, V, ps, L->outdeg.p + lo, rank + lo,
                                                                    nxt(it) + lo, acc, scal, it, damping);
    GG_LAUNCH_CHECK();
    ++launches;
  }
  void unpermute(double* ranks_out, cudaStream_t st) {
    k_unpermute<<<grid_for(V, 256, dev), 256, 0, st>>>(rank, L->newid.p, V, outv);
    GG_LAUNCH_CHECK();
    ++launches;
    GG_CUDA(cudaMemcpyAsync(ranks_out, outv, V * 8, cudaMemcpyDefault, st));
  }
};

template <class CT>
int64_t pagerank_blocked(const Graph& g, const gg_schedule& s, bool fusion, int64_t max_iters,
                         double tol, double damping, double* ranks_out, Runtime& rt, const double* init) {
  const int dev = g.dev;
  const int64_t V = g.V;
  cudaStream_t st = rt.stream;
  std::shared_ptr<PrBlockLayout> Lp =
      layout_for(g, pr_block_window(g, sizeof(CT), s.blocking_size), sizeof(CT));
  PrBlockLayout* L = Lp.get();
  const int64_t iters_cap = max_iters > 0 ? max_iters : 0;
  std::lock_guard<std::mutex> wlk(L->w_mu);
  PrRank<CT> R;
  R.bind(L, dev, iters_cap);
  R.rt_top = &rt;
  R.init(iters_cap, st, init);
  int64_t it = 0;
  if (!fusion) {
    double l1 = INFINITY;
    while (!(it >= max_iters || l1 < tol)) {
      rt.edge_begin();
      R.edges(it, st);
      rt.edge_end();
      R.vertex(it, damping, st, tol > 0.0 || it + 1 >= max_iters);
      rt.stats.dispatch_count += 1;
      rt.stats.direction_log.push_back(s.direction);
      ++it;
      if (tol > 0.0) {
        GG_CUDA(cudaMemcpyAsync(&l1, R.scal + 2 * (it - 1) + 1, 8, cudaMemcpyDeviceToHost, st));
        GG_CUDA(cudaStreamSynchronize(st));
      }
    }
  } else {
    DevBuf<int64_t> iters(1), segs(L->K + 1);
    GG_CUDA(cudaMemcpyAsync(segs.p, L->seg_edge.data(), (L->K + 1) * 8, cudaMemcpyHostToDevice, st));
    // small graphs: 2 CTAs per SM -- a grid barrier per segment and per vertex
    // pass dominates (C1 RMAT-16: 73 / 73 / 80 / 77 GTEPS at 8 / 4 / 2 / 1 per
    // SM); large ones keep every resident CTA for the edge stream
    int blocks = max_coop_blocks((const void*)k_prb_fused<CT>, 256, dev, 0, g.E < (int64_t(1) << 26) ? 2 : 0);
    const int32_t* sp = L->src.p;
    const int32_t* dp = L->dst.p;
    const int64_t* se = segs.p;
    int64_t K = L->K;
    int64_t Vv = V;
    const int32_t* od = L->outdeg.p;
    double* rk = R.rank;
    CT* p0 = R.c0;
    CT* p1 = R.c1;
    double* ac = R.acc;
    double* sc = R.scal;
    int64_t* ip = iters.p;
    void* args[] = {&sp, &dp, &se, &K, &Vv, &od, &rk, &p0, &p1, &ac, &sc, &max_iters, &tol, &damping, &ip};
    rt.edge_begin();
    GG_CUDA(cudaLaunchCooperativeKernel((const void*)k_prb_fused<CT>, blocks, 256, args, 0, st));
    rt.edge_end();
    ++R.launches;
    it = dget(iters.p);
    rt.stats.dispatch_count += 1;
    for (int64_t k = 0; k < it; ++k) rt.stats.direction_log.push_back(s.direction);
  }
  rt.stats.rounds += it;
  rt.stats.edges_traversed += it * g.E;
  R.unpermute(ranks_out, st);
  GG_CUDA(cudaStreamSynchronize(st));
  count_launch(R.launches);
  return it;
}

template int64_t pagerank_blocked<double>(const Graph&, const gg_schedule&, bool, int64_t, double,
                                          double, double*, Runtime&, const double*);
template int64_t pagerank_blocked<float>(const Graph&, const gg_schedule&, bool, int64_t, double,
                                         double, double*, Runtime&, const double*);

// ---------------------------------------------------------------------------
// Partitioned (multi-rank) run.  Per iteration: local edge phase over the
// owned destinations' in-edges, vertex pass over the owned slice, then the
// exchange: all-reduce of (L1 this iteration, dangling mass next iteration)
// -- adjacent doubles -- and all-gather of the owned next-contrib slices.
// ---------------------------------------------------------------------------
template <class CT>
int64_t pagerank_blocked_ranks(std::vector<PrRank<CT>*>& ranks, PrExchange& ex, int64_t max_iters, double tol,
                               double damping, int32_t direction_log, cudaStream_t st, Runtime& rt) {
  const PrBlockLayout* L0 = ranks[0]->L;
  int64_t it = 0;
  double l1 = INFINITY;
  std::vector<double*> sc(ranks.size());
  std::vector<void*> nx(ranks.size());
  // fused all-gather through peer memory when the exchange offers it
  std::vector<void*> c0s, c1s;
  for (auto* R : ranks) {
    c0s.push_back(R->c0);
    c1s.push_back(R->c1);
  }
  std::vector<std::vector<void*>> pc0, pc1;
  const bool p2p = ex.map_peers(c0s, c1s, (size_t)L0->V * sizeof(CT), pc0, pc1);
  if (p2p)
    for (size_t i = 0; i < ranks.size(); ++i) {
      if (pc0[i].size() > (size_t)kMaxPeers) fail(GG_ERR_VALUE, "too many peers for the fused all-gather");
      for (void* q : pc0[i]) ranks[i]->peer_c0.push_back(static_cast<CT*>(q));
      for (void* q : pc1[i]) ranks[i]->peer_c1.push_back(static_cast<CT*>(q));
    }
  // Without the fused all-gather the exchange overlaps the next iteration's
  // hot kernel: the hot window [0, ns) of every slice is gathered first (it
  // is small and all the hot kernel reads), the rest asynchronously; the
  // cold segments wait for it.  Hot first, cold after: acc sums commute.
  const bool split = !p2p && L0->P > 1;
  while (!(it >= max_iters || l1 < tol)) {
    rt.edge_begin();
    if (split) {
      for (auto* R : ranks) R->edges(it, st, 1);
      ex.wait_rest(st);
      for (auto* R : ranks) R->edges(it, st, 2);
    } else {
      for (auto* R : ranks) R->edges(it, st);
    }
    rt.edge_end();
    for (size_t i = 0; i < ranks.size(); ++i) {
      ranks[i]->vertex(it, damping, st, tol > 0.0 || it + 1 >= max_iters);
      sc[i] = ranks[i]->scal + 2 * it + 1;
      nx[i] = ranks[i]->nxt(it);
    }
    ex.allreduce2(sc, st);  // also the barrier after which peer stores are visible
    if (split)
      ex.allgather_split(nx, sizeof(CT), L0->bounds, L0->ns, st);
    else if (!p2p)
      ex.allgather(nx, sizeof(CT), L0->bounds, st);
    rt.stats.dispatch_count += 1;
    rt.stats.direction_log.push_back(direction_log);
    ++it;
    if (tol > 0.0) {
      GG_CUDA(cudaMemcpyAsync(&l1, ranks[0]->scal + 2 * (it - 1) + 1, 8, cudaMemcpyDeviceToHost, st));
      GG_CUDA(cudaStreamSynchronize(st));
    }
  }
  if (p2p) {
    GG_CUDA(cudaStreamSynchronize(st));
    for (auto* R : ranks) {
      R->peer_c0.clear();
      R->peer_c1.clear();
    }
    ex.unmap_peers();
  }
  if (split) ex.wait_rest(st);  // the last iteration's contributions: nobody reads them
  // every rank's owned rank slice to all ranks
  std::vector<void*> rk(ranks.size());
  for (size_t i = 0; i < ranks.size(); ++i) rk[i] = ranks[i]->rank;
  ex.allgather(rk, sizeof(double), L0->bounds, st);
  rt.stats.rounds += it;
  return it;
}

// Virtual ranks on one device (test mode for the multi-GPU path): P
// partitions, each with its own layout and buffers; the exchange copies.
struct CopyExchange : PrExchange {
  bool p2p = false;  // the vertex passes store into the other virtual ranks' buffers
  bool map_peers(const std::vector<void*>& c0s, const std::vector<void*>& c1s, size_t,
                 std::vector<std::vector<void*>>& pc0, std::vector<std::vector<void*>>& pc1) override {
    if (!p2p) return false;
    pc0.assign(c0s.size(), {});
    pc1.assign(c1s.size(), {});
    for (size_t i = 0; i < c0s.size(); ++i)
      for (size_t q = 0; q < c0s.size(); ++q)
        if (q != i) {
          pc0[i].push_back(c0s[q]);
          pc1[i].push_back(c1s[q]);
        }
    return true;
  }
  void allreduce2(std::vector<double*>& d, cudaStream_t st) override {
    std::vector<double> h(2 * d.size());
    for (size_t i = 0; i < d.size(); ++i)
      GG_CUDA(cudaMemcpyAsync(&h[2 * i], d[i], 16, cudaMemcpyDeviceToHost, st));
    GG_CUDA(cudaStreamSynchronize(st));
    double s[2] = {0, 0};
    for (size_t i = 0; i < d.size(); ++i) {  // rank order, as a ring reduce would
      s[0] += h[2 * i];
      s[1] += h[2 * i + 1];
    }
    for (size_t i = 0; i < d.size(); ++i) GG_CUDA(cudaMemcpyAsync(d[i], s, 16, cudaMemcpyHostToDevice, st));
    GG_CUDA(cudaStreamSynchronize(st));
  }
  void allgather(std::vector<void*>& bufs, size_t elt, const std::vector<int64_t>& bounds,
                 cudaStream_t st) override {
    for (size_t r = 0; r < bufs.size(); ++r) {
      const size_t off = (size_t)bounds[r] * elt, len = (size_t)(bounds[r + 1] - bounds[r]) * elt;
      for (size_t q = 0; q < bufs.size(); ++q)
        if (q != r && len)
          GG_CUDA(cudaMemcpyAsync((char*)bufs[q] + off, (char*)bufs[r] + off, len, cudaMemcpyDeviceToDevice, st));
    }
  }
};

template <class CT>
int64_t pagerank_blocked_virtual(const Graph& g, const gg_schedule& s, int nparts, int64_t max_iters, double tol,
                                 double damping, double* ranks_out, Runtime& rt, bool fused_allgather) {
  if (nparts < 1) fail(GG_ERR_VALUE, "nparts must be >= 1");
  const int64_t ns = pr_block_window(g, sizeof(CT), s.blocking_size);
  const int64_t iters_cap = max_iters > 0 ? max_iters : 0;
  std::vector<std::shared_ptr<PrBlockLayout>> lays;
  std::vector<PrRank<CT>> rs(nparts);
  std::vector<PrRank<CT>*> rp;
  int64_t local_edges = 0;
  for (int r = 0; r < nparts; ++r) {
    lays.push_back(build_layout(g, ns, sizeof(CT), PrPart{nparts, r}));
    rs[r].bind(lays.back().get(), g.dev, iters_cap);
    rs[r].init(iters_cap, rt.stream);
    rp.push_back(&rs[r]);
    local_edges += lays.back()->E;
  }
  if (local_edges != g.E) fail(GG_ERR_ENGINE, "partition lost edges");
  CopyExchange ex;
  ex.p2p = fused_allgather;
  int64_t it = pagerank_blocked_ranks<CT>(rp, ex, max_iters, tol, damping, s.direction, rt.stream, rt);
  rt.stats.edges_traversed += it * g.E;
  rs[0].unpermute(ranks_out, rt.stream);
  GG_CUDA(cudaStreamSynchronize(rt.stream));
  int launches = 0;
  for (auto& R : rs) launches += R.launches;
  count_launch(launches);
  return it;
}
template int64_t pagerank_blocked_virtual<double>(const Graph&, const gg_schedule&, int, int64_t, double, double,
                                                  double*, Runtime&, bool);
template int64_t pagerank_blocked_virtual<float>(const Graph&, const gg_schedule&, int, int64_t, double, double,
                                                 double*, Runtime&, bool);

// One rank of a multi-process run (dist.cu supplies the NCCL exchange).
template <class CT>
int64_t pagerank_blocked_rank(const Graph& g, const gg_schedule& s, int P, int r, PrExchange& ex,
                              int64_t max_iters, double tol, double damping, double* ranks_out, Runtime& rt,
                              int64_t* local_edges) {
  const int64_t ns = pr_block_window(g, sizeof(CT), s.blocking_size);
  std::shared_ptr<PrBlockLayout> Lp = layout_for(g, ns, sizeof(CT), PrPart{P, r});
  PrBlockLayout* L = Lp.get();
  const int64_t iters_cap = max_iters > 0 ? max_iters : 0;
  std::lock_guard<std::mutex> wlk(L->w_mu);
  PrRank<CT> R;
  R.bind(L, g.dev, iters_cap);
  R.rt_top = &rt;
  R.init(iters_cap, rt.stream);
  std::vector<PrRank<CT>*> rp{&R};
  int64_t it = pagerank_blocked_ranks<CT>(rp, ex, max_iters, tol, damping, s.direction, rt.stream, rt);
  rt.stats.edges_traversed += it * L->E;
  if (local_edges) *local_edges = L->E;
  R.unpermute(ranks_out, rt.stream);
  GG_CUDA(cudaStreamSynchronize(rt.stream));
  count_launch(R.launches);
  return it;
}
template int64_t pagerank_blocked_rank<double>(const Graph&, const gg_schedule&, int, int, PrExchange&, int64_t,
                                               double, double, double*, Runtime&, int64_t*);
template int64_t pagerank_blocked_rank<float>(const Graph&, const gg_schedule&, int, int, PrExchange&, int64_t,
                                              double, double, double*, Runtime&, int64_t*);

double pr_block_prep_part_ms(const Graph& g, int64_t blocking_size, int ct_bytes, int P, int r,
                             int64_t* bounds, int32_t* newid) {
  std::shared_ptr<PrBlockLayout> L =
      layout_for(g, pr_block_window(g, ct_bytes, blocking_size), ct_bytes, PrPart{P, r});
  if (bounds) memcpy(bounds, L->bounds.data(), (P + 1) * sizeof(int64_t));
  if (newid) GG_CUDA(cudaMemcpy(newid, L->newid.p, L->V * sizeof(int32_t), cudaMemcpyDefault));
  return L->prep_ms;
}

}  // namespace gg
