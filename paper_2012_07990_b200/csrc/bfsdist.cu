// bfsdist.cu — direction-optimizing BFS 1-D vertex-partitioned over ranks
// with bitmap frontier exchange (reference algos.bfs,
// algos.py:101-135, driven by engine.hybrid_apply, engine.py:622-636).
//
// Rank r owns vertices [lo_r, hi_r) (32-aligned so bitmap words never
// straddle owners; balanced by out-degree).  Every rank holds the whole graph
// (CSR-out and CSR-in), a replicated visited bitmap and a replicated frontier
// bitmap.  Per level, with the same hybrid rule as the single-GPU path
// (PULL iff |frontier| > threshold * V, engine.py:632):
//   top-down:  each rank expands the frontier vertices it owns over their
//              out-arcs and sets the bits of unvisited targets in a V-bit
//              discovered bitmap; the exchange is an all-to-all of bitmap
//              slices OR-ed at their owners (V/8 bytes per rank, not the
//              4*V-byte parent-candidate all-reduce of the first version);
//              each owner then gives its newly discovered vertices a parent
//              from the replicated frontier bitmap (first in-arc from the
//              frontier: a legal BFS parent) and all-gathers its owned words
//              of the next frontier;
//   bottom-up: each rank scans the in-arcs of its owned unvisited vertices
//              against the replicated frontier bitmap (first hit wins, which
//              is the reference's pull semantics: later arcs are no-ops once
//              parent[v] != -1, algos.py:121-125) and sets its owned words of
//              the next bitmap; the exchange is an all-gather of those words.
// The frontier size for the direction choice is a popcount of the replicated
// bitmap, so no extra collective is needed.  Depths equal the single-GPU BFS
// (level-synchronous); parents are a legal BFS tree.
#include "engine.cuh"
#include "prdist.cuh"

namespace gg {

__global__ void k_bfsd_init(int32_t* parent, int64_t V, uint32_t* vis, uint32_t* fr, uint32_t* nx, int64_t W,
                            int32_t source) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V; i += (int64_t)gridDim.x * blockDim.x)
    parent[i] = i == source ? source : -1;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W; w += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t b = (w == (source >> 5)) ? (1u << (source & 31)) : 0u;
    vis[w] = b;
    fr[w] = b;
    nx[w] = 0;
  }
}

__device__ __forceinline__ bool bit_of(const uint32_t* bm, int64_t v) { return (bm[v >> 5] >> (v & 31)) & 1u; }

// owned frontier vertices -> queue (word-parallel, warp-aggregated append)
__global__ void k_bfsd_queue(const uint32_t* fr, int64_t w0, int64_t w1, int32_t* q, unsigned long long* qn) {
  for (int64_t w = w0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < w1; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = fr[w];
    if (!x) continue;
    unsigned long long at = atomicAdd(qn, (unsigned long long)__popc(x));
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      q[at++] = (int32_t)(w * 32 + b);
    }
  }
}

// top-down, bitmap form: warp per queued vertex, unvisited targets set their
// bit in this rank's discovered bitmap
__global__ void __launch_bounds__(256) k_bfsd_push_bm(const int64_t* off, const int32_t* nbr, const int32_t* q,
                                                      const unsigned long long* qn, const uint32_t* vis,
                                                      uint32_t* disc, unsigned long long* scanned) {
  const int64_t n = (int64_t)*qn;
  const int lane = lane_id();
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long cnt = 0;
  for (int64_t i = warp; i < n; i += nw) {
    const int32_t u = q[i];
    const int64_t e0 = off[u], e1 = off[u + 1];
    cnt += e1 - e0;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int32_t v = __ldg(nbr + e);
      const uint32_t m = 1u << (v & 31);
      if (!(vis[v >> 5] & m) && !(*((volatile uint32_t*)disc + (v >> 5)) & m)) atomicOr(disc + (v >> 5), m);
    }
  }
  if (lane == 0 && cnt) atomicAdd(scanned, cnt);
}

// owner commit of a top-down level: the OR-ed discovered words of [w0, w1)
// minus the visited ones are the next frontier; each new vertex takes its
// first in-arc from the (replicated) frontier as parent
__global__ void __launch_bounds__(256) k_bfsd_td_commit(const int64_t* in_off, const int32_t* in_nbr, int64_t w0,
                                                        int64_t w1, const uint32_t* disc, const uint32_t* vis,
                                                        const uint32_t* fr, int32_t* parent, uint32_t* nx) {
  const int lane = lane_id();
  for (int64_t w = w0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); w < w1;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint32_t fresh = disc[w] & ~vis[w];
    if ((fresh >> lane) & 1u) {
      const int64_t v = w * 32 + lane;
      for (int64_t e = in_off[v], e1 = in_off[v + 1]; e < e1; ++e) {
        const int32_t u = __ldg(in_nbr + e);
        if (bit_of(fr, u)) {
          parent[v] = u;
          break;
        }
      }
    }
    if (lane == 0) nx[w] = fresh;
  }
}

__global__ void k_or_into(uint32_t* dst, const uint32_t* src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] |= src[i];
}

// bottom-up: thread per owned vertex; first in-arc from the frontier wins
__global__ void __launch_bounds__(256) k_bfsd_pull(const int64_t* off, const int32_t* nbr, int64_t lo, int64_t hi,
                                                   const uint32_t* vis, const uint32_t* fr, int32_t* parent,
                                                   uint32_t* nx, unsigned long long* scanned) {
  const int lane = lane_id();
  unsigned long long cnt = 0;
  for (int64_t base = lo + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~int64_t(31)); base < hi;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = base + lane;
    bool hit = false;
    if (v < hi && !bit_of(vis, v)) {
      const int64_t e0 = off[v], e1 = off[v + 1];
      for (int64_t e = e0; e < e1; ++e) {
        const int32_t u = __ldg(nbr + e);
        ++cnt;
        if (bit_of(fr, u)) {
          parent[v] = u;
          hit = true;
          break;
        }
      }
    }
    const uint32_t word = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) nx[base >> 5] = word;
  }
  cnt = warp_sum(cnt);
  if (lane == 0 && cnt) atomicAdd(scanned, cnt);
}

__global__ void k_bfsd_pull_commit(uint32_t* vis, const uint32_t* nx, int64_t W, unsigned long long* size) {
  unsigned long long c = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < W; w += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = nx[w];
    vis[w] |= x;
    c += __popc(x);
  }
  c = warp_sum(c);
  if (lane_id() == 0 && c) atomicAdd(size, c);
}

// vertex bounds balanced by out-degree, 32-aligned
__global__ void k_bfsd_bounds(const int64_t* off, int64_t V, int P, int64_t* bounds) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > P) return;
  if (r == 0) { bounds[0] = 0; return; }
  if (r == P) { bounds[r] = V; return; }
  const int64_t E = off[V];
  const int64_t target = (int64_t)((__int128)E * r / P);
  int64_t a = 0, b = V;
  while (a < b) {
    int64_t mid = (a + b) >> 1;
    if (off[mid] < target) a = mid + 1; else b = mid;
  }
  bounds[r] = a & ~int64_t(31);
}

// one rank's state
struct BfsRank {
  int dev = 0;
  int64_t V = 0, W = 0, lo = 0, hi = 0;
  DevBuf<int32_t> parent, q;
  DevBuf<uint32_t> vis, fr, nx, disc;  // disc: this rank's discovered bitmap of a top-down level
  DevBuf<unsigned long long> cnt;  // [0] queue length, [1] scanned arcs, [2] next frontier size
  int launches = 0;
  void alloc(int device, int64_t nv, int64_t l, int64_t h) {
    dev = device;
    V = nv;
    W = (V + 31) / 32;
    lo = l;
    hi = h;
    parent.alloc(V);
    q.alloc(std::max<int64_t>(h - l, 1));
    vis.alloc(W);
    fr.alloc(W);
    nx.alloc(W);
    disc.alloc(W);
    cnt.alloc(3);
  }
};

std::vector<int64_t> bfsd_bounds(const Graph& g, int P, cudaStream_t st) {
  CsrView out = g.out_view();
  DevBuf<int64_t> db(P + 1);
  k_bfsd_bounds<<<1, 256, 0, st>>>(out.off, g.V, P, db.p);
  GG_LAUNCH_CHECK();
  std::vector<int64_t> b(P + 1);
  GG_CUDA(cudaMemcpyAsync(b.data(), db.p, (P + 1) * 8, cudaMemcpyDeviceToHost, st));
  GG_CUDA(cudaStreamSynchronize(st));
  return b;
}

// Level-synchronous driver over the ranks this process holds.
int64_t bfs_dist_levels(const Graph& g, std::vector<BfsRank*>& rs, BfsExchange& ex, const std::vector<int64_t>& bounds,
                        int32_t source, double theta, cudaStream_t st, Runtime& rt, int64_t* scanned_out) {
  const int dev = g.dev;
  const int64_t V = g.V;
  CsrView out = g.out_view();
  CsrView in = g.in_view();
  const unsigned grid = (unsigned)sm_count(dev) * 8;
  std::vector<int64_t> wb(bounds.size());
  for (size_t i = 0; i < bounds.size(); ++i) wb[i] = (bounds[i] + 31) / 32;
  wb.back() = rs[0]->W;
  for (auto* R : rs) {
    k_bfsd_init<<<grid_for(V, 256, dev), 256, 0, st>>>(R->parent.p, V, R->vis.p, R->fr.p, R->nx.p, R->W, source);
    GG_LAUNCH_CHECK();
    ++R->launches;
  }
  int64_t size = 1, levels = 0, scanned = 0;
  while (size > 0) {
    const bool pull = (double)size > theta * (double)V;  // strictly greater (engine.py:632)
    rt.edge_begin();
    for (auto* R : rs) {
      GG_CUDA(cudaMemsetAsync(R->cnt.p, 0, 3 * sizeof(unsigned long long), st));
      if (!pull) {
        const int64_t w0 = R->lo / 32, w1 = (R->hi + 31) / 32;
        GG_CUDA(cudaMemsetAsync(R->disc.p, 0, R->W * sizeof(uint32_t), st));
        if (w1 > w0) k_bfsd_queue<<<grid_for(w1 - w0, 256, dev), 256, 0, st>>>(R->fr.p, w0, w1, R->q.p, R->cnt.p);
        k_bfsd_push_bm<<<grid, 256, 0, st>>>(out.off, out.nbr, R->q.p, R->cnt.p, R->vis.p, R->disc.p,
                                             R->cnt.p + 1);
      } else {
        k_bfsd_pull<<<grid, 256, 0, st>>>(in.off, in.nbr, R->lo, R->hi, R->vis.p, R->fr.p, R->parent.p, R->nx.p,
                                          R->cnt.p + 1);
      }
      GG_LAUNCH_CHECK();
      R->launches += 2;
    }
    if (!pull) {
      // discovered bits to their owners (OR), owners pick parents and form
      // their words of the next frontier
      std::vector<uint32_t*> discs;
      for (auto* R : rs) discs.push_back(R->disc.p);
      ex.alltoall_or_words(discs, wb, st);
      for (size_t i = 0; i < rs.size(); ++i) {
        BfsRank* R = rs[i];
        const int64_t w0 = R->lo / 32, w1 = (R->hi + 31) / 32;
        if (w1 > w0)
          k_bfsd_td_commit<<<grid_for((w1 - w0) * 32, 256, dev), 256, 0, st>>>(in.off, in.nbr, w0, w1, R->disc.p,
                                                                                R->vis.p, R->fr.p, R->parent.p,
                                                                                R->nx.p);
        ++R->launches;
      }
    }
    {  // owned next-frontier words to every rank, then vis |= next
      std::vector<void*> nxs;
      for (auto* R : rs) nxs.push_back(R->nx.p);
      ex.allgather_bytes(nxs, sizeof(uint32_t), wb, st);
      for (auto* R : rs) {
        k_bfsd_pull_commit<<<grid_for(R->W, 256, dev), 256, 0, st>>>(R->vis.p, R->nx.p, R->W, R->cnt.p + 2);
        ++R->launches;
      }
    }
    GG_LAUNCH_CHECK();
    rt.edge_end();
    for (auto* R : rs) {
      std::swap(R->fr, R->nx);
    }
    unsigned long long h[3];
    GG_CUDA(cudaMemcpyAsync(h, rs[0]->cnt.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    GG_CUDA(cudaStreamSynchronize(st));
    size = (int64_t)h[2];
    for (auto* R : rs) {
      unsigned long long sc = 0;
      GG_CUDA(cudaMemcpy(&sc, R->cnt.p + 1, 8, cudaMemcpyDeviceToHost));
      scanned += (int64_t)sc;
    }
    rt.stats.direction_log.push_back(pull ? GG_PULL : GG_PUSH);
    rt.stats.dispatch_count += 1;
    ++levels;
  }
  rt.stats.rounds += levels;
  rt.stats.edges_traversed += scanned;
  if (scanned_out) *scanned_out = scanned;
  // owners' parent slices to every rank (vertex bounds, 32-aligned)
  std::vector<void*> ps;
  for (auto* R : rs) ps.push_back(R->parent.p);
  ex.allgather_bytes(ps, sizeof(int32_t), bounds, st);
  return levels;
}

// Virtual ranks on one device (test mode of the multi-GPU path).
// Byte accounting (both exchanges): bytes RANK 0 receives, the per-rank
// exchange volume a real run moves (gg_bfs_exchange_bytes).
struct BfsCopyExchange : BfsExchange {
  int dev;
  explicit BfsCopyExchange(int d) : dev(d) {}
  void alltoall_or_words(std::vector<uint32_t*>& bufs, const std::vector<int64_t>& wb, cudaStream_t st) override {
    const int P = (int)bufs.size();
    for (int r = 0; r < P; ++r) {
      const int64_t n = wb[r + 1] - wb[r];
      for (int q = 0; q < P; ++q)
        if (q != r && n > 0) k_or_into<<<grid_for(n, 256, dev), 256, 0, st>>>(bufs[r] + wb[r], bufs[q] + wb[r], n);
    }
    GG_LAUNCH_CHECK();
    bytes += (uint64_t)(P - 1) * (uint64_t)(wb[1] - wb[0]) * 4;  // rank 0's slice from every peer
  }
  void allgather_bytes(std::vector<void*>& bufs, size_t elt, const std::vector<int64_t>& bounds,
                       cudaStream_t st) override {
    for (size_t r = 0; r < bufs.size(); ++r) {
      const size_t off = (size_t)bounds[r] * elt, len = (size_t)(bounds[r + 1] - bounds[r]) * elt;
      for (size_t q = 0; q < bufs.size(); ++q)
        if (q != r && len)
          GG_CUDA(cudaMemcpyAsync((char*)bufs[q] + off, (char*)bufs[r] + off, len, cudaMemcpyDeviceToDevice, st));
    }
    bytes += (uint64_t)(bounds.back() - bounds[0] - (bounds[1] - bounds[0])) * elt;  // all slices but its own
  }
};

void bfs_dist_check(const Graph& g, int64_t source) {
  if (source < 0 || source >= g.V)
    fail(GG_ERR_VALUE, strf("invalid source %lld for graph with %lld vertices", (long long)source,
                            (long long)g.V));
  if (g.V >= (int64_t)INT32_MAX) fail(GG_ERR_VALUE, "graph too large for int32 vertex ids");
}

int64_t bfs_virtual(const Graph& g, int nparts, int64_t source, double theta, int32_t* parents_out, Runtime& rt) {
  bfs_dist_check(g, source);
  if (nparts < 1) fail(GG_ERR_VALUE, "nparts must be >= 1");
  cudaStream_t st = rt.stream;
  std::vector<int64_t> bounds = bfsd_bounds(g, nparts, st);
  std::vector<BfsRank> rs(nparts);
  std::vector<BfsRank*> rp;
  for (int r = 0; r < nparts; ++r) {
    rs[r].alloc(g.dev, g.V, bounds[r], bounds[r + 1]);
    rp.push_back(&rs[r]);
  }
  BfsCopyExchange ex(g.dev);
  int64_t levels = bfs_dist_levels(g, rp, ex, bounds, (int32_t)source, theta, st, rt, nullptr);
  set_exchange_bytes(ex.bytes);
  GG_CUDA(cudaMemcpyAsync(parents_out, rs[0].parent.p, g.V * 4, cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
  int launches = 0;
  for (auto& R : rs) launches += R.launches;
  count_launch(launches);
  return levels;
}

int64_t bfs_rank(const Graph& g, int P, int r, BfsExchange& ex, int64_t source, double theta, int32_t* parents_out,
                 Runtime& rt) {
  bfs_dist_check(g, source);
  cudaStream_t st = rt.stream;
  std::vector<int64_t> bounds = bfsd_bounds(g, P, st);
  BfsRank R;
  R.alloc(g.dev, g.V, bounds[r], bounds[r + 1]);
  std::vector<BfsRank*> rp{&R};
  int64_t levels = bfs_dist_levels(g, rp, ex, bounds, (int32_t)source, theta, st, rt, nullptr);
  set_exchange_bytes(ex.bytes);
  GG_CUDA(cudaMemcpyAsync(parents_out, R.parent.p, g.V * 4, cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
  count_launch(R.launches);
  return levels;
}

}  // namespace gg
