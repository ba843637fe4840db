// prdist.cuh — the exchange step of a destination-partitioned PageRank run
// and the partitioned EdgeBlocking entry points (prblock.cu).
#pragma once
#include "engine.cuh"
#include <vector>

namespace gg {

// After each vertex pass every rank holds (a) two f64 partial sums -- the L1
// of this iteration and the dangling mass of the next, adjacent in memory --
// and (b) its owned slice [bounds[r], bounds[r+1]) of the next contribution
// vector.  The exchange sums (a) over ranks in place and gives (b) to every
// rank.  NCCL implements it across processes (dist.cu); CopyExchange across
// virtual ranks on one device (prblock.cu, test mode).  `d`/`bufs` hold one
// pointer per rank this process drives.
struct PrExchange {
  virtual ~PrExchange() {}
  virtual void allreduce2(std::vector<double*>& d, cudaStream_t st) = 0;
  virtual void allgather(std::vector<void*>& bufs, size_t elt, const std::vector<int64_t>& bounds,
                         cudaStream_t st) = 0;
  // Fused all-gather: for each rank this process drives (i), the pointers of
  // every OTHER rank's two contribution buffers (c0s/c1s hold this process's
  // ranks' own buffers, `bytes` long).  The vertex pass then stores each
  // owned contribution into all of them (P2P over NVLink) and allgather() is
  // skipped.  false = not available: allgather() after each vertex pass.
  virtual bool map_peers(const std::vector<void*>& c0s, const std::vector<void*>& c1s, size_t bytes,
                         std::vector<std::vector<void*>>& peer_c0, std::vector<std::vector<void*>>& peer_c1) {
    return false;
  }
  virtual void unmap_peers() {}
  // Split all-gather for overlap: the part of every slice below hot_end
  // (the hot source window the next iteration's first kernel gathers from)
  // on the main stream, the rest started asynchronously; wait_rest(st) makes
  // the main stream wait for it.  Default: everything on the main stream.
  virtual void allgather_split(std::vector<void*>& bufs, size_t elt, const std::vector<int64_t>& bounds,
                               int64_t hot_end, cudaStream_t st) {
    std::vector<int64_t> hb(bounds.size()), cb(bounds.size());
    split_bounds(bounds, hot_end, hb, cb);
    allgather(bufs, elt, hb, st);
    allgather(bufs, elt, cb, st);
  }
  virtual void wait_rest(cudaStream_t) {}
  // each slice [b_r, b_r+1) cut at h: [min(b_r,h), min(b_r+1,h)) and [max(b_r,h), max(b_r+1,h))
  static void split_bounds(const std::vector<int64_t>& b, int64_t h, std::vector<int64_t>& hot,
                           std::vector<int64_t>& rest) {
    for (size_t i = 0; i < b.size(); ++i) {
      hot[i] = b[i] < h ? b[i] : h;
      rest[i] = b[i] > h ? b[i] : h;
    }
  }
};

// Exchange of the partitioned BFS (bfsdist.cu): an element-wise max of an
// all-to-all of discovered-bitmap slices OR-ed at their owners (top-down) and
// an all-gather of owned slices (next-frontier words, final parents).
struct BfsExchange {
  uint64_t bytes = 0;  // received by one rank over the run (exchange volume)
  virtual ~BfsExchange() {}
  // top-down: every rank's V-bit discovered bitmap; the owner of word range
  // [wb[r], wb[r+1]) ends with the OR over all ranks in its slice
  virtual void alltoall_or_words(std::vector<uint32_t*>& bufs, const std::vector<int64_t>& wb,
                                 cudaStream_t st) = 0;
  virtual void allgather_bytes(std::vector<void*>& bufs, size_t elt, const std::vector<int64_t>& bounds,
                               cudaStream_t st) = 0;
};
int64_t bfs_virtual(const Graph& g, int nparts, int64_t source, double theta, int32_t* parents_out, Runtime& rt);
// bytes one rank received in the last partitioned / virtual run on this thread
void set_exchange_bytes(uint64_t b);
uint64_t last_exchange_bytes();
int64_t bfs_rank(const Graph& g, int P, int r, BfsExchange& ex, int64_t source, double theta, int32_t* parents_out,
                 Runtime& rt);

template <class CT>
int64_t pagerank_blocked_rank(const Graph& g, const gg_schedule& s, int P, int r, PrExchange& ex,
                              int64_t max_iters, double tol, double damping, double* ranks_out, Runtime& rt,
                              int64_t* local_edges);
template <class CT>
int64_t pagerank_blocked_virtual(const Graph& g, const gg_schedule& s, int nparts, int64_t max_iters, double tol,
                                 double damping, double* ranks_out, Runtime& rt, bool fused_allgather = false);
double pr_block_prep_part_ms(const Graph& g, int64_t blocking_size, int ct_bytes, int P, int r,
                             int64_t* bounds = nullptr, int32_t* newid = nullptr);
std::vector<int64_t> bfsd_bounds(const Graph& g, int P, cudaStream_t st);

}  // namespace gg
