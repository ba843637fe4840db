// graph.cuh — device-resident graph (reference graphio.Graph, graphio.py:19-92)
// and the EdgeBlocking layout (blocking.BlockedGraph, blocking.py:24-60).
#pragma once
#include "traverse.cuh"
#include <map>
#include <memory>

namespace gg {

// EdgeBlocking layout: COO stably partitioned by dst / n (Alg. 1).
// seg_end holds inclusive segment ends (blocking.py:24-30).
struct Blocked {
  int64_t n = 0, nseg = 0, E = 0;
  DevBuf<int64_t> seg_end;
  DevBuf<int32_t> src, dst;
  DevBuf<uint32_t> w;
  double prep_ms = 0;
};

// Cached pull work plan for the PageRank gather kernel (pagerank.cu).
struct PullPlan;

struct Graph {
  int dev = 0;
  int64_t V = 0, E = 0;
  bool symmetric = false, weighted = false, has_coo = true;
  DevBuf<int64_t> out_off, in_off;
  DevBuf<int32_t> out_nbr, in_nbr, coo_src, coo_dst;
  DevBuf<uint32_t> out_w, in_w, coo_w;
  std::mutex mu;
  std::map<int64_t, std::unique_ptr<Blocked>> blocked;
  std::shared_ptr<PullPlan> pull_plan;
  std::shared_ptr<void> pr_block;  // PageRank EdgeBlocking layout (prblock.cu)
  std::shared_ptr<void> pr_tiles;  // merge-path tile plan over CSR-in (pagerank.cu)
  std::shared_ptr<void> relabel;   // degree-ordered copy for CC / BC / BFS (relabel.cu)
  // CSR views are built on first use (a schedule that only streams the COO
  // never pays for the transpose); guarded by view_mu.
  bool has_out = false, has_in = false;
  int64_t max_out_degree = -1;  // set when CSR-out is built
  std::mutex view_mu;
  void ensure_out() const;
  void ensure_in() const;

  CsrView out_view() const {
    ensure_out();
    return {out_off.p, out_nbr.p, weighted ? out_w.p : nullptr, V};
  }
  CsrView in_view() const {
    ensure_in();
    return {in_off.p, in_nbr.p, weighted ? in_w.p : nullptr, V};
  }
  CooView coo_view() const { return {coo_src.p, coo_dst.p, weighted ? coo_w.p : nullptr, E}; }
};

// Build all views from device COO arrays (copied).  Throws gg::Error.
std::unique_ptr<Graph> graph_from_device_coo(int dev, int64_t V, int64_t E, const int32_t* src,
                                             const int32_t* dst, const uint32_t* w, bool symmetric);
// Takes ownership of already-allocated COO buffers (generators).
std::unique_ptr<Graph> graph_adopt_coo(int dev, int64_t V, DevBuf<int32_t>&& src,
                                       DevBuf<int32_t>&& dst, DevBuf<uint32_t>&& w, bool weighted,
                                       bool symmetric);
std::unique_ptr<Graph> generate_graph(int dev, int kind, int scale, int edge_factor, double a,
                                      double b, double c, uint64_t seed, int flags);

Blocked* blocked_for(Graph& g, int64_t n);  // blocking.blocked_for (blocking.py:69-75)
Blocked* blocked_install(Graph& g, int64_t n, int64_t nseg, const int64_t* seg_end, const int32_t* src,
                         const int32_t* dst, const uint32_t* w);
int64_t default_blocking_size(const Graph& g);

// Stable sort helper: returns the permutation that stably sorts `keys`
// (int32 keys in [0, key_limit)).  Used for CSR/CSC builds and Alg. 1.
void stable_order(int dev, const int32_t* keys, int64_t n, int64_t key_limit, DevBuf<uint32_t>& perm,
                  DevBuf<int32_t>* sorted_keys, cudaStream_t s);
// offsets[k] = first position of key >= k in sorted keys (length nkeys+1).
void offsets_from_sorted(int dev, const int32_t* sorted, int64_t n, int64_t nkeys, int64_t* off,
                         cudaStream_t s);

// Locality relabelling (relabel.cu): the graph renumbered by degree,
// descending, for the frontier algorithms; results map back to original ids.
struct Relabel;
constexpr int kRelabelCc = 0, kRelabelBc = 1, kRelabelBfs = 2;
bool relabel_wanted(const Graph& g, int algo);
std::shared_ptr<Relabel> relabel_for(const Graph& g);
const Graph* relabel_graph(const Relabel& R);
double relabel_prep_ms(const Relabel& R);
int32_t relabel_vertex(const Relabel& R, int64_t v);  // original id -> new id
void relabel_cc_out(const Relabel& R, const int32_t* labels_new, int32_t* out, cudaStream_t st);
void relabel_parents_out(const Relabel& R, const int32_t* par_new, int32_t* out, cudaStream_t st);
void relabel_scores_out(const Relabel& R, const double* x_new, double* out, cudaStream_t st);

}  // namespace gg
