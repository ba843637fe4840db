// api.cu — the extern "C" boundary (include/gg.h).  Every entry point catches
// library exceptions and maps them to gg_status codes + gg_last_error().
#include "engine.cuh"
#include "prdist.cuh"
#include <cstring>

namespace gg {
static thread_local std::string t_err;
static thread_local int64_t t_launches = 0;
static thread_local uint64_t t_exchange_bytes = 0;
void set_exchange_bytes(uint64_t b) { t_exchange_bytes = b; }
uint64_t last_exchange_bytes() { return t_exchange_bytes; }
void set_last_error(const std::string& m) { t_err = m; }
void count_launch(int n) { t_launches += n; }
int64_t launches_now() { return t_launches; }

static std::mutex g_dev_mu;
static std::vector<int> g_sm(64, 0);
static std::vector<int64_t> g_l2(64, 0);
int sm_count(int dev) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_sm[dev]) {
    int v = 0;
    GG_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    g_sm[dev] = v;
  }
  return g_sm[dev];
}
int64_t l2_bytes(int dev) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_l2[dev]) {
    int v = 0;
    GG_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev));
    g_l2[dev] = v;
  }
  return g_l2[dev];
}

void pagerank_run(const Graph& g, const gg_binding& b, bool fusion, const gg_exec* cfg,
                  int64_t max_iters, double tol, double damping, double* ranks_out, Runtime& rt,
                  bool fp32_contrib, const double* init_ranks = nullptr);
void bfs_run(const Graph& g, int64_t source, const gg_binding& b, bool fusion, Runtime& rt,
             int32_t* parents_out);
void sssp_run(const Graph& g, int64_t source, const gg_binding& b, bool fusion, Runtime& rt,
              uint64_t* dist_out);
void cc_run(const Graph& g, const gg_binding& b, bool fusion, Runtime& rt, int32_t* labels_out);
void bc_run(const Graph& g, const int64_t* sources, int64_t nsrc, const gg_binding& b, Runtime& rt,
            double* scores_out);
int64_t pagerank_dist_run(gg_comm* c, const Graph& g, int64_t max_iters, double tol, double damping,
                          double* ranks_out, Runtime& rt);
double pr_block_prep_ms(const Graph& g, int64_t blocking_size, int ct_bytes);
int64_t bfs_dist_run(gg_comm* c, const Graph& g, int64_t source, double theta, int32_t* parents_out, Runtime& rt);
int64_t pagerank_dist_blocked(gg_comm* c, const Graph& g, const gg_schedule& s, bool fp32, int64_t max_iters,
                              double tol, double damping, double* ranks_out, Runtime& rt);
inline void pr_block_prep(const Graph& g, int64_t blocking_size, int ct_bytes) {
  pr_block_prep_ms(g, blocking_size, ct_bytes);
}
}  // namespace gg

using namespace gg;

struct gg_graph { std::unique_ptr<Graph> g; };
struct gg_runtime { std::unique_ptr<Runtime> rt; };
struct gg_frontier {
  std::unique_ptr<Frontier> f;
  bool retired = false;
};
struct gg_blocked { Blocked* b; };
struct gg_bucket_queue { BucketQueueDev* q; };

static BucketQueueDev* bq(gg_bucket_queue* q) {
  if (!q || !q->q) fail(GG_ERR_VALUE, "null bucket queue");
  return q->q;
}

#define GG_API_BEGIN try {
#define GG_API_END                                                      \
  return GG_OK;                                                         \
  }                                                                     \
  catch (const gg::Error& e) {                                          \
    set_last_error(e.what());                                           \
    return e.code;                                                      \
  }                                                                     \
  catch (const std::bad_alloc&) {                                       \
    set_last_error("host allocation failed");                           \
    return GG_ERR_OOM;                                                  \
  }                                                                     \
  catch (const std::exception& e) {                                     \
    set_last_error(e.what());                                           \
    return GG_ERR_ENGINE;                                               \
  }

#define NEED(p)                                                         \
  if (!(p)) fail(GG_ERR_VALUE, "null argument: " #p)

static void fill_stats(Runtime& rt, gg_stats* out, double wall_ms, double kernel_ms, int64_t launches) {
  if (!out) return;
  out->dispatch_count = rt.stats.dispatch_count;
  out->rounds = rt.stats.rounds;
  out->edges_traversed = rt.edges_traversed();
  out->frontier_conversions = rt.stats.frontier_conversions;
  out->frontier_allocations = rt.stats.frontier_allocations;
  out->reused_frontiers = rt.stats.reused_frontiers;
  out->creation_passes = rt.stats.creation_passes;
  out->direction_log_len = (int64_t)rt.stats.direction_log.size();
  if (out->direction_log && out->direction_log_cap > 0) {
    int64_t n = std::min<int64_t>(out->direction_log_cap, out->direction_log_len);
    memcpy(out->direction_log, rt.stats.direction_log.data(), n * sizeof(int32_t));
  }
  out->wall_ms = wall_ms;
  out->kernel_ms = kernel_ms;
  out->gpu_launches = launches;
  out->edge_ms = rt.edge_ms(&out->edge_launches);
  out->top_ms = rt.top_ms(&out->top_launches);
  out->top_edges = rt.top_edges;
}

// Times a driver call: CUDA events around the device work, wall clock around all.
struct CallTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  double t0;
  int64_t l0;
  explicit CallTimer(int dev) {
    DeviceGuard g(dev);
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, 0);
    t0 = now_ms();
    l0 = launches_now();
  }
  void finish(int dev, Runtime& rt, gg_stats* st) {
    DeviceGuard g(dev);
    cudaEventRecord(b, 0);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    fill_stats(rt, st, now_ms() - t0, ms, launches_now() - l0);
  }
  ~CallTimer() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

extern "C" {

const char* gg_last_error(void) { return t_err.c_str(); }
int gg_release_cached_memory(void) {
  GG_API_BEGIN
  pool_trim();
  GG_API_END
}

int gg_pool_stats(int64_t* mallocs, int64_t* frees, int64_t* cached_bytes) {
  GG_API_BEGIN
  NEED(mallocs && frees && cached_bytes);
  pool_counters(mallocs, frees, cached_bytes);
  GG_API_END
}

const char* gg_version(void) { return "gg-b200 0.1.0 (sm_100a)"; }

int gg_device_count(int32_t* count) {
  GG_API_BEGIN
  NEED(count);
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) { cudaGetLastError(); n = 0; }
  *count = n;
  GG_API_END
}

int gg_device_info_get(int32_t device, gg_device_info* info) {
  GG_API_BEGIN
  NEED(info);
  cudaDeviceProp p;
  GG_CUDA(cudaGetDeviceProperties(&p, device));
  memset(info, 0, sizeof(*info));
  info->device = device;
  info->sm_count = p.multiProcessorCount;
  info->l2_bytes = p.l2CacheSize;
  info->hbm_bytes = (int64_t)p.totalGlobalMem;
  info->cc_major = p.major;
  info->cc_minor = p.minor;
  info->max_smem_per_block = (int32_t)p.sharedMemPerBlockOptin;
  memcpy(info->name, p.name, sizeof(info->name) - 1);
  GG_API_END
}

int gg_graph_create(int32_t device, int64_t V, int64_t E, const int32_t* src, const int32_t* dst,
                    const uint32_t* w, int32_t symmetric, gg_graph** out) {
  GG_API_BEGIN
  NEED(out);
  if (E > 0) { NEED(src); NEED(dst); }
  DeviceGuard guard(device);
  auto h = new gg_graph;
  try {
    h->g = graph_from_device_coo(device, V, E, src, dst, w, symmetric != 0);
  } catch (...) {
    delete h;
    throw;
  }
  *out = h;
  GG_API_END
}

int gg_graph_create_device(int32_t device, int64_t V, int64_t E, const int32_t* src, const int32_t* dst,
                           const uint32_t* w, int32_t symmetric, gg_graph** out) {
  return gg_graph_create(device, V, E, src, dst, w, symmetric, out);
}

int gg_graph_destroy(gg_graph* g) {
  GG_API_BEGIN
  if (g) {
    DeviceGuard guard(g->g->dev);
    delete g;
  }
  GG_API_END
}

int gg_graph_info(const gg_graph* g, int64_t* V, int64_t* E, int32_t* weighted, int32_t* symmetric,
                  int32_t* device) {
  GG_API_BEGIN
  NEED(g);
  if (V) *V = g->g->V;
  if (E) *E = g->g->E;
  if (weighted) *weighted = g->g->weighted;
  if (symmetric) *symmetric = g->g->symmetric;
  if (device) *device = g->g->dev;
  GG_API_END
}

int gg_graph_copy_array(const gg_graph* gh, int32_t which, void* out) {
  GG_API_BEGIN
  NEED(gh);
  NEED(out);
  const Graph& g = *gh->g;
  DeviceGuard guard(g.dev);
  if (which >= 0 && which <= 2) g.ensure_out();
  if (which >= 3 && which <= 5) g.ensure_in();
  const void* src = nullptr;
  size_t bytes = 0;
  const size_t eb4 = (size_t)g.E * 4, ob = (size_t)(g.V + 1) * 8;
  switch (which) {
    case 0: src = g.out_off.p; bytes = ob; break;
    case 1: src = g.out_nbr.p; bytes = eb4; break;
    case 2: src = g.out_w.p; bytes = g.weighted ? eb4 : 0; break;
    case 3: src = g.in_off.p; bytes = ob; break;
    case 4: src = g.in_nbr.p; bytes = eb4; break;
    case 5: src = g.in_w.p; bytes = g.weighted ? eb4 : 0; break;
    case 6: src = g.coo_src.p; bytes = g.has_coo ? eb4 : 0; break;
    case 7: src = g.coo_dst.p; bytes = g.has_coo ? eb4 : 0; break;
    case 8: src = g.coo_w.p; bytes = (g.has_coo && g.weighted) ? eb4 : 0; break;
    default: fail(GG_ERR_VALUE, "unknown array id");
  }
  if (bytes) GG_CUDA(cudaMemcpy(out, src, bytes, cudaMemcpyDefault));
  GG_API_END
}

int gg_graph_drop_coo(gg_graph* gh) {
  GG_API_BEGIN
  NEED(gh);
  DeviceGuard guard(gh->g->dev);
  gh->g->ensure_out();
  gh->g->ensure_in();
  gh->g->coo_src.release();
  gh->g->coo_dst.release();
  gh->g->coo_w.release();
  gh->g->has_coo = false;
  GG_API_END
}

int gg_generate(int32_t device, int32_t kind, int32_t scale, int32_t edge_factor, double a, double b,
                double c, uint64_t seed, int32_t flags, gg_graph** out) {
  GG_API_BEGIN
  NEED(out);
  auto h = new gg_graph;
  try {
    h->g = generate_graph(device, kind, scale, edge_factor, a, b, c, seed, flags);
  } catch (...) {
    delete h;
    throw;
  }
  *out = h;
  GG_API_END
}

int64_t gg_default_blocking_size(const gg_graph* g) {
  try {
    return default_blocking_size(*g->g);
  } catch (const gg::Error& e) {
    set_last_error(e.what());
    return e.code;
  }
}

int gg_block_edges(gg_graph* g, int64_t n, gg_blocked** out, double* prep_ms) {
  GG_API_BEGIN
  NEED(g);
  Blocked* b = blocked_for(*g->g, n);
  if (prep_ms) *prep_ms = b->prep_ms;
  if (out) *out = new gg_blocked{b};
  GG_API_END
}

int gg_blocked_install(gg_graph* g, int64_t n, int64_t num_segments, const int64_t* segment_start,
                       const int32_t* src, const int32_t* dst, const uint32_t* weights, gg_blocked** out) {
  GG_API_BEGIN
  NEED(g);
  NEED(segment_start);
  if (g->g->E > 0) { NEED(src); NEED(dst); }
  Blocked* b = blocked_install(*g->g, n, num_segments, segment_start, src, dst, weights);
  if (out) *out = new gg_blocked{b};
  GG_API_END
}

int gg_blocked_info(const gg_blocked* b, int64_t* nseg, int64_t* n) {
  GG_API_BEGIN
  NEED(b);
  if (nseg) *nseg = b->b->nseg;
  if (n) *n = b->b->n;
  GG_API_END
}

int gg_blocked_copy_array(const gg_blocked* bh, int32_t which, void* out) {
  GG_API_BEGIN
  NEED(bh);
  NEED(out);
  const Blocked& b = *bh->b;
  size_t eb4 = (size_t)b.E * 4;
  switch (which) {
    case 0: GG_CUDA(cudaMemcpy(out, b.seg_end.p, b.nseg * 8, cudaMemcpyDefault)); break;
    case 1: if (eb4) GG_CUDA(cudaMemcpy(out, b.src.p, eb4, cudaMemcpyDefault)); break;
    case 2: if (eb4) GG_CUDA(cudaMemcpy(out, b.dst.p, eb4, cudaMemcpyDefault)); break;
    case 3: if (eb4 && b.w.p) GG_CUDA(cudaMemcpy(out, b.w.p, eb4, cudaMemcpyDefault)); break;
    default: fail(GG_ERR_VALUE, "unknown array id");
  }
  GG_API_END
}

// ---- runtime / frontier ---------------------------------------------------
int gg_runtime_create(const gg_graph* g, const gg_exec* cfg, gg_runtime** out) {
  GG_API_BEGIN
  NEED(g);
  NEED(out);
  DeviceGuard guard(g->g->dev);
  auto h = new gg_runtime;
  try {
    h->rt = std::make_unique<Runtime>(g->g.get(), cfg);
  } catch (...) {
    delete h;
    throw;
  }
  *out = h;
  GG_API_END
}

int gg_runtime_destroy(gg_runtime* rt) {
  GG_API_BEGIN
  if (rt) {
    DeviceGuard guard(rt->rt->dev);
    delete rt;
  }
  GG_API_END
}

int gg_runtime_stats(gg_runtime* rt, gg_stats* out) {
  GG_API_BEGIN
  NEED(rt);
  DeviceGuard guard(rt->rt->dev);
  fill_stats(*rt->rt, out, 0, 0, 0);
  GG_API_END
}

int gg_frontier_new(gg_runtime* rt, const int32_t* ids, int64_t n, gg_frontier** out) {
  GG_API_BEGIN
  NEED(rt);
  NEED(out);
  if (n > 0) NEED(ids);
  DeviceGuard guard(rt->rt->dev);
  auto h = new gg_frontier;
  try {
    h->f = rt->rt->new_frontier(ids, n);
  } catch (...) {
    delete h;
    throw;
  }
  *out = h;
  GG_API_END
}

static Frontier* live(gg_frontier* f) {
  if (!f) fail(GG_ERR_VALUE, "null frontier");
  if (f->retired || !f->f) fail(GG_ERR_FRONTIER, "frontier was retired");
  return f->f.get();
}

int gg_frontier_release(gg_runtime* rt, gg_frontier* f) {
  GG_API_BEGIN
  NEED(rt);
  live(f);
  DeviceGuard guard(rt->rt->dev);
  rt->rt->release(std::move(f->f));
  f->retired = true;
  GG_API_END
}

int gg_frontier_free(gg_frontier* f) {
  GG_API_BEGIN
  if (f) {
    if (f->f) { DeviceGuard guard(f->f->dev); f->f.reset(); }
    delete f;
  }
  GG_API_END
}

int gg_frontier_size(gg_frontier* f, int64_t* size) {
  GG_API_BEGIN
  NEED(size);
  Frontier* fr = live(f);
  DeviceGuard guard(fr->dev);
  *size = frontier_size_raw(fr, 0);
  GG_API_END
}

int gg_frontier_repr(const gg_frontier* f, int32_t* repr) {
  GG_API_BEGIN
  NEED(repr);
  Frontier* fr = live(const_cast<gg_frontier*>(f));
  *repr = fr->repr;
  GG_API_END
}

int gg_frontier_members(gg_frontier* f, int32_t* out, int64_t cap, int64_t* n) {
  GG_API_BEGIN
  NEED(n);
  Frontier* fr = live(f);
  DeviceGuard guard(fr->dev);
  int64_t sz = frontier_size_raw(fr, 0);
  *n = sz;
  if (sz > cap) fail(GG_ERR_VALUE, "output buffer too small");
  if (sz) NEED(out);
  frontier_members(fr, out, sz, 0);
  GG_API_END
}

int gg_frontier_convert(gg_runtime* rt, gg_frontier* f, int32_t repr, gg_frontier** out) {
  GG_API_BEGIN
  NEED(rt);
  NEED(out);
  Frontier* fr = live(f);
  if (repr < 0 || repr > 2) fail(GG_ERR_FRONTIER, "unknown representation");
  DeviceGuard guard(fr->dev);
  auto h = new gg_frontier;
  h->f = frontier_alloc(fr->dev, fr->universe, repr,
                        repr == GG_SPARSE ? std::max<int64_t>(fr->universe, (int64_t)fr->ids.n) + 1 : 0);
  try {
    frontier_convert_into(rt->rt.get(), fr, h->f.get());
  } catch (...) {
    delete h;
    throw;
  }
  *out = h;
  GG_API_END
}

int gg_edgeset_apply(gg_runtime* rt, int32_t udf, const gg_udf_state* state, int32_t filter,
                     gg_frontier* input, const gg_binding* binding, int32_t reuse,
                     int32_t collect_output, gg_frontier** out) {
  GG_API_BEGIN
  NEED(rt);
  NEED(binding);
  if (input) live(input);
  gg_udf_state st{};
  if (state) st = *state;
  if (udf == GG_UDF_SSSP_RELAX) st.arr0 = bq(static_cast<gg_bucket_queue*>(st.arr0));  // handle -> queue
  DeviceGuard guard(rt->rt->dev);
  auto res = edgeset_apply(rt->rt.get(), udf, st, filter != 0, input ? &input->f : nullptr, *binding,
                           reuse != 0, collect_output != 0);
  if (input && !input->f) input->retired = true;
  if (out) {
    if (res) {
      auto h = new gg_frontier;
      h->f = std::move(res);
      *out = h;
    } else {
      *out = nullptr;
    }
  }
  GG_API_END
}

int gg_runtime_fused_region(gg_runtime* rt, int32_t enter) {
  GG_API_BEGIN
  NEED(rt);
  Runtime& r = *rt->rt;
  if (enter) {
    r.stats.dispatch_count += 1;  // the whole region is one dispatch (runtime.py:194-196)
    r.fused_depth += 1;
  } else {
    if (r.fused_depth <= 0) fail(GG_ERR_ENGINE, "no fused region to leave");
    r.fused_depth -= 1;
  }
  GG_API_END
}

int gg_runtime_add_rounds(gg_runtime* rt, int64_t n) {
  GG_API_BEGIN
  NEED(rt);
  rt->rt->stats.rounds += n;
  GG_API_END
}

int gg_partition_dump(gg_runtime* rt, gg_frontier* active, int32_t load_balance, int64_t* out,
                      int64_t cap, int64_t* n) {
  GG_API_BEGIN
  NEED(rt);
  NEED(n);
  Frontier* f = live(active);
  DeviceGuard guard(rt->rt->dev);
  *n = partition_dump(rt->rt.get(), f, load_balance, out, cap);
  GG_API_END
}

// ---- BucketQueue -------------------------------------------------------------

int gg_bucket_queue_create(int32_t device, int64_t universe, uint64_t delta, gg_bucket_queue** out) {
  GG_API_BEGIN
  NEED(out);
  auto h = new gg_bucket_queue{nullptr};
  try {
    h->q = bq_create(device, universe, delta);
  } catch (...) {
    delete h;
    throw;
  }
  *out = h;
  GG_API_END
}

int gg_bucket_queue_destroy(gg_bucket_queue* q) {
  GG_API_BEGIN
  if (q) {
    bq_destroy(q->q);
    delete q;
  }
  GG_API_END
}

int gg_bucket_queue_seed(gg_bucket_queue* q, int64_t v, uint64_t priority) {
  GG_API_BEGIN
  bq_seed(bq(q), v, priority);
  GG_API_END
}

int gg_bucket_queue_update_min(gg_bucket_queue* q, int64_t v, uint64_t candidate, int32_t* improved) {
  GG_API_BEGIN
  bool r = bq_update_min(bq(q), v, candidate);
  if (improved) *improved = r ? 1 : 0;
  GG_API_END
}

int gg_bucket_queue_take_current(gg_bucket_queue* q, gg_frontier** taken) {
  GG_API_BEGIN
  NEED(taken);
  auto h = new gg_frontier;
  try {
    h->f = bq_take_current(bq(q));
  } catch (...) {
    delete h;
    throw;
  }
  *taken = h;
  GG_API_END
}

int gg_bucket_queue_recycle(gg_bucket_queue* q, gg_frontier* taken) {
  GG_API_BEGIN
  live(taken);
  bq_recycle(bq(q), std::move(taken->f));
  taken->retired = true;
  GG_API_END
}

int gg_bucket_queue_advance(gg_bucket_queue* q, int32_t* nonempty) {
  GG_API_BEGIN
  bool r = bq_advance(bq(q));
  if (nonempty) *nonempty = r ? 1 : 0;
  GG_API_END
}

int gg_bucket_queue_info(gg_bucket_queue* q, uint64_t* index, int64_t* current_size, int64_t* far_size) {
  GG_API_BEGIN
  bq_info(bq(q), index, current_size, far_size);
  GG_API_END
}

int gg_bucket_queue_members(gg_bucket_queue* q, int32_t which, int32_t* out, int64_t cap, int64_t* n) {
  GG_API_BEGIN
  NEED(n);
  Frontier* f = bq_queue(bq(q), which ? 1 : 0);
  DeviceGuard guard(f->dev);
  const int64_t sz = frontier_size_raw(f, 0);
  *n = sz;
  if (sz > cap) fail(GG_ERR_VALUE, "output buffer too small");
  if (sz) NEED(out);
  frontier_members(f, out, sz, 0);
  GG_API_END
}

int gg_bucket_queue_priorities(gg_bucket_queue* q, uint64_t* out) {
  GG_API_BEGIN
  BucketQueueDev* d = bq(q);
  if (bq_universe(d)) NEED(out);
  bq_copy_priorities(d, out);
  GG_API_END
}

// ---- EdgeBlocking apply (blocking.py:116-186) ------------------------------------
int gg_apply_blocked(gg_runtime* rt, int64_t n, int32_t udf, const gg_udf_state* state, int64_t* edges) {
  GG_API_BEGIN
  NEED(rt);
  if (n < 1) fail(GG_ERR_VALUE, "vertices per segment must be >= 1");
  gg_binding b{};
  b.s1.direction = GG_PUSH;
  b.s1.pull_repr = GG_BITMAP;
  b.s1.load_balance = GG_LB_EDGE_ONLY;
  b.s1.blocking = 1;
  b.s1.blocking_size = n;
  b.s1.frontier_creation = GG_CREATE_FUSED;
  b.s1.delta = 1;
  b.s2 = b.s1;
  gg_udf_state st{};
  if (state) st = *state;
  DeviceGuard guard(rt->rt->dev);
  const int64_t before = rt->rt->stats.edges_traversed;
  if (udf == GG_UDF_SSSP_RELAX) st.arr0 = bq(static_cast<gg_bucket_queue*>(st.arr0));
  edgeset_apply(rt->rt.get(), udf, st, false, nullptr, b, false, false);
  if (edges) *edges = rt->rt->stats.edges_traversed - before;
  GG_API_END
}

// ---- algorithm drivers ---------------------------------------------------------
int gg_pagerank(const gg_graph* g, const gg_binding* binding, int32_t fusion, const gg_exec* cfg,
                int64_t max_iters, double tolerance, double damping, double* ranks, gg_stats* stats) {
  GG_API_BEGIN
  NEED(g);
  NEED(binding);
  NEED(ranks);
  DeviceGuard guard(g->g->dev);
  Runtime rt(g->g.get(), cfg);
  CallTimer t(g->g->dev);
  pagerank_run(*g->g, *binding, fusion != 0, cfg, max_iters, tolerance, damping, ranks, rt,
               /*fp32_contrib=*/false);
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_bfs(const gg_graph* g, int64_t source, const gg_binding* binding, int32_t fusion,
           const gg_exec* cfg, int32_t* parents, gg_stats* stats) {
  GG_API_BEGIN
  NEED(g);
  NEED(binding);
  NEED(parents);
  DeviceGuard guard(g->g->dev);
  // locality relabelling (relabel.cu): the query runs on the degree-ordered
  // copy and the parents map back (an invalid source passes through so the
  // driver reports it)
  std::shared_ptr<Relabel> R;
  const Graph* gp = g->g.get();
  if (relabel_wanted(*gp, kRelabelBfs)) {
    R = relabel_for(*gp);
    gp = relabel_graph(*R);
  }
  Runtime rt(gp, cfg);
  CallTimer t(g->g->dev);
  if (R) {
    const int64_t s2 = source >= 0 && source < gp->V ? relabel_vertex(*R, source) : source;
    DevBuf<int32_t> tmp(std::max<int64_t>(gp->V, 1));
    bfs_run(*gp, s2, *binding, fusion != 0, rt, tmp.p);
    relabel_parents_out(*R, tmp.p, parents, rt.stream);
  } else {
    bfs_run(*gp, source, *binding, fusion != 0, rt, parents);
  }
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_sssp_delta(const gg_graph* g, int64_t source, const gg_binding* binding, int32_t fusion,
                  const gg_exec* cfg, uint64_t* dist, gg_stats* stats) {
  GG_API_BEGIN
  NEED(g);
  NEED(binding);
  NEED(dist);
  DeviceGuard guard(g->g->dev);
  Runtime rt(g->g.get(), cfg);
  CallTimer t(g->g->dev);
  sssp_run(*g->g, source, *binding, fusion != 0, rt, dist);
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_cc(const gg_graph* g, const gg_binding* binding, int32_t fusion, const gg_exec* cfg,
          int32_t* labels, gg_stats* stats) {
  GG_API_BEGIN
  NEED(g);
  NEED(binding);
  NEED(labels);
  DeviceGuard guard(g->g->dev);
  std::shared_ptr<Relabel> R;  // locality relabelling (relabel.cu)
  const Graph* gp = g->g.get();
  if (relabel_wanted(*gp, kRelabelCc)) {
    R = relabel_for(*gp);
    gp = relabel_graph(*R);
  }
  Runtime rt(gp, cfg);
  CallTimer t(g->g->dev);
  if (R) {  // canonical labels: each component's minimum ORIGINAL id
    DevBuf<int32_t> tmp(std::max<int64_t>(gp->V, 1));
    cc_run(*gp, *binding, fusion != 0, rt, tmp.p);
    relabel_cc_out(*R, tmp.p, labels, rt.stream);
  } else {
    cc_run(*gp, *binding, fusion != 0, rt, labels);
  }
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_bc(const gg_graph* g, const int64_t* sources, int64_t num_sources, const gg_binding* binding,
          const gg_exec* cfg, double* scores, gg_stats* stats) {
  GG_API_BEGIN
  NEED(g);
  NEED(binding);
  NEED(scores);
  if (num_sources > 0) NEED(sources);
  DeviceGuard guard(g->g->dev);
  std::shared_ptr<Relabel> R;  // locality relabelling (relabel.cu)
  const Graph* gp = g->g.get();
  if (relabel_wanted(*gp, kRelabelBc)) {
    R = relabel_for(*gp);
    gp = relabel_graph(*R);
  }
  Runtime rt(gp, cfg);
  CallTimer t(g->g->dev);
  if (R) {
    std::vector<int64_t> s2(num_sources > 0 ? num_sources : 0);
    for (int64_t k = 0; k < num_sources; ++k)  // invalid ones pass through: the driver reports them
      s2[k] = sources[k] >= 0 && sources[k] < gp->V ? relabel_vertex(*R, sources[k]) : sources[k];
    DevBuf<double> tmp(std::max<int64_t>(gp->V, 1));
    bc_run(*gp, s2.data(), num_sources, *binding, rt, tmp.p);
    relabel_scores_out(*R, tmp.p, scores, rt.stream);
  } else {
    bc_run(*gp, sources, num_sources, *binding, rt, scores);
  }
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_relabel_prepare(const gg_graph* g, double* prep_ms) {
  GG_API_BEGIN
  NEED(g);
  DeviceGuard guard(g->g->dev);
  auto R = relabel_for(*g->g);
  if (prep_ms) *prep_ms = relabel_prep_ms(*R);
  GG_API_END
}

int gg_pagerank_dist(gg_comm* c, const gg_graph* g, int64_t max_iters, double tolerance,
                     double damping, double* ranks, gg_stats* stats) {
  GG_API_BEGIN
  NEED(c);
  NEED(g);
  NEED(ranks);
  DeviceGuard guard(g->g->dev);
  Runtime rt(g->g.get(), nullptr);
  CallTimer t(g->g->dev);
  pagerank_dist_run(c, *g->g, max_iters, tolerance, damping, ranks, rt);
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_pagerank_dist_ex(gg_comm* c, const gg_graph* g, const gg_binding* binding, int32_t fp32_contrib,
                        int64_t max_iters, double tolerance, double damping, double* ranks, gg_stats* stats) {
  GG_API_BEGIN
  NEED(c);
  NEED(g);
  NEED(binding);
  NEED(ranks);
  check_binding(*binding);
  if (binding->is_hybrid) fail(GG_ERR_SCHEDULE, "label 's0:s1' of pagerank takes a SimpleGPUSchedule");
  DeviceGuard guard(g->g->dev);
  Runtime rt(g->g.get(), nullptr);
  CallTimer t(g->g->dev);
  const gg_schedule& s = binding->s1;
  if (s.load_balance == GG_LB_EDGE_ONLY && s.blocking)
    pagerank_dist_blocked(c, *g->g, s, fp32_contrib != 0, max_iters, tolerance, damping, ranks, rt);
  else
    pagerank_dist_run(c, *g->g, max_iters, tolerance, damping, ranks, rt);
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_pagerank_dist_prepare(int32_t nranks, int32_t rank, const gg_graph* g, const gg_binding* binding,
                             int32_t fp32_contrib, double* prep_ms, int64_t* bounds, int32_t* newid) {
  GG_API_BEGIN
  NEED(g);
  NEED(binding);
  check_binding(*binding);
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(GG_ERR_VALUE, "bad rank/nranks");
  DeviceGuard guard(g->g->dev);
  double t0 = now_ms();
  const gg_schedule& s = binding->s1;
  if (s.load_balance == GG_LB_EDGE_ONLY && s.blocking) {
    pr_block_prep_part_ms(*g->g, s.blocking_size, fp32_contrib ? 4 : 8, nranks, rank, bounds, newid);
  } else {
    g->g->out_view();
    g->g->in_view();
    if (bounds || newid) fail(GG_ERR_VALUE, "partition bounds are reported for the EdgeBlocking schedule");
  }
  GG_CUDA(cudaDeviceSynchronize());
  if (prep_ms) *prep_ms = now_ms() - t0;
  GG_API_END
}

int gg_bfs_dist(gg_comm* c, const gg_graph* g, int64_t source, double threshold, int32_t* parents,
                gg_stats* stats) {
  GG_API_BEGIN
  NEED(c);
  NEED(g);
  NEED(parents);
  if (!(threshold > 0.0 && threshold < 1.0)) fail(GG_ERR_SCHEDULE, "threshold must lie in (0, 1)");
  DeviceGuard guard(g->g->dev);
  Runtime rt(g->g.get(), nullptr);
  CallTimer t(g->g->dev);
  bfs_dist_run(c, *g->g, source, threshold, parents, rt);
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_bfs_dist_bounds(const gg_graph* g, int32_t nranks, int64_t* bounds) {
  GG_API_BEGIN
  NEED(g);
  NEED(bounds);
  if (nranks < 1) fail(GG_ERR_VALUE, "bad nranks");
  DeviceGuard guard(g->g->dev);
  std::vector<int64_t> b = bfsd_bounds(*g->g, nranks, 0);
  memcpy(bounds, b.data(), (nranks + 1) * sizeof(int64_t));
  GG_API_END
}

int gg_last_exchange_bytes(uint64_t* bytes) {
  GG_API_BEGIN
  NEED(bytes);
  *bytes = last_exchange_bytes();
  GG_API_END
}

int gg_bfs_virtual(const gg_graph* g, int32_t nparts, int64_t source, double threshold, int32_t* parents,
                   gg_stats* stats) {
  GG_API_BEGIN
  NEED(g);
  NEED(parents);
  if (!(threshold > 0.0 && threshold < 1.0)) fail(GG_ERR_SCHEDULE, "threshold must lie in (0, 1)");
  DeviceGuard guard(g->g->dev);
  Runtime rt(g->g.get(), nullptr);
  CallTimer t(g->g->dev);
  bfs_virtual(*g->g, nparts, source, threshold, parents, rt);
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_pagerank_virtual(const gg_graph* g, int32_t nparts, const gg_binding* binding, int32_t fp32_contrib,
                        int32_t fused_allgather, int64_t max_iters, double tolerance, double damping,
                        double* ranks, gg_stats* stats) {
  GG_API_BEGIN
  NEED(g);
  NEED(binding);
  NEED(ranks);
  check_binding(*binding);
  const gg_schedule& s = binding->s1;
  if (binding->is_hybrid || !(s.load_balance == GG_LB_EDGE_ONLY && s.blocking))
    fail(GG_ERR_SCHEDULE, "virtual-rank PageRank runs the EdgeBlocking schedule (EDGE_ONLY + BLOCKED)");
  DeviceGuard guard(g->g->dev);
  Runtime rt(g->g.get(), nullptr);
  CallTimer t(g->g->dev);
  if (fp32_contrib)
    pagerank_blocked_virtual<float>(*g->g, s, nparts, max_iters, tolerance, damping, ranks, rt, fused_allgather != 0);
  else
    pagerank_blocked_virtual<double>(*g->g, s, nparts, max_iters, tolerance, damping, ranks, rt, fused_allgather != 0);
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_pagerank_prepare(const gg_graph* g, const gg_binding* binding, int32_t fp32_contrib,
                        double* prep_ms) {
  GG_API_BEGIN
  NEED(g);
  NEED(binding);
  DeviceGuard guard(g->g->dev);
  check_binding(*binding);
  double t0 = now_ms();
  const gg_schedule& s = binding->s1;
  if (s.load_balance == GG_LB_EDGE_ONLY && s.blocking) {
    pr_block_prep(*g->g, s.blocking_size, fp32_contrib ? 4 : 8);
  } else if (s.load_balance == GG_LB_EDGE_ONLY) {
    g->g->out_view();
  } else if (s.direction == GG_PULL) {
    g->g->out_view();
    g->g->in_view();
  } else {
    g->g->out_view();
  }
  GG_CUDA(cudaDeviceSynchronize());
  if (prep_ms) *prep_ms = now_ms() - t0;
  GG_API_END
}

int gg_pagerank_resume(const gg_graph* g, const gg_binding* binding, int32_t fusion, const gg_exec* cfg,
                       int64_t max_iters, double tolerance, double damping, const double* init_ranks,
                       double* ranks, gg_stats* stats) {
  GG_API_BEGIN
  NEED(g);
  NEED(binding);
  NEED(init_ranks);
  NEED(ranks);
  DeviceGuard guard(g->g->dev);
  Runtime rt(g->g.get(), cfg);
  CallTimer t(g->g->dev);
  const int64_t V = g->g->V;
  DevBuf<double> init(std::max<int64_t>(V, 1));
  if (V) GG_CUDA(cudaMemcpyAsync(init.p, init_ranks, V * 8, cudaMemcpyDefault, rt.stream));
  pagerank_run(*g->g, *binding, fusion != 0, cfg, max_iters, tolerance, damping, ranks, rt, false, init.p);
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

int gg_pagerank_ex(const gg_graph* g, const gg_binding* binding, int32_t fusion, const gg_exec* cfg,
                   int64_t max_iters, double tolerance, double damping, int32_t fp32_contrib,
                   double* ranks, gg_stats* stats) {
  GG_API_BEGIN
  NEED(g);
  NEED(binding);
  NEED(ranks);
  DeviceGuard guard(g->g->dev);
  Runtime rt(g->g.get(), cfg);
  CallTimer t(g->g->dev);
  pagerank_run(*g->g, *binding, fusion != 0, cfg, max_iters, tolerance, damping, ranks, rt,
               fp32_contrib != 0);
  t.finish(g->g->dev, rt, stats);
  GG_API_END
}

}  // extern "C"
