/* gg.h — C ABI of the B200-native edgeset.apply engine (libgg.so).
 *
 * This is the drop-in boundary for the reference's traversal hot path
 * (package `schedge`, /root/reference/pkg/src/schedge).  The reference is a
 * pure-Python package, so its "FFI" is the Python call surface; every entry
 * point below names the reference interface it replaces (file:line, relative
 * to /root/reference/pkg/src/schedge/).  The Python host package
 * `paper_2012_07990_b200` binds these symbols with ctypes (see
 * paper_2012_07990_b200/_lib.py and INTEGRATION.md).
 *
 * Conventions
 *  - plain pointers and sizes only; no torch / C++ types cross the boundary;
 *  - every function returns GG_OK (0) or a negative gg_status code, and the
 *    message of the last failure on the calling thread is gg_last_error();
 *  - "host or device" output pointers are written with cudaMemcpyDefault, so a
 *    caller may pass either pinned/pageable host memory or a device pointer;
 *  - a gg_graph is immutable after creation and may be shared by concurrent
 *    queries on different host threads (graphio.py:19-26); a gg_runtime is
 *    per query (algos.py:109, runtime.py:199-215).
 */
#ifndef GG_H
#define GG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (error conventions of SURVEY §8b) -------------------- */
typedef enum {
  GG_OK = 0,
  GG_ERR_SCHEDULE = -1, /* ScheduleError   sched.py:44, engine.py:434-436       */
  GG_ERR_ENGINE = -2,   /* EngineError     runtime.py:58, engine.py:439-441     */
  GG_ERR_VALUE = -3,    /* ValueError      algos.py:91-94, :222-224, :326-327   */
  GG_ERR_CUDA = -4,     /* device failure (no reference analogue)               */
  GG_ERR_NCCL = -5,     /* collective failure (no reference analogue)           */
  GG_ERR_FRONTIER = -6, /* FrontierError   frontier.py:26                       */
  GG_ERR_OOM = -7       /* device allocation failed                             */
} gg_status;

/* ---- schedule codes (sched.py:29-39 token order) ---------------------- */
enum { GG_PUSH = 0, GG_PULL = 1 };
enum { GG_SPARSE = 0, GG_BITMAP = 1, GG_BOOLMAP = 2 };
enum {
  GG_LB_VERTEX_BASED = 0, GG_LB_CM = 1, GG_LB_WM = 2, GG_LB_STRICT = 3,
  GG_LB_EDGE_ONLY = 4, GG_LB_ETWC = 5, GG_LB_TWC = 6
};
enum { GG_CREATE_FUSED = 0, GG_CREATE_UNFUSED_BOOLMAP = 1, GG_CREATE_UNFUSED_BITMAP = 2 };
enum { GG_DEDUP_MONOTONIC_COUNTERS = 0, GG_DEDUP_BITMAP = 1, GG_DEDUP_BOOLMAP = 2 };

/* POD mirror of sched.Schedule (sched.py:55-71). blocking_size 0 = default. */
typedef struct {
  int32_t direction;
  int32_t pull_repr;
  int32_t load_balance;
  int32_t blocking;
  int64_t blocking_size;
  int32_t frontier_creation;
  int32_t dedup;
  int32_t dedup_strategy;
  int32_t kernel_fusion;
  int64_t delta;
} gg_schedule;

/* A label binding: simple schedule or sched.HybridSchedule (sched.py:74-89). */
typedef struct {
  int32_t is_hybrid;
  double threshold; /* resolved hybrid threshold in (0,1) */
  gg_schedule s1;   /* the simple schedule when !is_hybrid */
  gg_schedule s2;
} gg_binding;

/* Shape of the CTA hierarchy (runtime.ExecConfig, runtime.py:26-50).
 * On the device cta_size is the block size used by the CTA-granular
 * load balancers (ETWC stage-2 chunk, TWC CTA threshold); warp_size must be
 * 32 there.  num_workers is a host-simulation knob of the reference and
 * only validated here; deterministic = 1 makes gg_pagerank sum in the
 * reference's fixed order (per destination in COO order, dangling mass and
 * L1 in vertex order, no FMA): ranks bitwise equal to the reference's for
 * EDGE_ONLY (+ BLOCKED) and PULL schedules (a slow correctness mode). */
typedef struct {
  int32_t num_workers;
  int32_t cta_size;
  int32_t warp_size;
  int32_t deterministic;
} gg_exec;

/* runtime.RunStats (runtime.py:53-67) + device timings. direction_log is a
 * caller buffer of direction codes; direction_log_len reports the full
 * length even when it exceeds direction_log_cap. */
typedef struct {
  int64_t dispatch_count;
  int64_t rounds;
  int64_t edges_traversed;
  int64_t frontier_conversions;
  int64_t frontier_allocations;
  int64_t reused_frontiers;
  int64_t creation_passes;
  int32_t* direction_log;
  int64_t direction_log_cap;
  int64_t direction_log_len;
  double kernel_ms;  /* device time of the algorithm (CUDA events) */
  double wall_ms;    /* host wall time of the call */
  int64_t gpu_launches; /* kernels this call launched */
  double edge_ms;       /* device time of the edge-traversal phase (events)  */
  int64_t edge_launches;/* number of edge-traversal phases timed in edge_ms */
  double top_ms;        /* device time of the call's dominant kernel (events; 0 if none) */
  int64_t top_launches; /* launches of that kernel timed in top_ms */
  int64_t top_edges;    /* edges one launch of it processes */
} gg_stats;

typedef struct {
  int32_t device;
  int32_t sm_count;
  int64_t l2_bytes;
  int64_t hbm_bytes;
  int32_t cc_major, cc_minor;
  int32_t max_smem_per_block;
  char name[128];
} gg_device_info;

typedef struct gg_graph gg_graph;       /* device-resident immutable graph   */
typedef struct gg_runtime gg_runtime;   /* per-query state (stats, pools)    */
typedef struct gg_frontier gg_frontier; /* device VertexSubset               */
typedef struct gg_blocked gg_blocked;   /* device EdgeBlocking layout        */

/* ---- library / device ---------------------------------------------------- */
const char* gg_last_error(void);
const char* gg_version(void);
int gg_device_count(int32_t* count);
/* Device buffers come from a per-device caching pool (per-query buffers are
 * reused across calls instead of cudaMalloc/cudaFree each time); this
 * returns every cached block to the driver.  GG_POOL_MAX_GB caps the cache
 * (default: 60% of the device's memory). */
int gg_release_cached_memory(void);
/* Pool counters since load: driver allocations, driver frees, bytes cached.
 * When a free would push the cache past the cap, the largest cached blocks
 * of other sizes are returned first, so per-call buffers stay cached. */
int gg_pool_stats(int64_t* mallocs, int64_t* frees, int64_t* cached_bytes);
int gg_device_info_get(int32_t device, gg_device_info* info);

/* ---- graph (graphio.Graph.from_coo, graphio.py:58-81) ------------------------
 * Builds CSR-out, CSR-in (CSC) and keeps the COO in load order, on `device`.
 * CSR views are a stable counting sort of the COO (graphio.py:95-102), so
 * neighbour order equals the reference's.  weights may be NULL.  Arrays are
 * host pointers; gg_graph_create_device takes device pointers (copied). */
int gg_graph_create(int32_t device, int64_t num_vertices, int64_t num_edges,
                    const int32_t* src, const int32_t* dst, const uint32_t* weights,
                    int32_t symmetric, gg_graph** out);
int gg_graph_create_device(int32_t device, int64_t num_vertices, int64_t num_edges,
                           const int32_t* d_src, const int32_t* d_dst,
                           const uint32_t* d_weights, int32_t symmetric, gg_graph** out);
int gg_graph_destroy(gg_graph* g);
int gg_graph_info(const gg_graph* g, int64_t* num_vertices, int64_t* num_edges,
                  int32_t* weighted, int32_t* symmetric, int32_t* device);
/* which: 0 out_offsets(int64,V+1) 1 out_neighbors(int32,E) 2 out_weights(uint32,E)
 *        3 in_offsets 4 in_neighbors 5 in_weights 6 coo_src 7 coo_dst 8 coo_weights */
int gg_graph_copy_array(const gg_graph* g, int32_t which, void* out);
/* Release the COO view (keeps CSR/CSC) to save HBM on the largest graphs. */
int gg_graph_drop_coo(gg_graph* g);

/* Synthetic inputs generated on the device (bench/test workloads, §8d).
 *  kind 0: RMAT(scale, edge_factor, a, b, c) directed, duplicates + loops kept
 *  kind 1: Graph500 Kronecker (same recursion, ids permuted)
 *  kind 2: 2-D 4-neighbour grid side x side, arcs both ways
 * flags: 1 = symmetrize+dedup (graphio._symmetrize semantics, graphio.py:118-140)
 *        2 = permute vertex ids (seeded)   4 = attach uint32 weights U[1,1000]
 *        8 = order the COO by source (edge-list-file order) */
int gg_generate(int32_t device, int32_t kind, int32_t scale, int32_t edge_factor,
                double a, double b, double c, uint64_t seed, int32_t flags,
                gg_graph** out);

/* ---- EdgeBlocking (blocking.py) ------------------------------------------ */
/* default_blocking_size (blocking.py:63-66) but from the queried L2 size. */
int64_t gg_default_blocking_size(const gg_graph* g);
/* Alg. 1 on the device (blocking.py:78-113): stable partition of the COO by
 * dst / n.  Cached on the graph per n (blocking.py:69-75). */
int gg_block_edges(gg_graph* g, int64_t n, gg_blocked** out, double* prep_ms);
/* Install a layout read from a blocked-graph sidecar (blocking.load_blocked,
 * blocking.py:200-217) instead of recomputing Alg. 1: host (or device)
 * arrays, inclusive segment ends; validated against the graph (segment
 * bounds, every edge in its segment, same edge multiset) and cached as
 * gg_block_edges(g, n) would have cached it. */
int gg_blocked_install(gg_graph* g, int64_t n, int64_t num_segments, const int64_t* segment_start,
                       const int32_t* src, const int32_t* dst, const uint32_t* weights,
                       gg_blocked** out);
int gg_blocked_info(const gg_blocked* b, int64_t* num_segments, int64_t* n);
/* which: 0 segment_start(int64,S) 1 src(int32,E) 2 dst(int32,E) 3 weight(uint32,E) */
int gg_blocked_copy_array(const gg_blocked* b, int32_t which, void* out);

/* ---- runtime + frontier (runtime.py:160-248, frontier.py:129-269) ------- */
int gg_runtime_create(const gg_graph* g, const gg_exec* cfg, gg_runtime** out);
int gg_runtime_destroy(gg_runtime* rt);
int gg_runtime_stats(gg_runtime* rt, gg_stats* out);
/* FrontierPool.new_frontier (runtime.py:151-157): SPARSE subset of ids. */
int gg_frontier_new(gg_runtime* rt, const int32_t* ids, int64_t n, gg_frontier** out);
int gg_frontier_release(gg_runtime* rt, gg_frontier* f); /* FrontierPool.release */
int gg_frontier_free(gg_frontier* f);
int gg_frontier_size(gg_frontier* f, int64_t* size);      /* VertexSubset.size   */
int gg_frontier_repr(const gg_frontier* f, int32_t* repr);
/* VertexSubset.members (frontier.py:186-201): insertion order for SPARSE,
 * ascending for dense.  out must hold `size` ids. */
int gg_frontier_members(gg_frontier* f, int32_t* out, int64_t cap, int64_t* n);
int gg_frontier_convert(gg_runtime* rt, gg_frontier* f, int32_t repr, gg_frontier** out);

/* ---- edgeset.apply with a named device UDF (engine.py:418-460) ------------
 * The reference accepts an arbitrary Python udf(ctx); on the device each udf
 * is a named functor (SURVEY §7 hard part 1) -- every UDF the reference's
 * algorithms define is one.  udf ids (state fields are device pointers):
 *   GG_UDF_BFS        arr0 int32 parent[V]       push CAS / pull store + enqueue,
 *                                                 filter parent[v] == -1 (algos.py:114-125)
 *   GG_UDF_COUNT      arr0 int64 counts[V]       atomic_add(counts[dst], 1)
 *   GG_UDF_ENQUEUE    -                          enqueue(dst)
 *   GG_UDF_PR         arr0 double acc[V],        atomic_add(acc[dst], contrib[src]) (algos.py:180-181)
 *                     arr1 double contrib[V]
 *   GG_UDF_CC_HOOK    arr0 int32 label[V],       la, lb = label[src], label[dst];
 *                     arr1 int changed            atomic_min(label, max, min) -> changed = 1
 *                                                 (algos.py:283-293)
 *   GG_UDF_BC_FORWARD arr0 int32 depth[V],       CAS depth -1 -> level+1 + enqueue; sigma[dst] +=
 *                     arr1 double sigma[V],       sigma[src] when depth[dst] == level+1; filter
 *                     i0 level                    depth == -1 or level+1 (algos.py:353-365)
 *   GG_UDF_BC_BACKWARD arr0 depth, arr1 sigma,   delta[src] += sigma[src]/sigma[dst]*(1+delta[dst])
 *                     arr2 double delta[V]        when depth[dst] == depth[src]+1 (algos.py:378-382)
 *   GG_UDF_SSSP_RELAX arr0 gg_bucket_queue*      q.update_priority_min(dst, prio[src] + w)
 *                                                 (algos.py:233-234)
 * `filter` 0 = none, 1 = the udf's own filter. */
enum {
  GG_UDF_BFS = 0, GG_UDF_COUNT = 1, GG_UDF_ENQUEUE = 2, GG_UDF_PR = 3, GG_UDF_CC_HOOK = 4,
  GG_UDF_BC_FORWARD = 5, GG_UDF_BC_BACKWARD = 6, GG_UDF_SSSP_RELAX = 7
};
typedef struct {
  void* arr0;
  void* arr1;
  int64_t i0;
  void* arr2;
} gg_udf_state;
int gg_edgeset_apply(gg_runtime* rt, int32_t udf, const gg_udf_state* state, int32_t filter,
                     gg_frontier* input /* NULL = all vertices */, const gg_binding* binding,
                     int32_t reuse, int32_t collect_output, gg_frontier** out);

/* The device balancers' split of a SPARSE active list, for pinning against
 * the reference partitioners (engine.py:51-142): ETWC -> 3 values per entry
 * (stage 0 / 1 / 2 edge counts, engine.py:62-85), TWC -> the bin per entry
 * (0 thread, 1 warp, 2 CTA; engine.py:131-142), STRICT -> the exclusive
 * degree prefix, n + 1 values (engine.py:116-122).  *n = values written. */
int gg_partition_dump(gg_runtime* rt, gg_frontier* active, int32_t load_balance, int64_t* out,
                      int64_t cap, int64_t* n);

/* engine.fused_loop / Runtime.fused_dispatch (engine.py:639-662,
 * runtime.py:194-209): enter = 1 opens a fused region (one dispatch for
 * everything inside, counted now), enter = 0 closes it; add_rounds adds loop
 * bodies to RunStats.rounds. */
int gg_runtime_fused_region(gg_runtime* rt, int32_t enter);
int gg_runtime_add_rounds(gg_runtime* rt, int64_t n);

/* ---- BucketQueue on the device (priority.py:17-118) --------------------------
 * Priorities u64 (GG_UNREACHED = 2^64-1), current / far buckets as SPARSE
 * queues with the reference's dedup (per round for current, until advance
 * for far).  take_current hands out the current bucket as a frontier (input
 * of a GG_UDF_SSSP_RELAX apply), recycle returns its storage.  advance
 * reports *nonempty = 0 when drained (the reference returns None) and fails
 * with GG_ERR_ENGINE while current is non-empty. */
typedef struct gg_bucket_queue gg_bucket_queue;
int gg_bucket_queue_create(int32_t device, int64_t universe, uint64_t delta,
                           gg_bucket_queue** out);
int gg_bucket_queue_destroy(gg_bucket_queue* q);
int gg_bucket_queue_seed(gg_bucket_queue* q, int64_t v, uint64_t priority);
int gg_bucket_queue_update_min(gg_bucket_queue* q, int64_t v, uint64_t candidate,
                               int32_t* improved);
int gg_bucket_queue_take_current(gg_bucket_queue* q, gg_frontier** taken);
int gg_bucket_queue_recycle(gg_bucket_queue* q, gg_frontier* taken);
int gg_bucket_queue_advance(gg_bucket_queue* q, int32_t* nonempty);
int gg_bucket_queue_info(gg_bucket_queue* q, uint64_t* index, int64_t* current_size,
                         int64_t* far_size);
int gg_bucket_queue_members(gg_bucket_queue* q, int32_t which /* 0 current, 1 far */,
                            int32_t* out, int64_t cap, int64_t* n);
int gg_bucket_queue_priorities(gg_bucket_queue* q, uint64_t* out /* V, host or device */);

/* ---- EdgeBlocking apply (blocking.py:116-186) -------------------------------
 * Alg. 2 over the graph's blocked layout of width n (built and cached on
 * first use, or installed from a sidecar): segments in order, each split
 * evenly over the grid, a grid barrier between segments, the named udf's
 * atomic form per edge; one dispatch.  *edges = edges processed. */
int gg_apply_blocked(gg_runtime* rt, int64_t n, int32_t udf, const gg_udf_state* state,
                     int64_t* edges);

/* ---- algorithm drivers (algos.py) ------------------------------------------
 * fusion = the "s0" loop binding's kernel fusion (engine.fused_loop).  All
 * outputs may be host or device pointers. */
int gg_bfs(const gg_graph* g, int64_t source, const gg_binding* binding, int32_t fusion,
           const gg_exec* cfg, int32_t* parents, gg_stats* stats);            /* algos.py:101 */
int gg_pagerank(const gg_graph* g, const gg_binding* binding, int32_t fusion,
                const gg_exec* cfg, int64_t max_iters, double tolerance, double damping,
                double* ranks, gg_stats* stats);                              /* algos.py:163 */
/* gg_pagerank with the contribution vector stored as f32 (accumulation stays
 * f64); halves the bytes of the random gathers on the largest graphs. */
/* Build (and cache on the graph) whatever layout the bound PageRank schedule
 * uses -- the EdgeBlocking source-segment layout for EDGE_ONLY+BLOCKED, the
 * pull plan for PULL -- and report its preprocessing time, which the
 * reference's CLI also times apart from the runs (cli.py:178-192). */
int gg_pagerank_prepare(const gg_graph* g, const gg_binding* binding, int32_t fp32_contrib,
                        double* prep_ms);
int gg_pagerank_ex(const gg_graph* g, const gg_binding* binding, int32_t fusion,
                   const gg_exec* cfg, int64_t max_iters, double tolerance, double damping,
                   int32_t fp32_contrib, double* ranks, gg_stats* stats);
/* Locality relabelling for the frontier algorithms (no reference
 * counterpart; a layout choice like EdgeBlocking): gg_bc runs on a copy of
 * the graph renumbered by degree (descending) when
 * the graph has >= 2^20 vertices, gg_cc / gg_bfs only when GG_RELABEL=1
 * (GG_RELABEL=0 turns it off everywhere); results map back to the original
 * ids -- canonical CC labels stay each component's minimum original id.
 * This builds the copy ahead of the queries (cached on the graph) and
 * reports its preprocessing time. */
int gg_relabel_prepare(const gg_graph* g, double* prep_ms);
/* gg_pagerank continued from a given rank vector (host or device, original
 * ids) instead of rank_0 = 1/n: the power iteration's whole state between
 * iterations is the rank vector, so k calls of one iteration each equal one
 * call of k.  pagerank(on_iteration=...) drives it one iteration per call
 * (algos.py:163-208 observes every iteration). */
int gg_pagerank_resume(const gg_graph* g, const gg_binding* binding, int32_t fusion,
                       const gg_exec* cfg, int64_t max_iters, double tolerance, double damping,
                       const double* init_ranks, double* ranks, gg_stats* stats);
int gg_sssp_delta(const gg_graph* g, int64_t source, const gg_binding* binding,
                  int32_t fusion, const gg_exec* cfg, uint64_t* dist, gg_stats* stats); /* algos.py:215 */
int gg_cc(const gg_graph* g, const gg_binding* binding, int32_t fusion, const gg_exec* cfg,
          int32_t* labels, gg_stats* stats);                                  /* algos.py:267 */
int gg_bc(const gg_graph* g, const int64_t* sources, int64_t num_sources,
          const gg_binding* binding, const gg_exec* cfg, double* scores,
          gg_stats* stats);                                                   /* algos.py:314 */

/* ---- multi-GPU (1-D vertex partition, NCCL over NVLink) --------
 * One process per GPU.  gg_nccl_unique_id fills 128 bytes on rank 0; the
 * caller broadcasts it (torch.distributed) and every rank calls
 * gg_comm_init.  gg_pagerank_dist runs PageRank on this rank's partition:
 * the rank owns destinations [lo, hi) (balanced by in-edge count) and
 * allgathers contributions every iteration. */
typedef struct gg_comm gg_comm;
int gg_nccl_unique_id(char out[128]);
int gg_comm_init(int32_t device, int32_t nranks, int32_t rank, const char id[128],
                 gg_comm** out);
int gg_comm_destroy(gg_comm* c);
int gg_pagerank_dist(gg_comm* c, const gg_graph* g, int64_t max_iters, double tolerance,
                     double damping, double* ranks /* V, gathered on every rank */,
                     gg_stats* stats);
/* The same with the bound schedule: EDGE_ONLY + BLOCKED runs the
 * EdgeBlocking layout over this rank's destinations (renumbered ids,
 * partition balanced by in-edges), any other schedule the PULL gather above.
 * Replaces blocking.apply_blocked (blocking.py:116-186) driven by
 * algos.pagerank (algos.py:163-208) for one partition of a multi-GPU run. */
int gg_pagerank_dist_ex(gg_comm* c, const gg_graph* g, const gg_binding* binding,
                        int32_t fp32_contrib, int64_t max_iters, double tolerance, double damping,
                        double* ranks, gg_stats* stats);
/* Build (and cache) rank `rank` of `nranks`'s layout without running.
 * Optionally reports the destination partition (bounds: nranks+1 entries,
 * in renumbered ids) and the renumbering (newid: V entries, original id ->
 * renumbered id); both may be NULL (EdgeBlocking schedule only). */
int gg_pagerank_dist_prepare(int32_t nranks, int32_t rank, const gg_graph* g,
                             const gg_binding* binding, int32_t fp32_contrib, double* prep_ms,
                             int64_t* bounds, int32_t* newid);
/* Direction-optimizing BFS, 1-D vertex partition (32-aligned, balanced by
 * out-degree), bitmap frontier exchange: top-down levels all-reduce(max)
 * parent candidates, bottom-up levels all-gather the owned next-frontier
 * words; PULL iff |frontier| > threshold*V (engine.hybrid_apply,
 * engine.py:622-636; algos.bfs, algos.py:101-135).  parents: V, gathered on
 * every rank; a legal BFS tree with the single-GPU depths. */
int gg_bfs_dist(gg_comm* c, const gg_graph* g, int64_t source, double threshold,
                int32_t* parents, gg_stats* stats);
/* The vertex partition gg_bfs_dist uses (nranks+1 entries). */
int gg_bfs_dist_bounds(const gg_graph* g, int32_t nranks, int64_t* bounds);
/* The same with `nparts` virtual ranks on the graph's one device (test mode). */
/* Bytes one rank received through the exchange in the last gg_bfs_dist /
 * gg_bfs_virtual call on this thread (top-down: V/8 of discovered bitmap
 * slices, bottom-up: V/8 of frontier words, per level; plus the final
 * V*4-byte parent all-gather). */
int gg_last_exchange_bytes(uint64_t* bytes);
int gg_bfs_virtual(const gg_graph* g, int32_t nparts, int64_t source, double threshold,
                   int32_t* parents, gg_stats* stats);
/* Test mode of the partitioned run: `nparts` virtual ranks on the graph's
 * one device, each with its own layout and buffers, exchanging by copies in
 * the same order as the NCCL exchange (fused_allgather = 0), or with the
 * vertex pass storing into the other ranks' buffers as the multi-GPU fused
 * all-gather does over NVLink (fused_allgather = 1).  EDGE_ONLY + BLOCKED. */
int gg_pagerank_virtual(const gg_graph* g, int32_t nparts, const gg_binding* binding,
                        int32_t fp32_contrib, int32_t fused_allgather, int64_t max_iters,
                        double tolerance, double damping, double* ranks, gg_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* GG_H */
