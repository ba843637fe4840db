// engine.cuh — host side of edgeset.apply: per-query runtime, device frontiers
// and the dispatcher (reference engine.py:418-460, runtime.py:124-248,
// frontier.py:129-284).
#pragma once
#include "graph.cuh"
#include "ops.cuh"

namespace gg {

struct Frontier {
  int dev = 0;
  int64_t universe = 0;
  int repr = GG_SPARSE;
  bool retired = false;
  DevBuf<int32_t> ids;                 // SPARSE queue (capacity = ids.n)
  DevBuf<unsigned long long> count;    // SPARSE entry count (device)
  DevBuf<uint32_t> bits;               // BITMAP words
  DevBuf<uint8_t> bools;               // BOOLMAP bytes (padded to 4)
  int64_t size_cache = -1;             // host cache of size (dense reprs)
  bool size_known_zero = false;

  InView view() const {
    InView v{};
    v.repr = repr;
    v.ids = ids.p;
    v.count = count.p;
    v.bits = bits.p;
    v.bools = bools.p;
    return v;
  }
};

// RunStats (runtime.py:53-67) accumulated on the host.
struct Stats {
  int64_t dispatch_count = 0, rounds = 0, edges_traversed = 0, frontier_conversions = 0,
          frontier_allocations = 0, reused_frontiers = 0, creation_passes = 0;
  std::vector<int32_t> direction_log;
};

struct Runtime {
  const Graph* g = nullptr;
  int dev = 0;
  gg_exec cfg{1, 256, 32, 0};
  cudaStream_t stream = 0;
  Stats stats;
  int fused_depth = 0;
  DevBuf<unsigned long long> scanned;  // device accumulator of edges_traversed
  // FrontierPool: one spare per representation (runtime.py:124-157)
  std::unique_ptr<Frontier> spare[3];
  // MonotonicCounters / DenseMarks (frontier.py:34-118), allocated lazily
  DevBuf<int32_t> stamps;
  int32_t round = 0;
  DevBuf<uint32_t> mark_bits;
  DevBuf<uint8_t> mark_bytes;
  // scratch
  DevBuf<int32_t> twc_q;               // 3 * V
  DevBuf<unsigned long long> twc_cnt;  // 3
  DevBuf<EtwcEntry> etwc_q;            // ETWC huge CTA-stage ranges
  DevBuf<unsigned long long> etwc_n;
  DevBuf<int64_t> prefix;              // STRICT push prefix (V+1)
  DevBuf<int64_t> spans;               // STRICT pull spans
  int64_t spans_n = -1;
  Scratch cub_tmp;
  std::unique_ptr<Frontier> conv;      // temporary converted view

  // CUDA-event timing of every edge-traversal phase (stats.edge_ms)
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> edge_events;
  cudaEvent_t edge_open = nullptr;
  void edge_begin();
  void edge_end();
  double edge_ms(int64_t* launches);   // syncs; sums all recorded phases
  // the call's dominant kernel (PageRank EB: the hot-segment gather), timed
  // the same way; top_edges = edges one launch processes
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> top_events;
  int64_t top_edges = 0;
  void top_record(cudaEvent_t a, cudaEvent_t b) { top_events.emplace_back(a, b); }
  double top_ms(int64_t* launches);

  Runtime(const Graph* graph, const gg_exec* c);
  ~Runtime();
  int64_t edges_traversed();           // syncs the device accumulator

  std::unique_ptr<Frontier> acquire(int repr);
  void release(std::unique_ptr<Frontier> f);
  std::unique_ptr<Frontier> new_frontier(const int32_t* host_ids, int64_t n);
};

// Frontier helpers
int64_t frontier_size(Runtime* rt, Frontier* f);
int64_t frontier_size_raw(Frontier* f, cudaStream_t s);
void frontier_members(Frontier* f, int32_t* out_host, int64_t n, cudaStream_t s);
std::unique_ptr<Frontier> frontier_alloc(int dev, int64_t universe, int repr, int64_t sparse_cap);
void frontier_clear(Frontier* f, cudaStream_t s);
// convert into `dst` (allocated by caller with the target repr)
void frontier_convert_into(Runtime* rt, Frontier* src, Frontier* dst);
// members of a BITMAP / BOOLMAP frontier, ascending, into out[0..*count)
void dense_to_sparse(const Frontier* src, int32_t* out, unsigned long long* count, cudaStream_t s);

// Host-side schedule validation (sched.validate, sched.py:123-142).
void check_schedule(const gg_schedule& s);
void check_binding(const gg_binding& b);

enum UdfKind { UDF_BFS = GG_UDF_BFS, UDF_COUNT = GG_UDF_COUNT, UDF_ENQUEUE = GG_UDF_ENQUEUE,
               UDF_PR = GG_UDF_PR, UDF_CC_HOOK = GG_UDF_CC_HOOK, UDF_BC_FORWARD = GG_UDF_BC_FORWARD,
               UDF_BC_BACKWARD = GG_UDF_BC_BACKWARD, UDF_SSSP_RELAX = GG_UDF_SSSP_RELAX,
               UDF_PR32 = 100 };

// One edgeset.apply round with a named UDF; returns the output frontier
// (null when collect_output is false).  `input` may be null (all active).
// When reuse is set, the input is released to the pool.
// Device BucketQueue (priority.py:17-118), sssp.cu
struct BucketQueueDev;
BucketQueueDev* bq_create(int dev, int64_t universe, uint64_t delta);
void bq_destroy(BucketQueueDev* q);
void bq_seed(BucketQueueDev* q, int64_t v, uint64_t priority);
std::unique_ptr<Frontier> bq_take_current(BucketQueueDev* q);
void bq_recycle(BucketQueueDev* q, std::unique_ptr<Frontier> taken);
bool bq_update_min(BucketQueueDev* q, int64_t v, uint64_t candidate);
bool bq_advance(BucketQueueDev* q);
void bq_info(BucketQueueDev* q, uint64_t* index, int64_t* ncur, int64_t* nfar);
void bq_copy_priorities(BucketQueueDev* q, uint64_t* dst);
Frontier* bq_queue(BucketQueueDev* q, int which);  // 0 current, 1 far
int64_t bq_universe(const BucketQueueDev* q);

// The device balancers' per-vertex split of an active list (test hook):
// ETWC -> (e0, e1, e2) stage sizes per entry, TWC -> bin per entry, STRICT ->
// the exclusive degree prefix (n + 1).  Returns the number of values.
int64_t partition_dump(Runtime* rt, Frontier* active, int lb, int64_t* out, int64_t cap);

std::unique_ptr<Frontier> edgeset_apply(Runtime* rt, int udf, const gg_udf_state& st, bool use_filter,
                                        std::unique_ptr<Frontier>* input, const gg_binding& b,
                                        bool reuse, bool collect_output);

}  // namespace gg
