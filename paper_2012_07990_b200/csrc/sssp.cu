// sssp.cu — algos.sssp_delta (reference algos.py:215-247) with the two-bucket
// queue of priority.BucketQueue (priority.py:17-118) kept on the device.
//
// Device state: dist u64[V] (UNREACHED = 2^64-1), bucket queues as SPARSE
// id lists: current, far (+ a spare for advance), per-round dedup marks for
// current and persistent marks for far (DenseMarks BOOLMAP, priority.py:33-35).
// Round (fused_loop body, algos.py:236-243):
//   current empty -> advance(): drop stale far entries (bucket <= index), pick
//                    the minimum far bucket, split far into current / far;
//   else          -> take current, relax its out-edges with the schedule's
//                    load balancer (PUSH forced), re-bucketing improvements.
// Unfused: one kernel sequence per round with host-side control.
// Fused (s0 kernel fusion): the whole loop, including advance(), is ONE
// cooperative launch with per-bucket frontiers and grid barriers.
#include "fused.cuh"
#include <cstdio>

namespace gg {

static constexpr unsigned long long kUnreached = ~0ULL;

__global__ void k_adv_min(const int32_t* far, const unsigned long long* nfar,
                          const unsigned long long* dist, unsigned long long delta,
                          unsigned long long index, uint8_t* fmark, unsigned long long* best) {
  unsigned long long b_min = kUnreached;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*nfar;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = far[i];
    fmark[v] = 0;
    unsigned long long b = dist[v] / delta;
    if (b > index && b < b_min) b_min = b;
  }
  if (b_min != kUnreached) atomicMin(best, b_min);
}

__global__ void k_adv_split(const int32_t* far, const unsigned long long* nfar,
                            const unsigned long long* dist, unsigned long long delta,
                            unsigned long long index, const unsigned long long* bestp,
                            OutBuilder cur, OutBuilder far2) {
  const unsigned long long best = *bestp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*nfar;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = far[i];
    unsigned long long b = dist[v] / delta;
    if (b <= index) continue;  // stale: handled in an earlier bucket (priority.py:101-105)
    if (b == best) cur.emit(v);
    else far2.emit(v);
  }
}

__global__ void k_clear_byte_marks(const int32_t* ids, const unsigned long long* n, uint8_t* m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)*n;
       i += (int64_t)gridDim.x * blockDim.x)
    m[ids[i]] = 0;
}

static OutBuilder queue_builder(Frontier* q, uint8_t* marks) {
  OutBuilder ob{};
  ob.mode = GG_CREATE_FUSED;
  ob.dedup = DEDUP_MARK_BYTES;
  ob.queue = q->ids.p;
  ob.qcount = q->count.p;
  ob.mark_bytes = marks;
  return ob;
}

// ---------------------------------------------------------------------------
// Fused delta-stepping: one cooperative launch for the whole loop.
// ---------------------------------------------------------------------------
struct SsspFusedArgs {
  gg_schedule s;
  CsrView out;
  CooView coo;
  FusedScratch sc;
  unsigned long long* dist;
  unsigned long long delta;
  int32_t* q[5];                  // current-bucket ring [0..2], far pair [3..4]
  unsigned long long* qn;         // counts [5]
  uint8_t* cmark;
  uint8_t* fmark;
  int32_t* stamps;                // fused relax rounds: current-bucket dedup by round stamp
  uint8_t* member;                // EDGE_ONLY input membership (boolmap)
  unsigned long long* best;       // advance scratch
  unsigned long long* scanned;
  long long* counters;            // [0] rounds [1] relax rounds
  int cta;
  unsigned long long* prof;       // GG_SSSP_PROFILE: [0] top-barrier wait [1] prep+barrier
                                  // [2] max edge-phase time of any thread per round (summed) (ns)
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) k_sssp_fused(SsspFusedArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  // Queues: a ring of three for the current bucket (q[0..2]) and a pair for
  // far (q[3], q[4]).  One grid barrier per relax round: every thread reads
  // the counts right after the barrier; a relax round reads ring slot `ci`
  // (its size stays in a register), appends to slot ci+1, and thread 0
  // zeroes slot ci+2 -- the previous round's input, which nobody reads or
  // writes in this round and which becomes the next round's output.  The
  // output's per-round dedup is a round stamp (no marks to clear).  An
  // advance refills the (empty) current slot behind its own barrier.
  int ci = 0, far = 3, far2 = 4;
  unsigned long long index = 0;
  long long rounds = 0, relax = 0, advances = 0;
  unsigned long long t0 = a.prof ? gtime() : 0;
  while (true) {
    grid.sync();
    unsigned long long t1 = 0;
    if (a.prof && tid == 0) {
      t1 = gtime();
      a.prof[0] += t1 - t0;
    }
    const unsigned long long ncur = *((volatile unsigned long long*)a.qn + ci);
    const unsigned long long nfar = *((volatile unsigned long long*)a.qn + far);
    if (ncur == 0 && nfar == 0) break;  // BucketQueue.done()
    ++rounds;
    if (ncur == 0) {
      // advance(): minimum live far bucket, then split far
      unsigned long long* bestp = a.best + (advances & 1);
      unsigned long long b_min = kUnreached;
      for (int64_t i = tid; i < (int64_t)nfar; i += nth) {
        int32_t v = a.q[far][i];
        a.fmark[v] = 0;
        unsigned long long b = a.dist[v] / a.delta;
        if (b > index && b < b_min) b_min = b;
      }
      if (b_min != kUnreached) atomicMin(bestp, b_min);
      grid.sync();
      const unsigned long long best = *((volatile unsigned long long*)bestp);
      if (best != kUnreached) {
        OutBuilder oc{}, of{};
        oc.mode = of.mode = GG_CREATE_FUSED;
        oc.dedup = DEDUP_NONE;  // far holds each vertex once (fmark), so the split does too
        of.dedup = DEDUP_MARK_BYTES;
        oc.queue = a.q[ci]; oc.qcount = a.qn + ci;
        of.queue = a.q[far2]; of.qcount = a.qn + far2; of.mark_bytes = a.fmark;
        for (int64_t i = tid; i < (int64_t)nfar; i += nth) {
          int32_t v = a.q[far][i];
          unsigned long long b = a.dist[v] / a.delta;
          if (b <= index) continue;
          if (b == best) oc.emit(v);
          else of.emit(v);
        }
        index = best;
      }
      if (tid == 0) {
        a.qn[far] = 0;                            // read into registers before the barrier
        a.best[(advances + 1) & 1] = kUnreached;  // next advance's slot
      }
      ++advances;
      int t = far; far = far2; far2 = t;
      if (a.prof) t0 = gtime();
      continue;
    }
    const int in = ci, out = ci == 2 ? 0 : ci + 1, spare = ci == 0 ? 2 : ci - 1;
    if (tid == 0) a.qn[spare] = 0;
    InView iv{};
    iv.coherent = 1;
    if (a.s.load_balance == GG_LB_EDGE_ONLY) {
      for (int64_t i = tid; i < (int64_t)ncur; i += nth) a.member[a.q[in][i]] = 1;
      iv.repr = GG_BOOLMAP;
      iv.bools = a.member;
      grid.sync();
    } else {
      iv.repr = GG_SPARSE;
      iv.ids = a.q[in];
      iv.count = a.qn + in;
      iv.n_fixed = (int64_t)ncur;
    }
    unsigned long long t2 = a.prof ? gtime() : 0;
    if (a.prof && tid == 0) a.prof[1] += t2 - t1;
    OpRelax op{a.dist, a.delta, index, OutBuilder{}, OutBuilder{}};
    op.cur.mode = op.far.mode = GG_CREATE_FUSED;
    op.cur.dedup = DEDUP_COUNTERS;
    op.cur.stamps = a.stamps;
    op.cur.round = (int32_t)(relax + 1);
    op.far.dedup = DEDUP_MARK_BYTES;
    op.cur.queue = a.q[out]; op.cur.qcount = a.qn + out;
    op.far.queue = a.q[far]; op.far.qcount = a.qn + far; op.far.mark_bytes = a.fmark;
    OutBuilder none{};
    none.mode = OUT_NONE;
    fused_edge_phase(a.s, a.out, a.out, a.coo, iv, op, none, false, a.scanned, a.sc, a.cta, grid);
    if (a.prof) {
      const unsigned long long t3 = gtime();
      if (relax < 1024) atomicMax(a.prof + 3 + relax, t3 - t2);  // slowest thread of the round
      t0 = t3;
    }
    if (a.s.load_balance == GG_LB_EDGE_ONLY) {
      grid.sync();  // membership is read by the edge phase
      for (int64_t i = tid; i < (int64_t)ncur; i += nth) a.member[a.q[in][i]] = 0;
    }
    ci = out;
    ++relax;
  }
  if (tid == 0) {
    a.counters[0] = rounds;
    a.counters[1] = relax;
  }
}

// ---------------------------------------------------------------------------
// BucketQueue as a device object (priority.py:17-118) for custom loops:
// priorities u64[V] (UNREACHED = 2^64-1), current / far SPARSE queues with
// byte-mark dedup (per round for current, until advance for far), a spare
// for recycle().  Host calls order on the legacy stream like every driver.
// ---------------------------------------------------------------------------
struct BucketQueueDev {
  int dev = 0;
  int64_t V = 0;
  unsigned long long delta = 1;
  unsigned long long index = 0;
  DevBuf<unsigned long long> prio, best;
  DevBuf<uint8_t> cmark, fmark;
  DevBuf<int> flag;
  std::unique_ptr<Frontier> cur, far, far2, spare;
};

__global__ void k_bq_update(unsigned long long* prio, int64_t v, unsigned long long cand,
                            unsigned long long delta, unsigned long long index, OutBuilder cur,
                            OutBuilder far, int* improved, int seed) {
  if (seed) {  // seed(): the priority is set, the vertex enters current (priority.py:35-39)
    prio[v] = cand;
    cur.emit((int32_t)v);
    *improved = 1;
    return;
  }
  unsigned long long old = atomicMin(prio + v, cand);
  *improved = cand < old;
  if (cand < old) {
    if (cand / delta == index) cur.emit((int32_t)v);
    else far.emit((int32_t)v);
  }
}

BucketQueueDev* bq_create(int dev, int64_t V, uint64_t delta) {
  if (delta < 1) fail(GG_ERR_VALUE, "delta must be >= 1");
  if (V < 0) fail(GG_ERR_VALUE, "universe must be >= 0");
  DeviceGuard guard(dev);
  auto q = std::make_unique<BucketQueueDev>();
  q->dev = dev;
  q->V = V;
  q->delta = delta;
  q->prio.alloc(V);
  GG_CUDA(cudaMemsetAsync(q->prio.p, 0xff, std::max<int64_t>(V, 1) * 8, 0));
  const int64_t mb = ((V + 3) & ~int64_t(3)) + 4;
  q->cmark.alloc(mb);
  q->fmark.alloc(mb);
  q->cmark.zero();
  q->fmark.zero();
  q->best.alloc(1);
  q->flag.alloc(1);
  q->cur = frontier_alloc(dev, V, GG_SPARSE, V + 1);
  q->far = frontier_alloc(dev, V, GG_SPARSE, V + 1);
  q->far2 = frontier_alloc(dev, V, GG_SPARSE, V + 1);
  return q.release();
}

void bq_destroy(BucketQueueDev* q) {
  if (!q) return;
  DeviceGuard guard(q->dev);
  GG_CUDA(cudaStreamSynchronize(0));
  delete q;
}

static void bq_check_vertex(const BucketQueueDev* q, int64_t v) {
  if (v < 0 || v >= q->V)
    fail(GG_ERR_VALUE, strf("vertex %lld out of range [0, %lld)", (long long)v, (long long)q->V));
}

static bool bq_point_update(BucketQueueDev* q, int64_t v, uint64_t cand, int seed) {
  DeviceGuard guard(q->dev);
  k_bq_update<<<1, 1>>>(q->prio.p, v, cand, q->delta, q->index, queue_builder(q->cur.get(), q->cmark.p),
                        queue_builder(q->far.get(), q->fmark.p), q->flag.p, seed);
  GG_LAUNCH_CHECK();
  count_launch();
  q->cur->size_cache = -1;
  q->far->size_cache = -1;
  int h = 0;
  GG_CUDA(cudaMemcpy(&h, q->flag.p, sizeof(int), cudaMemcpyDeviceToHost));
  return h != 0;
}

void bq_seed(BucketQueueDev* q, int64_t v, uint64_t priority) {
  bq_check_vertex(q, v);
  q->index = priority / q->delta;  // the bucket index snaps to the seed's bucket
  bq_point_update(q, v, priority, 1);
}

bool bq_update_min(BucketQueueDev* q, int64_t v, uint64_t candidate) {
  bq_check_vertex(q, v);
  return bq_point_update(q, v, candidate, 0);
}

std::unique_ptr<Frontier> bq_take_current(BucketQueueDev* q) {
  DeviceGuard guard(q->dev);
  std::unique_ptr<Frontier> taken = std::move(q->cur);
  // clear the per-round marks of the taken ids (priority.py:47)
  k_clear_byte_marks<<<grid_for(std::max<int64_t>(q->V, 1), 256, q->dev), 256>>>(
      taken->ids.p, taken->count.p, q->cmark.p);
  GG_LAUNCH_CHECK();
  count_launch();
  if (q->spare) {
    q->cur = std::move(q->spare);
    q->cur->retired = false;
  } else {
    q->cur = frontier_alloc(q->dev, q->V, GG_SPARSE, q->V + 1);
  }
  frontier_clear(q->cur.get(), 0);
  taken->size_cache = -1;
  return taken;
}

void bq_recycle(BucketQueueDev* q, std::unique_ptr<Frontier> taken) {
  if (!taken) return;
  if (taken->universe != q->V || taken->repr != GG_SPARSE || (int64_t)taken->ids.n < q->V + 1)
    fail(GG_ERR_FRONTIER, "recycle takes a bucket handed out by take_current");
  frontier_clear(taken.get(), 0);
  if (!q->spare) q->spare = std::move(taken);
}

bool bq_advance(BucketQueueDev* q) {
  DeviceGuard guard(q->dev);
  if (frontier_size_raw(q->cur.get(), 0) != 0)
    fail(GG_ERR_ENGINE, "advance with a non-empty current bucket");
  const unsigned grid = (unsigned)sm_count(q->dev) * 8;
  GG_CUDA(cudaMemsetAsync(q->best.p, 0xff, 8, 0));
  k_adv_min<<<grid, 256>>>(q->far->ids.p, q->far->count.p, q->prio.p, q->delta, q->index, q->fmark.p,
                           q->best.p);
  GG_LAUNCH_CHECK();
  unsigned long long hb = 0;
  GG_CUDA(cudaMemcpy(&hb, q->best.p, 8, cudaMemcpyDeviceToHost));
  frontier_clear(q->far2.get(), 0);
  if (hb != kUnreached) {
    k_adv_split<<<grid, 256>>>(q->far->ids.p, q->far->count.p, q->prio.p, q->delta, q->index, q->best.p,
                               queue_builder(q->cur.get(), q->cmark.p),
                               queue_builder(q->far2.get(), q->fmark.p));
    GG_LAUNCH_CHECK();
    q->index = hb;
  }
  count_launch(hb != kUnreached ? 2 : 1);
  frontier_clear(q->far.get(), 0);
  std::swap(q->far, q->far2);
  q->cur->size_cache = -1;
  q->far->size_cache = -1;
  return hb != kUnreached;
}

void bq_info(BucketQueueDev* q, uint64_t* index, int64_t* ncur, int64_t* nfar) {
  DeviceGuard guard(q->dev);
  if (index) *index = q->index;
  if (ncur) *ncur = frontier_size_raw(q->cur.get(), 0);
  if (nfar) *nfar = frontier_size_raw(q->far.get(), 0);
}

void bq_copy_priorities(BucketQueueDev* q, uint64_t* dst) {
  DeviceGuard guard(q->dev);
  if (q->V) GG_CUDA(cudaMemcpy(dst, q->prio.p, q->V * 8, cudaMemcpyDefault));
}

Frontier* bq_queue(BucketQueueDev* q, int which) { return which ? q->far.get() : q->cur.get(); }
int64_t bq_universe(const BucketQueueDev* q) { return q->V; }

// gg_edgeset_apply(GG_UDF_SSSP_RELAX): update_priority_min(dst, prio[src] + w)
// for every arc of the input (algos.py:233-234); state arr0 = the queue.
std::unique_ptr<Frontier> apply_sssp_relax(Runtime* rt, const gg_udf_state& st, bool use_filter,
                                           std::unique_ptr<Frontier>* in, const gg_binding& b,
                                           bool reuse, bool collect) {
  auto* q = static_cast<BucketQueueDev*>(st.arr0);
  if (!q) fail(GG_ERR_VALUE, "sssp relax needs a bucket queue");
  if (q->V != rt->g->V)
    fail(GG_ERR_ENGINE, strf("bucket queue universe %lld does not match graph (%lld vertices)",
                             (long long)q->V, (long long)rt->g->V));
  if (!rt->g->weighted) fail(GG_ERR_VALUE, "sssp relax needs edge weights");
  OpRelax op{q->prio.p, q->delta, q->index, queue_builder(q->cur.get(), q->cmark.p),
             queue_builder(q->far.get(), q->fmark.p)};
  auto out = apply_op(rt, op, use_filter, in, b, reuse, collect);
  q->cur->size_cache = -1;
  q->far->size_cache = -1;
  return out;
}

void sssp_run(const Graph& g, int64_t source, const gg_binding& b, bool fusion, Runtime& rt,
              uint64_t* dist_out) {
  if (source < 0 || source >= g.V)
    fail(GG_ERR_VALUE, strf("invalid source %lld for graph with %lld vertices", (long long)source,
                            (long long)g.V));
  if (!g.weighted) fail(GG_ERR_VALUE, "sssp needs edge weights (load weighted or inject random weights)");
  if (b.is_hybrid)
    fail(GG_ERR_SCHEDULE, "label 's0:s1' of sssp takes a SimpleGPUSchedule (hybrid direction "
                          "switching applies to bfs/bc)");
  check_binding(b);
  DeviceGuard guard(g.dev);
  const int64_t V = g.V;
  const int dev = g.dev;
  cudaStream_t st = rt.stream;
  gg_binding pb = b;
  pb.s1.direction = GG_PUSH;  // relaxation is source-driven (algos.py:226-227)
  const gg_schedule& s = pb.s1;
  const unsigned long long delta = (unsigned long long)s.delta;
  DevBuf<unsigned long long> dist(V);
  GG_CUDA(cudaMemsetAsync(dist.p, 0xff, V * 8, st));
  unsigned long long zero = 0;
  GG_CUDA(cudaMemcpyAsync(dist.p + source, &zero, 8, cudaMemcpyHostToDevice, st));
  const int64_t mb = ((V + 3) & ~int64_t(3)) + 4;
  DevBuf<uint8_t> cmark(mb), fmark(mb);
  cmark.zero(st);
  fmark.zero(st);
  const uint8_t one = 1;
  GG_CUDA(cudaMemcpyAsync(cmark.p + source, &one, 1, cudaMemcpyHostToDevice, st));
  int32_t src32 = (int32_t)source;

  if (fusion) {
    SsspFusedArgs a{};
    a.s = s;
    if (s.load_balance == GG_LB_EDGE_ONLY) {
      if (!s.blocking) a.coo = g.coo_view();
    } else {
      a.out = g.out_view();
    }
    a.out.V = V;
    a.dist = dist.p;
    a.delta = delta;
    DevBuf<int32_t> q[5];
    DevBuf<unsigned long long> qn(5), best(2);
    qn.zero(st);
    GG_CUDA(cudaMemsetAsync(best.p, 0xff, 2 * sizeof(unsigned long long), st));
    for (int k = 0; k < 5; ++k) {
      q[k].alloc(V + 1);
      a.q[k] = q[k].p;
    }
    GG_CUDA(cudaMemcpyAsync(q[0].p, &src32, 4, cudaMemcpyHostToDevice, st));
    unsigned long long n1 = 1;
    GG_CUDA(cudaMemcpyAsync(qn.p, &n1, 8, cudaMemcpyHostToDevice, st));
    DevBuf<uint8_t> member(mb);
    member.zero(st);
    DevBuf<int32_t> stamps(V);
    stamps.zero(st);
    a.stamps = stamps.p;
    DevBuf<long long> counters(2);
    a.qn = qn.p;
    a.cmark = cmark.p;
    a.fmark = fmark.p;
    a.member = member.p;
    a.best = best.p;
    a.scanned = rt.scanned.p;
    a.counters = counters.p;
    a.cta = rt.cfg.cta_size;
    DevBuf<unsigned long long> prof;
    if (getenv("GG_SSSP_PROFILE")) {
      prof.alloc(3 + 1024);
      prof.zero(st);
      a.prof = prof.p;
    }
    int blocks = max_coop_blocks((const void*)k_sssp_fused, 256, dev, 0, 1);  // barrier-bound
    FusedHost fh;
    const gg_schedule* ss[1] = {&s};
    fh.prepare(rt, ss, 1, blocks);
    a.sc = fh.sc;
    void* args[] = {&a};
    rt.edge_begin();
    GG_CUDA(cudaLaunchCooperativeKernel((const void*)k_sssp_fused, blocks, 256, args, 0, st));
    rt.edge_end();
    count_launch();
    long long h[2];
    GG_CUDA(cudaMemcpyAsync(h, counters.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    GG_CUDA(cudaStreamSynchronize(st));
    if (a.prof) {  // diagnostic: where a fused round's time goes (stderr)
      std::vector<unsigned long long> hp(3 + 1024);
      GG_CUDA(cudaMemcpy(hp.data(), prof.p, hp.size() * 8, cudaMemcpyDeviceToHost));
      unsigned long long mx = 0;
      for (int k = 0; k < 1024; ++k) mx += hp[3 + k];
      const long long nr = h[1] < 1024 ? h[1] : 1024;
      fprintf(stderr, "sssp fused profile: rounds %lld relax %lld | thread0: top-barrier wait %.3f ms, "
              "prep+barrier %.3f ms | slowest-thread edge phase, mean of first %lld rounds: %.3f us\n",
              h[0], h[1], hp[0] / 1e6, hp[1] / 1e6, nr, nr ? mx / 1e3 / nr : 0.0);
    }
    rt.stats.dispatch_count += 1;
    rt.stats.rounds += h[0];
    for (long long k = 0; k < h[1]; ++k) rt.stats.direction_log.push_back(GG_PUSH);
    if (s.load_balance == GG_LB_EDGE_ONLY) rt.stats.frontier_conversions += h[1];
  } else {
    std::unique_ptr<Frontier> cur = frontier_alloc(dev, V, GG_SPARSE, V + 1);
    std::unique_ptr<Frontier> take = frontier_alloc(dev, V, GG_SPARSE, V + 1);
    std::unique_ptr<Frontier> far = frontier_alloc(dev, V, GG_SPARSE, V + 1);
    std::unique_ptr<Frontier> far2 = frontier_alloc(dev, V, GG_SPARSE, V + 1);
    GG_CUDA(cudaMemcpyAsync(cur->ids.p, &src32, 4, cudaMemcpyHostToDevice, st));
    unsigned long long n1 = 1;
    GG_CUDA(cudaMemcpyAsync(cur->count.p, &n1, 8, cudaMemcpyHostToDevice, st));
    DevBuf<unsigned long long> best(1);
    unsigned long long index = 0;
    const unsigned grid = (unsigned)sm_count(dev) * 8;
    while (true) {
      unsigned long long n[2];
      GG_CUDA(cudaMemcpyAsync(&n[0], cur->count.p, 8, cudaMemcpyDeviceToHost, st));
      GG_CUDA(cudaMemcpyAsync(&n[1], far->count.p, 8, cudaMemcpyDeviceToHost, st));
      GG_CUDA(cudaStreamSynchronize(st));
      if (n[0] == 0 && n[1] == 0) break;
      rt.stats.rounds += 1;
      if (n[0] == 0) {  // advance()
        GG_CUDA(cudaMemsetAsync(best.p, 0xff, 8, st));
        k_adv_min<<<grid, 256, 0, st>>>(far->ids.p, far->count.p, dist.p, delta, index, fmark.p, best.p);
        GG_LAUNCH_CHECK();
        unsigned long long hb = 0;
        GG_CUDA(cudaMemcpyAsync(&hb, best.p, 8, cudaMemcpyDeviceToHost, st));
        GG_CUDA(cudaStreamSynchronize(st));
        if (hb != kUnreached) {
          OutBuilder oc = queue_builder(cur.get(), cmark.p);
          OutBuilder of = queue_builder(far2.get(), fmark.p);
          k_adv_split<<<grid, 256, 0, st>>>(far->ids.p, far->count.p, dist.p, delta, index, best.p,
                                            oc, of);
          GG_LAUNCH_CHECK();
          index = hb;
        }
        count_launch(hb != kUnreached ? 2 : 1);
        GG_CUDA(cudaMemsetAsync(far->count.p, 0, 8, st));
        std::swap(far, far2);
        continue;
      }
      std::swap(cur, take);  // take_current()
      GG_CUDA(cudaMemsetAsync(cur->count.p, 0, 8, st));
      k_clear_byte_marks<<<grid, 256, 0, st>>>(take->ids.p, take->count.p, cmark.p);
      GG_LAUNCH_CHECK();
      count_launch();
      take->size_cache = (int64_t)n[0];
      OpRelax op{dist.p, delta, index, queue_builder(cur.get(), cmark.p), queue_builder(far.get(), fmark.p)};
      rt.edge_begin();
      apply_op(&rt, op, false, &take, pb, false, false);
      rt.edge_end();
      take->size_cache = -1;
    }
  }
  GG_CUDA(cudaMemcpyAsync(dist_out, dist.p, V * 8, cudaMemcpyDefault, st));
  GG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gg
